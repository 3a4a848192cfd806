// common.hpp — shared host-side types and the error model behind the C ABI.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>

#include "gpm.h"

namespace gpm {

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;

// Internal exception; converted to a gpm_status at the ABI (exceptions never
// cross extern "C").  Mirrors gpmine::error / parse_error
// (error.hpp:10-25): parse errors carry a 1-based line number.
struct Error : std::runtime_error {
  int code;
  u64 line;
  Error(int c, const std::string& m, u64 l = 0) : std::runtime_error(m), code(c), line(l) {}
};

void set_last_error(const std::string& msg);

// Runs f(), converting exceptions into status codes + thread-local message.
template <class F>
int guarded(F&& f, u64* err_line = nullptr) {
  try {
    f();
    return GPM_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    if (err_line) *err_line = e.line;
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return GPM_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GPM_EINVAL;
  }
}

}  // namespace gpm
