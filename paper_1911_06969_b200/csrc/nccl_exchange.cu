// nccl_exchange.cu — the multi-GPU exchange hook (gpm_exchange_fn) implemented
// inside libgpm.so over NCCL (NVLink / NVSwitch on a B200 node), so a C++
// host needs no Python.  SURVEY §8(e): the only collectives of the path are
//   op 0  sum of u64 count vectors                      -> ncclAllReduce(sum)
//   op 1  bitwise OR of u32 FSM domain bitmaps          -> owner-based OR:
//         every rank owns 1/N of the words; one grouped all-to-all
//         (ncclSend/ncclRecv) delivers each owner the N copies of its slice,
//         a device kernel ORs them, and ncclAllGather returns the ORed
//         slices.  Per GPU that moves 2(N-1)/N of the bitmap bytes instead of
//         the (N-1)x of an all-gather + local OR (NCCL has no bitwise op).
//   op 2  all-gather of per-rank slots (FSM pattern-key union) -> in-place
//         ncclAllGather.
// The engine calls the hook with the stream idle (exchange_device syncs it)
// and orders its later work on the same stream, so no extra host syncs here.
#include <nccl.h>

#include <cstring>
#include <memory>

#include "engine.hpp"

namespace gpm {
namespace {

struct NcclEx {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  bool owned = false;
};

#define GPM_NCCL(x)                                                                           \
  do {                                                                                        \
    ncclResult_t r_ = (x);                                                                    \
    if (r_ != ncclSuccess) throw Error(GPM_ENCCL, std::string("nccl: ") + ncclGetErrorString(r_)); \
  } while (0)

// own[i] = OR over ranks q of parts[q * per + i]
__global__ void or_slices_kernel(const u32* __restrict__ parts, int world, u64 per, u32* __restrict__ own) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < per; i += (u64)gridDim.x * blockDim.x) {
    u32 v = 0;
    for (int q = 0; q < world; ++q) v |= parts[(u64)q * per + i];
    own[i] = v;
  }
}

unsigned grid_for(u64 n) { return (unsigned)std::max<u64>(1, std::min<u64>(4096, (n + 255) / 256)); }

void owner_or(NcclEx& x, u32* buf, u64 count, cudaStream_t s) {
  const int W = x.world;
  const u64 per = (count + W - 1) / W;
  // padded copy when count is not a multiple of the world size
  DBuf<u32> pad;
  u32* src = buf;
  if (per * W != count) {
    pad.alloc(per * W, s);
    GPM_CUDA(cudaMemsetAsync(pad.get(), 0, sizeof(u32) * per * W, s));
    GPM_CUDA(cudaMemcpyAsync(pad.get(), buf, sizeof(u32) * count, cudaMemcpyDeviceToDevice, s));
    src = pad.get();
  }
  DBuf<u32> parts(per * W, s), own(per, s);
  GPM_NCCL(ncclGroupStart());
  for (int q = 0; q < W; ++q) {
    GPM_NCCL(ncclSend(src + (u64)q * per, per, ncclUint32, q, x.comm, s));
    GPM_NCCL(ncclRecv(parts.get() + (u64)q * per, per, ncclUint32, q, x.comm, s));
  }
  GPM_NCCL(ncclGroupEnd());
  or_slices_kernel<<<grid_for(per), 256, 0, s>>>(parts.get(), W, per, own.get());
  GPM_CUDA(cudaGetLastError());
  GPM_NCCL(ncclAllGather(own.get(), src, per, ncclUint32, x.comm, s));
  if (src != buf) GPM_CUDA(cudaMemcpyAsync(buf, src, sizeof(u32) * count, cudaMemcpyDeviceToDevice, s));
}

int nccl_exchange(void* ctx, void* dev_buf, uint64_t count, int elem_bytes, int op, void* stream) {
  auto* x = static_cast<NcclEx*>(ctx);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return guarded([&] {
    if (!x || !x->comm) throw Error(GPM_ENCCL, "nccl exchange: no communicator");
    if (count == 0) return;
    switch (op) {
      case 0:
        if (elem_bytes != 8) throw Error(GPM_EINVAL, "exchange sum: u64 elements");
        GPM_NCCL(ncclAllReduce(dev_buf, dev_buf, count, ncclUint64, ncclSum, x->comm, s));
        break;
      case 1:
        if (elem_bytes != 4) throw Error(GPM_EINVAL, "exchange OR: u32 words");
        if (x->world > 1) owner_or(*x, static_cast<u32*>(dev_buf), count, s);
        break;
      case 2: {
        const size_t nb = (size_t)count * elem_bytes;
        char* b = static_cast<char*>(dev_buf);
        GPM_NCCL(ncclAllGather(b + (size_t)x->rank * nb, b, nb, ncclUint8, x->comm, s));
        break;
      }
      default:
        throw Error(GPM_EINVAL, "exchange: unknown op");
    }
  });
}

}  // namespace
}  // namespace gpm

using namespace gpm;

extern "C" {

int gpm_nccl_unique_id(void* id_out) {
  return guarded([&] {
    if (!id_out) throw Error(GPM_EINVAL, "null argument");
    ncclUniqueId id;
    GPM_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == GPM_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof id);
  });
}

int gpm_exchange_nccl_create(const void* unique_id, int rank, int world, int device, void** ctx) {
  return guarded([&] {
    if (!unique_id || !ctx || world < 1 || rank < 0 || rank >= world) throw Error(GPM_EINVAL, "bad argument");
    GPM_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    auto x = std::make_unique<NcclEx>();
    GPM_NCCL(ncclCommInitRank(&x->comm, world, id, rank));
    x->rank = rank;
    x->world = world;
    x->device = device;
    x->owned = true;
    *ctx = x.release();
  });
}

int gpm_exchange_nccl_wrap(void* nccl_comm, void** ctx) {
  return guarded([&] {
    if (!nccl_comm || !ctx) throw Error(GPM_EINVAL, "null argument");
    auto x = std::make_unique<NcclEx>();
    x->comm = static_cast<ncclComm_t>(nccl_comm);
    GPM_NCCL(ncclCommCount(x->comm, &x->world));
    GPM_NCCL(ncclCommUserRank(x->comm, &x->rank));
    GPM_NCCL(ncclCommCuDevice(x->comm, &x->device));
    *ctx = x.release();
  });
}

gpm_exchange_fn gpm_exchange_nccl_fn(void) { return &gpm::nccl_exchange; }

int gpm_exchange_nccl_destroy(void* ctx) {
  return guarded([&] {
    auto* x = static_cast<NcclEx*>(ctx);
    if (!x) return;
    if (x->owned && x->comm) GPM_NCCL(ncclCommDestroy(x->comm));
    delete x;
  });
}

}  // extern "C"
