// pattern.cuh — packed quick/canonical pattern codes, shared by the vertex
// and edge engines (__host__ __device__).
//
// a pattern is (position labels, position edge set); the
// canonical form is the lexicographic minimum of (labels, sorted edge list)
// over all permutations, the first minimiser in next_permutation order giving
// the PositionMap.  We pack a pattern into one u64 whose INTEGER order equals
// that lexicographic order:
//
//   code = nv << 60 | labels << NP | E          (nv <= 8; labels + E <= 60 bits)
//   labels = L[0] << LB*(nv-1) | ... | L[nv-1]        (L[0] most significant)
//   E      = ~M & (2^NP - 1),  M bit (NP-1-p) set iff pair p is an edge,
//            pairs p in lexicographic order (0,1),(0,2),..,(nv-2,nv-1)
//
// For two sorted edge lists of equal length, the lexicographically smaller
// list has the LARGER M (its first differing pair is a smaller pair, i.e. a
// more significant bit), hence the smaller E.  So min(code) over permutations
// == the SPEC's lexicographic minimum, and ties (automorphisms) keep the
// first permutation.  The CPU oracle implements the literal vector compare;
// tests hold the two to each other.
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace gpm {
namespace pat {

__host__ __device__ __forceinline__ int npairs(int nv) { return nv * (nv - 1) / 2; }

__host__ __device__ __forceinline__ int pair_index(int i, int j, int nv) {
  // i < j
  return i * nv - i * (i + 1) / 2 + (j - i - 1);
}

// mask: bit p set iff pair p is an edge (natural bit order).
__host__ __device__ __forceinline__ uint64_t make_code(int nv, const uint32_t* lab, uint32_t mask, int LB) {
  const int NP = npairs(nv);
  uint64_t lab_packed = 0;
  for (int i = 0; i < nv; ++i) lab_packed = (lab_packed << LB) | (uint64_t)lab[i];
  uint64_t M = 0;
  for (int p = 0; p < NP; ++p)
    if (mask >> p & 1u) M |= (uint64_t)1 << (NP - 1 - p);
  const uint64_t E = (~M) & (((uint64_t)1 << NP) - 1);
  return ((uint64_t)nv << 60) | (lab_packed << NP) | E;
}

#ifdef __CUDACC__
// Device fast paths of the same packing (no per-pair loop): E = complement of
// the bit-reversed natural mask; labels already packed (L[0] most significant).
__device__ __forceinline__ uint64_t make_code_packed(int nv, uint64_t lab_packed, uint32_t mask) {
  const int NP = npairs(nv);
  const uint32_t full = NP >= 32 ? 0xffffffffu : ((1u << NP) - 1u);
  const uint32_t M = NP ? (__brev(mask) >> (32 - NP)) : 0u;
  return ((uint64_t)nv << 60) | (lab_packed << NP) | (uint64_t)(~M & full);
}
// natural pair mask over nv positions -> the same pairs over nv + 1 positions
// (pair (i, j) moves from index p to p + i: row i shifts by i)
__device__ __forceinline__ uint32_t widen_mask(uint32_t mask, int nv) {
  uint32_t out = 0;
  int start = 0;
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    if (i < nv - 1) {
      const int len = nv - 1 - i;
      const uint32_t row = (mask >> start) & ((1u << len) - 1u);
      out |= row << (start + i);
      start += len;
    }
  }
  return out;
}
#endif

__host__ __device__ __forceinline__ bool next_perm(uint8_t* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return false;
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  uint8_t t = a[i];
  a[i] = a[j];
  a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) {
    t = a[l];
    a[l] = a[r];
    a[r] = t;
  }
  return true;
}

// canonicalize: returns canonical code; perm[i] = canonical
// position of quick position i.
//
// Labels compare first, so every minimiser sorts the labels: only
// permutations sending each position into its label's block of the sorted
// label sequence can win (the exact label-partition pre-filter of
// SPEC.md:245).  They are enumerated depth-first with increasing slots, i.e.
// in the lexicographic (next_permutation) order of the full enumeration, so
// the first minimiser -- the PositionMap tie-break -- is unchanged.  With
// distinct labels this is one permutation; unlabeled 8-vertex patterns still
// visit all 40320.
__host__ __device__ inline uint64_t canonicalize(int nv, const uint32_t* lab, uint32_t mask, int LB, uint8_t* perm_out) {
  uint32_t sl[8];
  for (int i = 0; i < nv; ++i) sl[i] = lab[i];
  for (int i = 1; i < nv; ++i) {  // insertion sort: the canonical label sequence
    const uint32_t x = sl[i];
    int j = i - 1;
    while (j >= 0 && sl[j] > x) {
      sl[j + 1] = sl[j];
      --j;
    }
    sl[j + 1] = x;
  }
  uint8_t lo[8], hi[8];
  for (int i = 0; i < nv; ++i) {
    int a = 0;
    while (sl[a] != lab[i]) ++a;
    int b = a;
    while (b < nv && sl[b] == lab[i]) ++b;
    lo[i] = (uint8_t)a;
    hi[i] = (uint8_t)b;
  }
  // the pattern's edges as (i, j) position pairs
  uint8_t ea[28], eb[28];
  int ne = 0;
  for (int a = 0; a < nv; ++a)
    for (int b = a + 1; b < nv; ++b)
      if (mask >> pair_index(a, b, nv) & 1u) {
        ea[ne] = (uint8_t)a;
        eb[ne] = (uint8_t)b;
        ++ne;
      }
  uint64_t best = ~(uint64_t)0;
  uint8_t p[8], nxt[8];
  uint32_t used = 0;
  int i = 0;
  nxt[0] = lo[0];
  for (;;) {
    int sv = nxt[i];
    while (sv < hi[i] && (used >> sv & 1u)) ++sv;
    if (sv >= hi[i]) {  // position i exhausted: backtrack
      if (i == 0) break;
      --i;
      used &= ~(1u << p[i]);
      nxt[i] = (uint8_t)(p[i] + 1);
      continue;
    }
    p[i] = (uint8_t)sv;
    used |= 1u << sv;
    if (i + 1 < nv) {
      ++i;
      nxt[i] = lo[i];
      continue;
    }
    uint32_t pm = 0;
    for (int e = 0; e < ne; ++e) {
      int x = p[ea[e]], y = p[eb[e]];
      if (x > y) { const int t = x; x = y; y = t; }
      pm |= 1u << pair_index(x, y, nv);
    }
    const uint64_t c = make_code(nv, sl, pm, LB);
    if (c < best) {
      best = c;
      if (perm_out)
        for (int j = 0; j < nv; ++j) perm_out[j] = p[j];
    }
    used &= ~(1u << sv);
    nxt[i] = (uint8_t)(sv + 1);
  }
  return best;
}

// Automorphism orbits of a pattern (full-automorphism MNI):
// rep[i] = smallest position j such that some automorphism (a label- and
// edge-preserving permutation) maps i to j.  Label-preserving permutations are
// enumerated depth-first as in canonicalize (each position stays inside its
// label block); those that map the edge mask onto itself are automorphisms.
__host__ __device__ inline void orbits(int nv, const uint32_t* lab, uint32_t mask, uint8_t* rep) {
  for (int i = 0; i < nv; ++i) rep[i] = (uint8_t)i;
  uint8_t ea[28], eb[28];
  int ne = 0;
  for (int a = 0; a < nv; ++a)
    for (int b = a + 1; b < nv; ++b)
      if (mask >> pair_index(a, b, nv) & 1u) {
        ea[ne] = (uint8_t)a;
        eb[ne] = (uint8_t)b;
        ++ne;
      }
  uint8_t p[8], nxt[8];
  uint32_t used = 0;
  int i = 0;
  nxt[0] = 0;
  for (;;) {
    int sv = nxt[i];
    while (sv < nv && ((used >> sv & 1u) || lab[sv] != lab[i])) ++sv;
    if (sv >= nv) {
      if (i == 0) break;
      --i;
      used &= ~(1u << p[i]);
      nxt[i] = (uint8_t)(p[i] + 1);
      continue;
    }
    p[i] = (uint8_t)sv;
    used |= 1u << sv;
    if (i + 1 < nv) {
      ++i;
      nxt[i] = 0;
      continue;
    }
    uint32_t pm = 0;
    for (int e = 0; e < ne; ++e) {
      int x = p[ea[e]], y = p[eb[e]];
      if (x > y) { const int t = x; x = y; y = t; }
      pm |= 1u << pair_index(x, y, nv);
    }
    if (pm == mask) {  // automorphism: merge the orbits of j and p[j]
      for (int j = 0; j < nv; ++j) {
        const uint8_t a = rep[j], b = rep[p[j]];
        const uint8_t lo = a < b ? a : b, hi = a < b ? b : a;
        if (lo != hi)
          for (int t = 0; t < nv; ++t)
            if (rep[t] == hi) rep[t] = lo;
      }
    }
    used &= ~(1u << sv);
    nxt[i] = (uint8_t)(sv + 1);
  }
}

__host__ __device__ __forceinline__ int code_nv(uint64_t code) { return (int)(code >> 60); }
// bits a code of nv positions with LB-bit labels needs below the nv field
__host__ __device__ __forceinline__ int code_bits(int nv, int LB) { return nv * LB + npairs(nv); }
constexpr int kCodeBits = 60;

// Decode labels and natural-order edge mask from a code.
__host__ __device__ inline void decode(uint64_t code, int LB, int* nv_out, uint32_t* lab, uint32_t* mask) {
  const int nv = code_nv(code);
  const int NP = npairs(nv);
  const uint64_t E = code & (((uint64_t)1 << NP) - 1);
  const uint64_t M = (~E) & (((uint64_t)1 << NP) - 1);
  uint32_t m = 0;
  for (int p = 0; p < NP; ++p)
    if (M >> (NP - 1 - p) & 1u) m |= 1u << p;
  uint64_t lp = (code & (((uint64_t)1 << 60) - 1)) >> NP;
  for (int i = nv - 1; i >= 0; --i) {
    lab[i] = LB ? (uint32_t)(lp & ((((uint64_t)1) << LB) - 1)) : 0u;
    lp = LB ? (lp >> LB) : 0;
  }
  *nv_out = nv;
  *mask = m;
}

}  // namespace pat
}  // namespace gpm
