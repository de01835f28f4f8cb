// Per-snapshot top-k peak selection (K6 in SURVEY.md).
//
// Order = extract_support's (reference: pkg/src/bccblasso/solvers.py:494-499): descending
// |c| in float64 (np.abs of the complex128 estimate), ties to the lower flat index (stable
// argsort of -|c|).  Encoded in a 96-bit key compared lexicographically:
//     key.a = double_bits(hypot(re, im)),  key.b = 0xFFFFFFFF - index
// so "largest key" is exactly that order (|c| >= 0 => IEEE bits order like integers).  The
// magnitude is float64 for complex64 input too (exact products of the float components).
// Key (0, 0) is a sentinel below every real key (index < 2^32 - 1).
//
// Phase 1: grid (chunks, batch); every thread keeps its own sorted top-KT list in
// registers, then the CTA merges the 256 lists by k rounds of block-wide argmax.
// Phase 2: one CTA per snapshot merges the chunk candidates the same way.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bccb {

inline int topk_chunks(int batch, long long length) {
  long long by_len = (length + 8191) / 8192;
  long long by_occ = (592 + batch - 1) / batch;  // ~4 CTAs per SM over 148 SMs
  long long c = by_len < by_occ ? by_len : by_occ;
  if (c < 1) c = 1;
  if (c > 4096) c = 4096;
  return (int)c;
}

struct TKey {
  unsigned long long a;   // float64 bits of |c|
  unsigned int b;         // 0xFFFFFFFF - index
};
__device__ __forceinline__ bool key_gt(const TKey& x, const TKey& y) { return x.a > y.a || (x.a == y.a && x.b > y.b); }
__device__ __forceinline__ bool key_eq(const TKey& x, const TKey& y) { return x.a == y.a && x.b == y.b; }
__device__ __forceinline__ TKey key_zero() { return TKey{0ull, 0u}; }

template <int KT>
__device__ __forceinline__ void topk_insert(TKey (&lst)[KT], TKey key) {
  if (!key_gt(key, lst[KT - 1])) return;
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    if (key_gt(key, lst[i])) {
      const TKey t = lst[i];
      lst[i] = key;
      key = t;
    }
  }
}

__device__ __forceinline__ TKey warp_max_key(TKey v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    TKey w;
    w.a = __shfl_xor_sync(0xffffffffu, v.a, o);
    w.b = __shfl_xor_sync(0xffffffffu, v.b, o);
    if (key_gt(w, v)) v = w;
  }
  return v;
}

// k rounds of block argmax over the per-thread sorted lists; writes winners to out[0..k).
template <int KT>
__device__ void topk_block_merge(TKey (&lst)[KT], int k, TKey* out) {
  __shared__ TKey warp_best[32];
  __shared__ TKey best;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int r = 0; r < k; ++r) {
    TKey v = warp_max_key(lst[0]);
    if (lane == 0) warp_best[wid] = v;
    __syncthreads();
    if (wid == 0) {
      TKey u = lane < nw ? warp_best[lane] : key_zero();
      u = warp_max_key(u);
      if (lane == 0) best = u;
    }
    __syncthreads();
    const TKey b = best;
    if (threadIdx.x == 0) out[r] = b;
    if (b.a | b.b) {
      if (key_eq(lst[0], b)) {
#pragma unroll
        for (int i = 0; i + 1 < KT; ++i) lst[i] = lst[i + 1];
        lst[KT - 1] = key_zero();
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ TKey topk_key(double mag, unsigned int idx) {
  return TKey{(unsigned long long)__double_as_longlong(mag), 0xFFFFFFFFu - idx};
}

template <int KT>
__global__ void __launch_bounds__(256) topk_partial_kernel(const void* __restrict__ values, int is_double,
                                                           long long length, int k, int nchunk,
                                                           TKey* __restrict__ cand) {
  const int b = blockIdx.y, ch = blockIdx.x;
  const long long per = (length + nchunk - 1) / nchunk;
  const long long lo = (long long)ch * per;
  const long long hi = lo + per < length ? lo + per : length;
  TKey lst[KT];
#pragma unroll
  for (int i = 0; i < KT; ++i) lst[i] = key_zero();
  if (is_double) {
    const double2* v = (const double2*)values + (long long)b * length;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const double2 x = v[i];
      topk_insert<KT>(lst, topk_key(hypot(x.x, x.y), (unsigned int)i));
    }
  } else {
    const float2* v = (const float2*)values + (long long)b * length;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const float2 x = v[i];
      topk_insert<KT>(lst, topk_key(hypot((double)x.x, (double)x.y), (unsigned int)i));
    }
  }
  topk_block_merge<KT>(lst, k, cand + ((long long)b * nchunk + ch) * k);
}

// Phase 2: one CTA per snapshot; k rounds, each a block-wide argmax over the candidates
// strictly below the previous winner (keys are unique: the index is part of the key).  No
// per-thread lists: the candidate set (chunks x k) is re-scanned each round.
__global__ void __launch_bounds__(256) topk_merge_kernel(const TKey* __restrict__ cand, int ncand, int k,
                                                         int* __restrict__ idx, float* __restrict__ mag) {
  __shared__ TKey warp_best[32];
  __shared__ TKey best;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const TKey* c = cand + (long long)b * ncand;
  TKey bound{~0ull, ~0u};                 // exclusive upper bound (above every finite key)
  for (int r = 0; r < k; ++r) {
    TKey v = key_zero();
    for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
      const TKey x = c[i];
      if (key_gt(bound, x) && key_gt(x, v)) v = x;
    }
    v = warp_max_key(v);
    if (lane == 0) warp_best[wid] = v;
    __syncthreads();
    if (wid == 0) {
      TKey u = lane < nw ? warp_best[lane] : key_zero();
      u = warp_max_key(u);
      if (lane == 0) best = u;
    }
    __syncthreads();
    const TKey w = best;
    if (threadIdx.x == 0) {
      idx[(long long)b * k + r] = (int)(0xFFFFFFFFu - w.b);
      if (mag) mag[(long long)b * k + r] = (float)__longlong_as_double((long long)w.a);
    }
    bound = w;
    __syncthreads();
  }
}

}  // namespace bccb
