// Per-snapshot top-k peak selection (K6 in SURVEY.md).
//
// Order = extract_support's (reference: pkg/src/bccblasso/solvers.py:494-499): descending
// |c|, ties to the lower flat index (stable argsort of -|c|).  Encoded in one 64-bit key
//     key = (float_bits(|c|) << 32) | (0xFFFFFFFF - index)
// so "largest key" is exactly that order (|c| >= 0 => IEEE bits order like integers).
// Key 0 is a sentinel below every real key.
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

template <int KT>
__device__ __forceinline__ void topk_insert(unsigned long long (&lst)[KT], unsigned long long key) {
  if (key <= lst[KT - 1]) return;
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    if (key > lst[i]) {
      const unsigned long long t = lst[i];
      lst[i] = key;
      key = t;
    }
  }
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// k rounds of block argmax over the per-thread sorted lists; writes winners to out[0..k).
template <int KT>
__device__ void topk_block_merge(unsigned long long (&lst)[KT], int k, unsigned long long* out) {
  __shared__ unsigned long long warp_best[32];
  __shared__ unsigned long long best;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int r = 0; r < k; ++r) {
    unsigned long long v = warp_max_u64(lst[0]);
    if (lane == 0) warp_best[wid] = v;
    __syncthreads();
    if (wid == 0) {
      unsigned long long u = lane < nw ? warp_best[lane] : 0ull;
      u = warp_max_u64(u);
      if (lane == 0) best = u;
    }
    __syncthreads();
    const unsigned long long b = best;
    if (threadIdx.x == 0) out[r] = b;
    if (b != 0ull && lst[0] == b) {
#pragma unroll
      for (int i = 0; i + 1 < KT; ++i) lst[i] = lst[i + 1];
      lst[KT - 1] = 0ull;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ unsigned long long topk_key(float mag, unsigned int idx) {
  return ((unsigned long long)__float_as_uint(mag) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
}

template <int KT>
__global__ void __launch_bounds__(256) topk_partial_kernel(const void* __restrict__ values, int is_double,
                                                           long long length, int k, int nchunk,
                                                           unsigned long long* __restrict__ cand) {
  const int b = blockIdx.y, ch = blockIdx.x;
  const long long per = (length + nchunk - 1) / nchunk;
  const long long lo = (long long)ch * per;
  const long long hi = lo + per < length ? lo + per : length;
  unsigned long long lst[KT];
#pragma unroll
  for (int i = 0; i < KT; ++i) lst[i] = 0ull;
  if (is_double) {
    const double2* v = (const double2*)values + (long long)b * length;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const double2 x = v[i];
      const float m = (float)sqrt(x.x * x.x + x.y * x.y);
      topk_insert<KT>(lst, topk_key(m, (unsigned int)i));
    }
  } else {
    const float2* v = (const float2*)values + (long long)b * length;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const float2 x = v[i];
      const float m = (float)sqrt((double)x.x * x.x + (double)x.y * x.y);
      topk_insert<KT>(lst, topk_key(m, (unsigned int)i));
    }
  }
  topk_block_merge<KT>(lst, k, cand + ((long long)b * nchunk + ch) * k);
}

template <int KT>
__global__ void __launch_bounds__(256) topk_merge_kernel(const unsigned long long* __restrict__ cand,
                                                         int ncand, int k, int* __restrict__ idx,
                                                         float* __restrict__ mag) {
  __shared__ unsigned long long res[64];
  const int b = blockIdx.x;
  unsigned long long lst[KT];
#pragma unroll
  for (int i = 0; i < KT; ++i) lst[i] = 0ull;
  const unsigned long long* c = cand + (long long)b * ncand;
  for (int i = threadIdx.x; i < ncand; i += blockDim.x) topk_insert<KT>(lst, c[i]);
  topk_block_merge<KT>(lst, k, res);
  __syncthreads();
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const unsigned long long key = res[r];
    idx[(long long)b * k + r] = (int)(0xFFFFFFFFu - (unsigned int)(key & 0xFFFFFFFFull));
    if (mag) mag[(long long)b * k + r] = __uint_as_float((unsigned int)(key >> 32));
  }
}

}  // namespace bccb
