// Self-test of the tcgen05 primitives in tcgen05.cuh (built as libbccb_tcprobe.so, used only by
// tests/test_gpu_tc.py): one CTA of 128 threads computes D = A . B^T with kind::tf32 MMAs,
// A (128 x 8k) and B (N x 8k) staged in the canonical K-major no-swizzle layout, D (128 x N)
// read back from TMEM with tcgen05.ld.  passes = 1: plain tf32 product; passes = 3: the
// hi/lo split product A_hi B_hi + A_lo B_hi + A_hi B_lo used by the band engine.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tcgen05.cuh"

using namespace bccb;

template <int N>
__global__ void __launch_bounds__(128, 1) tc_probe_kernel(const float* A, const float* B, float* D, int ksteps,
                                                          int passes) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int M = 128;
  // per K step: A_hi, A_lo (M x 8 each, 4 KB), B_hi, B_lo (N x 8 each)
  const int a_bytes = M * 32, b_bytes = N * 32;
  const int step_bytes = 2 * a_bytes + 2 * b_bytes;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  const int K = 8 * ksteps;
  for (int ks = 0; ks < ksteps; ++ks) {
    unsigned char* base = smem + ks * step_bytes;
    for (int i = tid; i < M * 8; i += 128) {
      const int r = i / 8, k = i % 8;
      float hi, lo;
      tc::split_tf32(A[r * K + ks * 8 + k], hi, lo);
      *reinterpret_cast<float*>(base + tc::km_off(r, k)) = hi;
      *reinterpret_cast<float*>(base + a_bytes + tc::km_off(r, k)) = lo;
    }
    for (int i = tid; i < N * 8; i += 128) {
      const int r = i / 8, k = i % 8;
      float hi, lo;
      tc::split_tf32(B[r * K + ks * 8 + k], hi, lo);
      *reinterpret_cast<float*>(base + 2 * a_bytes + tc::km_off(r, k)) = hi;
      *reinterpret_cast<float*>(base + 2 * a_bytes + b_bytes + tc::km_off(r, k)) = lo;
    }
  }
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  if (tid < 32) tc::tmem_alloc(&tmem_base, N < 32 ? 32 : N);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    constexpr uint32_t idesc = tc::idesc_tf32<M, N>();
    int acc = 0;
    for (int ks = 0; ks < ksteps; ++ks) {
      unsigned char* base = smem + ks * step_bytes;
      const uint64_t ahi = tc::desc_kmajor(base, tc::KM_LBO, tc::KM_SBO);
      const uint64_t alo = tc::desc_kmajor(base + a_bytes, tc::KM_LBO, tc::KM_SBO);
      const uint64_t bhi = tc::desc_kmajor(base + 2 * a_bytes, tc::KM_LBO, tc::KM_SBO);
      const uint64_t blo = tc::desc_kmajor(base + 2 * a_bytes + b_bytes, tc::KM_LBO, tc::KM_SBO);
      tc::mma_tf32(tmem, ahi, bhi, idesc, acc++);
      if (passes == 3) {
        tc::mma_tf32(tmem, alo, bhi, idesc, 1);
        tc::mma_tf32(tmem, ahi, blo, idesc, 1);
      }
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  const int warp = tid >> 5, lane = tid & 31;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) D[(warp * 32 + lane) * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (tid < 32) tc::tmem_dealloc(tmem, N < 32 ? 32 : N);
}

extern "C" int bccb_tc_probe(const float* A, const float* B, float* D, int n, int ksteps, int passes,
                             void* stream) {
  const int smem = ksteps * (2 * 128 * 32 + 2 * n * 32);
  cudaStream_t st = (cudaStream_t)stream;
#define PROBE_CASE(N_)                                                                              \
  if (n == N_) {                                                                                    \
    cudaFuncSetAttribute(tc_probe_kernel<N_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);   \
    tc_probe_kernel<N_><<<1, 128, smem, st>>>(A, B, D, ksteps, passes);                            \
    return (int)cudaGetLastError();                                                                 \
  }
  PROBE_CASE(32) PROBE_CASE(64) PROBE_CASE(128) PROBE_CASE(256)
#undef PROBE_CASE
  return -1;
}
