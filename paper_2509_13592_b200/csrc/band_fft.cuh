// Band-limited 1D DFT engine for the BCCB Gram operator (sm_100a).
//
// The reference applies the Gram operator as ifft2(eig_t * fft2(x)) with numpy's
// pocketfft (reference: pkg/src/bccblasso/bccb.py:113-125).  For the Gram of a
// sparse array the spectrum eig_t is supported on the occupied corner
// [0,M1) x [0,M2) (reference pin: pkg/tests/test_bccb.py:116-125), so every 1D
// pass only needs a BAND of K outputs (forward) or K inputs (inverse) out of N.
//
// Decomposition of one length-N line (N = KP * R, band K = KP * Mo):
//   position n = R*r + s      (r < KP: register index, s < R: thread in the line team)
//   X[j + KP*m] = sum_s  w_R^{s m} * w_N^{s j} * DFT_KP( x[R*r + s] )[j]
//   x[R*r + s]  = IDFT_KP_r( w_N^{-s j} * sum_m X[j + KP*m] * w_R^{-s m} )
// Level 1 (the KP-point DFT) runs fully unrolled in registers; level 2 is an
// R-term reduction (forward) or broadcast (inverse) through shared memory.
// With K << N (K1/L1 = 1/32 at config 5) this is far cheaper than a full FFT
// and keeps every HBM access 128-bit / coalesced (lanes own consecutive s).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bccb {

constexpr int KP_MAX = 32;

// Forward 64th roots of unity: c_roots64[t] = exp(-2 pi i t / 64).  Filled once
// per device by the host (plan creation); indexed with compile-time constants so
// every access becomes a constant-bank operand of the FFMA.  (Single translation
// unit: the library is built from bccb_capi.cu alone, no -rdc needed.)
__constant__ float2 c_roots64[64];

template <int P> struct Log2 { static constexpr int v = Log2<P / 2>::v + 1; };
template <> struct Log2<1> { static constexpr int v = 0; };

__host__ __device__ constexpr int bit_reverse(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r = (r << 1) | ((x >> i) & 1);
  return r;
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
// acc += a * b
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
  return acc;
}

// In-register radix-2 DIT DFT of size P (P divides 64), natural order in/out.
// INV=false: A[j] = sum_r a[r] e^{-2 pi i r j / P};  INV=true: e^{+...} (unnormalised).
template <int P, bool INV>
__device__ __forceinline__ void reg_dft(float2 (&a)[P]) {
  constexpr int LG = Log2<P>::v;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const int j = bit_reverse(i, LG);
    if (j > i) {
      const float2 t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
#pragma unroll
  for (int half = 1; half < P; half <<= 1) {
#pragma unroll
    for (int k = 0; k < half; ++k) {
      const int t = k * (64 / (2 * half));
#pragma unroll
      for (int i = 0; i < P; i += 2 * half) {
        const float2 u = a[i + k];
        float2 v = a[i + k + half];
        if (t == 16) {
          // w = -i (forward) / +i (inverse)
          v = INV ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
        } else if (t != 0) {
          float2 w = c_roots64[t];
          if (INV) w.y = -w.y;
          v = cmul(v, w);
        }
        a[i + k] = make_float2(u.x + v.x, u.y + v.y);
        a[i + k + half] = make_float2(u.x - v.x, u.y - v.y);
      }
    }
  }
}

// Runtime geometry of one axis (built on the host, see bccb_capi.cu: make_axis).
struct Axis {
  int N;      // line length (L1 for rows, L2 for columns)
  int K;      // band (multiple of KP, <= N)
  int KP;     // register DFT size (compile-time copy in the kernels)
  int R;      // N / KP: threads per line team
  int Mo;     // K / KP
  int pitch;  // shared-memory row pitch for the level-2 transpose (odd)
  const float2* tw1;  // [KP][R]  w_N^{s j}
  const float2* tw2;  // [Mo][R]  w_R^{s m}
};

// Level-2 forward, part 1: thread s scatters T[j] = A[j] * w_N^{s j} into the
// line's transpose buffer S[j][s] (pitch = axis.pitch, odd => conflict-free reads).
template <int KP>
__device__ __forceinline__ void band_fwd_scatter(const float2 (&A)[KP], int s, const Axis& ax,
                                                 float2* __restrict__ S) {
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const float2 w = __ldg(ax.tw1 + j * ax.R + s);
    S[j * ax.pitch + s] = cmul(A[j], w);
  }
}

// Level-2 forward, part 2: band output o = j + KP*m of a line from its S buffer.
__device__ __forceinline__ float2 band_fwd_output(const float2* __restrict__ S, int o, int KP,
                                                  const Axis& ax) {
  const int j = o % KP;
  const int m = o / KP;
  const float2* row = S + j * ax.pitch;
  float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
  const int R = ax.R;
  if (m == 0) {
    int s = 0;
#pragma unroll 4
    for (; s + 1 < R; s += 2) {
      acc0 = cadd(acc0, row[s]);
      acc1 = cadd(acc1, row[s + 1]);
    }
    if (s < R) acc0 = cadd(acc0, row[s]);
  } else {
    const float2* tw = ax.tw2 + m * R;
    int s = 0;
#pragma unroll 4
    for (; s + 1 < R; s += 2) {
      acc0 = cfma(row[s], __ldg(tw + s), acc0);
      acc1 = cfma(row[s + 1], __ldg(tw + s + 1), acc1);
    }
    if (s < R) acc0 = cfma(row[s], __ldg(tw + s), acc0);
  }
  return cadd(acc0, acc1);
}

// Level-2 inverse + level-1 inverse DFT: thread s of a line team turns the K band
// values Y (shared memory, one line) into its KP outputs g[r] = x[R*r + s]
// (unnormalised inverse).
template <int KP>
__device__ __forceinline__ void band_inverse(const float2* __restrict__ Y, int s, const Axis& ax,
                                             float2 (&g)[KP]) {
  if (ax.Mo == 1) {
#pragma unroll
    for (int j = 0; j < KP; ++j) g[j] = cmulc(Y[j], __ldg(ax.tw1 + j * ax.R + s));
  } else {
#pragma unroll
    for (int j = 0; j < KP; ++j) g[j] = Y[j];
    for (int m = 1; m < ax.Mo; ++m) {
      const float2 w2 = __ldg(ax.tw2 + m * ax.R + s);
#pragma unroll
      for (int j = 0; j < KP; ++j) {
        const float2 t = cmulc(Y[j + KP * m], w2);
        g[j] = cadd(g[j], t);
      }
    }
#pragma unroll
    for (int j = 0; j < KP; ++j) g[j] = cmulc(g[j], __ldg(ax.tw1 + j * ax.R + s));
  }
  reg_dft<KP, true>(g);
}

}  // namespace bccb
