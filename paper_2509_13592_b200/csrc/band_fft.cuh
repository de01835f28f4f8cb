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
//
// The engine is generic over the complex type: float2 (FISTA / ISTA / matvec) or
// double2 (ADMM, whose dual grows like t*|q| in the degenerate config-3 regime and
// cancels against the band correction — see DESIGN.md "precision").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bccb {

constexpr int KP_MAX = 32;     // register DFT size cap, complex64
constexpr int KP_MAX_D = 16;   // register DFT size cap, complex128

// Forward 64th roots of unity exp(-2 pi i t / 64).  Filled once per device by the host;
// indexed with compile-time constants so each access is a constant-bank operand.
// (Single translation unit: the library is built from bccb_capi.cu alone, no -rdc.)
__constant__ float2 c_roots64[64];
__constant__ double2 c_roots64d[64];

template <int P> struct Log2 { static constexpr int v = Log2<P / 2>::v + 1; };
template <> struct Log2<1> { static constexpr int v = 0; };

__host__ __device__ constexpr int bit_reverse(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r = (r << 1) | ((x >> i) & 1);
  return r;
}

// ---- complex helpers (float2 / double2 overloads)
__device__ __forceinline__ float2 cmake(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 cmake(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// acc += a * b
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ float2 to_c(float2 v, float2) { return v; }
__device__ __forceinline__ double2 to_c(float2 v, double2) { return make_double2(v.x, v.y); }
__device__ __forceinline__ double2 to_c(double2 v, double2) { return v; }
__device__ __forceinline__ float2 to_c(double2 v, float2) { return make_float2((float)v.x, (float)v.y); }

template <typename C> __device__ __forceinline__ C root64(int t);
template <> __device__ __forceinline__ float2 root64<float2>(int t) { return c_roots64[t]; }
template <> __device__ __forceinline__ double2 root64<double2>(int t) { return c_roots64d[t]; }

// In-register radix-2 DIT DFT of size P (P divides 64), natural order in/out.
// INV=false: A[j] = sum_r a[r] e^{-2 pi i r j / P};  INV=true: e^{+...} (unnormalised).
template <int P, bool INV, typename C>
__device__ __forceinline__ void reg_dft(C (&a)[P]) {
  constexpr int LG = Log2<P>::v;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const int j = bit_reverse(i, LG);
    if (j > i) {
      const C t = a[i];
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
        const C u = a[i + k];
        C v = a[i + k + half];
        if (t == 16) {
          // w = -i (forward) / +i (inverse)
          v = INV ? cmake(-v.y, v.x) : cmake(v.y, -v.x);
        } else if (t != 0) {
          C w = root64<C>(t);
          if (INV) w.y = -w.y;
          v = cmul(v, w);
        }
        a[i + k] = cadd(u, v);
        a[i + k + half] = csub(u, v);
      }
    }
  }
}

// Screened inverse register DFT (complex64, P = 16 or 32): a radix-4 decimation-in-frequency
// first stage splits the P outputs into four residue classes r = 4p + q, each the (P/4)-point
// inverse DFT of u_q[l] = W_P^{+ql} * sum_i a[(P/4) i + l] (+i)^{qi}.  Parseval bounds every
// output of class q: |x[4p + q]|^2 <= (P/4) * sum_l |u_q[l]|^2, so when that energy is below
// the soft threshold for all 32 lanes of the warp (and the class holds no live state: `live`
// has a bit per register slot), the class's twiddles, sub-DFT and per-point tests are skipped:
// its points provably stay exactly zero (the bound carries a 2^-10 margin over the per-point
// fp32 test `|g|^2 < kap2_lo`, far above fp32 rounding of the skipped stages).  Returns the
// per-lane mask of slots proven below the threshold (all lanes agree on skipped classes);
// a[] holds x in natural order for the computed classes and unspecified values for skipped
// ones.  thr_scale <= 0 disables skipping (same arithmetic, every class computed).
template <int P>
__device__ __forceinline__ unsigned reg_idft_screened(float2 (&a)[P], float kap2_lo, float thr_scale, unsigned live,
                                                      bool active) {
  static_assert(P == 16 || P == 32, "screened inverse DFT: P = 16 or 32");
  constexpr int Q = P / 4;
  float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int l = 0; l < Q; ++l) {
    const float2 s02 = cadd(a[l], a[2 * Q + l]), d02 = csub(a[l], a[2 * Q + l]);
    const float2 s13 = cadd(a[Q + l], a[3 * Q + l]), d13 = csub(a[Q + l], a[3 * Q + l]);
    a[l] = cadd(s02, s13);
    a[2 * Q + l] = csub(s02, s13);
    a[Q + l] = make_float2(d02.x - d13.y, d02.y + d13.x);       // d02 + i d13
    a[3 * Q + l] = make_float2(d02.x + d13.y, d02.y - d13.x);   // d02 - i d13
#pragma unroll
    for (int q = 0; q < 4; ++q) e[q] = fmaf(a[q * Q + l].x, a[q * Q + l].x, fmaf(a[q * Q + l].y, a[q * Q + l].y, e[q]));
  }
  const float thr = kap2_lo * thr_scale;     // thr_scale = (1 - 2^-10) / Q, or <= 0: never skip
  unsigned ok = 0u;
#pragma unroll
  for (int q = 0; q < 4; ++q) ok |= ((e[q] < thr) || !active ? 1u : 0u) << q;
  ok = __reduce_and_sync(0xffffffffu, ok);
  constexpr unsigned ALL = P >= 32 ? 0xffffffffu : ((1u << P) - 1u);
  unsigned pass = 0u;
  float2 o[P];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    constexpr unsigned CLS = 0x11111111u;
    const unsigned gm = (CLS << q) & ALL;
    float2 v[Q];
#pragma unroll
    for (int l = 0; l < Q; ++l) v[l] = a[q * Q + l];
    if (((ok >> q) & 1u) && !(live & gm)) {
      pass |= gm;
    } else {
#pragma unroll
      for (int l = 1; l < Q; ++l) {
        const int t = (q * l * (64 / P)) % 64;   // W_P^{+ql} = conj(root64(t))
        if (t == 0) {
        } else if (t == 16) {
          v[l] = make_float2(-v[l].y, v[l].x);
        } else if (t == 32) {
          v[l] = make_float2(-v[l].x, -v[l].y);
        } else if (t == 48) {
          v[l] = make_float2(v[l].y, -v[l].x);
        } else {
          v[l] = cmulc(v[l], c_roots64[t]);
        }
      }
      reg_dft<Q, true>(v);
#pragma unroll
      for (int p = 0; p < Q; ++p)
        pass |= (fmaf(v[p].x, v[p].x, v[p].y * v[p].y) < kap2_lo ? 1u : 0u) << (4 * p + q);
    }
#pragma unroll
    for (int p = 0; p < Q; ++p) o[4 * p + q] = v[p];
  }
#pragma unroll
  for (int r = 0; r < P; ++r) a[r] = o[r];
  return pass;
}

// Runtime geometry of one axis at one precision (built on the host: make_axis).
template <typename C>
struct AxisT {
  int N;      // line length (L1 for rows, L2 for columns)
  int K;      // band (multiple of KP, <= N)
  int KP;     // register DFT size (compile-time copy in the kernels)
  int R;      // N / KP: threads per line team
  int Mo;     // K / KP
  int pitch;  // shared-memory row pitch for the level-2 transpose (odd)
  const C* tw1;  // [KP][R]  w_N^{s j}
  const C* tw2;  // [Mo][R]  w_R^{s m}
};

// Level-2 forward, part 1: thread s scatters T[j] = A[j] * w_N^{s j} into the
// line's transpose buffer S[j][s] (odd pitch => conflict-free reads in part 2).
template <int KP, typename C>
__device__ __forceinline__ void band_fwd_scatter(const C (&A)[KP], int s, const AxisT<C>& ax,
                                                 C* __restrict__ S) {
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const C w = __ldg(ax.tw1 + j * ax.R + s);
    S[j * ax.pitch + s] = cmul(A[j], w);
  }
}

// Level-2 forward, part 2: band output o = j + KP*m of a line from its S buffer, summed over
// the thread range s in [s0, s1) (the whole line: 0, R).  Four independent accumulators keep
// the dependent-add chain at a quarter of the range.
template <typename C>
__device__ __forceinline__ C band_fwd_partial(const C* __restrict__ S, int o, int KP, const AxisT<C>& ax, int s0,
                                              int s1) {
  const int j = o % KP;
  const int m = o / KP;
  const C* row = S + j * ax.pitch;
  const C zero = cmake(decltype(C::x)(0), decltype(C::x)(0));
  C acc0 = zero, acc1 = zero, acc2 = zero, acc3 = zero;
  int s = s0;
  if (m == 0) {
#pragma unroll 2
    for (; s + 3 < s1; s += 4) {
      acc0 = cadd(acc0, row[s]);
      acc1 = cadd(acc1, row[s + 1]);
      acc2 = cadd(acc2, row[s + 2]);
      acc3 = cadd(acc3, row[s + 3]);
    }
    for (; s < s1; ++s) acc0 = cadd(acc0, row[s]);
  } else {
    const C* tw = ax.tw2 + m * ax.R;
#pragma unroll 2
    for (; s + 3 < s1; s += 4) {
      acc0 = cfma(row[s], __ldg(tw + s), acc0);
      acc1 = cfma(row[s + 1], __ldg(tw + s + 1), acc1);
      acc2 = cfma(row[s + 2], __ldg(tw + s + 2), acc2);
      acc3 = cfma(row[s + 3], __ldg(tw + s + 3), acc3);
    }
    for (; s < s1; ++s) acc0 = cfma(row[s], __ldg(tw + s), acc0);
  }
  return cadd(cadd(acc0, acc1), cadd(acc2, acc3));
}

template <typename C>
__device__ __forceinline__ C band_fwd_output(const C* __restrict__ S, int o, int KP, const AxisT<C>& ax) {
  return band_fwd_partial(S, o, KP, ax, 0, ax.R);
}

// Level-2 inverse + level-1 inverse DFT: thread s of a line team turns the K band
// values Y (shared memory, one line) into its KP outputs g[r] = x[R*r + s]
// (unnormalised inverse).
template <int KP, typename C>
__device__ __forceinline__ void band_inverse(const C* __restrict__ Y, int s, const AxisT<C>& ax,
                                             C (&g)[KP]) {
  if (ax.Mo == 1) {
#pragma unroll
    for (int j = 0; j < KP; ++j) g[j] = cmulc(Y[j], __ldg(ax.tw1 + j * ax.R + s));
  } else {
#pragma unroll
    for (int j = 0; j < KP; ++j) g[j] = Y[j];
    for (int m = 1; m < ax.Mo; ++m) {
      const C w2 = __ldg(ax.tw2 + m * ax.R + s);
#pragma unroll
      for (int j = 0; j < KP; ++j) g[j] = cadd(g[j], cmulc(Y[j + KP * m], w2));
    }
#pragma unroll
    for (int j = 0; j < KP; ++j) g[j] = cmulc(g[j], __ldg(ax.tw1 + j * ax.R + s));
  }
  reg_dft<KP, true>(g);
}

}  // namespace bccb
