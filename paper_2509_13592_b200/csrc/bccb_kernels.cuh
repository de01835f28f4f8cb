// Pass kernels of the fused BCCB Gram iteration (sm_100a).
//
// One solver iteration = two launches:
//   rows_*_kernel (pass A, one L1-line per team): band inverse of V -> g, fused solver
//                 epilogue (gradient step + complex soft-threshold + FISTA momentum or
//                 ADMM z/v update + non-finite flag), band forward of the next operator
//                 input -> U.
//   cols_kernel   (pass B, one L2-line per (snapshot, k1) team): band forward of U,
//                 spectral multiply-add  Y = D*X + P*Bhat  on the K1 x K2 box, band
//                 inverse -> V.
// Intermediates U, V are [B][K1][L2] (transposed so pass-B lines are contiguous);
// Bhat / D / P boxes are [.][K1][K2].  The full-grid state never leaves its
// [B][L2][L1] layout.  See DESIGN.md for the byte model.
#pragma once
#include <cooperative_groups.h>

#include <type_traits>

#include "band_fft.cuh"
#include "tcgen05.cuh"

namespace bccb {

// Programmatic dependent launch (PDL).  The per-pass kernels are launched with the
// programmatic-stream-serialization attribute (bccb_capi.cu launch_pass), so the next pass's
// CTAs are scheduled while this pass drains.  griddepcontrol.wait blocks until the previous
// grid on the stream has completed and its writes are visible (a no-op without the
// attribute); nothing before it may touch memory another pass writes.  With c_pdl_trigger
// set, each CTA then releases its dependents at once.
__constant__ int c_pdl_trigger;
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (c_pdl_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

struct Geo {
  int L1, L2;
  long long rows;  // total lines in this launch
  int TR;          // lines per CTA
  int do_inv, do_fwd;
  int screen = 0;  // rows passes, BCCB_SCREEN bits: 1 = energy-screened register IDFT (CUDA-core
                   // engines, default), 2 = TMEM energy screen of the tensor-core tiles (off by
                   // default: a tile waits for its slowest warp, and a warp that fails the screen
                   // runs screen + full path: 346 vs 358 G gpi/s at config 5, profiles/r2/r2l_*)
  int l2_shift = -1;  // log2(L2) when L2 is a power of two (rows passes: snapshot of a line by shift)
  int dbg = 0;     // BCCB_DEBUG bits: 1 = barrier between tensor-core tiles, 2 = unsplit column sums (4: host, L1 split; 8/16/32/64: timing probes of the TC tile, results invalid)
};

// ------------------------------------------------------------------ epilogues
// Every epilogue provides
//   C load(pos, b)          : operator input x_t from the current state (first pass)
//   ... update/step         : consume g (the ifft2 part) at pos, update the state and
//                             return the next operator input x_{t+1}
// `pos` is the flat index b*L + l2*L1 + l1; `b` the snapshot.

// Plain vectors (matvec / spectrum / synthesis).  update() returns
// out = alpha*x + scale*g; the kernel stores it and optionally reduces max|out|.
template <typename C>
struct EpiVector {
  using R = decltype(C::x);
  const C* __restrict__ in;   // may be null when alpha == 0
  C* __restrict__ out;        // may be null (only maxabs wanted)
  float* __restrict__ maxabs; // may be null
  R alpha, scale;
  __device__ __forceinline__ C load(long long pos, int) const { return in[pos]; }
  __device__ __forceinline__ C update(long long pos, int, C g) const {
    C o = cmake(scale * g.x, scale * g.y);
    if (alpha != R(0)) {
      const C x = in[pos];
      o.x = fma(alpha, x.x, o.x);
      o.y = fma(alpha, x.y, o.y);
    }
    if (out) out[pos] = o;
    return o;
  }
};

// max over lanes that share the same snapshot b, then one atomicMax per group.
// |.| >= 0, so IEEE bit patterns order like unsigned ints (NaN sorts high).
__device__ __forceinline__ void group_atomic_max(float* maxabs, int b, float m) {
  const unsigned act = __activemask();
  const unsigned grp = __match_any_sync(act, b);
  const unsigned v = __reduce_max_sync(grp, __float_as_uint(m));
  if ((threadIdx.x & 31) == (__ffs(grp) - 1)) atomicMax(reinterpret_cast<unsigned int*>(maxabs) + b, v);
}

// ISTA (momentum=false) and FISTA (momentum=true).
// State: c (complex128) and, for FISTA, d = c_t - c_{t-1} (complex64).
// x_t = c_t + beta_t * d_t ;  w = a*x_t + g (+ extra_scale*extra) ;
// c_{t+1} = S_kappa(w) ;  d_{t+1} = c_{t+1} - c_t ;  x_{t+1} = c_{t+1} + beta_{t+1} d_{t+1}.
// reference: pkg/src/bccblasso/solvers.py:245-249 (prox step), 131-145 (soft threshold),
//            311-355 (FISTA loop), 252-291 (ISTA loop), 222-224 (finite check).
struct EpiFista {
  double2* c;
  float2* d;
  const float2* __restrict__ extra;
  const double* __restrict__ tau;  // [B]
  int* first_bad;                  // [B]
  double a, kscale, extra_scale, beta_cur, beta_next;
  int it, momentum;
  // fused objective trace (record_objective): tau_b ||c_{t+1}||_1 is added to
  // trace[b * trace_stride + it] by the rows pass (null: off)
  double* trace;
  long long trace_stride;

  __device__ __forceinline__ float2 load(long long pos, int) const {
    double2 cc = c[pos];
    if (momentum) {
      const float2 dd = d[pos];
      cc.x = __fma_rn(beta_cur, (double)dd.x, cc.x);
      cc.y = __fma_rn(beta_cur, (double)dd.y, cc.y);
    }
    return make_float2((float)cc.x, (float)cc.y);
  }
  __device__ __forceinline__ float2 step(double2 cc, float2 dd, float2 g, float2 e, int b,
                                         double2& cn, float2& dn) const {
    double xr = cc.x, xi = cc.y;
    if (momentum) {
      xr = __fma_rn(beta_cur, (double)dd.x, xr);
      xi = __fma_rn(beta_cur, (double)dd.y, xi);
    }
    double wr = __fma_rn(a, xr, (double)g.x);
    double wi = __fma_rn(a, xi, (double)g.y);
    if (extra) {
      wr = __fma_rn(extra_scale, (double)e.x, wr);
      wi = __fma_rn(extra_scale, (double)e.y, wi);
    }
    if (!isfinite(wr) || !isfinite(wi)) atomicMin(first_bad + b, it);
    const double kap = kscale * tau[b];
    const double m2 = wr * wr + wi * wi;
    if (m2 <= kap * kap) {
      cn.x = 0.0;
      cn.y = 0.0;
    } else {
      const double f = 1.0 - kap / sqrt(m2);
      cn.x = wr * f;
      cn.y = wi * f;
    }
    if (momentum) {
      dn.x = (float)(cn.x - cc.x);
      dn.y = (float)(cn.y - cc.y);
      const double nx = __fma_rn(beta_next, (double)dn.x, cn.x);
      const double ny = __fma_rn(beta_next, (double)dn.y, cn.y);
      return make_float2((float)nx, (float)ny);
    }
    return make_float2((float)cn.x, (float)cn.y);
  }
};

// ADMM (complex128 engine): state z and v both complex128 (z - v cancels when the threshold is
// small and z ~ c + v, so z needs the dual's precision).
// u = z - v is the operator input; c = a*u + g (+extra); z' = S_kappa(c + v);
// v' = v + (c - z'); u' = z' - v'.   reference: pkg/src/bccblasso/solvers.py:385-448.
struct EpiAdmm {
  double2* z;
  double2* v;
  double2* c_out;                  // optional: c of this iteration (last iteration only)
  const float2* __restrict__ extra;
  const double* __restrict__ tau;
  int* first_bad;
  double a, kscale, extra_scale;
  int it;
  __device__ __forceinline__ double2 load(long long pos, int) const {
    const double2 zz = z[pos];
    const double2 vv = v[pos];
    return make_double2(zz.x - vv.x, zz.y - vv.y);
  }
  __device__ __forceinline__ double2 step(double2 zz, double2 vv, double2 g, float2 e, int b,
                                          double2& zn, double2& vn, double2& cc) const {
    const double ur = zz.x - vv.x, ui = zz.y - vv.y;
    double cr = __fma_rn(a, ur, g.x);
    double ci = __fma_rn(a, ui, g.y);
    if (extra) {
      cr = __fma_rn(extra_scale, (double)e.x, cr);
      ci = __fma_rn(extra_scale, (double)e.y, ci);
    }
    if (!isfinite(cr) || !isfinite(ci)) atomicMin(first_bad + b, it);
    const double sr = cr + vv.x, si = ci + vv.y;
    const double kap = kscale * tau[b];
    const double m2 = sr * sr + si * si;
    double nzr, nzi;
    if (m2 <= kap * kap) {
      nzr = 0.0;
      nzi = 0.0;
    } else {
      const double f = 1.0 - kap / sqrt(m2);
      nzr = sr * f;
      nzi = si * f;
    }
    zn = make_double2(nzr, nzi);
    // v' = v + (c - z'): the reference identity v_t = v_{t-1} + (c_t - z_t)
    // (pkg/tests/test_solvers.py:283-295) holds bitwise in float64.
    vn = make_double2(vv.x + (cr - nzr), vv.y + (ci - nzi));
    cc = make_double2(cr, ci);
    return make_double2(nzr - vn.x, nzi - vn.y);
  }
};

// ------------------------------------------------------------------ pass A helpers
template <typename C>
struct RowsIO {
  const C* __restrict__ V;  // [B][K1][L2]  (inverse input)
  C* __restrict__ U;        // [B][K1][L2]  (forward output)
};

template <typename C>
__device__ __forceinline__ void rows_load_band(const Geo& G, const AxisT<C>& ax, const RowsIO<C>& io,
                                               C* Xs, long long row0) {
  const int K = ax.K, TR = G.TR, XP = K + 1;
  for (int idx = threadIdx.x; idx < TR * K; idx += blockDim.x) {
    const int k = idx / TR, ii = idx - k * TR;
    const long long gr = row0 + ii;
    if (gr < G.rows) {
      const long long b = gr / G.L2, l2 = gr - b * G.L2;
      Xs[ii * XP + k] = io.V[(b * K + k) * G.L2 + l2];
    }
  }
}

template <int KP, typename C>
__device__ __forceinline__ void rows_forward_store(const Geo& G, const AxisT<C>& ax, const RowsIO<C>& io,
                                                   C (&a)[KP], bool active, int ii_self, int s, C* Xs,
                                                   C* S, long long row0) {
  const int K = ax.K, TR = G.TR, XP = K + 1;
  const int SP = KP * ax.pitch;  // per-line transpose buffer size
  if (active) {
    reg_dft<KP, false>(a);
    band_fwd_scatter<KP>(a, s, ax, S + ii_self * SP);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TR * K; idx += blockDim.x) {
    const int ii = idx / K, o = idx - ii * K;
    if (row0 + ii < G.rows) Xs[ii * XP + o] = band_fwd_output(S + ii * SP, o, KP, ax);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TR * K; idx += blockDim.x) {
    const int k = idx / TR, ii = idx - k * TR;
    const long long gr = row0 + ii;
    if (gr < G.rows) {
      const long long b = gr / G.L2, l2 = gr - b * G.L2;
      io.U[(b * K + k) * G.L2 + l2] = Xs[ii * XP + k];
    }
  }
}

// ------------------------------------------------------------------ fused objective trace
// The reference's objective (solvers.py:233-242)
//   f(c) = ||y||^2 - 2 Re<b, c> + Re<c, G c> + tau ||c||_1
// is evaluated for every iterate c_{t+1} without a host round trip.  By Parseval, with
// C = FFT2(c) (unnormalised) on the spectral box that carries both Lambda and FFT2(b):
//   -2 Re<b, c> + <c, G c> = (1/L) sum_box ( Lambda |C|^2 - 2 Re(conj(Bhat) C) ).
// The column pass already forms X = FFT2(x_t) on the box for the FISTA point
// x_t = c_t + beta_t (c_t - c_{t-1}); linearity gives C_t = (X_t + beta_t C_{t-1}) / (1 + beta_t)
// (ISTA: beta = 0, C = X), kept in float64 per box value.  tau ||c||_1 is summed by the rows
// pass over the points its exact float64 update touched (every other point is exactly zero).
struct ObjBox {
  double2* chat;            // [B][K1][K2] C_{t-1} in, C_t out (null: off)
  const double2* lam;       // [K1][K2] eigenvalues on the box (real for a Gram operator)
  const float2* bh;         // [B][K1][K2] FFT2(b) on the box
  double* trace;            // [B][stride]: column `col` receives the quadratic part (null: store only)
  long long stride;
  double beta, inv_L;
  int col, K2;
};

// quadratic part contributed by band value o of column line `line` (= b K1 + k1)
__device__ __forceinline__ double obj_term(const ObjBox& ob, long long line, int o, int K1, float2 x) {
  const long long bi = line * ob.K2 + o;
  double cr = x.x, ci = x.y;
  if (ob.beta != 0.0) {
    const double2 prev = ob.chat[bi];
    const double inv = 1.0 / (1.0 + ob.beta);
    cr = (cr + ob.beta * prev.x) * inv;
    ci = (ci + ob.beta * prev.y) * inv;
  }
  ob.chat[bi] = make_double2(cr, ci);
  if (!ob.trace) return 0.0;
  const double lam = __ldg(&ob.lam[(line % K1) * ob.K2 + o].x);
  const float2 bh = ob.bh[bi];
  return ob.inv_L * (lam * (cr * cr + ci * ci) - 2.0 * ((double)bh.x * cr + (double)bh.y * ci));
}

// sum v over the lanes of the warp that share key `b` and add it to dst[b * stride] once per
// group (every lane of the warp calls this; b < 0: no contribution)
__device__ __forceinline__ void warp_group_add(double* dst, long long stride, long long b, double v) {
  const unsigned grp = __match_any_sync(0xffffffffu, b);
  if (grp == 0xffffffffu) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && b >= 0) atomicAdd(dst + b * stride, v);
  } else if (b >= 0 && v != 0.0) {
    atomicAdd(dst + b * stride, v);
  }
}

// ------------------------------------------------------------------ pass B
template <typename C>
struct ColsIO {
  const C* __restrict__ U;          // [B][K1][L2] forward input (do_fwd)
  C* __restrict__ V;                // [B][K1][L2] inverse output (do_inv)
  const C* __restrict__ D;          // [K1][K2] multiplier (null => identity)
  const C* __restrict__ P;          // [K1][K2] rhs multiplier (null => 1)
  const float2* __restrict__ Bh;    // [B][K1][K2] rhs box, complex64 data (null => none)
  C* __restrict__ box_out;          // [B][K1][K2] (used when !do_inv; may be null)
  int K1;
  ObjBox ob;                        // fused objective trace (ob.chat null: off; complex64 only)
};

// Default band stage of the column pass: Y = D*X + P*Bh from ColsIO.
struct BandMulAdd {};

// Band operands of a thread's first output (idx = threadIdx.x) of the default band stage,
// D[k1][o] and P*Bh: they do not depend on the previous pass, so cols_kernel fetches them
// before its grid-dependency wait.
template <typename C>
struct ColsPre {
  C d, pb;
  bool ok;
};

template <typename C>
__device__ __forceinline__ ColsPre<C> cols_prefetch(const Geo& G, const AxisT<C>& ax, const ColsIO<C>& io,
                                                    long long row0, int TR) {
  ColsPre<C> pre;
  pre.ok = false;
  const int K = ax.K;
  const int idx = threadIdx.x;
  if (idx >= TR * K) return pre;
  const int i2 = idx / K, o = idx - i2 * K;
  const long long g2 = row0 + i2;
  if (g2 >= G.rows) return pre;
  const long long k1 = g2 % io.K1;
  if (io.D) pre.d = __ldg(io.D + k1 * K + o);
  pre.pb = cmake(decltype(C::x)(0), decltype(C::x)(0));
  if (io.Bh) {
    pre.pb = to_c(io.Bh[g2 * K + o], C{});
    if (io.P) pre.pb = cmul(pre.pb, __ldg(io.P + k1 * K + o));
  }
  pre.ok = true;
  return pre;
}

// Column lines [row0, row0 + TR) (line = (snapshot b, column k1): length L2, band K2) processed
// by one CTA of TR * ax.R threads (threads beyond that idle).  Shared by cols_kernel and the
// fused rows kernel.  smem: TR x (K+1) band tile + TR x KP x pitch transpose buffer.
// Op (other than BandMulAdd) replaces the band stage: y = op(line, o, X or 0).
template <int KP, typename C, bool U_GLOBAL = true, typename Op = BandMulAdd>
__device__ __forceinline__ void cols_block(const Geo& G, const AxisT<C>& ax, const ColsIO<C>& io, long long row0,
                                           int TR, C* smem, const Op& op = Op{},
                                           const ColsPre<C>& pre = ColsPre<C>{}, C* part = nullptr) {
  const int R = ax.R, K = ax.K, N = ax.N;
  const int XP = K + 1, SP = KP * ax.pitch;
  const int nthr = TR * R;
  const int tid = threadIdx.x;
  const int ii = tid / R, s = tid - ii * R;
  const long long gr = row0 + ii;
  const bool active = (tid < nthr) && (gr < G.rows);
  C* Xs = smem;
  C* S = smem + TR * XP;
  C a[KP];
  if (G.do_fwd) {
    if (active) {
      const C* line = io.U + gr * N + s;
#pragma unroll
      for (int r = 0; r < KP; ++r) a[r] = U_GLOBAL ? __ldcg(line + (long long)R * r) : line[(long long)R * r];
      reg_dft<KP, false>(a);
      band_fwd_scatter<KP>(a, s, ax, S + ii * SP);
    }
    __syncthreads();
  }
  // Split level-2 forward sums (long lines, few outputs per thread: config 5's column pass has
  // TR*K = 128 outputs of R = 256 terms for 256 threads): NP threads share each output's
  // range of s, the partial sums meet in `part` ([NP][TR*K]) and are added in the band loop.
  const int n_out = TR * K;
  const int NP = (part && G.do_fwd) ? min(4, (int)blockDim.x / n_out) : 1;
  if (NP > 1) {
    for (int idx = tid; idx < NP * n_out; idx += blockDim.x) {
      const int q = idx / n_out, oi = idx - q * n_out;
      const int i2 = oi / K, o = oi - i2 * K;
      part[idx] = band_fwd_partial(S + i2 * SP, o, KP, ax, (q * R) / NP, ((q + 1) * R) / NP);
    }
    __syncthreads();
  }
  auto fwd_value = [&](int i2, int o) {
    if (NP == 1) return band_fwd_output(S + i2 * SP, o, KP, ax);
    C v = part[i2 * K + o];
    for (int q = 1; q < NP; ++q) v = cadd(v, part[q * n_out + i2 * K + o]);
    return v;
  };
  // band values: Y = D*X + P*Bh   (+ the objective's box terms of X when io.ob.chat is set)
  constexpr bool OBJ = std::is_same<C, float2>::value && std::is_same<Op, BandMulAdd>::value;
  long long ob_b = -1;       // snapshot of the running objective sum
  double ob_v = 0.0;
  for (int idx = tid; idx < TR * K; idx += blockDim.x) {
    const int i2 = idx / K, o = idx - i2 * K;
    const long long g2 = row0 + i2;
    if (g2 >= G.rows) continue;
    C y = cmake(decltype(C::x)(0), decltype(C::x)(0));
    if constexpr (std::is_same<Op, BandMulAdd>::value) {
      if (G.do_fwd) y = fwd_value(i2, o);
      if constexpr (OBJ) {
        if (G.do_fwd && io.ob.chat) {
          const long long bb = g2 / io.K1;
          if (bb != ob_b) {
            if (ob_b >= 0 && io.ob.trace && ob_v != 0.0) atomicAdd(io.ob.trace + ob_b * io.ob.stride + io.ob.col, ob_v);
            ob_b = bb;
            ob_v = 0.0;
          }
          ob_v += obj_term(io.ob, g2, o, io.K1, y);
        }
      }
      if (pre.ok && idx == tid) {
        if (G.do_fwd && io.D) y = cmul(y, pre.d);
        Xs[i2 * XP + o] = io.Bh ? cadd(y, pre.pb) : y;
        continue;
      }
      const long long k1 = g2 % io.K1;
      if (G.do_fwd && io.D) y = cmul(y, __ldg(io.D + k1 * K + o));
      if (io.Bh) {
        C bh = to_c(io.Bh[g2 * K + o], C{});
        if (io.P) bh = cmul(bh, __ldg(io.P + k1 * K + o));
        y = cadd(y, bh);
      }
    } else {
      y = op(g2, o, G.do_fwd ? fwd_value(i2, o) : y);
    }
    Xs[i2 * XP + o] = y;
  }
  if constexpr (OBJ) {
    if (G.do_fwd && io.ob.chat && io.ob.trace)
      warp_group_add(io.ob.trace + io.ob.col, io.ob.stride, ob_b, ob_v);
  }
  __syncthreads();
  if (G.do_inv) {
    if (active) {
      band_inverse<KP>(Xs + ii * XP, s, ax, a);
      C* line = io.V + gr * N + s;
#pragma unroll
      for (int r = 0; r < KP; ++r) line[(long long)R * r] = a[r];
    }
  } else {
    for (int idx = tid; idx < TR * K; idx += blockDim.x) {
      const int i2 = idx / K, o = idx - i2 * K;
      const long long g2 = row0 + i2;
      if (g2 < G.rows && io.box_out) io.box_out[g2 * K + o] = Xs[i2 * XP + o];
    }
  }
}

template <int KP, typename C>
__global__ void __launch_bounds__(KP <= 8 ? 1024 : 256) cols_kernel(Geo G, AxisT<C> ax, ColsIO<C> io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const long long row0 = (long long)blockIdx.x * G.TR;
  const ColsPre<C> pre = cols_prefetch(G, ax, io, row0, G.TR);
  pdl_wait();
  // split forward sums when the launch reserved room for them (cols_split_smem)
  C* base = reinterpret_cast<C*>(smem_raw);
  C* part = ((int)blockDim.x >= 2 * G.TR * ax.K && !(G.dbg & 2)) ? base + G.TR * (ax.K + 1) + G.TR * KP * ax.pitch : nullptr;
  cols_block<KP>(G, ax, io, row0, G.TR, base, BandMulAdd{}, pre, part);
}

// Warp-per-line column pass (complex64 streaming axis with R = 32 threads per line and a band
// of K = 32 NSET: config 2's L2 = 256 with KP = 8, the split ADMM's L2 = 512 with KP = 16 and
// K = 64).  The level-2 sums run across the warp instead of through shared memory: each lane
// forms its twiddled products T_s[j] w_32^{s m}; per set of 32 band values a recursive-halving
// reduce-scatter over the 32 lanes leaves band value 32 set + lane on the lane, the band stage
// (D X + P Bh, or the split ADMM's float64 box update Op) runs there, and shuffles broadcast the
// band back for the inverse.  No shared memory and no block barrier: a line's latency chain is
// one warp's.  Same arithmetic per term as cols_block (fp32 products, then sums; only the
// summation order over the 32 lanes differs).
template <int KP, int NSET, typename Op = BandMulAdd>
__global__ void __launch_bounds__(256) cols_warp_kernel(Geo G, AxisT<float2> ax, ColsIO<float2> io, Op op) {
  constexpr int R = 32, K = 32 * NSET, MO = K / KP;
  constexpr bool MULADD = std::is_same<Op, BandMulAdd>::value;
  static_assert(KP * MO == K, "band");
  const int lane = threadIdx.x & 31;
  const long long line = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool live = line < G.rows;
  // loop-invariant operands (before the grid-dependency wait): twiddles and, for D X + P Bh,
  // the lane's band multipliers D[k1][o], P Bh[line][o]
  float2 tw1[KP], tw2[MO];
#pragma unroll
  for (int j = 0; j < KP; ++j) tw1[j] = __ldg(ax.tw1 + j * R + lane);
#pragma unroll
  for (int m = 0; m < MO; ++m) tw2[m] = __ldg(ax.tw2 + m * R + lane);
  float2 d[NSET], pb[NSET];
#pragma unroll
  for (int q = 0; q < NSET; ++q) {
    d[q] = make_float2(1.f, 0.f);
    pb[q] = make_float2(0.f, 0.f);
    if (MULADD && live) {
      const long long k1 = line % io.K1;
      const int o = 32 * q + lane;
      if (io.D) d[q] = __ldg(io.D + k1 * K + o);
      if (io.Bh) {
        pb[q] = io.Bh[line * K + o];
        if (io.P) pb[q] = cmul(pb[q], __ldg(io.P + k1 * K + o));
      }
    }
  }
  pdl_wait();
  if (!live) return;   // whole warps only
  const int N = ax.N;
  float2 x[NSET];
#pragma unroll
  for (int q = 0; q < NSET; ++q) x[q] = make_float2(0.f, 0.f);
  if (G.do_fwd) {
    float2 t[KP];
    const float2* src = io.U + line * N + lane;
#pragma unroll
    for (int r = 0; r < KP; ++r) t[r] = __ldcg(src + R * r);
    reg_dft<KP, false>(t);
#pragma unroll
    for (int j = 0; j < KP; ++j) t[j] = cmul(t[j], tw1[j]);
#pragma unroll
    for (int q = 0; q < NSET; ++q) {
      float2 v[32];   // v[i]: band value o = 32 q + i = j + KP m
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int o = 32 * q + i, j = o % KP, m = o / KP;
        v[i] = m == 0 ? t[j] : cmul(t[j], tw2[m]);
      }
      // reduce-scatter: after the stage of width h the lane keeps the half its bit h selects
#pragma unroll
      for (int h = 16; h >= 1; h >>= 1) {
        const bool upper = (lane & h) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
          const float2 send = upper ? v[i] : v[i + h];
          const float2 keep = upper ? v[i + h] : v[i];
          const float2 recv = make_float2(__shfl_xor_sync(0xffffffffu, send.x, h),
                                          __shfl_xor_sync(0xffffffffu, send.y, h));
          v[i] = cadd(keep, recv);
        }
      }
      x[q] = v[0];
    }
  }
  if constexpr (MULADD) {
    if (G.do_fwd && io.ob.chat) {   // fused objective trace: box terms of this line (one snapshot)
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < NSET; ++q) v += obj_term(io.ob, line, 32 * q + lane, io.K1, x[q]);
      if (io.ob.trace) warp_group_add(io.ob.trace + io.ob.col, io.ob.stride, line / io.K1, v);
    }
  }
  float2 y[NSET];
#pragma unroll
  for (int q = 0; q < NSET; ++q) {
    if constexpr (MULADD) {
      y[q] = (G.do_fwd && io.D) ? cmul(x[q], d[q]) : x[q];
      if (io.Bh) y[q] = cadd(y[q], pb[q]);
      if (!G.do_inv && io.box_out) io.box_out[line * K + 32 * q + lane] = y[q];
    } else {
      y[q] = op(line, 32 * q + lane, x[q]);
    }
  }
  if (!G.do_inv) return;
  // inverse: g_j = IDFT_KP( conj(w_N^{s j}) sum_m Y[j + KP m] conj(w_32^{s m}) )
  float2 g[KP];
#pragma unroll
  for (int j = 0; j < KP; ++j) {
#pragma unroll
    for (int m = 0; m < MO; ++m) {
      const int o = j + KP * m;
      const float2 ym = make_float2(__shfl_sync(0xffffffffu, y[o / 32].x, o % 32),
                                    __shfl_sync(0xffffffffu, y[o / 32].y, o % 32));
      g[j] = m == 0 ? ym : cadd(g[j], cmulc(ym, tw2[m]));
    }
    g[j] = cmulc(g[j], tw1[j]);
  }
  reg_dft<KP, true>(g);
  float2* dst = io.V + line * N + lane;
#pragma unroll
  for (int r = 0; r < KP; ++r) dst[R * r] = g[r];
}

// ------------------------------------------------------------------ pass A kernels
// Generic pass A for plain-vector epilogues.
template <int KP, typename C, typename E = EpiVector<C>>
__global__ void __launch_bounds__(256) rows_vector_kernel(Geo G, AxisT<C> ax, RowsIO<C> io, E epi) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* smem = reinterpret_cast<C*>(smem_raw);
  const int R = ax.R, K = ax.K;
  const int ii = threadIdx.x / R, s = threadIdx.x - ii * R;
  const long long row0 = (long long)blockIdx.x * G.TR;
  const long long gr = row0 + ii;
  const bool active = (ii < G.TR) && (gr < G.rows);
  C* Xs = smem;
  C* S = smem + G.TR * (K + 1);
  C a[KP];
  if (G.do_inv) {
    rows_load_band(G, ax, io, Xs, row0);
    __syncthreads();
    if (active) band_inverse<KP>(Xs + ii * (K + 1), s, ax, a);
  }
  if (active) {
    const long long base = gr * G.L1 + s;
    const int b = (int)(gr / G.L2);
    float mx = 0.f;
#pragma unroll
    for (int r = 0; r < KP; ++r) {
      const long long pos = base + (long long)R * r;
      a[r] = G.do_inv ? epi.update(pos, b, a[r]) : epi.load(pos, b);
      mx = fmaxf(mx, (float)sqrt((double)a[r].x * a[r].x + (double)a[r].y * a[r].y));
    }
    if constexpr (std::is_same<E, EpiVector<C>>::value)
      if (G.do_inv && epi.maxabs) group_atomic_max(epi.maxabs, b, mx);
  }
  if (G.do_fwd) {
    if (G.do_inv) __syncthreads();
    rows_forward_store<KP>(G, ax, io, a, active, ii, s, Xs, S, row0);
  }
}

// Pass A for ISTA / FISTA (complex64 engine) with a software-pipelined state stream:
// the first chunk of state is requested before the band inverse runs (its latency hides
// behind the V-tile load and the inverse DFT), and every later chunk is requested before
// the stores of the current one (state is updated in place).  MINB = CTAs per SM the
// register allocation is capped for.
template <int KP, int CH, int MINB>
__global__ void __launch_bounds__(256, MINB) rows_fista_kernel(Geo G, AxisT<float2> ax, RowsIO<float2> io,
                                                               EpiFista epi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* smem = reinterpret_cast<float2*>(smem_raw);
  pdl_wait();
  const int R = ax.R, K = ax.K;
  const int ii = threadIdx.x / R, s = threadIdx.x - ii * R;
  const long long row0 = (long long)blockIdx.x * G.TR;
  const long long gr = row0 + ii;
  const bool active = (ii < G.TR) && (gr < G.rows);
  float2* Xs = smem;
  float2* S = smem + G.TR * (K + 1);
  float2 a[KP];
  const long long base = gr * G.L1 + s;
  const int b = (int)(gr / G.L2);
  double2 cb[CH];
  float2 db[CH], eb[CH];
  if (active && G.do_inv) {
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const long long pos = base + (long long)R * q;
      cb[q] = epi.c[pos];
      db[q] = epi.momentum ? epi.d[pos] : make_float2(0.f, 0.f);
      eb[q] = epi.extra ? epi.extra[pos] : make_float2(0.f, 0.f);
    }
  }
  if (G.do_inv) {
    rows_load_band(G, ax, io, Xs, row0);
    __syncthreads();
    if (active) band_inverse<KP>(Xs + ii * (K + 1), s, ax, a);
  }
  if (active) {
    if (!G.do_inv) {
#pragma unroll
      for (int r = 0; r < KP; ++r) a[r] = epi.load(base + (long long)R * r, b);
    } else {
#pragma unroll
      for (int r0 = 0; r0 < KP; r0 += CH) {
        double2 cn[CH];
        float2 dn[CH], en[CH];
        if (r0 + CH < KP) {
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const long long pos = base + (long long)R * (r0 + CH + q);
            cn[q] = epi.c[pos];
            dn[q] = epi.momentum ? epi.d[pos] : make_float2(0.f, 0.f);
            en[q] = epi.extra ? epi.extra[pos] : make_float2(0.f, 0.f);
          }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const long long pos = base + (long long)R * (r0 + q);
          double2 cnew;
          float2 dnew;
          a[r0 + q] = epi.step(cb[q], db[q], a[r0 + q], eb[q], b, cnew, dnew);
          epi.c[pos] = cnew;
          if (epi.momentum) epi.d[pos] = dnew;
        }
        if (r0 + CH < KP) {
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            cb[q] = cn[q];
            db[q] = dn[q];
            eb[q] = en[q];
          }
        }
      }
    }
  }
  if (G.do_fwd) {
    if (G.do_inv) __syncthreads();
    rows_forward_store<KP>(G, ax, io, a, active, ii, s, Xs, S, row0);
  }
}

// ---------------------------------------------------------------- specialised pass A (FISTA/ISTA)
// Compile-time line shape: KP (register DFT), R (threads per line), MO (band / KP), so every
// stride and loop bound is a constant.  Rows of a CTA never straddle snapshots (host checks
// L2 % TR == 0), so all per-row scalars are hoisted and indices are 32-bit offsets from
// per-row base pointers.
//
// Zero fast path (bitwise identical to the full update): when c_t = 0 and d_t = 0 the
// operator input is x_t = 0, so w = g exactly; if fp32 |g|^2 is below kappa^2 by more than
// its rounding bound the exact float64 test m2 <= kappa^2 must hold too, giving c_{t+1} = 0,
// d_{t+1} = 0, x_{t+1} = 0 — state unchanged, so its stores are skipped.  After the first
// few dozen iterations ~99% of the iterate is exactly zero (LASSO sparsity).
//
// Zero-segment skipping (ZS): flags[warp] bit r says whether the 32 state elements held by
// the warp's lanes at register slot r may be nonzero.  Clear segments are not read (they are
// exactly zero) and not written while they stay zero; a segment that is (or becomes) nonzero
// is written whole.  zero_segments_kernel writes the skipped zeros back at the end of a run.
struct FistaScalars {
  double kap, a_id, bc;
  int b, it;
  int* first_bad;
};

// Full float64 update of one point (solvers.py:245-249, 131-145, 336-337): returns c_{t+1}
// and d_{t+1} (FISTA).  Out of line to keep the unrolled kernel small: only points with a
// nonzero state or with |g| near / above the threshold take it.
template <bool MOM>
__device__ __noinline__ double2 fista_point_slow(double2 cc, float2 dd, float2 g, const FistaScalars sc,
                                                  float2* dnew) {
  double xr = cc.x, xi = cc.y;
  if (MOM) {
    xr = __fma_rn(sc.bc, (double)dd.x, xr);
    xi = __fma_rn(sc.bc, (double)dd.y, xi);
  }
  const double wr = __fma_rn(sc.a_id, xr, (double)g.x);
  const double wi = __fma_rn(sc.a_id, xi, (double)g.y);
  if (!isfinite(wr + wi)) atomicMin(sc.first_bad + sc.b, sc.it);
  const double m2 = wr * wr + wi * wi;
  double nr = 0.0, ni = 0.0;
  if (!(m2 <= sc.kap * sc.kap)) {
    const double f = 1.0 - sc.kap * rsqrt(m2);
    nr = wr * f;
    ni = wi * f;
  }
  if (MOM) *dnew = make_float2((float)(nr - cc.x), (float)(ni - cc.y));
  return make_double2(nr, ni);
}

// Fused column pass (KP2 > 0): the column work of one snapshot (K1 lines of length L2) is at
// most one CTA's rows work for small grids (config 2: 32 x 256 vs 32 x 256 points), so the last
// rows CTA to finish a snapshot (threadfence + atomic counter) runs that snapshot's column
// lines in place, overlapping other snapshots' rows work and halving the launches.
struct FusedCols {
  ColsIO<float2> io;
  AxisT<float2> ax;
  Geo G;          // column-line geometry (rows = B * K1)
  int* counter;   // [B] arrival counters (monotonic; last arrival when count % cps == 0)
  int cps;        // rows CTAs per snapshot
  int TRc;        // column lines per block pass (divides K1)
  int K1;
};

// Shared-memory twiddle staging of the specialised rows pass: tables of at most 8 KB are
// staged (short-latency LDS instead of L1 round trips, measured +1% at config 2); larger ones
// are read through L1 (a 36 KB table at L1 = 4096 would cost a resident CTA per SM, measured
// -18% at config 5).
// threads per CTA of the tensor-core rows tiles: two line teams.  Single-line tiles (128 threads,
// 4 CTAs per SM, N = KP) measured slower at config 5, 284 vs 330 G gpi/s: the per-tile flag /
// staging / MMA round trip is paid per line (profiles/r2/r2h_*).
__host__ __device__ constexpr int tc_threads(int KP) { return 256; }

template <int KP, int R, int MO, int NTMIN = 256>
struct TileShape {
  static constexpr int NT = R > NTMIN ? R : NTMIN;   // threads per CTA
  static constexpr int TR = NT / R;              // lines per CTA
  static constexpr int K = KP * MO;
  static constexpr int XP = K + 2;   // even: 16-byte aligned band rows (LDS.128 pairs)
  static constexpr int PITCH = (R % 2 == 1) ? R : R + 1;
  static constexpr int SP = KP * PITCH;
  static constexpr bool STAGE_TW = (KP + MO) * R * 8 <= 8192;
};

template <int KP, int R, int MO>
__device__ __forceinline__ void stage_twiddles(const AxisT<float2>& ax, float2* dst, const float2*& tw1s,
                                               const float2*& tw2s) {
  using TS = TileShape<KP, R, MO>;
  tw1s = ax.tw1;
  tw2s = ax.tw2;
  if constexpr (TS::STAGE_TW) {
    float2* t1 = dst;     // [KP][R] then [MO][R]
    float2* t2 = t1 + KP * R;
    for (int i2 = threadIdx.x; i2 < KP * R; i2 += TS::NT) t1[i2] = ax.tw1[i2];
    for (int i2 = threadIdx.x; i2 < MO * R; i2 += TS::NT) t2[i2] = ax.tw2[i2];
    tw1s = t1;
    tw2s = t2;
  }
}

// State policies of the specialised rows tile.  A policy is built per tile (state offset of
// the thread's first point, snapshot b) and defines the per-point state S, its loads and
// stores, the exact float64 update (out of line: only points with a nonzero state or |g| near
// the threshold take it) and the next operator input.  A zero state with fp32 |g|^2 below
// kappa^2 (1 - 2^-18) must stay exactly zero under the update (the zero fast path).
template <bool MOM>
struct FistaPolicy {
  using Args = EpiFista;
  struct S {
    double2 c;
    float2 d;
  };
  double2* cp;
  float2* dp;
  FistaScalars sc;
  float bn;
  __device__ __forceinline__ FistaPolicy(const EpiFista& e, long long off, int b, const double* tau_pre = nullptr) {
    cp = e.c + off;
    dp = MOM ? e.d + off : nullptr;
    sc = FistaScalars{e.kscale * (tau_pre ? *tau_pre : e.tau[b]), e.a, e.beta_cur, b, e.it, e.first_bad};
    bn = (float)e.beta_next;
  }
  // fused objective: |c_{t+1}| of an updated point (float: summed over at most KP points per
  // thread, then in float64 across threads)
  __device__ __forceinline__ static float l1_term(const S& n) {
    return sqrtf((float)(n.c.x * n.c.x + n.c.y * n.c.y));
  }
  __device__ __forceinline__ double kap() const { return sc.kap; }
  __device__ __forceinline__ S load(int o, bool live) const {
    S s;
    s.c = live ? __ldcg(cp + o) : make_double2(0.0, 0.0);
    s.d = (MOM && live) ? __ldcg(dp + o) : make_float2(0.f, 0.f);
    return s;
  }
  __device__ __forceinline__ static bool zero(const S& s) {
    return (s.c.x == 0.0) & (s.c.y == 0.0) & (!MOM | ((s.d.x == 0.f) & (s.d.y == 0.f)));
  }
  __device__ __forceinline__ static S empty() { return S{make_double2(0.0, 0.0), make_float2(0.f, 0.f)}; }
  __device__ __forceinline__ S update(const S& s, float2 g) const {
    S n = empty();
    n.c = fista_point_slow<MOM>(s.c, s.d, g, sc, &n.d);
    return n;
  }
  __device__ __forceinline__ void store(int o, const S& n) const {
    cp[o] = n.c;
    if (MOM) dp[o] = n.d;
  }
  // x_{t+1} = c_{t+1} + beta_{t+1} d_{t+1}
  __device__ __forceinline__ float2 next_x(const S& n) const {
    return MOM ? make_float2(fmaf(bn, n.d.x, (float)n.c.x), fmaf(bn, n.d.y, (float)n.c.y))
               : make_float2((float)n.c.x, (float)n.c.y);
  }
  // x_t = c_t + beta_t d_t (first pass of a run)
  __device__ __forceinline__ float2 first_x(const S& s) const {
    double2 cc = s.c;
    if (MOM) {
      cc.x = __fma_rn(sc.bc, (double)s.d.x, cc.x);
      cc.y = __fma_rn(sc.bc, (double)s.d.y, cc.y);
    }
    return make_float2((float)cc.x, (float)cc.y);
  }
};

// ADMM with the dual split into a spatial part r and a spectral box part vs:
// v = r + IFFT2u(vs).  The column pass accumulates vs in float64 on the box
// (vs' = vs + Cb, Cb = D FFT2(w) + P Bhat - rho/(lam+rho) vs, w = z - r), so the part of the
// dual that grows with t (SURVEY finding 7) never enters a spatial sum; the rows pass sees
// V = IFFT2u(vs') and forms
//   s = a w + r + IFFT2u(vs')   (= c + v),   z' = S_kappa(s),   r' = r + a w - z'
// and the next operator input w' = z' - r'.  reference: pkg/src/bccblasso/solvers.py:403-436.
struct EpiAdmmSplit {
  double2* z;
  double2* r;
  const double* __restrict__ tau;  // [B]
  int* first_bad;                  // [B]
  double a, kscale;
  int it;
};

__device__ __noinline__ void admm_split_point_slow(double2 z, double2 r, float2 g, double a, double kap,
                                                   int* first_bad, int it, double2* zn, double2* rn) {
  const double wr = z.x - r.x, wi = z.y - r.y;
  const double awr = a * wr, awi = a * wi;
  const double sr = (awr + r.x) + (double)g.x, si = (awi + r.y) + (double)g.y;
  if (!isfinite(sr + si)) atomicMin(first_bad, it);
  const double m2 = sr * sr + si * si;
  double nr = 0.0, ni = 0.0;
  if (!(m2 <= kap * kap)) {
    const double f = 1.0 - kap * rsqrt(m2);
    nr = sr * f;
    ni = si * f;
  }
  *zn = make_double2(nr, ni);
  *rn = make_double2((r.x + awr) - nr, (r.y + awi) - ni);
}

struct AdmmSplitPolicy {
  using Args = EpiAdmmSplit;
  struct S {
    double2 z, r;
  };
  double2* zp;
  double2* rp;
  double a, kp;
  int* fb;
  int it;
  __device__ __forceinline__ AdmmSplitPolicy(const EpiAdmmSplit& e, long long off, int b) {
    zp = e.z + off;
    rp = e.r + off;
    a = e.a;
    kp = e.kscale * e.tau[b];
    fb = e.first_bad + b;
    it = e.it;
  }
  __device__ __forceinline__ double kap() const { return kp; }
  __device__ __forceinline__ S load(int o, bool live) const {
    S s;
    s.z = live ? __ldcg(zp + o) : make_double2(0.0, 0.0);
    s.r = live ? __ldcg(rp + o) : make_double2(0.0, 0.0);
    return s;
  }
  __device__ __forceinline__ static bool zero(const S& s) {
    return (s.z.x == 0.0) & (s.z.y == 0.0) & (s.r.x == 0.0) & (s.r.y == 0.0);
  }
  __device__ __forceinline__ static S empty() { return S{make_double2(0.0, 0.0), make_double2(0.0, 0.0)}; }
  __device__ __forceinline__ S update(const S& s, float2 g) const {
    S n;
    admm_split_point_slow(s.z, s.r, g, a, kp, fb, it, &n.z, &n.r);
    return n;
  }
  __device__ __forceinline__ void store(int o, const S& n) const {
    zp[o] = n.z;
    rp[o] = n.r;
  }
  __device__ __forceinline__ float2 next_x(const S& n) const {
    return make_float2((float)(n.z.x - n.r.x), (float)(n.z.y - n.r.y));
  }
  __device__ __forceinline__ float2 first_x(const S& s) const {
    return make_float2((float)(s.z.x - s.r.x), (float)(s.z.y - s.r.y));
  }
  __device__ __forceinline__ static float l1_term(const S&) { return 0.f; }
};

// fused objective trace slot of the rows pass, read from the kernel parameters (constant
// bank) only where it is used, so the untraced pass keeps its register budget
__device__ __forceinline__ void trace_add(const EpiFista& e, int b, double v) {
  atomicAdd(e.trace + (long long)b * e.trace_stride + e.it, e.tau[b] * v);
}
__device__ __forceinline__ void trace_add(const EpiAdmmSplit&, int, double) {}

// Tensor-core level 2 of the band inverse (TCI rows tiles, R = 128 threads per line).
// For each line and register slot j the level-2 sum is
//   Z_s[j] = sum_m  A0[s][m] * Y[j + KP m],   A0[s][m] = exp(+2 pi i s m / R),
// i.e. one [R x MO] x [MO x (TR KP)] complex product per tile, shared by every (line, j).
// As real tf32 GEMMs (K = 8 per step q: m = 4q..4q+3, re then im):
//   D_re[s][n] = sum_k [A0re | -A0im][s][k] B[n][k],  D_im[s][n] = sum_k [A0im | A0re][s][k] B[n][k]
// with B[n = ii KP + j] = [Re Y[j + KP m], Im Y[j + KP m]] (m = 4q..4q+3).  Every operand is
// split into tf32 hi + lo and the product taken as A_hi B_hi + A_lo B_hi + A_hi B_lo (3 MMAs),
// fp32-grade (tests/test_gpu_tc.py).  D_re sits in TMEM columns [0, N), D_im in [N, 2N),
// N = TR KP; TMEM lane s belongs to thread s of each line team (warp w reads lanes 32 (w % 4)..).
// Per tile: the band is staged into B (each thread's value was prefetched during the previous
// tile), one thread issues the MMAs, every thread waits on the mbarrier and reads its lane of D.
// B and D are single-buffered: the next tile stages B only after every thread has waited for
// this tile's MMAs, and issues its MMAs after a barrier that follows every thread's D reads.
// per-thread asynchronous global -> shared copies (LDGSTS): nothing is held in registers while
// the copy is in flight (a register prefetch gets spilled by the 128-register budget, and the
// spill store then blocks on the load: profiles/r2/r2i_*)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(tc::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(tc::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// a thread's prefetch slot for its CTA's next tile (written and read by that thread only)
struct TcPrefetch {
  float2 pv;           // the thread's band value of the tile
  unsigned fl, tw;     // its warp's flag word, the tile word
  double tau;          // tau of the tile's snapshot
};

struct TcInv {
  unsigned char* At;   // [MO/4][re_hi | re_lo | im_hi | im_lo][128 x 8 tf32] (K-major, 4 KB each)
  unsigned char* Bt;   // [MO/4][hi | lo][N x 8 tf32]
  uint64_t* mbar;      // MMA completion (tcgen05.commit)
  uint32_t tmem;       // TMEM base column (lane 0)
  uint32_t phase;      // mbarrier parity of the next completion
  int next;            // next tile of this CTA (-1: none)
  // prefetched during the previous tile (pre != 0): this thread's band value of the tile and
  // the tile's flag words
  int pre;
  TcPrefetch* slot;    // shared memory
  float2 w8[3];        // this lane's level-1 twiddles tw[8], tw[16], tw[24] (KP = 32: TMEM energy screen)
};

template <int KP, int MO, int TR>
struct TcShape {
  static constexpr int N = KP * TR;
  static constexpr int QS = MO / 4;                 // K steps of 8 tf32
  static constexpr int A_BYTES = QS * 4 * 128 * 32;
  static constexpr int B_BYTES = QS * 2 * N * 32;
  // TMEM columns: D_re [0, N), D_im [N, 2N), then the level-1 twiddles conj(w_N^{s j}) of lane s
  // (re [2N, 2N + KP), im [2N + KP, 2N + 2KP)): resident for the CTA's lifetime, read with
  // tcgen05.ld instead of KP global/L1 loads per line
  static constexpr int TW = 2 * N;
  static constexpr int USED = 2 * N + 2 * KP;
  static constexpr int COLS = USED <= 32 ? 32 : (USED <= 64 ? 64 : (USED <= 128 ? 128 : (USED <= 256 ? 256 : 512)));
  static_assert(MO % 4 == 0 && MO <= 16, "tensor-core band: MO must be 4, 8, 12 or 16");
  static_assert(N % 16 == 0 && N <= 256, "tensor-core band: N = KP * TR must be a multiple of 16, <= 256");
};

// A tiles of the tensor-core level 2 (constant per line length): exp(+2 pi i s m / 128), split.
template <int MO>
__device__ __forceinline__ void tc_stage_a(unsigned char* At, int tid, int nthreads) {
  for (int idx = tid; idx < 128 * MO; idx += nthreads) {
    const int s = idx % 128, m = idx / 128;
    const int q = m >> 2, k = m & 3;
    double sn, cs;
    sincospi((double)((s * m) % 128) / 64.0, &sn, &cs);   // angle 2 pi s m / 128
    const float c = (float)cs, si = (float)sn;
    unsigned char* base = At + q * 4 * 4096;
    float hi, lo;
    // D_re row: [cos | -sin];  D_im row: [sin | cos]
    tc::split_tf32(c, hi, lo);
    *reinterpret_cast<float*>(base + 0 * 4096 + tc::km_off(s, k)) = hi;
    *reinterpret_cast<float*>(base + 1 * 4096 + tc::km_off(s, k)) = lo;
    *reinterpret_cast<float*>(base + 2 * 4096 + tc::km_off(s, 4 + k)) = hi;
    *reinterpret_cast<float*>(base + 3 * 4096 + tc::km_off(s, 4 + k)) = lo;
    tc::split_tf32(-si, hi, lo);
    *reinterpret_cast<float*>(base + 0 * 4096 + tc::km_off(s, 4 + k)) = hi;
    *reinterpret_cast<float*>(base + 1 * 4096 + tc::km_off(s, 4 + k)) = lo;
    tc::split_tf32(si, hi, lo);
    *reinterpret_cast<float*>(base + 2 * 4096 + tc::km_off(s, k)) = hi;
    *reinterpret_cast<float*>(base + 3 * 4096 + tc::km_off(s, k)) = lo;
  }
}

// band value Y[k] of tile line i2 -> B tiles (hi/lo split), k = j + KP m
template <int KP, int MO, int TR>
__device__ __forceinline__ void tc_put_b(unsigned char* Bt, int k, int i2, float2 v) {
  using TSH = TcShape<KP, MO, TR>;
  const int j = k % KP, m = k / KP;
  const int q = m >> 2, mm = m & 3;
  const int n = i2 * KP + j;
  unsigned char* hi_t = Bt + q * 2 * TSH::N * 32;
  unsigned char* lo_t = hi_t + TSH::N * 32;
  float hi, lo;
  tc::split_tf32(v.x, hi, lo);
  *reinterpret_cast<float*>(hi_t + tc::km_off(n, mm)) = hi;
  *reinterpret_cast<float*>(lo_t + tc::km_off(n, mm)) = lo;
  tc::split_tf32(v.y, hi, lo);
  *reinterpret_cast<float*>(hi_t + tc::km_off(n, 4 + mm)) = hi;
  *reinterpret_cast<float*>(lo_t + tc::km_off(n, 4 + mm)) = lo;
}

// one elected thread: the tile's 6 * MO/4 MMAs, then commit to the mbarrier
template <int KP, int MO, int TR>
__device__ __forceinline__ void tc_issue(const TcInv& t) {
  using TSH = TcShape<KP, MO, TR>;
  constexpr uint32_t idesc = tc::idesc_tf32<128, TSH::N>();
  tc::fence_after_sync();
#pragma unroll
  for (int q = 0; q < TSH::QS; ++q) {
    const unsigned char* a = t.At + q * 4 * 4096;
    const unsigned char* b = t.Bt + q * 2 * TSH::N * 32;
    const uint64_t are_hi = tc::desc_kmajor(a, tc::KM_LBO, tc::KM_SBO);
    const uint64_t are_lo = tc::desc_kmajor(a + 4096, tc::KM_LBO, tc::KM_SBO);
    const uint64_t aim_hi = tc::desc_kmajor(a + 2 * 4096, tc::KM_LBO, tc::KM_SBO);
    const uint64_t aim_lo = tc::desc_kmajor(a + 3 * 4096, tc::KM_LBO, tc::KM_SBO);
    const uint64_t b_hi = tc::desc_kmajor(b, tc::KM_LBO, tc::KM_SBO);
    const uint64_t b_lo = tc::desc_kmajor(b + TSH::N * 32, tc::KM_LBO, tc::KM_SBO);
    tc::mma_tf32(t.tmem, are_hi, b_hi, idesc, q > 0);
    tc::mma_tf32(t.tmem, are_lo, b_hi, idesc, 1);
    tc::mma_tf32(t.tmem, are_hi, b_lo, idesc, 1);
    tc::mma_tf32(t.tmem + TSH::N, aim_hi, b_hi, idesc, q > 0);
    tc::mma_tf32(t.tmem + TSH::N, aim_lo, b_hi, idesc, 1);
    tc::mma_tf32(t.tmem + TSH::N, aim_hi, b_lo, idesc, 1);
  }
  tc::commit(t.mbar);
}

// once per CTA: lane s's level-1 twiddles conj(w_N^{s j}), j < KP, into TMEM (warps of the
// first line team; the second team reads the same lanes)
template <int KP, int MO, int TR>
__device__ __forceinline__ void tc_put_twiddles(const TcInv& t, const float2* tw1, int R) {
  using TSH = TcShape<KP, MO, TR>;
  if (threadIdx.x >= 128) return;
  const int s = threadIdx.x;
  const uint32_t base = t.tmem + ((uint32_t)((threadIdx.x >> 5) & 3) * 32u << 16) + TSH::TW;
#pragma unroll
  for (int q = 0; q < KP / 8; ++q) {
    float re[8], im[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 w = __ldg(tw1 + (8 * q + i) * R + s);
      re[i] = w.x;
      im[i] = -w.y;                       // conjugate: the inverse transform
    }
    tc::tmem_st8(base + 8 * q, re);
    tc::tmem_st8(base + KP + 8 * q, im);
  }
  tc::tmem_st_wait();
}

// forward level-1 twiddle from the TMEM copy: a[j] *= w_N^{s j} (the stored value is its conjugate)
template <int KP, int MO, int TR>
__device__ __forceinline__ void tc_twiddle_fwd(const TcInv& t, float2 (&a)[KP]) {
  using TSH = TcShape<KP, MO, TR>;
  const uint32_t lane = t.tmem + ((uint32_t)((threadIdx.x >> 5) & 3) * 32u << 16);
#pragma unroll
  for (int q = 0; q < KP / 8; ++q) {
    float wr[8], wi[8];
    tc::tmem_ld8(lane + TSH::TW + 8 * q, wr);
    tc::tmem_ld8(lane + TSH::TW + KP + 8 * q, wi);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 8; ++i) a[8 * q + i] = cmulc(a[8 * q + i], make_float2(wr[i], wi[i]));
  }
}

// every thread: wait for the tile's MMAs
__device__ __forceinline__ void tc_wait(TcInv& t) {
  tc::mbar_wait(t.mbar, t.phase);
  t.phase ^= 1u;
  tc::fence_after_sync();
}

// thread (ii, s): its KP level-2 values of line ii from TMEM, times the level-1 twiddles
template <int KP, int MO, int TR>
__device__ __forceinline__ void tc_read(const TcInv& t, int ii, float2 (&a)[KP]) {
  using TSH = TcShape<KP, MO, TR>;
  static_assert(KP % 8 == 0, "tensor-core band: KP 8, 16 or 32");
  const uint32_t lane = t.tmem + ((uint32_t)((threadIdx.x >> 5) & 3) * 32u << 16);
  const uint32_t col = lane + (uint32_t)(ii * KP);
#pragma unroll
  for (int q = 0; q < KP / 8; ++q) {      // quarters of 8 slots: 32 live temporaries
    float re[8], im[8], wr[8], wi[8];
    tc::tmem_ld8(col + 8 * q, re);
    tc::tmem_ld8(col + TSH::N + 8 * q, im);
    tc::tmem_ld8(lane + TSH::TW + 8 * q, wr);
    tc::tmem_ld8(lane + TSH::TW + KP + 8 * q, wi);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 8; ++i) a[8 * q + i] = cmul(make_float2(re[i], im[i]), make_float2(wr[i], wi[i]));
  }
}

// Second-level screen of one residue class q (warp-uniform) of the TMEM energy screen: the
// class's eight first-stage values u[l] are formed again from TMEM, one more decimation-in-
// frequency split gives the two 4-output sub-classes (even / odd p of x[4 p + q]) with the
// Parseval bounds 4 sum_l' |u[l'] +- u[l' + 4] phi|^2, phi = tw[4] W_8^q the twiddle ratio of
// slots l' + 4 and l' (unit-modulus common factors dropped).  `thr4` = threshold / 4.
template <int KP, int MO, int TR>
__device__ __forceinline__ bool tc_class_rescreen(const TcInv& t, int ii, int q, const float2 (&w)[3], float thr4,
                                                  bool active) {
  using TSH = TcShape<KP, MO, TR>;
  const uint32_t lane = t.tmem + ((uint32_t)((threadIdx.x >> 5) & 3) * 32u << 16);
  const uint32_t col = lane + (uint32_t)(ii * KP);
  // i^q as (cq, sq); W_8^q = exp(+i pi q / 4)
  const float cq = (q == 0) ? 1.f : ((q == 2) ? -1.f : 0.f);
  const float sq = (q == 1) ? 1.f : ((q == 3) ? -1.f : 0.f);
  const float r = 0.70710678118654752f;
  const float2 w8 = (q == 0) ? make_float2(1.f, 0.f)
                             : ((q == 1) ? make_float2(r, r) : ((q == 2) ? make_float2(0.f, 1.f) : make_float2(-r, r)));
  const float2 phi = cmul(make_float2(tc::tmem_ld1(lane + TSH::TW + 4), tc::tmem_ld1(lane + TSH::TW + KP + 4)), w8);
  float2 u[8];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float re[4][4], im[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      tc::tmem_ld4(col + 8 * i + 4 * h, re[i]);
      tc::tmem_ld4(col + TSH::N + 8 * i + 4 * h, im[i]);
    }
    tc::tmem_ld_wait();
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const float2 a0 = make_float2(re[0][l], im[0][l]);
      const float2 a1 = cmul(make_float2(re[1][l], im[1][l]), w[0]);
      const float2 a2 = cmul(make_float2(re[2][l], im[2][l]), w[1]);
      const float2 a3 = cmul(make_float2(re[3][l], im[3][l]), w[2]);
      // u = a0 + i^q a1 + (-1)^q a2 + (-i)^q a3 = (a0 + (-1)^q a2) + i^q (a1 + (-1)^q a3)
      const float sg = (q & 1) ? -1.f : 1.f;
      const float2 p02 = make_float2(fmaf(sg, a2.x, a0.x), fmaf(sg, a2.y, a0.y));
      const float2 p13 = make_float2(fmaf(sg, a3.x, a1.x), fmaf(sg, a3.y, a1.y));
      u[4 * h + l] = make_float2(p02.x + cq * p13.x - sq * p13.y, p02.y + cq * p13.y + sq * p13.x);
    }
  }
  float ee = 0.f, eo = 0.f;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const float2 v = cmul(u[l + 4], phi);
    const float2 a = cadd(u[l], v), b = csub(u[l], v);
    ee = fmaf(a.x, a.x, fmaf(a.y, a.y, ee));
    eo = fmaf(b.x, b.x, fmaf(b.y, b.y, eo));
  }
  return __all_sync(0xffffffffu, !active || fmaxf(ee, eo) < thr4);
}

// Energy screen straight from TMEM (KP = 32; the thread's state is known to be all zero): the
// radix-4 first stage of the screened inverse DFT (band_fft.cuh reg_idft_screened) on the
// level-2 values Z[8 i + l], i < 4, without keeping any of them.  Only the energy of each residue
// class matters and the level-1 twiddle factors as tw[8 i + l] = tw[8 i] tw[l] with |tw[l]| = 1, so
// the class sums are formed from Z[8 i + l] tw[8 i] (three per-thread constants read from the TMEM
// twiddle table).  Returns true when all four class bounds of every lane of the warp lie below
// the threshold: none of the warp's points can leave zero, and nothing else of the tile's
// inverse transform is needed.
template <int KP, int MO, int TR>
__device__ __forceinline__ bool tc_energy_screen(const TcInv& t, int ii, float thr, bool active) {
  using TSH = TcShape<KP, MO, TR>;
  static_assert(KP == 32, "TMEM energy screen: KP = 32");
  const uint32_t lane = t.tmem + ((uint32_t)((threadIdx.x >> 5) & 3) * 32u << 16);
  const uint32_t col = lane + (uint32_t)(ii * KP);
  const float2 w[3] = {t.w8[0], t.w8[1], t.w8[2]};
  float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float re[4][4], im[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      tc::tmem_ld4(col + 8 * i + 4 * h, re[i]);
      tc::tmem_ld4(col + TSH::N + 8 * i + 4 * h, im[i]);
    }
    tc::tmem_ld_wait();
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const float2 a0 = make_float2(re[0][l], im[0][l]);
      const float2 a1 = cmul(make_float2(re[1][l], im[1][l]), w[0]);
      const float2 a2 = cmul(make_float2(re[2][l], im[2][l]), w[1]);
      const float2 a3 = cmul(make_float2(re[3][l], im[3][l]), w[2]);
      const float2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
      const float2 u0 = cadd(s02, s13), u2 = csub(s02, s13);
      const float2 u1 = make_float2(d02.x - d13.y, d02.y + d13.x), u3 = make_float2(d02.x + d13.y, d02.y - d13.x);
      e[0] = fmaf(u0.x, u0.x, fmaf(u0.y, u0.y, e[0]));
      e[1] = fmaf(u1.x, u1.x, fmaf(u1.y, u1.y, e[1]));
      e[2] = fmaf(u2.x, u2.x, fmaf(u2.y, u2.y, e[2]));
      e[3] = fmaf(u3.x, u3.x, fmaf(u3.y, u3.y, e[3]));
    }
  }
  // classes whose bound fails somewhere in the warp get a second look (tc_class_rescreen)
  unsigned ok = 0u;
#pragma unroll
  for (int q = 0; q < 4; ++q) ok |= ((!active || e[q] < thr) ? 1u : 0u) << q;
  ok = __reduce_and_sync(0xffffffffu, ok);
  if (ok == 0xfu) return true;
  bool all = true;
  for (int q = 0; q < 4 && all; ++q)
    if (!((ok >> q) & 1u)) all = tc_class_rescreen<KP, MO, TR>(t, ii, q, w, 2.0f * thr, active);
  return all;
}

template <typename Pol, typename Args>
__device__ __forceinline__ Pol make_policy(const Args& e, long long off, int b, const double* tau_pre) {
  if constexpr (std::is_constructible<Pol, const Args&, long long, int, const double*>::value)
    return Pol(e, off, b, tau_pre);
  else
    return Pol(e, off, b);
}

// One tile (TR lines of one snapshot) of the specialised rows pass, complex64 band engine,
// state policy Pol.  `tile` indexes the tile (and its flag words); with KP2 > 0 and do_fwd,
// the last tile of a snapshot to arrive runs that snapshot's column pass.  Streaming state /
// band loads bypass L1 (ld.global.cg): they are read once.
template <int KP, int R, int MO, typename Pol, bool ZS, int KP2, bool TCI = false, bool TRACE = false>
__device__ __forceinline__ void rows_tile(const Geo& G, const AxisT<float2>& ax, const RowsIO<float2>& io,
                                          const typename Pol::Args& epi, unsigned* __restrict__ flags,
                                          const FusedCols& fc, int tile, const float2* tw1s, const float2* tw2s,
                                          float2* Xs, TcInv* tci = nullptr) {
  static_assert(!TCI || (R == 128 && KP2 == 0), "tensor-core tiles: R = 128, no fused column pass");
  using TS = TileShape<KP, R, MO, TCI ? tc_threads(KP) : 256>;
  using St = typename Pol::S;
  constexpr int NT = TS::NT, TR = TS::TR, K = TS::K, XP = TS::XP, PITCH = TS::PITCH, SP = TS::SP;
  constexpr int CH = 2;
  static_assert(KP % CH == 0, "chunking");
  float2* S = Xs + TR * XP;
  const int tid = threadIdx.x;
  const int ii = tid / R, s = tid % R;
  const int row0 = tile * TR;                  // rows < 2^31 (host check)
  const int gr = row0 + ii;
  const bool active = gr < (int)G.rows;
  const int L2 = G.L2;
  const int b = G.l2_shift >= 0 ? (row0 >> G.l2_shift) : row0 / L2;   // whole CTA lies in one snapshot
  const int l20 = row0 - b * L2;
  const long long vbase = (long long)b * K * L2 + l20;   // io.V/U index of (k=0, ii=0)
  // tensor-core tiles: the flag words, the band value and tau of this tile were copied into the
  // thread's shared-memory slot during the CTA's previous tile
  const double* tau_pre = nullptr;
  if constexpr (TCI) {
    if (tci->pre) {
      cp_async_wait_group0();
      tau_pre = &tci->slot->tau;
    }
  }
  const Pol pol = make_policy<Pol>(epi, (long long)gr * G.L1 + s, b, tau_pre);
  const double kap = pol.kap();
  const float kap2_lo = (float)(kap * kap) * (1.0f - 1.0f / 262144.0f);
  const int lane = tid & 31;
  // flag words per tile: NT/32 warp words (zero segments), then one tile word (bit 0: the
  // tile's U band may be nonzero; clear = U already holds zeros, the store can be skipped)
  unsigned* fw = ZS ? flags + ((long long)tile * (NT / 32 + 1) + (tid >> 5)) : nullptr;
  unsigned* tword = ZS ? flags + ((long long)tile * (NT / 32 + 1) + NT / 32) : nullptr;
  // Reads before the dependency wait are safe only when a separate column pass runs between
  // two rows passes (it waited for the previous rows pass).  With the fused column pass
  // (KP2 > 0) the previous grid on the stream IS the previous rows pass, still writing the
  // flags and the state when PDL releases this grid, so everything waits first.
  constexpr bool PRE_WAIT_READS = KP2 == 0;
  if constexpr (!PRE_WAIT_READS) pdl_wait();
  unsigned fl = 0xffffffffu, u_maybe_nonzero = 1u;
  if constexpr (TCI) {                 // prefetched during the CTA's previous tile
    if (tci->pre) {
      fl = tci->slot->fl;
      u_maybe_nonzero = tci->slot->tw;
    } else {
      fl = __ldcg(fw);
      u_maybe_nonzero = __ldcg(tword);
    }
  } else if constexpr (ZS) {
    fl = __ldcg(fw);
    u_maybe_nonzero = __ldcg(tword);
  }
  bool warp_zero = false;   // the whole warp's next operator input is zero
  float2 a[KP];
  __shared__ unsigned live_rows[(TR + 31) / 32];   // lines whose next operator input is nonzero
  auto live_rows_zero = [&](int i) { live_rows[i] = 0u; };

  // first state chunk in flight while the band tile loads and the inverse DFT runs.  The
  // flags and the state were last written by the previous rows pass, which completed before
  // the column pass between them released this grid (pdl_wait there), so they are read before
  // this grid's own dependency wait; the band tile V comes from that column pass (after it).
  // Early only for short lines (config 2: +2.7%); the long-line shapes keep the load order
  // band tile -> state (configs 4/5 measured 1-2% slower with the state first).
  constexpr bool EARLY = PRE_WAIT_READS && R <= 16;
  St sb[CH];
  if (EARLY && G.do_inv) {
#pragma unroll
    for (int q = 0; q < CH; ++q) sb[q] = pol.load(q * R, active && ((fl >> q) & 1u));
  }
  if constexpr (PRE_WAIT_READS) pdl_wait();
  if (G.do_inv) {
    // Level-1 register IDFT.  With zero-segment flags (ZS) and KP >= 16 it is the screened
    // variant: residue classes of outputs whose Parseval energy bound lies below the threshold
    // for the whole warp skip their sub-DFT and per-point tests (band_fft.cuh).
    // (tensor-core tiles screen from TMEM instead and keep the plain register DFT for the warps
    // that fail it: the screened register variant measured slower there, 300 vs 365 G gpi/s
    // with every class computed, profiles/r2/r2g_bench_cfg5_screen0.json vs r2d)
    constexpr bool SCREEN = ZS && !TCI && (KP == 16 || KP == 32);
    constexpr bool TSCREEN = ZS && TCI && KP == 32;
    unsigned pass = 0u;
    const float thr_scale = (G.screen & 1) ? (1.0f - 1.0f / 1024.0f) / (float)(KP / 4) : -1.0f;
    bool ez = false;          // TMEM energy screen: the whole warp provably stays zero
    constexpr bool ONE = TR * K == NT;     // tensor-core tiles with one band value per thread: prefetched
    if constexpr (TCI) {
      // tensor-core level 2: this tile's band V[b][k][l20 + i] -> B tiles (tf32 hi/lo)
      if (ONE && tci->pre) {
        tc_put_b<KP, MO, TR>(tci->Bt, tid / TR, tid % TR, tci->slot->pv);
      } else {
        for (int idx = tid; idx < TR * K; idx += NT) {
          const int k = idx / TR, i2 = idx % TR;
          tc_put_b<KP, MO, TR>(tci->Bt, k, i2, __ldcg(io.V + vbase + (long long)k * L2 + i2));
        }
      }
      tc::fence_async_smem();   // B writes -> visible to the tensor core
    } else {
      // band tile V[b][k][l20 + ii] -> Xs[ii][k]
      for (int idx = tid; idx < TR * K; idx += NT) {
        const int k = idx / TR, i2 = idx % TR;
        Xs[i2 * XP + k] = __ldcg(io.V + vbase + (long long)k * L2 + i2);
      }
    }
    if (!EARLY) {
      if (fl & ((1u << CH) - 1u)) {          // warp-uniform: a clear flag word loads nothing
#pragma unroll
        for (int q = 0; q < CH; ++q) sb[q] = pol.load(q * R, active && ((fl >> q) & 1u));
      } else {
#pragma unroll
        for (int q = 0; q < CH; ++q) sb[q] = Pol::empty();
      }
    }
    if (G.do_fwd && tid < (TR + 31) / 32) live_rows_zero(tid);
    __syncthreads();
    unsigned nfl = 0;
    float l1 = 0.f;           // fused objective: sum of |c_{t+1}| over this thread's updated points
    if constexpr (TCI) {
      if (tid == 0 && !(G.dbg & 32)) tc_issue<KP, MO, TR>(*tci);
      // while the MMAs run: the next tile's flag words and this thread's band value of it
      tci->pre = 0;
      if (tci->next >= 0) {
        const int nrow0 = tci->next * TR;
        const int nb = G.l2_shift >= 0 ? (nrow0 >> G.l2_shift) : nrow0 / L2;
        static_assert(ZS, "tensor-core tiles run with zero-segment flags");
        cp_async4(&tci->slot->fl, flags + ((long long)tci->next * (NT / 32 + 1) + (tid >> 5)));
        cp_async4(&tci->slot->tw, flags + ((long long)tci->next * (NT / 32 + 1) + NT / 32));
        cp_async8(&tci->slot->tau, epi.tau + nb);
        if constexpr (ONE)
          cp_async8(&tci->slot->pv,
                    io.V + (long long)nb * K * L2 + (nrow0 - nb * L2) + (long long)(tid / TR) * L2 + tid % TR);
        cp_async_commit_group();
        tci->pre = 1;
      }
      // ---- band inverse, level 2 of this tile from TMEM (times the level-1 twiddle)
      if (!(G.dbg & (16 | 32))) tc_wait(*tci);
      if (G.dbg & 64) ez = fl == 0u;     // timing probe only: no TMEM reads, no transform
      if constexpr (TSCREEN) {
        if (fl == 0u && (G.screen & 2))
          ez = tc_energy_screen<KP, MO, TR>(*tci, ii, kap2_lo * (1.0f - 1.0f / 1024.0f) / (float)(KP / 4), active);
      }
      if (!ez) {
        tc_read<KP, MO, TR>(*tci, ii, a);
        reg_dft<KP, true>(a);
      }
      tc::fence_before_sync();   // these TMEM reads precede the next tile's MMAs (barrier between)
    }
    {
      // ---- band inverse (level 2 broadcast + twiddle, level 1 register IDFT); the band row
      // is read as 16-byte pairs
      if constexpr (!TCI) {
      const float4* Y4 = reinterpret_cast<const float4*>(Xs + ii * XP);
#pragma unroll
      for (int j = 0; j < KP; j += 2) {
        const float4 q = Y4[j / 2];
        a[j] = make_float2(q.x, q.y);
        a[j + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int m = 1; m < MO; ++m) {
        const float2 w2 = tw2s[m * R + s];
#pragma unroll
        for (int j = 0; j < KP; j += 2) {
          const float4 q = Y4[(j + KP * m) / 2];
          a[j] = cadd(a[j], cmulc(make_float2(q.x, q.y), w2));
          a[j + 1] = cadd(a[j + 1], cmulc(make_float2(q.z, q.w), w2));
        }
      }
#pragma unroll
      for (int j = 0; j < KP; ++j) a[j] = cmulc(a[j], tw1s[j * R + s]);
      if constexpr (SCREEN) pass = reg_idft_screened<KP>(a, kap2_lo, thr_scale, fl, active);
      else reg_dft<KP, true>(a);
      }
      // ---- fused epilogue, register-pipelined state stream.
      // Warp-level fast path: a clear segment whose 32 points all stay below the threshold
      // stays exactly zero (same test as the per-point fast path below).  One warp AND-reduce
      // covers all KP segments; when every segment qualifies the loop is skipped.
      unsigned fast = 0u;
      if constexpr (ZS) {
        if (ez) {
          fast = 0xffffffffu;
        } else {
          if constexpr (!SCREEN) {
            // one predicate chain and one vote first: when every point of the warp is below the
            // threshold (nearly all warps once the iterate is sparse) the per-slot bits are all
            // ones (a NaN compares false, so it still reaches the per-slot path and the slow path)
            bool below = true;
#pragma unroll
            for (int r = 0; r < KP; ++r) below = below & (fmaf(a[r].x, a[r].x, a[r].y * a[r].y) < kap2_lo);
            if (__all_sync(0xffffffffu, !active || below)) {
              pass = 0xffffffffu;
            } else {
#pragma unroll
              for (int r = 0; r < KP; ++r)
                pass |= (fmaf(a[r].x, a[r].x, a[r].y * a[r].y) < kap2_lo ? 1u : 0u) << r;
            }
          }
          if (!active) pass = 0xffffffffu;
          fast = __reduce_and_sync(0xffffffffu, pass) & ~fl;
        }
      }
      constexpr unsigned ALL = KP >= 32 ? 0xffffffffu : ((1u << KP) - 1u);
      if (ZS && (fast & ALL) == ALL) {
        warp_zero = true;   // a[] is not used again (the forward part writes zeros for this warp)
      } else
#pragma unroll
      for (int r0 = 0; r0 < KP; r0 += CH) {
        St sn[CH];
        if (r0 + CH < KP) {
#pragma unroll
          for (int q = 0; q < CH; ++q) sn[q] = pol.load((r0 + CH + q) * R, active && ((fl >> (r0 + CH + q)) & 1u));
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int r = r0 + q;
          const float2 g = a[r];
          if (ZS && ((fast >> r) & 1u)) {
            a[r] = make_float2(0.f, 0.f);
            continue;
          }
          St n = Pol::empty();
          if (active && !(Pol::zero(sb[q]) && fmaf(g.x, g.x, g.y * g.y) < kap2_lo)) {
            n = pol.update(sb[q], g);
            if (!ZS) pol.store(r * R, n);
            if constexpr (TRACE) l1 += Pol::l1_term(n);
          }
          if (ZS) {
            if (__any_sync(0xffffffffu, !Pol::zero(n))) {  // segment (still / newly) nonzero: write it whole
              if (active) pol.store(r * R, n);
              nfl |= 1u << r;
            }
          }
          a[r] = pol.next_x(n);
        }
        if (r0 + CH < KP) {
#pragma unroll
          for (int q = 0; q < CH; ++q) sb[q] = sn[q];
        }
      }
    }
    if (ZS && lane == 0 && (nfl | fl)) *fw = nfl;   // (a clear word stays clear: no store)
    if constexpr (TRACE) {   // whole CTA in one snapshot: one atomic per warp
      double v = (double)l1;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v != 0.0) trace_add(epi, b, v);
    }
  } else if (active) {
#pragma unroll
    for (int r = 0; r < KP; ++r) {
      if (!((fl >> r) & 1u)) {
        a[r] = make_float2(0.f, 0.f);
        continue;
      }
      a[r] = pol.first_x(pol.load(r * R, true));
    }
  }
  if (!G.do_fwd) return;
  if constexpr (TCI) {
    if (G.dbg & 8) return;               // timing probe only: no forward part, no tile barrier
  }
  // ---- band forward: register DFT, twiddle + transpose scatter, R-term reductions.
  // A line whose next operator input is entirely zero (most lines once the iterate is sparse)
  // has a zero band: its DFT, scatter and reductions are skipped.
  if (!G.do_inv) {                        // (zeroed before the band-load barrier otherwise)
    if (tid < (TR + 31) / 32) live_rows_zero(tid);
    __syncthreads();
  }
  bool nzx = false;
  if (!warp_zero) {
#pragma unroll
    for (int r = 0; r < KP; ++r) nzx |= (a[r].x != 0.f) | (a[r].y != 0.f);
    if (active && nzx) atomicOr(&live_rows[ii >> 5], 1u << (ii & 31));
  }
  const bool tile_live = __syncthreads_or(active && nzx);
  if (ZS && !tile_live) {
    // the whole tile's next operator input is zero, so is its band: store zeros unless U
    // already holds them from the previous step
    if (u_maybe_nonzero) {
      for (int idx = tid; idx < TR * K; idx += NT) {
        const int k = idx / TR, i2 = idx % TR;
        if (row0 + i2 < (int)G.rows) io.U[vbase + (long long)k * L2 + i2] = make_float2(0.f, 0.f);
      }
      if (tid == 0) *tword = 0u;
    }
  } else {
    const bool my_live = (live_rows[ii >> 5] >> (ii & 31)) & 1u;
    if (active && my_live && warp_zero) {    // this warp's slice of a live line is zero
      float2* Srow = S + ii * SP;
#pragma unroll
      for (int j = 0; j < KP; ++j) Srow[j * PITCH + s] = make_float2(0.f, 0.f);
    } else if (active && my_live) {
      reg_dft<KP, false>(a);
      float2* Srow = S + ii * SP;
      if constexpr (TCI) {     // warp-uniform branch (a warp lies in one line): TMEM twiddles
        tc_twiddle_fwd<KP, MO, TR>(*tci, a);
#pragma unroll
        for (int j = 0; j < KP; ++j) Srow[j * PITCH + s] = a[j];
      } else {
#pragma unroll
        for (int j = 0; j < KP; ++j) Srow[j * PITCH + s] = cmul(a[j], tw1s[j * R + s]);
      }
    }
    __syncthreads();
    for (int idx = tid; idx < TR * K; idx += NT) {
      const int i2 = idx / K, o = idx % K;
      if (!((live_rows[i2 >> 5] >> (i2 & 31)) & 1u)) {
        Xs[i2 * XP + o] = make_float2(0.f, 0.f);
        continue;
      }
      const int j = o % KP, m = o / KP;
      const float2* row = S + i2 * SP + j * PITCH;
      float2 acc = make_float2(0.f, 0.f);
      if (m == 0) {
#pragma unroll
        for (int t = 0; t < R; ++t) acc = cadd(acc, row[t]);
      } else {
        const float2* tw = tw2s + m * R;
#pragma unroll
        for (int t = 0; t < R; ++t) acc = cfma(row[t], tw[t], acc);
      }
      Xs[i2 * XP + o] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < TR * K; idx += NT) {
      const int k = idx / TR, i2 = idx % TR;
      if (row0 + i2 < (int)G.rows) io.U[vbase + (long long)k * L2 + i2] = Xs[i2 * XP + k];
    }
    if (ZS && tid == 0 && !u_maybe_nonzero) *tword = 1u;
  }
  if constexpr (KP2 > 0) {
    __shared__ int s_last;
    __threadfence();                       // publish this CTA's U tile
    __syncthreads();
    if (tid == 0) s_last = ((atomicAdd(fc.counter + b, 1) + 1) % fc.cps) == 0;
    __syncthreads();
    if (s_last) {
      __threadfence();                     // acquire the other CTAs' U tiles
      for (int l0 = 0; l0 < fc.K1; l0 += fc.TRc)
        cols_block<KP2>(fc.G, fc.ax, fc.io, (long long)b * fc.K1 + l0, fc.TRc, Xs);
    }
  }
}

// TRACE: the fused objective trace variant (tau ||c||_1 summed over the updated points);
// a separate instantiation so the plain pass keeps its register budget.
template <int KP, int R, int MO, bool MOM, bool ZS, int KP2 = 0, int MINB = 2, bool TRACE = false>
__global__ void __launch_bounds__(R > 256 ? R : 256, R > 256 ? 1 : MINB)
    rows_fista_fast_kernel(Geo G, AxisT<float2> ax, RowsIO<float2> io, EpiFista epi, unsigned* __restrict__ flags,
                           FusedCols fc) {
  using TS = TileShape<KP, R, MO>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* Xs = reinterpret_cast<float2*>(smem_raw);
  const float2* tw1s;
  const float2* tw2s;
  stage_twiddles<KP, R, MO>(ax, Xs + TS::TR * TS::XP + TS::TR * TS::SP, tw1s, tw2s);
  rows_tile<KP, R, MO, FistaPolicy<MOM>, ZS, KP2, false, TRACE>(G, ax, io, epi, flags, fc, blockIdx.x, tw1s, tw2s,
                                                               Xs);
}

// Tensor-core variant of the specialised FISTA/ISTA rows pass (lines of L1 = 128 KP points, band
// K = KP MO): the level-2 stage of the band inverse runs as kind::tf32 MMAs (TcInv), the rest
// of rows_tile is unchanged.  Persistent: each CTA stages the constant A tiles, allocates its
// TMEM columns and initialises its mbarrier once, then walks tiles blockIdx.x, +gridDim.x, ...
template <int KP, int MO, bool MOM, int MINB, bool TRACE = false>
__global__ void __launch_bounds__(tc_threads(KP), MINB)
    rows_fista_tc_kernel(Geo G, AxisT<float2> ax, RowsIO<float2> io, EpiFista epi, unsigned* __restrict__ flags,
                         int ntiles) {
  constexpr int R = 128;
  using TS = TileShape<KP, R, MO, tc_threads(KP)>;
  using TSH = TcShape<KP, MO, TS::TR>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* Xs = reinterpret_cast<float2*>(smem_raw);
  const float2* tw1s;
  const float2* tw2s;
  size_t off = (size_t)(TS::TR * TS::XP + TS::TR * TS::SP) * sizeof(float2);
  stage_twiddles<KP, R, MO>(ax, reinterpret_cast<float2*>(smem_raw + off), tw1s, tw2s);
  if constexpr (TS::STAGE_TW) off += (size_t)(KP + MO) * R * sizeof(float2);
  off = (off + 127) & ~(size_t)127;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  __shared__ TcPrefetch prefetch_slots[TS::NT];
  TcInv t;
  t.slot = &prefetch_slots[threadIdx.x];
  t.At = smem_raw + off;
  t.Bt = t.At + TSH::A_BYTES;
  t.mbar = &mbar;
  t.phase = 0;
  t.pre = 0;
  tc_stage_a<MO>(t.At, threadIdx.x, TS::NT);
  if (threadIdx.x == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tmem_base, TSH::COLS);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  t.tmem = tmem_base;
  tc_put_twiddles<KP, MO, TS::TR>(t, ax.tw1, R);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if constexpr (KP == 32) {
    const uint32_t lane = t.tmem + ((uint32_t)((threadIdx.x >> 5) & 3) * 32u << 16);
#pragma unroll
    for (int i = 1; i < 4; ++i)
      t.w8[i - 1] = make_float2(tc::tmem_ld1(lane + TSH::TW + 8 * i), tc::tmem_ld1(lane + TSH::TW + KP + 8 * i));
    tc::tmem_ld_wait();
  }
  const FusedCols nofc{};
  // No barrier between tiles: the next tile writes shared memory only after barriers every
  // thread passes after its last read of it here (B is rewritten after every thread's mbarrier
  // wait of this tile; live_rows, Xs and S are last read before this tile's final
  // __syncthreads), and its MMAs overwrite D only after the barrier that follows every
  // thread's TMEM reads.
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    t.next = tile + (int)gridDim.x < ntiles ? tile + (int)gridDim.x : -1;
    rows_tile<KP, R, MO, FistaPolicy<MOM>, true, 0, true, TRACE>(G, ax, io, epi, flags, nofc, tile, tw1s, tw2s, Xs,
                                                                 &t);
    if (G.dbg & 1) __syncthreads();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (threadIdx.x < 32) tc::tmem_dealloc(t.tmem, TSH::COLS);
}

// ---------------------------------------------------------------- ADMM, spectral dual split
// Rows pass of the split ADMM (AdmmSplitPolicy): complex64 band engine, zero-segment skipping on
// the (z, r) state, which stays sparse because the growing part of the dual lives on the box.
template <int KP, int R, int MO, int MINB = 2>
__global__ void __launch_bounds__(R > 256 ? R : 256, R > 256 ? 1 : MINB)
    rows_admm_split_kernel(Geo G, AxisT<float2> ax, RowsIO<float2> io, EpiAdmmSplit epi,
                           unsigned* __restrict__ flags) {
  using TS = TileShape<KP, R, MO>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* Xs = reinterpret_cast<float2*>(smem_raw);
  const float2* tw1s;
  const float2* tw2s;
  stage_twiddles<KP, R, MO>(ax, Xs + TS::TR * TS::XP + TS::TR * TS::SP, tw1s, tw2s);
  const FusedCols nofc{};
  rows_tile<KP, R, MO, AdmmSplitPolicy, true, 0>(G, ax, io, epi, flags, nofc, blockIdx.x, tw1s, tw2s, Xs);
}

// Band stage of the split ADMM column pass (float64 on the box):
//   Cb = D X + P Bh - rho L P vs,   vs' = vs + Cb,   Y = vs'  (-> V = IFFT_col(vs'))
// and, on the last iteration, Cb is kept for c = a w + IFFT2u(Cb).
struct AdmmSplitBand {
  const double2* __restrict__ D;   // [K1][K2]
  const double2* __restrict__ P;   // [K1][K2]
  const float2* __restrict__ Bh;   // [B][K1][K2]
  double2* vs;                     // [B][K1][K2]
  double2* cb_out;                 // [B][K1][K2] or null
  double rhoL;
  int K1, K2;
  __device__ __forceinline__ float2 operator()(long long line, int o, float2 x) const {
    const long long k1 = line % K1;
    const long long bi = line * K2 + o;
    const double2 d = __ldg(D + k1 * K2 + o), pp = __ldg(P + k1 * K2 + o);
    const float2 bh = Bh[bi];
    const double2 v = vs[bi];
    const double xr = x.x, xi = x.y, br = bh.x, bim = bh.y;
    const double rr = rhoL * pp.x, ri = rhoL * pp.y;
    double cr = __fma_rn(d.x, xr, -d.y * xi) + __fma_rn(pp.x, br, -pp.y * bim);
    double ci = __fma_rn(d.x, xi, d.y * xr) + __fma_rn(pp.x, bim, pp.y * br);
    cr -= __fma_rn(rr, v.x, -ri * v.y);
    ci -= __fma_rn(rr, v.y, ri * v.x);
    const double2 vn = make_double2(v.x + cr, v.y + ci);
    vs[bi] = vn;
    if (cb_out) cb_out[bi] = make_double2(cr, ci);
    return make_float2((float)vn.x, (float)vn.y);
  }
};

template <int KP>
__global__ void __launch_bounds__(KP <= 8 ? 1024 : 256) cols_admm_split_kernel(Geo G, AxisT<float2> ax,
                                                                             ColsIO<float2> io, AdmmSplitBand op) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cols_block<KP, float2, true, AdmmSplitBand>(G, ax, io, (long long)blockIdx.x * G.TR, G.TR,
                                               reinterpret_cast<float2*>(smem_raw), op);
}

// Box input at engine precision for a synthesis column pass (y = box[line][o]).
template <typename C>
struct BoxIn {
  const C* __restrict__ box;   // [B][K1][K2]
  int K2;
  __device__ __forceinline__ C operator()(long long line, int o, C) const { return box[line * K2 + o]; }
};

template <int KP, typename C>
__global__ void __launch_bounds__(KP <= 8 ? 1024 : 256) cols_box_kernel(Geo G, AxisT<C> ax, ColsIO<C> io,
                                                                      BoxIn<C> op) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cols_block<KP, C, true, BoxIn<C>>(G, ax, io, (long long)blockIdx.x * G.TR, G.TR, reinterpret_cast<C*>(smem_raw),
                                    op);
}

// Epilogue of the split-ADMM finalisation: out = alpha (x1 - x2) + g (c = a (z - r) + IFFT2u(Cb))
// or, with x2 = null, out = x1 + g (v = r + IFFT2u(vs)).
struct EpiCombine {
  const double2* x1;
  const double2* x2;
  double2* out;
  double alpha;
  __device__ __forceinline__ double2 load(long long pos, int) const { return x1[pos]; }
  __device__ __forceinline__ double2 update(long long pos, int, double2 g) const {
    const double2 a1 = x1[pos];
    double2 o;
    if (x2) {
      const double2 a2 = x2[pos];
      o = make_double2(__fma_rn(alpha, a1.x - a2.x, g.x), __fma_rn(alpha, a1.y - a2.y, g.y));
    } else {
      o = make_double2(a1.x + g.x, a1.y + g.y);
    }
    out[pos] = o;
    return o;
  }
};

// cp.async (LDGSTS): per-thread asynchronous global -> shared copies that hold no registers
// while in flight.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// ---------------------------------------------------------------- specialised pass A (ADMM)
// Complex128 engine, compile-time line shape (KP <= 16, R, MO).  State: z (complex64, sparse:
// zero-segment flags as in the FISTA kernel) and the scaled dual v (complex128, dense, always
// streamed).  Per point (solvers.py:426-430): u = z - v; c = a*u + g (+ q folded in g);
// z' = S_{rho tau}(c + v); v' = v + (c - z'); next operator input u' = z' - v'.
template <int KP, int R, int MO, bool ZS>
__global__ void __launch_bounds__(R > 256 ? R : 256, R > 256 ? 1 : 2)
    rows_admm_fast_kernel(Geo G, AxisT<double2> ax, RowsIO<double2> io, EpiAdmm epi, unsigned* __restrict__ flags) {
  pdl_wait();
  constexpr int NT = R > 256 ? R : 256;
  constexpr int TR = NT / R;
  constexpr int K = KP * MO;
  constexpr int XP = K + 1;
  constexpr int PITCH = (R % 2 == 1) ? R : R + 1;
  constexpr int SP = KP * PITCH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Xs = reinterpret_cast<double2*>(smem_raw);
  double2* S = Xs + TR * XP;
  const int tid = threadIdx.x, lane = tid & 31;
  const int ii = tid / R, s = tid % R;
  const int row0 = blockIdx.x * TR;
  const int gr = row0 + ii;
  const bool active = gr < (int)G.rows;
  const int L2 = G.L2;
  const int b = row0 / L2;
  const int l20 = row0 - b * L2;
  const long long vbase = (long long)b * K * L2 + l20;
  double2* zp = epi.z + (long long)gr * G.L1 + s;
  double2* vp = epi.v + (long long)gr * G.L1 + s;
  double2* cop = epi.c_out ? epi.c_out + (long long)gr * G.L1 + s : nullptr;
  const double kap = epi.kscale * epi.tau[b];
  const double kap2 = kap * kap;
  const double a_id = epi.a;
  unsigned* fw = ZS ? flags + ((long long)blockIdx.x * (NT / 32) + (tid >> 5)) : nullptr;
  const unsigned fl = ZS ? __ldcg(fw) : 0xffffffffu;
  double2 a[KP];

  // The dense dual v streams through shared memory: all KP values of a thread are requested
  // with cp.async before the band inverse runs (no registers held; the fp64 inverse DFT hides
  // the latency).  The staging aliases the transpose buffer S, which is free until the forward.
  double2* vstage = S;   // [KP][NT]
  if (G.do_inv) {
    if (active) {
#pragma unroll
      for (int r = 0; r < KP; ++r) cp_async16(vstage + r * NT + tid, vp + r * R);
    }
    cp_async_commit();
    for (int idx = tid; idx < TR * K; idx += NT) {
      const int k = idx / TR, i2 = idx % TR;
      Xs[i2 * XP + k] = io.V[vbase + (long long)k * L2 + i2];
    }
    double2 z0 = make_double2(0.0, 0.0), z1 = z0;
    if (active) {
      if (fl & 1u) z0 = zp[0];
      if ((fl >> 1) & 1u) z1 = zp[R];
    }
    __syncthreads();
    {
      const double2* Y = Xs + ii * XP;
#pragma unroll
      for (int j = 0; j < KP; ++j) a[j] = Y[j];
#pragma unroll
      for (int m = 1; m < MO; ++m) {
        const double2 w2 = __ldg(ax.tw2 + m * R + s);
#pragma unroll
        for (int j = 0; j < KP; ++j) a[j] = cadd(a[j], cmulc(Y[j + KP * m], w2));
      }
#pragma unroll
      for (int j = 0; j < KP; ++j) a[j] = cmulc(a[j], __ldg(ax.tw1 + j * R + s));
      reg_dft<KP, true>(a);
    }
    cp_async_wait_all();   // this thread's v values have landed
    unsigned nfl = 0;
#pragma unroll
    for (int r = 0; r < KP; ++r) {
      const double2 zz = z0;
      const double2 vv = active ? vstage[r * NT + tid] : make_double2(0.0, 0.0);
      z0 = z1;
      if (r + 2 < KP && active) z1 = ((fl >> (r + 2)) & 1u) ? zp[(r + 2) * R] : make_double2(0.0, 0.0);
      const double2 g = a[r];
      const double cr = __fma_rn(a_id, zz.x - vv.x, g.x);
      const double ci = __fma_rn(a_id, zz.y - vv.y, g.y);
      if (active && !isfinite(cr + ci)) atomicMin(epi.first_bad + b, epi.it);
      const double sr = cr + vv.x, si = ci + vv.y;
      const double m2 = sr * sr + si * si;
      double2 zn = make_double2(0.0, 0.0);
      if (!(m2 <= kap2)) {
        const double f = 1.0 - kap * rsqrt(m2);
        zn = make_double2(sr * f, si * f);
      }
      // v' = v + (c - z') (bitwise identity of test_solvers.py:283-295)
      const double2 vn = make_double2(vv.x + (cr - zn.x), vv.y + (ci - zn.y));
      if (active) {
        vp[r * R] = vn;
        if (cop) cop[r * R] = make_double2(cr, ci);
      }
      if (ZS) {
        const bool nzv = (zn.x != 0.0) | (zn.y != 0.0);
        if (__any_sync(0xffffffffu, nzv)) {
          if (active) zp[r * R] = zn;
          nfl |= 1u << r;
        }
      } else if (active) {
        zp[r * R] = zn;
      }
      a[r] = make_double2(zn.x - vn.x, zn.y - vn.y);
    }
    if (ZS && lane == 0 && (nfl | fl)) *fw = nfl;   // (a clear word stays clear: no store)
  } else if (active) {
#pragma unroll
    for (int r = 0; r < KP; ++r) {
      const double2 zz = ((fl >> r) & 1u) ? zp[r * R] : make_double2(0.0, 0.0);
      const double2 vv = vp[r * R];
      a[r] = make_double2(zz.x - vv.x, zz.y - vv.y);
    }
  }
  if (!G.do_fwd) return;
  __syncthreads();   // every thread is done with its v staging (aliases S)
  if (active) {
    reg_dft<KP, false>(a);
    double2* Srow = S + ii * SP;
#pragma unroll
    for (int j = 0; j < KP; ++j) Srow[j * PITCH + s] = cmul(a[j], __ldg(ax.tw1 + j * R + s));
  }
  __syncthreads();
  for (int idx = tid; idx < TR * K; idx += NT) {
    const int i2 = idx / K, o = idx % K;
    const int j = o % KP, m = o / KP;
    const double2* row = S + i2 * SP + j * PITCH;
    double2 acc = make_double2(0.0, 0.0);
    if (m == 0) {
#pragma unroll 8
      for (int t = 0; t < R; ++t) acc = cadd(acc, row[t]);
    } else {
      const double2* tw = ax.tw2 + m * R;
#pragma unroll 8
      for (int t = 0; t < R; ++t) acc = cfma(row[t], __ldg(tw + t), acc);
    }
    Xs[i2 * XP + o] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < TR * K; idx += NT) {
    const int k = idx / TR, i2 = idx % TR;
    if (row0 + i2 < (int)G.rows) io.U[vbase + (long long)k * L2 + i2] = Xs[i2 * XP + k];
  }
}

// Final zero pass for z of a zero-skipping ADMM run.
template <int KP, int R>
__global__ void __launch_bounds__(R > 256 ? R : 256) zero_segments_z_kernel(Geo G, double2* z,
                                                                            const unsigned* __restrict__ flags) {
  pdl_wait();
  constexpr int NT = R > 256 ? R : 256;
  constexpr int TR = NT / R;
  const int tid = threadIdx.x;
  const int ii = tid / R, s = tid % R;
  const int gr = blockIdx.x * TR + ii;
  if (gr >= (int)G.rows) return;
  const unsigned fl = flags[(long long)blockIdx.x * (NT / 32) + (tid >> 5)];
  double2* zp = z + (long long)gr * G.L1 + s;
#pragma unroll
  for (int r = 0; r < KP; ++r)
    if (!((fl >> r) & 1u)) zp[r * R] = make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------- small-grid persistent solver
// K5 of SURVEY.md: when a snapshot's whole state fits in shared memory (config 1: 64 x 64,
// c 64 KB + d 32 KB), one CTA per snapshot runs ALL T iterations in one launch: rows pass
// (band IFFT of V, fused epilogue, band FFT -> U), then the column pass (U -> V), both out of
// shared memory, separated only by __syncthreads.  No HBM traffic and no launches per iteration.
struct SmallArgs {
  AxisT<float2> ax1;      // rows axis (complex64 engine)
  AxisT<float2> ax2;      // columns axis (KP <= 16 engine)
  ColsIO<float2> cio;     // D, P, Bh (global); U, V replaced by shared arrays in the kernel
  EpiFista epi;           // c, d (global, per batch), tau, first_bad, a, kscale
  const double* beta;     // [T + 1] momentum coefficients (FISTA)
  int L1, L2, K1, K2;
  int iterations, first_iteration;
  int TRc;                // column lines per block pass
};

template <int KP1, int KP2, bool MOM>
__global__ void __launch_bounds__(1024, 1) small_fista_kernel(SmallArgs A) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L1 = A.L1, L2 = A.L2, L = L1 * L2, K1 = A.K1;
  const int b = blockIdx.x;
  // shared layout: c [L] double2 | d [L] float2 | U [K1*L2] | V [K1*L2] | scratch
  double2* cs = reinterpret_cast<double2*>(smem_raw);
  float2* ds = reinterpret_cast<float2*>(cs + L);
  float2* Us = ds + (MOM ? L : 0);
  float2* Vs = Us + K1 * L2;
  float2* scratch = Vs + K1 * L2;
  const int tid = threadIdx.x, nthr = blockDim.x;
  double2* cg = A.epi.c + (long long)b * L;
  float2* dg = MOM ? A.epi.d + (long long)b * L : nullptr;
  for (int i = tid; i < L; i += nthr) {
    cs[i] = cg[i];
    if (MOM) ds[i] = dg[i];
  }
  EpiFista e = A.epi;
  e.c = cs;                      // shared-memory state; positions are local to the snapshot
  e.d = MOM ? ds : nullptr;
  e.extra = nullptr;
  e.tau = A.epi.tau + b;         // the epilogue indexes tau[0] / first_bad[0] for this CTA
  e.first_bad = A.epi.first_bad + b;
  const AxisT<float2>& ax = A.ax1;
  const int R = ax.R, K = ax.K, TR = L2;   // all rows of the snapshot at once
  const double kap = e.kscale * e.tau[0];
  const float kap2_lo = (float)(kap * kap) * (1.0f - 1.0f / 262144.0f);
  const int ii = tid / R, s = tid % R;
  const bool active = tid < TR * R;
  float2* Xs = scratch;
  float2* S = scratch + TR * (K + 1);
  const int SP = KP1 * ax.pitch;
  // column pass geometry (one snapshot, lines = K1), shared-memory U / V
  ColsIO<float2> cio = A.cio;
  cio.U = Us;
  cio.V = Vs;
  cio.Bh = A.cio.Bh + (long long)b * K1 * A.K2;
  Geo gc;
  gc.L1 = L1;
  gc.L2 = L2;
  gc.rows = K1;
  gc.TR = A.TRc;
  gc.do_fwd = 1;
  gc.do_inv = 1;
  __syncthreads();
  const int t_end = A.first_iteration + A.iterations;
  for (int t = A.first_iteration - 1; t < t_end; ++t) {
    const bool inv = t >= A.first_iteration;
    const bool fwd = t + 1 < t_end;
    float2 a[KP1];
    // ---- rows pass: V (shared, [k1][l2]) -> per-line band tile -> g -> epilogue -> forward
    if (inv) {
      for (int idx = tid; idx < TR * K; idx += nthr) {
        const int k = idx / TR, i2 = idx % TR;
        Xs[i2 * (K + 1) + k] = Vs[k * L2 + i2];
      }
      __syncthreads();
      if (active) band_inverse<KP1>(Xs + ii * (K + 1), s, ax, a);
    }
    if (active) {
      e.it = t;
      e.beta_cur = MOM ? A.beta[inv ? t : A.first_iteration] : 0.0;
      e.beta_next = MOM ? A.beta[t + 1] : 0.0;
#pragma unroll
      for (int r = 0; r < KP1; ++r) {
        const int pos = ii * L1 + s + R * r;
        if (inv) {
          const double2 cc = cs[pos];
          const float2 dd = MOM ? ds[pos] : make_float2(0.f, 0.f);
          const float2 g = a[r];
          // zero fast path (bitwise identical, see rows_fista_fast_kernel)
          if ((cc.x == 0.0) & (cc.y == 0.0) & (!MOM | ((dd.x == 0.f) & (dd.y == 0.f))) &&
              fmaf(g.x, g.x, g.y * g.y) < kap2_lo) {
            a[r] = make_float2(0.f, 0.f);
            continue;
          }
          double2 cn;
          float2 dn;
          a[r] = e.step(cc, dd, g, make_float2(0.f, 0.f), 0, cn, dn);
          cs[pos] = cn;
          if (MOM) ds[pos] = dn;
        } else {
          a[r] = e.load(pos, 0);
        }
      }
    }
    if (!fwd) break;
    __syncthreads();
    if (active) {
      reg_dft<KP1, false>(a);
      band_fwd_scatter<KP1>(a, s, ax, S + ii * SP);
    }
    __syncthreads();
    for (int idx = tid; idx < TR * K; idx += nthr) {
      const int i2 = idx / K, o = idx % K;
      Xs[i2 * (K + 1) + o] = band_fwd_output(S + i2 * SP, o, KP1, ax);
    }
    __syncthreads();
    for (int idx = tid; idx < TR * K; idx += nthr) {
      const int k = idx / TR, i2 = idx % TR;
      Us[k * L2 + i2] = Xs[i2 * (K + 1) + k];
    }
    __syncthreads();
    // ---- column pass: U -> V (all K1 lines of this snapshot)
    for (int l0 = 0; l0 < K1; l0 += A.TRc) cols_block<KP2, float2, false>(gc, A.ax2, cio, l0, A.TRc, scratch);
    __syncthreads();
  }
  __syncthreads();
  for (int i = tid; i < L; i += nthr) {
    cg[i] = cs[i];
    if (MOM) dg[i] = ds[i];
  }
}

// ---------------------------------------------------------------- 64 x 64 cluster solver
// Config-1 shape (L1 = L2 = 64, band K1, K2 <= 16, multiples of 8): one thread-block CLUSTER of
// 8 CTAs per snapshot runs all T iterations in one launch.  CTA r owns rows [8r, 8r+8) and the
// column lines k1 in [r*K1/8, (r+1)*K1/8).  Band tiles move between CTAs through distributed
// shared memory (map_shared_rank), two cluster barriers per iteration; the state never leaves
// shared memory.  With lines of 64 points and bands of 16, direct band DFTs on the constant
// 64th-root table are shorter dependency chains than FFT stages.
struct ClusterArgs {
  const float2* D;       // [K1][K2]
  const float2* P;       // [K1][K2]
  const float2* Bh;      // [B][K1][K2]
  EpiFista epi;
  const double* beta;    // [T + 1]
  int K1, K2, iterations, first_iteration;
};


template <bool MOM>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256, 1) cluster64_fista_kernel(ClusterArgs A) {
  pdl_wait();
  namespace cgp = cooperative_groups;
  constexpr int L = 64, CL = 8, RPC = L / CL;
  cgp::cluster_group cluster = cgp::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CL;
  const int K1 = A.K1, K2 = A.K2, LPC = K1 / CL;   // column lines per CTA
  const int tid = threadIdx.x;
  __shared__ double2 cs[RPC * L];
  __shared__ float2 ds[RPC * L];
  __shared__ float2 xs[RPC * L];       // next operator input (forward DFT input)
  __shared__ float2 Ul[16 * RPC];      // my rows' band: [k1][row]
  __shared__ float2 Vl[16 * RPC];      // band input of my rows: [k1][row]
  __shared__ float2 Vline[2 * L];      // my column lines after the column pass: [j][l2]
  __shared__ float2 line[2 * L];       // my column lines gathered from U: [j][l2]
  __shared__ float2 Yb[2 * 16];        // band values of my lines: [j][k2]
  __shared__ float2 roots[64];         // e^{-2 pi i t / 64}: lane-varying indices -> shared, not constant
  if (tid < 64) roots[tid] = c_roots64[tid];
  auto w64 = [&](int t) { return roots[t & 63]; };
  const long long base = ((long long)b * L + rank * RPC) * L;
  for (int i = tid; i < RPC * L; i += 256) {
    cs[i] = A.epi.c[base + i];
    ds[i] = MOM ? A.epi.d[base + i] : make_float2(0.f, 0.f);
  }
  EpiFista e = A.epi;
  e.c = cs;
  e.d = MOM ? ds : nullptr;
  e.extra = nullptr;
  e.tau = A.epi.tau + b;
  e.first_bad = A.epi.first_bad + b;
  const double kap = e.kscale * e.tau[0];
  const float kap2_lo = (float)(kap * kap) * (1.0f - 1.0f / 262144.0f);
  const float2* Bh = A.Bh + (long long)b * K1 * K2;
  // loop-invariant spectral data of my column lines, hoisted out of global memory
  __shared__ float2 Dl[2 * 16], PB[2 * 16];
  for (int q = tid; q < LPC * K2; q += 256) {
    const int j = q / K2, k2 = q % K2, k1 = rank * LPC + j;
    Dl[j * 16 + k2] = A.D[k1 * K2 + k2];
    PB[j * 16 + k2] = cmul(Bh[k1 * K2 + k2], A.P[k1 * K2 + k2]);
  }
  FistaScalars sc{kap, e.a, 0.0, 0, 0, e.first_bad};
  __syncthreads();
  const int t_end = A.first_iteration + A.iterations;
  for (int t = A.first_iteration - 1; t < t_end; ++t) {
    const bool inv = t >= A.first_iteration;
    const bool fwd = t + 1 < t_end;
    e.it = t;
    e.beta_cur = MOM ? A.beta[inv ? t : A.first_iteration] : 0.0;
    e.beta_next = MOM ? A.beta[t + 1] : 0.0;
    sc.bc = e.beta_cur;
    sc.it = t;
    const float bn = (float)e.beta_next;
    // ---- rows: inverse band DFT (direct), fused epilogue -> xs
    for (int p = tid; p < RPC * L; p += 256) {
      const int i = p / L, l1 = p % L;
      float2 x;
      if (inv) {
        float2 g = make_float2(0.f, 0.f);
        for (int k = 0; k < K1; ++k) g = cfma(Vl[k * RPC + i], cmake(w64(l1 * k).x, -w64(l1 * k).y), g);
        const double2 cc = cs[p];
        const float2 dd = MOM ? ds[p] : make_float2(0.f, 0.f);
        if ((cc.x == 0.0) & (cc.y == 0.0) & (!MOM | ((dd.x == 0.f) & (dd.y == 0.f))) &&
            fmaf(g.x, g.x, g.y * g.y) < kap2_lo) {
          x = make_float2(0.f, 0.f);
        } else {
          float2 dn = make_float2(0.f, 0.f);
          const double2 cn = fista_point_slow<MOM>(cc, dd, g, sc, &dn);
          cs[p] = cn;
          if (MOM) ds[p] = dn;
          x = MOM ? make_float2(fmaf(bn, dn.x, (float)cn.x), fmaf(bn, dn.y, (float)cn.y))
                  : make_float2((float)cn.x, (float)cn.y);
        }
      } else {
        x = e.load(p, 0);
      }
      xs[p] = x;
    }
    if (!fwd) break;
    __syncthreads();
    // ---- rows: forward band DFT, U[k1][row] (2 lanes per output, 32 terms each)
    for (int q = tid; q < 2 * K1 * RPC; q += 256) {
      const int o = q >> 1, h = q & 1;
      const int k = o / RPC, i = o % RPC;
      float2 acc = make_float2(0.f, 0.f);
      for (int l1 = h * 32; l1 < h * 32 + 32; ++l1) acc = cfma(xs[i * L + l1], w64(l1 * k), acc);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      if (h == 0) Ul[k * RPC + i] = acc;
    }
    cluster.sync();   // every CTA's U tile is published
    // ---- columns: gather my lines from the 8 row owners (DSMEM)
    for (int q = tid; q < LPC * L; q += 256) {
      const int j = q / L, l2 = q % L;
      const int k1 = rank * LPC + j;
      const float2* src = cluster.map_shared_rank(Ul, l2 / RPC);
      line[j * L + l2] = src[k1 * RPC + (l2 % RPC)];
    }
    __syncthreads();
    // forward column DFT to the band (8 lanes per output), spectral multiply-add
    for (int q = tid; q < LPC * K2 * 8; q += 256) {
      const int o = q >> 3, h = q & 7;
      const int j = o / K2, k2 = o % K2;
      float2 acc = make_float2(0.f, 0.f);
      for (int l2 = h * 8; l2 < h * 8 + 8; ++l2) acc = cfma(line[j * L + l2], w64(l2 * k2), acc);
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      }
      if (h == 0) Yb[j * 16 + k2] = cadd(cmul(acc, Dl[j * 16 + k2]), PB[j * 16 + k2]);
    }
    __syncthreads();
    // inverse column DFT of the band -> Vline[j][l2]
    for (int q = tid; q < LPC * L; q += 256) {
      const int j = q / L, l2 = q % L;
      float2 acc = make_float2(0.f, 0.f);
      for (int k2 = 0; k2 < K2; ++k2) acc = cfma(Yb[j * 16 + k2], cmake(w64(l2 * k2).x, -w64(l2 * k2).y), acc);
      Vline[q] = acc;
    }
    cluster.sync();   // every CTA's column lines are published
    // ---- gather the band input of my rows from the line owners (DSMEM)
    for (int q = tid; q < K1 * RPC; q += 256) {
      const int k1 = q / RPC, i = q % RPC;
      const float2* src = cluster.map_shared_rank(Vline, k1 / LPC);
      Vl[q] = src[(k1 % LPC) * L + rank * RPC + i];
    }
    __syncthreads();
  }
  cluster.sync();   // no CTA may exit while others still read its shared memory
  for (int i = tid; i < RPC * L; i += 256) {
    A.epi.c[base + i] = cs[i];
    if (MOM) A.epi.d[base + i] = ds[i];
  }
}

// Final pass of a zero-skipping run: write the zeros of every clear segment back so c (and d)
// are dense, consistent arrays again.
template <int KP, int R, typename T2 = float2, int NTMIN = 256>
__global__ void __launch_bounds__(R > NTMIN ? R : NTMIN) zero_segments_kernel(Geo G, double2* c, T2* d,
                                                                              const unsigned* __restrict__ flags) {
  pdl_wait();
  constexpr int NT = R > NTMIN ? R : NTMIN;
  constexpr int TR = NT / R;
  const int tid = threadIdx.x;
  const int ii = tid / R, s = tid % R;
  const int gr = blockIdx.x * TR + ii;
  if (gr >= (int)G.rows) return;
  const unsigned fl = flags[(long long)blockIdx.x * (NT / 32 + 1) + (tid >> 5)];   // rows_tile layout
  double2* cp = c + (long long)gr * G.L1 + s;
  T2* dp = d ? d + (long long)gr * G.L1 + s : nullptr;
#pragma unroll
  for (int r = 0; r < KP; ++r)
    if (!((fl >> r) & 1u)) {
      cp[r * R] = make_double2(0.0, 0.0);
      if (dp) dp[r * R] = T2{};
    }
}

// Pass A for ADMM (complex128 engine).
template <int KP, int CH>
__global__ void __launch_bounds__(256) rows_admm_kernel(Geo G, AxisT<double2> ax, RowsIO<double2> io,
                                                        EpiAdmm epi) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw);
  const int R = ax.R, K = ax.K;
  const int ii = threadIdx.x / R, s = threadIdx.x - ii * R;
  const long long row0 = (long long)blockIdx.x * G.TR;
  const long long gr = row0 + ii;
  const bool active = (ii < G.TR) && (gr < G.rows);
  double2* Xs = smem;
  double2* S = smem + G.TR * (K + 1);
  double2 a[KP];
  if (G.do_inv) {
    rows_load_band(G, ax, io, Xs, row0);
    __syncthreads();
    if (active) band_inverse<KP>(Xs + ii * (K + 1), s, ax, a);
  }
  if (active) {
    const long long base = gr * G.L1 + s;
    const int b = (int)(gr / G.L2);
    if (!G.do_inv) {
#pragma unroll
      for (int r = 0; r < KP; ++r) a[r] = epi.load(base + (long long)R * r, b);
    } else {
      double2 zb[CH], vb[CH];
      float2 eb[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const long long pos = base + (long long)R * q;
        zb[q] = epi.z[pos];
        vb[q] = epi.v[pos];
        eb[q] = epi.extra ? epi.extra[pos] : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int r0 = 0; r0 < KP; r0 += CH) {
        double2 zn[CH], vn[CH];
        float2 en[CH];
        if (r0 + CH < KP) {
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const long long pos = base + (long long)R * (r0 + CH + q);
            zn[q] = epi.z[pos];
            vn[q] = epi.v[pos];
            en[q] = epi.extra ? epi.extra[pos] : make_float2(0.f, 0.f);
          }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const long long pos = base + (long long)R * (r0 + q);
          double2 znew, vnew, cc;
          a[r0 + q] = epi.step(zb[q], vb[q], a[r0 + q], eb[q], b, znew, vnew, cc);
          epi.z[pos] = znew;
          epi.v[pos] = vnew;
          if (epi.c_out) epi.c_out[pos] = cc;
        }
        if (r0 + CH < KP) {
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            zb[q] = zn[q];
            vb[q] = vn[q];
            eb[q] = en[q];
          }
        }
      }
    }
  }
  if (G.do_fwd) {
    if (G.do_inv) __syncthreads();
    rows_forward_store<KP>(G, ax, io, a, active, ii, s, Xs, S, row0);
  }
}

}  // namespace bccb
