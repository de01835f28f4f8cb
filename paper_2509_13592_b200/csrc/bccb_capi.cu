// C ABI + launch sequencing for the B200-native BCCB Gram operator.
// See include/bccb_b200.h for the interface and the reference functions replaced.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bccb_b200.h"
#include "bccb_kernels.cuh"
#include "topk.cuh"

using namespace bccb;

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(BCCB_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define LAUNCH_CHECK()                                                                   \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(BCCB_ERR_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                   \
  } while (0)

extern "C" const char* bccb_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* bccb_version(void) { return "bccb_b200 0.1.0 (sm_100a)"; }

// ------------------------------------------------------------------ device init
static std::mutex g_init_mu;
static bool g_roots_ready[64];

static int ensure_device_constants(int device) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (device < 0 || device >= 64) return fail(BCCB_ERR_INVALID, "bad device %d", device);
  if (g_roots_ready[device]) return BCCB_OK;
  float2 roots[64];
  for (int t = 0; t < 64; ++t) {
    const double ang = -2.0 * M_PI * t / 64.0;
    roots[t] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  CUDA_TRY(cudaMemcpyToSymbol(c_roots64, roots, sizeof(roots)));
  g_roots_ready[device] = true;
  return BCCB_OK;
}

// ------------------------------------------------------------------ plan
struct AxisHost {
  int N = 0, K = 0, KP = 1, R = 1, Mo = 1, pitch = 1;
  float2* tw1 = nullptr;
  float2* tw2 = nullptr;
  Axis dev() const {
    Axis a;
    a.N = N;
    a.K = K;
    a.KP = KP;
    a.R = R;
    a.Mo = Mo;
    a.pitch = pitch;
    a.tw1 = tw1;
    a.tw2 = tw2;
    return a;
  }
};

struct bccb_plan_s {
  int device = 0;
  int L1 = 0, L2 = 0;
  AxisHost ax1, ax2;               // rows (N = L1, K = K1), columns (N = L2, K = K2)
  std::vector<std::complex<double>> box;  // [K1][K2]
  std::complex<double> lam_out{0.0, 0.0};
  double2* lam_box_dev = nullptr;  // [K1][K2]
  int M = 0;                       // occupied elements (Gram plans)
  int* occ_dev = nullptr;          // [3][M]: m1, m2 (reduced mod L1 / L2), (m1 + m2) & 1
  int occ_alias = 0;               // some occupied cells alias (M1 > L1 or M2 > L2)
  bool full() const { return ax1.K == L1 && ax2.K == L2; }
};

static int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}
static int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p *= 2;
  return p;
}

// Choose the register DFT size KP (largest power of two dividing N, <= 32 and <= the band),
// round the band up to a multiple of KP and build the twiddle tables in double precision.
static int make_axis(int N, int Kreq, AxisHost& ax) {
  int KP = 1;
  while (KP < KP_MAX && N % (KP * 2) == 0) KP *= 2;
  KP = std::min(KP, pow2_ceil(std::max(1, Kreq)));
  int K = ((Kreq + KP - 1) / KP) * KP;
  K = std::min(K, N);
  if (K % KP != 0) K = N;  // N is a multiple of KP
  const int R = N / KP;
  if (R > 1024)
    return fail(BCCB_ERR_UNSUPPORTED,
                "grid length %d needs %d threads per line (> 1024); use a length with a larger "
                "power-of-two factor",
                N, R);
  ax.N = N;
  ax.K = K;
  ax.KP = KP;
  ax.R = R;
  ax.Mo = K / KP;
  ax.pitch = (R % 2 == 1) ? R : R + 1;
  std::vector<float2> t1((size_t)KP * R), t2((size_t)ax.Mo * R);
  for (int j = 0; j < KP; ++j)
    for (int s = 0; s < R; ++s) {
      // w_N^{s j}; reduce the exponent mod N in integers for accuracy
      const long long e = ((long long)s * j) % N;
      const double ang = -2.0 * M_PI * (double)e / (double)N;
      t1[(size_t)j * R + s] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
  for (int m = 0; m < ax.Mo; ++m)
    for (int s = 0; s < R; ++s) {
      const long long e = ((long long)s * m) % R;
      const double ang = -2.0 * M_PI * (double)e / (double)R;
      t2[(size_t)m * R + s] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
  CUDA_TRY(cudaMalloc(&ax.tw1, t1.size() * sizeof(float2)));
  CUDA_TRY(cudaMalloc(&ax.tw2, t2.size() * sizeof(float2)));
  CUDA_TRY(cudaMemcpy(ax.tw1, t1.data(), t1.size() * sizeof(float2), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(ax.tw2, t2.data(), t2.size() * sizeof(float2), cudaMemcpyHostToDevice));
  return BCCB_OK;
}

static void free_plan(bccb_plan_s* p) {
  if (!p) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(p->device);
  cudaFree(p->ax1.tw1);
  cudaFree(p->ax1.tw2);
  cudaFree(p->ax2.tw1);
  cudaFree(p->ax2.tw2);
  cudaFree(p->lam_box_dev);
  cudaFree(p->occ_dev);
  cudaSetDevice(cur);
  delete p;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Common tail of plan creation: axes, box upload.
static int finish_plan(bccb_plan_s* p, int k1req, int k2req) {
  int rc = ensure_device_constants(p->device);
  if (rc) return rc;
  if ((rc = make_axis(p->L1, k1req, p->ax1))) return rc;
  if ((rc = make_axis(p->L2, k2req, p->ax2))) return rc;
  return BCCB_OK;
}

static int upload_box(bccb_plan_s* p, const std::vector<std::complex<double>>& box_req, int k1req,
                      int k2req) {
  // re-embed the requested box into the (possibly rounded-up) plan box
  const int K1 = p->ax1.K, K2 = p->ax2.K;
  p->box.assign((size_t)K1 * K2, p->lam_out);
  for (int a = 0; a < std::min(k1req, K1); ++a)
    for (int b = 0; b < std::min(k2req, K2); ++b) p->box[(size_t)a * K2 + b] = box_req[(size_t)a * k2req + b];
  if (p->full()) p->lam_out = 0.0;
  std::vector<double2> h(p->box.size());
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_double2(p->box[i].real(), p->box[i].imag());
  CUDA_TRY(cudaMalloc(&p->lam_box_dev, h.size() * sizeof(double2)));
  CUDA_TRY(cudaMemcpy(p->lam_box_dev, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  return BCCB_OK;
}

extern "C" int bccb_plan_create(int l1, int l2, int k1, int k2, const double* box_t,
                                double lam_out_re, double lam_out_im, int device,
                                bccb_plan_t* out) {
  if (!out) return fail(BCCB_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (l1 < 1 || l2 < 1) return fail(BCCB_ERR_INVALID, "block sizes must be positive");
  if (k1 < 1 || k2 < 1 || k1 > l1 || k2 > l2)
    return fail(BCCB_ERR_INVALID, "box (%d, %d) outside the grid (%d, %d)", k1, k2, l1, l2);
  if (!box_t) return fail(BCCB_ERR_INVALID, "box is NULL");
  DeviceGuard dg(device);
  auto* p = new bccb_plan_s();
  p->device = device;
  p->L1 = l1;
  p->L2 = l2;
  p->lam_out = {lam_out_re, lam_out_im};
  std::vector<std::complex<double>> req((size_t)k1 * k2);
  for (size_t i = 0; i < req.size(); ++i) req[i] = {box_t[2 * i], box_t[2 * i + 1]};
  // A complex value outside a partial box would need a complex identity coefficient in the
  // fused epilogues; use the full grid instead (rare: shifted operators with complex beta).
  const bool partial = (k1 < l1 || k2 < l2);
  int kk1 = k1, kk2 = k2;
  if (partial && lam_out_im != 0.0) {
    std::vector<std::complex<double>> fullbox((size_t)l1 * l2, p->lam_out);
    for (int a = 0; a < k1; ++a)
      for (int b = 0; b < k2; ++b) fullbox[(size_t)a * l2 + b] = req[(size_t)a * k2 + b];
    req.swap(fullbox);
    kk1 = l1;
    kk2 = l2;
  }
  int rc = finish_plan(p, kk1, kk2);
  if (!rc) rc = upload_box(p, req, kk1, kk2);
  if (rc) {
    free_plan(p);
    return rc;
  }
  *out = p;
  return BCCB_OK;
}

extern "C" int bccb_plan_create_gram(int l1, int l2, int m1_count, int m2_count,
                                     const uint8_t* occupancy, int device, bccb_plan_t* out) {
  if (!out) return fail(BCCB_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (l1 < 1 || l2 < 1) return fail(BCCB_ERR_INVALID, "grid lengths must be positive");
  if (m1_count < 1 || m2_count < 1 || !occupancy)
    return fail(BCCB_ERR_INVALID, "geometry needs positive extents and an occupancy array");
  // occupied coordinates in scan order (m2 outer, m1 inner) — arrays.py:55-62
  std::vector<int> m1s, m2s;
  for (int b = 0; b < m2_count; ++b)
    for (int a = 0; a < m1_count; ++a)
      if (occupancy[(size_t)a * m2_count + b]) {
        m1s.push_back(a);
        m2s.push_back(b);
      }
  if (m1s.empty()) return fail(BCCB_ERR_INVALID, "geometry needs at least one occupied element");
  DeviceGuard dg(device);
  auto* p = new bccb_plan_s();
  p->device = device;
  p->L1 = l1;
  p->L2 = l2;
  p->lam_out = 0.0;
  p->M = (int)m1s.size();
  // eigenvalues = L * (number of occupied cells aliasing to (k1, k2)); finding 3 of SURVEY.md
  const int e1 = std::min(m1_count, l1), e2 = std::min(m2_count, l2);
  std::vector<std::complex<double>> req((size_t)e1 * e2, 0.0);
  const double L = (double)l1 * (double)l2;
  for (size_t i = 0; i < m1s.size(); ++i) req[(size_t)(m1s[i] % l1) * e2 + (m2s[i] % l2)] += L;
  p->occ_alias = (m1_count > l1 || m2_count > l2) ? 1 : 0;
  int rc = finish_plan(p, e1, e2);
  if (!rc) rc = upload_box(p, req, e1, e2);
  if (!rc) {
    std::vector<int> occ(3 * (size_t)p->M);
    for (int i = 0; i < p->M; ++i) {
      occ[i] = m1s[i] % l1;
      occ[p->M + i] = m2s[i] % l2;
      occ[2 * p->M + i] = (m1s[i] + m2s[i]) & 1;  // sign (-1)^(m1+m2) of the unreduced cell
    }
    cudaError_t e = cudaMalloc(&p->occ_dev, occ.size() * sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(p->occ_dev, occ.data(), occ.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) rc = fail(BCCB_ERR_CUDA, "occupancy upload: %s", cudaGetErrorString(e));
  }
  if (rc) {
    free_plan(p);
    return rc;
  }
  *out = p;
  return BCCB_OK;
}

extern "C" int bccb_plan_destroy(bccb_plan_t plan) {
  free_plan(plan);
  return BCCB_OK;
}

extern "C" int bccb_plan_info(bccb_plan_t p, int* l1, int* l2, int* k1, int* k2, int* m) {
  if (!p) return fail(BCCB_ERR_INVALID, "plan is NULL");
  if (l1) *l1 = p->L1;
  if (l2) *l2 = p->L2;
  if (k1) *k1 = p->ax1.K;
  if (k2) *k2 = p->ax2.K;
  if (m) *m = p->M;
  return BCCB_OK;
}

extern "C" int bccb_plan_eigen_box(bccb_plan_t p, double* box_t, double* re, double* im) {
  if (!p) return fail(BCCB_ERR_INVALID, "plan is NULL");
  if (box_t)
    for (size_t i = 0; i < p->box.size(); ++i) {
      box_t[2 * i] = p->box[i].real();
      box_t[2 * i + 1] = p->box[i].imag();
    }
  if (re) *re = p->lam_out.real();
  if (im) *im = p->lam_out.imag();
  return BCCB_OK;
}

// ------------------------------------------------------------------ workspace
struct Workspace {
  float2* U;
  float2* V;
  float2* D;
  float2* P;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t ws_bytes(const bccb_plan_s* p, int batch) {
  const size_t inter = (size_t)batch * p->ax1.K * p->L2 * sizeof(float2);
  const size_t box = (size_t)p->ax1.K * p->ax2.K * sizeof(float2);
  return 2 * align_up(inter) + 2 * align_up(box);
}

static Workspace carve(const bccb_plan_s* p, int batch, void* base) {
  Workspace w;
  char* ptr = (char*)base;
  const size_t inter = align_up((size_t)batch * p->ax1.K * p->L2 * sizeof(float2));
  const size_t box = align_up((size_t)p->ax1.K * p->ax2.K * sizeof(float2));
  w.U = (float2*)ptr;
  ptr += inter;
  w.V = (float2*)ptr;
  ptr += inter;
  w.D = (float2*)ptr;
  ptr += box;
  w.P = (float2*)ptr;
  return w;
}

extern "C" size_t bccb_workspace_bytes(bccb_plan_t p, int batch) {
  if (!p || batch < 1) return 0;
  return ws_bytes(p, batch);
}

// ------------------------------------------------------------------ launch helpers
struct LaunchShape {
  int TR, threads;
  size_t smem;
};

static LaunchShape shape_for(const AxisHost& ax) {
  LaunchShape s;
  s.TR = std::max(1, 256 / ax.R);
  s.threads = s.TR * ax.R;
  s.smem = ((size_t)s.TR * (ax.K + 1) + (size_t)s.TR * ax.KP * ax.pitch) * sizeof(float2);
  return s;
}

template <typename KernelT>
static int prep_smem(KernelT kernel, size_t smem) {
  if (smem > 48 * 1024) {
    if (smem > 227 * 1024) return fail(BCCB_ERR_UNSUPPORTED, "shared memory need %zu B > 227 KB", smem);
    CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  return BCCB_OK;
}

#define KP_DISPATCH(KPVAL, ...)            \
  switch (KPVAL) {                          \
    case 1: { constexpr int KPC = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int KPC = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int KPC = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int KPC = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int KPC = 16; __VA_ARGS__; } break; \
    case 32: { constexpr int KPC = 32; __VA_ARGS__; } break; \
    default: return fail(BCCB_ERR_UNSUPPORTED, "register DFT size %d", KPVAL); \
  }

static Geo rows_geo(const bccb_plan_s* p, int batch, const LaunchShape& sh, bool inv, bool fwd) {
  Geo G;
  G.L1 = p->L1;
  G.L2 = p->L2;
  G.rows = (long long)batch * p->L2;
  G.TR = sh.TR;
  G.do_inv = inv ? 1 : 0;
  G.do_fwd = fwd ? 1 : 0;
  return G;
}

static int launch_rows_vector(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                              const EpiVector& epi, cudaStream_t st) {
  const LaunchShape sh = shape_for(p->ax1);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO io{w.V, w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  KP_DISPATCH(p->ax1.KP, {
    auto k = rows_vector_kernel<KPC>;
    int rc = prep_smem(k, sh.smem);
    if (rc) return rc;
    k<<<grid, sh.threads, sh.smem, st>>>(G, p->ax1.dev(), io, epi);
  });
  LAUNCH_CHECK();
  return BCCB_OK;
}

static int launch_rows_fista(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                             const EpiFista& epi, cudaStream_t st) {
  const LaunchShape sh = shape_for(p->ax1);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO io{w.V, w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  KP_DISPATCH(p->ax1.KP, {
    constexpr int CH = KPC < 4 ? KPC : 4;
    auto k = rows_fista_kernel<KPC, CH>;
    int rc = prep_smem(k, sh.smem);
    if (rc) return rc;
    k<<<grid, sh.threads, sh.smem, st>>>(G, p->ax1.dev(), io, epi);
  });
  LAUNCH_CHECK();
  return BCCB_OK;
}

static int launch_rows_admm(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                            const EpiAdmm& epi, cudaStream_t st) {
  const LaunchShape sh = shape_for(p->ax1);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO io{w.V, w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  KP_DISPATCH(p->ax1.KP, {
    constexpr int CH = KPC < 4 ? KPC : 4;
    auto k = rows_admm_kernel<KPC, CH>;
    int rc = prep_smem(k, sh.smem);
    if (rc) return rc;
    k<<<grid, sh.threads, sh.smem, st>>>(G, p->ax1.dev(), io, epi);
  });
  LAUNCH_CHECK();
  return BCCB_OK;
}

static int launch_cols(const bccb_plan_s* p, int batch, bool fwd, bool inv, const Workspace& w,
                       const float2* D, const float2* P, const float2* Bh, float2* box_out,
                       cudaStream_t st) {
  const LaunchShape sh = shape_for(p->ax2);
  Geo G;
  G.L1 = p->L1;
  G.L2 = p->L2;
  G.rows = (long long)batch * p->ax1.K;
  G.TR = sh.TR;
  G.do_fwd = fwd ? 1 : 0;
  G.do_inv = inv ? 1 : 0;
  ColsIO io;
  io.U = w.U;
  io.V = w.V;
  io.D = D;
  io.P = P;
  io.Bh = Bh;
  io.box_out = box_out;
  io.K1 = p->ax1.K;
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  KP_DISPATCH(p->ax2.KP, {
    auto k = cols_kernel<KPC>;
    int rc = prep_smem(k, sh.smem);
    if (rc) return rc;
    k<<<grid, sh.threads, sh.smem, st>>>(G, p->ax2.dev(), io);
  });
  LAUNCH_CHECK();
  return BCCB_OK;
}

// D / P boxes for one operation (complex64 [K1][K2]), from the complex128 eigenvalue box.
//   mode 0 (matvec):  D = (lam - lam_out) / L,               P = -
//   mode 1 (ISTA):    D = -mu (lam - lam_out) / L,           P = mu / L
//   mode 2 (ADMM):    D = (rho/(lam+rho) - a) / L,           P = 1 / ((lam + rho) L)
//   mode 3 (synth):   D = -,                                  P = scale
__global__ void coef_kernel(const double2* __restrict__ lam, int n, int mode, double s1,
                            double lam_out, double a, double invL, float2* D, float2* P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lr = lam[i].x, li = lam[i].y;
  if (mode == 0) {
    D[i] = make_float2((float)((lr - lam_out) * invL), (float)(li * invL));
  } else if (mode == 1) {
    D[i] = make_float2((float)(-s1 * (lr - lam_out) * invL), (float)(-s1 * li * invL));
    P[i] = make_float2((float)(s1 * invL), 0.f);
  } else if (mode == 2) {
    // q = 1/(lam + rho) ; D = rho*q - a
    const double dr = lr + s1, di = li;
    const double den = dr * dr + di * di;
    const double qr = dr / den, qi = -di / den;
    D[i] = make_float2((float)((s1 * qr - a) * invL), (float)(s1 * qi * invL));
    P[i] = make_float2((float)(qr * invL), (float)(qi * invL));
  }
}

static int launch_coef(const bccb_plan_s* p, int mode, double s1, double a, const Workspace& w,
                       cudaStream_t st) {
  const int n = p->ax1.K * p->ax2.K;
  const double invL = 1.0 / ((double)p->L1 * (double)p->L2);
  coef_kernel<<<(n + 255) / 256, 256, 0, st>>>(p->lam_box_dev, n, mode, s1, p->lam_out.real(), a,
                                                invL, w.D, w.P);
  LAUNCH_CHECK();
  return BCCB_OK;
}

static int check_common(const bccb_plan_s* p, int batch, void* workspace) {
  if (!p) return fail(BCCB_ERR_INVALID, "plan is NULL");
  if (batch < 1) return fail(BCCB_ERR_INVALID, "batch must be positive");
  if (!workspace) return fail(BCCB_ERR_INVALID, "workspace is NULL");
  return BCCB_OK;
}

// ------------------------------------------------------------------ operator entry points
extern "C" int bccb_matvec(bccb_plan_t p, int batch, const void* x, void* y, void* workspace,
                           void* stream) {
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!x || !y) return fail(BCCB_ERR_INVALID, "x / y is NULL");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  if ((rc = launch_coef(p, 0, 0.0, 0.0, w, st))) return rc;
  EpiVector e{(const float2*)x, nullptr, nullptr, 0.f, 1.f};
  if ((rc = launch_rows_vector(p, batch, false, true, w, e, st))) return rc;
  if ((rc = launch_cols(p, batch, true, true, w, w.D, nullptr, nullptr, nullptr, st))) return rc;
  const float lo = (float)p->lam_out.real();
  EpiVector e2{(const float2*)x, (float2*)y, nullptr, lo, 1.f};
  return launch_rows_vector(p, batch, true, false, w, e2, st);
}

extern "C" int bccb_spectrum_box(bccb_plan_t p, int batch, const void* x, void* out_box,
                                 void* workspace, void* stream) {
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!x || !out_box) return fail(BCCB_ERR_INVALID, "x / out_box is NULL");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  EpiVector e{(const float2*)x, nullptr, nullptr, 0.f, 1.f};
  if ((rc = launch_rows_vector(p, batch, false, true, w, e, st))) return rc;
  return launch_cols(p, batch, true, false, w, nullptr, nullptr, nullptr, (float2*)out_box, st);
}

extern "C" int bccb_synthesize(bccb_plan_t p, int batch, const void* box, float scale, const void* x,
                               float alpha, void* out, float* maxabs, void* workspace,
                               void* stream) {
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!box) return fail(BCCB_ERR_INVALID, "box is NULL");
  if (alpha != 0.f && !x) return fail(BCCB_ERR_INVALID, "x is NULL with alpha != 0");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  if ((rc = launch_cols(p, batch, false, true, w, nullptr, nullptr, (const float2*)box, nullptr, st)))
    return rc;
  EpiVector e{(const float2*)x, (float2*)out, maxabs, alpha, scale};
  return launch_rows_vector(p, batch, true, false, w, e, st);
}

// signed scatter of y into the spectral box: Bh[b][m1][m2] = L (-1)^(m1+m2) y[b][m]
__global__ void adjoint_scatter_kernel(const float2* __restrict__ y, const int* __restrict__ occ,
                                       int M, int K1, int K2, long long total, float L, int alias,
                                       float2* __restrict__ Bh) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const long long b = i / M;
  const int m = (int)(i - b * M);
  const int m1 = occ[m], m2 = occ[M + m];
  const int sgn = occ[2 * M + m];
  const float2 v = y[i];
  const float f = (sgn & 1) ? -L : L;
  float2* dst = Bh + (b * K1 + m1) * K2 + m2;
  if (alias) {
    atomicAdd(&dst->x, f * v.x);
    atomicAdd(&dst->y, f * v.y);
  } else {
    *dst = make_float2(f * v.x, f * v.y);
  }
}

extern "C" int bccb_adjoint(bccb_plan_t p, int batch, const void* y, void* bhat_box, void* b,
                            float* maxabs, void* workspace, void* stream) {
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!p->occ_dev || p->M < 1) return fail(BCCB_ERR_INVALID, "bccb_adjoint needs a Gram plan");
  if (!y || !bhat_box) return fail(BCCB_ERR_INVALID, "y / bhat_box is NULL");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  const int K1 = p->ax1.K, K2 = p->ax2.K;
  CUDA_TRY(cudaMemsetAsync(bhat_box, 0, (size_t)batch * K1 * K2 * sizeof(float2), st));
  const long long total = (long long)batch * p->M;
  const float L = (float)((double)p->L1 * (double)p->L2);
  adjoint_scatter_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      (const float2*)y, p->occ_dev, p->M, K1, K2, total, L, p->occ_alias, (float2*)bhat_box);
  LAUNCH_CHECK();
  if (maxabs) CUDA_TRY(cudaMemsetAsync(maxabs, 0, (size_t)batch * sizeof(float), st));
  if (!b && !maxabs) return BCCB_OK;
  const float invL = (float)(1.0 / ((double)p->L1 * (double)p->L2));
  if ((rc = launch_cols(p, batch, false, true, w, nullptr, nullptr, (const float2*)bhat_box, nullptr,
                        st)))
    return rc;
  EpiVector e{nullptr, (float2*)b, maxabs, 0.f, invL};
  return launch_rows_vector(p, batch, true, false, w, e, st);
}

// ------------------------------------------------------------------ solvers
__global__ void fill_int_kernel(int* p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

static int reset_first_bad(int* first_bad, int batch, cudaStream_t st) {
  fill_int_kernel<<<(batch + 255) / 256, 256, 0, st>>>(first_bad, batch, INT_MAX);
  LAUNCH_CHECK();
  return BCCB_OK;
}

static int check_singular_admm(const bccb_plan_s* p, double rho) {
  // bccb_inverse(bccb_scale_add_identity(G, 1, rho)) guard — bccb.py:133-148
  double mx = 0.0, mn = INFINITY;
  for (const auto& v : p->box) {
    const double m = std::abs(v + rho);
    mx = std::max(mx, m);
    mn = std::min(mn, m);
  }
  if (!p->full()) {
    const double m = std::abs(p->lam_out + rho);
    mx = std::max(mx, m);
    mn = std::min(mn, m);
  }
  const double thr = 1e-12 * mx;
  if (mn <= thr)
    return fail(BCCB_ERR_SINGULAR,
                "operator is numerically singular: min |eigenvalue| = %.6e is below the guard "
                "threshold %.6e|%.17g|%.17g",
                mn, thr, mn, thr);
  return BCCB_OK;
}

extern "C" int bccb_fista_run(bccb_plan_t p, int batch, int first_iteration, int iterations,
                              double mu, const double* tau,
                              const void* bhat_box, const void* extra, void* c, void* d,
                              int* first_bad, void* workspace, void* stream) {
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (iterations < 1) return fail(BCCB_ERR_INVALID, "iteration count must be positive");
  if (first_iteration < 0) return fail(BCCB_ERR_INVALID, "first iteration must be >= 0");
  if (!(mu > 0)) return fail(BCCB_ERR_INVALID, "step size must be positive");
  if (!tau || !bhat_box || !c || !first_bad) return fail(BCCB_ERR_INVALID, "NULL argument");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  const double lo = p->lam_out.real();
  if ((rc = launch_coef(p, 1, mu, 0.0, w, st))) return rc;
  if (first_iteration == 0 && (rc = reset_first_bad(first_bad, batch, st))) return rc;
  EpiFista e;
  e.c = (double2*)c;
  e.d = (float2*)d;
  e.extra = (const float2*)extra;
  e.tau = tau;
  e.first_bad = first_bad;
  e.a = 1.0 - mu * lo;
  e.kscale = mu;
  e.extra_scale = mu;
  e.momentum = d ? 1 : 0;
  // momentum coefficients: beta_t = (alpha_{t-1} - 1) / alpha_t, alpha_0 = 1 (solvers.py:294-337)
  const int t_end = first_iteration + iterations;
  std::vector<double> beta((size_t)t_end + 1, 0.0);
  {
    double alpha = 1.0;
    for (int t = 1; t <= t_end; ++t) {
      const double an = 0.5 * (std::sqrt(1.0 + 4.0 * alpha * alpha) + 1.0);
      beta[t] = (alpha - 1.0) / an;
      alpha = an;
    }
  }
  e.it = first_iteration;
  e.beta_cur = e.momentum ? beta[first_iteration] : 0.0;
  e.beta_next = 0.0;
  if ((rc = launch_rows_fista(p, batch, false, true, w, e, st))) return rc;
  for (int t = first_iteration; t < t_end; ++t) {
    if ((rc = launch_cols(p, batch, true, true, w, w.D, w.P, (const float2*)bhat_box, nullptr, st)))
      return rc;
    e.it = t;
    e.beta_cur = e.momentum ? beta[t] : 0.0;
    e.beta_next = e.momentum ? beta[t + 1] : 0.0;
    if ((rc = launch_rows_fista(p, batch, true, t + 1 < t_end, w, e, st))) return rc;
  }
  return BCCB_OK;
}

extern "C" int bccb_admm_run(bccb_plan_t p, int batch, int first_iteration, int iterations,
                             double rho, const double* tau,
                             const void* bhat_box, const void* extra, void* z, void* v, void* c_last,
                             int* first_bad, void* workspace, void* stream) {
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (iterations < 1) return fail(BCCB_ERR_INVALID, "iteration count must be positive");
  if (first_iteration < 0) return fail(BCCB_ERR_INVALID, "first iteration must be >= 0");
  if (!(rho > 0)) return fail(BCCB_ERR_INVALID, "rho must be positive");
  if (!tau || !bhat_box || !z || !v || !first_bad) return fail(BCCB_ERR_INVALID, "NULL argument");
  if ((rc = check_singular_admm(p, rho))) return rc;
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  const double lo = p->lam_out.real();
  const double a = rho / (lo + rho);
  if ((rc = launch_coef(p, 2, rho, a, w, st))) return rc;
  if (first_iteration == 0 && (rc = reset_first_bad(first_bad, batch, st))) return rc;
  EpiAdmm e;
  e.z = (float2*)z;
  e.v = (float2*)v;
  e.c_out = nullptr;
  e.extra = (const float2*)extra;
  e.tau = tau;
  e.first_bad = first_bad;
  e.a = a;
  e.kscale = rho;
  e.extra_scale = 1.0 / (lo + rho);
  e.it = first_iteration;
  const int t_end = first_iteration + iterations;
  if ((rc = launch_rows_admm(p, batch, false, true, w, e, st))) return rc;
  for (int t = first_iteration; t < t_end; ++t) {
    if ((rc = launch_cols(p, batch, true, true, w, w.D, w.P, (const float2*)bhat_box, nullptr, st)))
      return rc;
    e.it = t;
    e.c_out = (t + 1 == t_end) ? (float2*)c_last : nullptr;
    if ((rc = launch_rows_admm(p, batch, true, t + 1 < t_end, w, e, st))) return rc;
  }
  return BCCB_OK;
}

// ------------------------------------------------------------------ top-k
extern "C" size_t bccb_topk_workspace_bytes(int batch, long long length, int k) {
  if (batch < 1 || length < 1 || k < 1) return 0;
  const int nchunk = topk_chunks(batch, length);
  return (size_t)batch * nchunk * pow2_ceil(k) * sizeof(unsigned long long) + 256;
}

extern "C" int bccb_topk(int batch, long long length, const void* values, int is_double, int k,
                         int* idx, float* mag, void* workspace, void* stream) {
  if (batch < 1 || length < 1) return fail(BCCB_ERR_INVALID, "empty input");
  if (k < 1 || k > 64) return fail(BCCB_ERR_INVALID, "k must lie in [1, 64]");
  if (k > length) return fail(BCCB_ERR_INVALID, "k exceeds the vector length");
  if (length > 0xFFFFFFFFLL) return fail(BCCB_ERR_UNSUPPORTED, "vector longer than 2^32");
  if (!values || !idx || !workspace) return fail(BCCB_ERR_INVALID, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int nchunk = topk_chunks(batch, length);
  unsigned long long* cand = (unsigned long long*)workspace;
  const int kt = std::max(4, pow2_ceil(k));
#define TOPK_CASE(KT)                                                                            \
  case KT:                                                                                       \
    topk_partial_kernel<KT><<<dim3(nchunk, batch), 256, 0, st>>>(values, is_double, length, k,   \
                                                                 nchunk, cand);                  \
    topk_merge_kernel<KT><<<batch, 256, 0, st>>>(cand, nchunk * k, k, idx, mag);                 \
    break;
  switch (kt) {
    TOPK_CASE(4)
    TOPK_CASE(8)
    TOPK_CASE(16)
    TOPK_CASE(32)
    TOPK_CASE(64)
    default:
      return fail(BCCB_ERR_UNSUPPORTED, "k = %d", k);
  }
#undef TOPK_CASE
  LAUNCH_CHECK();
  return BCCB_OK;
}
