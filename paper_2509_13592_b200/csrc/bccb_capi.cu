// C ABI + launch sequencing for the B200-native BCCB Gram operator.
// See include/bccb_b200.h for the interface and the reference functions replaced.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <type_traits>
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

// ------------------------------------------------------------------ launch accounting
// Every kernel launch is counted (bccb_launch_count); between bccb_profile_begin/end each
// launch is also bracketed by CUDA events on its own stream, grouped by kernel kind.
enum KernelKind { KIND_ROWS = 0, KIND_COLS = 1, KIND_OTHER = 2, KIND_COUNT = 3 };
static std::atomic<long long> g_launches{0};
struct ProfEvent {
  cudaEvent_t a, b;
  int kind;
};
static thread_local bool g_prof_on = false;
static thread_local std::vector<ProfEvent> g_prof_events;
static thread_local size_t g_prof_used = 0;

static void prof_before(int kind, cudaStream_t st, ProfEvent** slot) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  *slot = nullptr;
  if (!g_prof_on) return;
  if (g_prof_used == g_prof_events.size()) {
    ProfEvent e;
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
    g_prof_events.push_back(e);
  }
  ProfEvent* e = &g_prof_events[g_prof_used++];
  e->kind = kind;
  cudaEventRecord(e->a, st);
  *slot = e;
}
static void prof_after(ProfEvent* e, cudaStream_t st) {
  if (e) cudaEventRecord(e->b, st);
}

extern "C" long long bccb_launch_count(void) { return g_launches.load(); }

// Set at the top of every public entry point that launches kernels (EntryScope); consumed by
// the first launch_pass of the call.  The scope is also an NVTX range named after the entry
// point (header-only NVTX 3: free unless a profiler is attached), so nsys / ncu timelines
// group each call's kernels.
static thread_local bool t_entry_fresh = false;
struct EntryScope {
  explicit EntryScope(const char* name) {
    t_entry_fresh = true;
    nvtxRangePushA(name);
  }
  ~EntryScope() {
    t_entry_fresh = false;
    nvtxRangePop();
  }
};

extern "C" int bccb_profile_begin(void) {
  g_prof_on = true;
  g_prof_used = 0;
  return BCCB_OK;
}

extern "C" int bccb_profile_end(double* ms_by_kind, long long* launches_by_kind) {
  g_prof_on = false;
  for (int k = 0; k < KIND_COUNT; ++k) {
    if (ms_by_kind) ms_by_kind[k] = 0.0;
    if (launches_by_kind) launches_by_kind[k] = 0;
  }
  for (size_t i = 0; i < g_prof_used; ++i) {
    ProfEvent& e = g_prof_events[i];
    cudaError_t err = cudaEventSynchronize(e.b);
    if (err != cudaSuccess) return fail(BCCB_ERR_CUDA, "profile sync: %s", cudaGetErrorString(err));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    if (ms_by_kind) ms_by_kind[e.kind] += ms;
    if (launches_by_kind) launches_by_kind[e.kind] += 1;
  }
  g_prof_used = 0;
  return BCCB_OK;
}
extern "C" const char* bccb_version(void) { return "bccb_b200 0.1.0 (sm_100a)"; }

// ------------------------------------------------------------------ launch mode
// Programmatic dependent launch of the pass kernels (BCCB_PDL): 0 off, 1 on with each CTA
// releasing its dependents right after its griddepcontrol.wait, 2 on with the implicit
// release at grid completion (default: measured +0.6 % at config 2, +0.3 % at config 3,
// neutral at configs 4/5 against mode 1, profiles/ab/r1_pdl_modes.txt).
static int pdl_mode() {
  static const int m = [] {
    const char* e = getenv("BCCB_PDL");
    return e ? atoi(e) : 2;
  }();
  return m;
}

// ------------------------------------------------------------------ device init
static std::mutex g_init_mu;
static bool g_roots_ready[64];

static int ensure_device_constants(int device) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (device < 0 || device >= 64) return fail(BCCB_ERR_INVALID, "bad device %d", device);
  if (g_roots_ready[device]) return BCCB_OK;
  float2 roots[64];
  double2 rootsd[64];
  for (int t = 0; t < 64; ++t) {
    const double ang = -2.0 * M_PI * t / 64.0;
    roots[t] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    rootsd[t] = make_double2(std::cos(ang), std::sin(ang));
  }
  CUDA_TRY(cudaMemcpyToSymbol(c_roots64, roots, sizeof(roots)));
  CUDA_TRY(cudaMemcpyToSymbol(c_roots64d, rootsd, sizeof(rootsd)));
  const int trig = pdl_mode() == 1 ? 1 : 0;
  CUDA_TRY(cudaMemcpyToSymbol(c_pdl_trigger, &trig, sizeof(trig)));
  g_roots_ready[device] = true;
  return BCCB_OK;
}

// ------------------------------------------------------------------ plan
// One axis at one precision (register DFT size, band, team size, twiddles).
struct AxisPrec {
  int KP = 1, R = 1, Mo = 1, pitch = 1;
  void* tw1 = nullptr;  // [KP][R]  w_N^{s j}   (float2 or double2)
  void* tw2 = nullptr;  // [Mo][R]  w_R^{s m}
};

struct AxisHost {
  int N = 0, K = 0;
  // complex64 engine (KP <= 32), complex128 engine (KP <= 16), complex64 streaming engine
  // (KP <= 16: the KP16 rows engine and the column pass) and its KP <= 8 variant (column
  // passes with few lines: twice the threads per line, shorter latency chains)
  AxisPrec f, d, s, s8;
  // tensor-core rows engine (rows axis only): R = 128 threads per line, KP = N / 128,
  // Mo = K / KP a multiple of 4 (KP = 0: not eligible)
  AxisPrec t;
  template <typename C>
  const AxisPrec& prec() const;
  template <typename C>
  AxisT<C> dev() const {
    const AxisPrec& p = prec<C>();
    AxisT<C> a;
    a.N = N;
    a.K = K;
    a.KP = p.KP;
    a.R = p.R;
    a.Mo = p.Mo;
    a.pitch = p.pitch;
    a.tw1 = (const C*)p.tw1;
    a.tw2 = (const C*)p.tw2;
    return a;
  }
  AxisT<float2> dev_t() const {
    AxisT<float2> a;
    a.N = N;
    a.K = K;
    a.KP = t.KP;
    a.R = t.R;
    a.Mo = t.Mo;
    a.pitch = t.pitch;
    a.tw1 = (const float2*)t.tw1;
    a.tw2 = (const float2*)t.tw2;
    return a;
  }
  AxisT<float2> dev_s(bool narrow = false) const {
    const AxisPrec& q = narrow ? s8 : s;
    AxisT<float2> a;
    a.N = N;
    a.K = K;
    a.KP = q.KP;
    a.R = q.R;
    a.Mo = q.Mo;
    a.pitch = q.pitch;
    a.tw1 = (const float2*)q.tw1;
    a.tw2 = (const float2*)q.tw2;
    return a;
  }
};
template <> const AxisPrec& AxisHost::prec<float2>() const { return f; }
template <> const AxisPrec& AxisHost::prec<double2>() const { return d; }

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
  static constexpr int MAX_SUB = 8;
  // Threading: after creation a plan is read-only.  Everything a call
  // mutates lives in the caller's workspace, in per-thread state (the sub-batch streams and
  // events, SubStreams) or in the process-wide, grow-only momentum table (beta_table).
  bool full() const { return ax1.K == L1 && ax2.K == L2; }
};

static int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p *= 2;
  return p;
}

template <typename C>
static int upload_twiddles(int N, AxisPrec& ap) {
  std::vector<C> t1((size_t)ap.KP * ap.R), t2((size_t)ap.Mo * ap.R);
  for (int j = 0; j < ap.KP; ++j)
    for (int s = 0; s < ap.R; ++s) {
      // w_N^{s j}; the exponent is reduced mod N in integers for accuracy
      const long long e = ((long long)s * j) % N;
      const double ang = -2.0 * M_PI * (double)e / (double)N;
      t1[(size_t)j * ap.R + s] = C{(decltype(C::x))std::cos(ang), (decltype(C::x))std::sin(ang)};
    }
  for (int m = 0; m < ap.Mo; ++m)
    for (int s = 0; s < ap.R; ++s) {
      const long long e = ((long long)s * m) % ap.R;
      const double ang = -2.0 * M_PI * (double)e / (double)ap.R;
      t2[(size_t)m * ap.R + s] = C{(decltype(C::x))std::cos(ang), (decltype(C::x))std::sin(ang)};
    }
  CUDA_TRY(cudaMalloc(&ap.tw1, t1.size() * sizeof(C)));
  CUDA_TRY(cudaMalloc(&ap.tw2, t2.size() * sizeof(C)));
  CUDA_TRY(cudaMemcpy(ap.tw1, t1.data(), t1.size() * sizeof(C), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(ap.tw2, t2.data(), t2.size() * sizeof(C), cudaMemcpyHostToDevice));
  return BCCB_OK;
}

// Choose the register DFT size KP (largest power of two dividing N, <= 32 and <= the band),
// round the band up to a multiple of KP and build both precisions' twiddle tables.
static int make_axis(int N, int Kreq, AxisHost& ax, bool cols) {
  int KP = 1;
  while (KP < KP_MAX && N % (KP * 2) == 0) KP *= 2;
  KP = std::min(KP, pow2_ceil(std::max(1, Kreq)));
  int K = ((Kreq + KP - 1) / KP) * KP;
  K = std::min(K, N);
  if (K % KP != 0) K = N;  // N is a multiple of KP
  ax.N = N;
  ax.K = K;
  // streaming-axis register DFT size: 16 (the KP16 rows engine and the column pass);
  // BCCB_COLS_KP overrides it for the column axis (tuning)
  static const int cols_kp = [] {
    const char* e = getenv("BCCB_COLS_KP");
    const int v = e ? atoi(e) : 16;
    return (v == 4 || v == 8 || v == 16 || v == 32) ? v : 16;
  }();
  const int kps[4] = {KP, std::min(KP, KP_MAX_D), std::min(KP, cols ? cols_kp : 16), std::min(KP, 8)};
  AxisPrec* aps[4] = {&ax.f, &ax.d, &ax.s, &ax.s8};
  for (int q = 0; q < 4; ++q) {
    AxisPrec& ap = *aps[q];
    ap.KP = kps[q];
    ap.R = N / ap.KP;
    if (ap.R > 1024)
      return fail(BCCB_ERR_UNSUPPORTED,
                  "grid length %d needs %d threads per line (> 1024); use a length with a larger "
                  "power-of-two factor",
                  N, ap.R);
    ap.Mo = K / ap.KP;
    ap.pitch = (ap.R % 2 == 1) ? ap.R : ap.R + 1;
  }
  int rc = upload_twiddles<float2>(N, ax.f);
  if (!rc) rc = upload_twiddles<double2>(N, ax.d);
  if (!rc) rc = upload_twiddles<float2>(N, ax.s);
  if (!rc) rc = upload_twiddles<float2>(N, ax.s8);
  ax.t = AxisPrec{};
  ax.t.KP = 0;
  if (!rc && !cols && N % 128 == 0) {
    const int kp = N / 128;
    if ((kp == 8 || kp == 16 || kp == 32) && K % kp == 0 && (K / kp) % 4 == 0 && K / kp <= 16) {
      ax.t.KP = kp;
      ax.t.R = 128;
      ax.t.Mo = K / kp;
      ax.t.pitch = 129;
      rc = upload_twiddles<float2>(N, ax.t);
    }
  }
  return rc;
}

static void free_axis(AxisHost& a) {
  for (AxisPrec* p : {&a.f, &a.d, &a.s, &a.s8, &a.t}) {
    cudaFree(p->tw1);
    cudaFree(p->tw2);
  }
}

static void free_plan(bccb_plan_s* p) {
  if (!p) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(p->device);
  free_axis(p->ax1);
  free_axis(p->ax2);
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
  if ((rc = make_axis(p->L1, k1req, p->ax1, false))) return rc;
  if ((rc = make_axis(p->L2, k2req, p->ax2, true))) return rc;
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
// U, V hold [batch][K1][L2] band intermediates and D, P the [K1][K2] multipliers; all are
// sized for complex128 so one workspace serves both engines.
struct Workspace {
  void* U;
  void* V;
  void* D;
  void* P;
  unsigned char* flags;  // zero-segment flags of the streaming FISTA pass
  int* counters;         // [batch] arrival counters of the fused column pass
  void* vs;              // [batch][K1][K2] complex128: spectral part of the ADMM dual
  void* cb;              // [batch][K1][K2] complex128: last column-pass box of the split ADMM
};

// Rows engine of the specialised FISTA pass: the KP = 16 axis at 3 CTAs / SM for the shapes
// that have it (half the register DFT => more resident warps to hide latency once the
// iterate is sparse; measured +2-3% on configs 2 and 4), else the complex64 axis (KP <= 32).
// BCCB_ROWS_KP16=0 selects the KP <= 32 engine everywhere.
static int rows_kp16_env() {
  static const int v = [] {
    const char* e = getenv("BCCB_ROWS_KP16");
    return e ? atoi(e) : 1;
  }();
  return v;
}
static bool kp16_shape(const AxisPrec& a) {
  return a.KP == 16 && ((a.R == 16 && a.Mo == 2) || (a.R == 64 && a.Mo == 4));
}
static bool rows_use_kp16(const AxisHost& ax) { return rows_kp16_env() && kp16_shape(ax.s); }

// Tensor-core rows engine of the specialised FISTA/ISTA pass (BCCB_ROWS_TC, default on): the
// level-2 stage of the band inverse runs as tcgen05 kind::tf32 MMAs (bccb_kernels.cuh TcInv).
// Shapes with an instantiation: (KP, Mo) at R = 128.
#define TC_SHAPES(X)                                       \
  X(32, 4)   /* L1 = 4096, band 128 (config 5) */          \
  X(8, 8)    /* L1 = 1024, band 64  (config 4) */
static int rows_tc_env() {
  static const int v = [] {
    const char* e = getenv("BCCB_ROWS_TC");
    return e ? atoi(e) : 1;
  }();
  return v;
}
static bool tc_shape(const AxisPrec& a) {
  if (a.KP == 0 || a.R != 128) return false;
#define TC_KEY(KP_, MO_) \
  if (a.KP == KP_ && a.Mo == MO_) return true;
  TC_SHAPES(TC_KEY)
#undef TC_KEY
  return false;
}
// 1 (default): the shapes where the tensor-core engine measured faster (KP = 32: config 5,
// 365 vs 310 G gpi/s; at KP = 8 (config 4) the CUDA-core KP16 engine stays ahead, 296 vs 236,
// profiles/r2/r2d_*); 2: every TC shape; 0: off
static bool rows_use_tc(const AxisHost& ax) {
  const int env = rows_tc_env();
  return env && tc_shape(ax.t) && (env == 2 || ax.t.KP == 32);
}

// rows engine of the specialised passes: tc = the FISTA/ISTA tensor-core engine
static const AxisPrec& rows_axis(const AxisHost& ax, bool tc = false) {
  return tc ? ax.t : (rows_use_kp16(ax) ? ax.s : ax.f);
}

// threads per CTA of the specialised FISTA rows pass (flags: one 32-bit word per warp)
static int zs_threads(const AxisHost& ax, bool tc = false) {
  return tc ? tc_threads(ax.t.KP) : std::max(256, rows_axis(ax, tc).R);
}
static size_t zs_flag_bytes(const bccb_plan_s* p, int batch, bool tc = false);

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t flag_bytes_for(const bccb_plan_s* p, int batch, int R, int extra_words = 0, int ntmin = 256) {
  const int nt = std::max(ntmin, R);
  const int tr = nt / R;
  const long long rows = (long long)batch * p->L2;
  const long long ctas = (rows + tr - 1) / tr;
  return (size_t)ctas * (nt / 32 + extra_words) * sizeof(unsigned);
}

// flags of the specialised FISTA rows pass (complex64 axis): per tile, one word per warp and
// one tile word (rows_tile)
// flags of the specialised ADMM rows pass (complex128 axis)
static size_t zs_flag_bytes_d(const bccb_plan_s* p, int batch) { return flag_bytes_for(p, batch, p->ax1.d.R); }

static size_t zs_flag_bytes(const bccb_plan_s* p, int batch, bool tc) {
  return flag_bytes_for(p, batch, rows_axis(p->ax1, tc).R, 1, tc ? tc_threads(p->ax1.t.KP) : 256);
}
static size_t zs_flag_bytes_max(const bccb_plan_s* p, int batch) {
  size_t b = std::max(zs_flag_bytes(p, batch), zs_flag_bytes_d(p, batch));
  if (p->ax1.t.KP > 0) b = std::max(b, zs_flag_bytes(p, batch, true));
  return b;
}


static size_t ws_bytes(const bccb_plan_s* p, int batch) {
  const size_t inter = (size_t)batch * p->ax1.K * p->L2 * sizeof(double2);
  const size_t box = (size_t)p->ax1.K * p->ax2.K * sizeof(double2);
  return 2 * align_up(inter) + 2 * align_up(box) +
         align_up(zs_flag_bytes_max(p, batch)) +
         align_up((size_t)batch * sizeof(int)) + 2 * align_up((size_t)batch * box);
}

static Workspace carve(const bccb_plan_s* p, int batch, void* base) {
  Workspace w;
  char* ptr = (char*)base;
  const size_t inter = align_up((size_t)batch * p->ax1.K * p->L2 * sizeof(double2));
  const size_t box = align_up((size_t)p->ax1.K * p->ax2.K * sizeof(double2));
  w.U = ptr;
  ptr += inter;
  w.V = ptr;
  ptr += inter;
  w.D = ptr;
  ptr += box;
  w.P = ptr;
  ptr += box;
  w.flags = (unsigned char*)ptr;
  ptr += align_up(zs_flag_bytes_max(p, batch));
  w.counters = (int*)ptr;
  ptr += align_up((size_t)batch * sizeof(int));
  w.vs = ptr;
  ptr += align_up((size_t)batch * p->ax1.K * p->ax2.K * sizeof(double2));
  w.cb = ptr;
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

// Lines per CTA: 256 threads by default; when the launch would leave SMs idle (few lines,
// e.g. the column pass of config 2: 2048 lines) shrink the CTA so the grid covers >= 2 waves.
static LaunchShape shape_for_prec(const AxisHost& ax, const AxisPrec& ap, size_t elem, long long lines) {
  LaunchShape s;
  s.TR = std::max(1, 256 / ap.R);
  if (lines > 0)
    while (s.TR > 1 && s.TR * ap.R > 64 && (lines + s.TR - 1) / s.TR < 2 * 148) s.TR /= 2;
  s.threads = s.TR * ap.R;
  s.smem = ((size_t)s.TR * (ax.K + 1) + (size_t)s.TR * ap.KP * ap.pitch) * elem;
  return s;
}

template <typename C>
static LaunchShape shape_for(const AxisHost& ax, long long lines = 0) {
  const AxisPrec& ap = ax.prec<C>();
  LaunchShape s;
  s.TR = std::max(1, 256 / ap.R);
  if (lines > 0)
    while (s.TR > 1 && s.TR * ap.R > 64 && (lines + s.TR - 1) / s.TR < 2 * 148) s.TR /= 2;
  s.threads = s.TR * ap.R;
  s.smem = ((size_t)s.TR * (ax.K + 1) + (size_t)s.TR * ap.KP * ap.pitch) * sizeof(C);
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

// Register DFT size dispatch: complex64 engine up to 32, complex128 engine up to 16.
#define KP_CASES_COMMON(...)                               \
  case 1: { constexpr int KPC = 1; __VA_ARGS__; } break;   \
  case 2: { constexpr int KPC = 2; __VA_ARGS__; } break;   \
  case 4: { constexpr int KPC = 4; __VA_ARGS__; } break;   \
  case 8: { constexpr int KPC = 8; __VA_ARGS__; } break;   \
  case 16: { constexpr int KPC = 16; __VA_ARGS__; } break;
#define KP_DISPATCH_F(KPVAL, ...)                                               \
  switch (KPVAL) {                                                              \
    KP_CASES_COMMON(__VA_ARGS__)                                                \
    case 32: { constexpr int KPC = 32; __VA_ARGS__; } break;                    \
    default: return fail(BCCB_ERR_UNSUPPORTED, "register DFT size %d", KPVAL);  \
  }
#define KP_DISPATCH_D(KPVAL, ...)                                               \
  switch (KPVAL) {                                                              \
    KP_CASES_COMMON(__VA_ARGS__)                                                \
    default: return fail(BCCB_ERR_UNSUPPORTED, "register DFT size %d", KPVAL);  \
  }

// Energy screen of the level-1 inverse DFT in the zero-skipping rows passes, bitwise neutral.
// BCCB_SCREEN bits: 1 (default) = the register screen of the CUDA-core engines (band_fft.cuh
// reg_idft_screened), 2 = the TMEM screen of the tensor-core tiles (tc_energy_screen); 0 computes
// every residue class.
static int rows_screen_env() {
  static const int v = [] {
    const char* e = getenv("BCCB_SCREEN");
    return e ? atoi(e) : 1;
  }();
  return v;
}

static int debug_env() {
  static const int v = [] {
    const char* e = getenv("BCCB_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

static Geo rows_geo(const bccb_plan_s* p, int batch, const LaunchShape& sh, bool inv, bool fwd) {
  Geo G;
  G.screen = rows_screen_env();
  G.dbg = debug_env();
  if ((p->L2 & (p->L2 - 1)) == 0) {
    G.l2_shift = 0;
    while ((1 << G.l2_shift) < p->L2) ++G.l2_shift;
  }
  G.L1 = p->L1;
  G.L2 = p->L2;
  G.rows = (long long)batch * p->L2;
  G.TR = sh.TR;
  G.do_inv = inv ? 1 : 0;
  G.do_fwd = fwd ? 1 : 0;
  return G;
}

template <typename C, typename KernelT, typename... Args>
static int launch_pass(KernelT k, int kind, unsigned grid, const LaunchShape& sh, cudaStream_t st,
                       Args... args) {
  int rc = prep_smem(k, sh.smem);
  if (rc) return rc;
  ProfEvent* pe;
  prof_before(kind, st, &pe);
  // The first kernel of a public entry point follows work this library did not launch (or an
  // earlier call whose kernels may release dependents before their last stores): it is
  // launched without the programmatic-serialization attribute, so every read it makes, even
  // one placed before its griddepcontrol.wait, sees the finished predecessor.
  const bool entry_first = t_entry_fresh;
  t_entry_fresh = false;
  if (pdl_mode() > 0 && !entry_first) {
    // programmatic dependent launch: every kernel of bccb_kernels.cuh starts with pdl_wait()
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(sh.threads);
    cfg.dynamicSmemBytes = sh.smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, k, args...));
  } else {
    k<<<grid, sh.threads, sh.smem, st>>>(args...);
  }
  prof_after(pe, st);
  LAUNCH_CHECK();
  return BCCB_OK;
}

template <typename C>
static int launch_rows_vector(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                              const EpiVector<C>& epi, cudaStream_t st) {
  const LaunchShape sh = shape_for<C>(p->ax1);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO<C> io{(const C*)w.V, (C*)w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<C> ax = p->ax1.dev<C>();
  if constexpr (std::is_same<C, float2>::value) {
    KP_DISPATCH_F(ax.KP, return launch_pass<C>(rows_vector_kernel<KPC, C>, KIND_ROWS, grid, sh, st, G, ax, io, epi));
  } else {
    KP_DISPATCH_D(ax.KP, return launch_pass<C>(rows_vector_kernel<KPC, C>, KIND_ROWS, grid, sh, st, G, ax, io, epi));
  }
  return BCCB_OK;
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// Kernel-path selection: 0 = automatic (small-grid persistent solver, specialised + fused
// shapes, generic fallback); 1 = generic runtime-shape kernels only.  Env BCCB_ROWS_VARIANT
// sets the default; bccb_set_path() overrides it (used by the tests to cross-check paths).
static std::atomic<int> g_path{-1};

static int rows_variant() {
  int v = g_path.load();
  if (v < 0) {
    const char* e = getenv("BCCB_ROWS_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

extern "C" int bccb_set_path(int path) {
  if (path < 0 || path > 1) return fail(BCCB_ERR_INVALID, "path must be 0 (auto) or 1 (generic)");
  g_path.store(path);
  return BCCB_OK;
}

// Specialised line shapes (compile-time KP, R, Mo) of the FISTA/ISTA rows pass.
#define FAST_SHAPES(X)                                                \
  X(16, 4, 1)    /* L1 = 64,   band 16  (config 1) */                 \
  X(32, 4, 1)    /* L1 = 128,  band 32 */                             \
  X(32, 8, 1)    /* L1 = 256,  band 32  (config 2) */                 \
  X(32, 8, 2)    /* L1 = 256,  band 64 */                             \
  X(32, 16, 1)   /* L1 = 512,  band 32 */                             \
  X(32, 16, 2)   /* L1 = 512,  band 64  (config 3 shape) */           \
  X(32, 32, 1)   /* L1 = 1024, band 32 */                             \
  X(32, 32, 2)   /* L1 = 1024, band 64  (config 4) */                 \
  X(32, 64, 4)   /* L1 = 2048, band 128 */                            \
  X(32, 128, 4)  /* L1 = 4096, band 128 (config 5) */

static int fast_key(const AxisPrec& a) { return a.KP * 100000 + a.R * 10 + a.Mo; }

static bool fast_supported(const bccb_plan_s* p, int batch, const void* extra) {
  if (extra || rows_variant() != 0) return false;
  const AxisPrec& a = rows_axis(p->ax1);
  if (rows_use_kp16(p->ax1))
    return (long long)batch * p->L2 < (1LL << 31) && p->L2 % (zs_threads(p->ax1) / a.R) == 0;
  const int tr = zs_threads(p->ax1) / a.R;
  if ((long long)batch * p->L2 >= (1LL << 31) || p->L2 % tr != 0) return false;
  const int key = fast_key(a);
#define FAST_KEY(KP_, R_, MO_) \
  if (key == KP_ * 100000 + R_ * 10 + MO_) return true;
  FAST_SHAPES(FAST_KEY)
#undef FAST_KEY
  return false;
}

static LaunchShape fast_shape(const bccb_plan_s* p) {
  const AxisPrec& a = rows_axis(p->ax1);
  LaunchShape sh;
  sh.threads = zs_threads(p->ax1);
  sh.TR = sh.threads / a.R;
  const int pitch = (a.R % 2 == 1) ? a.R : a.R + 1;
  // band tile + transpose buffer (+ staged twiddles [KP][R], [Mo][R] when <= 8 KB: STAGE_TW)
  const size_t tw = (size_t)(a.KP + a.Mo) * a.R;
  sh.smem = ((size_t)sh.TR * (p->ax1.K + 2) + (size_t)sh.TR * a.KP * pitch + (tw * 8 <= 8192 ? tw : 0)) *
            sizeof(float2);   // TileShape: band rows of K + 2
  return sh;
}

// Fused column pass: enabled when one snapshot's column work (K1 x L2 points) is no more than
// one rows CTA's work (TR x L1 points) and the shape has a fused specialisation.
#define FUSED_SHAPES(X)                            \
  X(16, 4, 1, 16, 2)  /* config 1 */              \
  X(32, 8, 1, 16, 2)  /* config 2, KP 32 engine */ \
  X(16, 16, 2, 16, 3) /* config 2, KP 16 engine */ \
  X(16, 16, 2, 16, 4) /* same, 4 CTAs/SM (BCCB_FUSED_MINB=4) */

// The last CTA's column tail must not dominate: one snapshot's column work (K1 x L2 points) is
// at most one rows CTA's work (TR x L1 points).
static bool fused_supported(const bccb_plan_s* p) {
  static const int env = [] {
    const char* e = getenv("BCCB_FUSE_COLS");
    return e ? atoi(e) : 1;
  }();
  if (!env) return false;
  const AxisPrec& a = rows_axis(p->ax1);
  const int tr = zs_threads(p->ax1) / a.R;
  if ((long long)p->ax1.K * p->L2 > (long long)tr * p->L1) return false;
  const AxisPrec& c = p->ax2.s;
  const int trc = std::min(zs_threads(p->ax1) / c.R, p->ax1.K);
  if (trc < 1 || p->ax1.K % trc != 0) return false;
  const int key = fast_key(a);
#define FUSED_KEY(KP_, R_, MO_, KP2_, MINB_) \
  if (key == KP_ * 100000 + R_ * 10 + MO_ && c.KP == KP2_) return true;
  FUSED_SHAPES(FUSED_KEY)
#undef FUSED_KEY
  return false;
}

static int fused_minb() {
  static const int v = [] {
    const char* e = getenv("BCCB_FUSED_MINB");
    return e ? atoi(e) : 3;
  }();
  return v;
}

static FusedCols make_fused(const bccb_plan_s* p, int batch, const Workspace& w, const float2* D, const float2* P,
                            const float2* Bh) {
  FusedCols fc{};
  const AxisPrec& c = p->ax2.s;
  fc.ax = p->ax2.dev_s();
  fc.io.U = (const float2*)w.U;
  fc.io.V = (float2*)w.V;
  fc.io.D = D;
  fc.io.P = P;
  fc.io.Bh = Bh;
  fc.io.box_out = nullptr;
  fc.io.K1 = p->ax1.K;
  fc.G.L1 = p->L1;
  fc.G.L2 = p->L2;
  fc.G.rows = (long long)batch * p->ax1.K;
  fc.G.do_fwd = 1;
  fc.G.do_inv = 1;
  fc.TRc = std::min(zs_threads(p->ax1) / c.R, p->ax1.K);
  fc.G.TR = fc.TRc;
  fc.counter = w.counters;
  fc.cps = p->L2 / (zs_threads(p->ax1) / rows_axis(p->ax1).R);
  fc.K1 = p->ax1.K;
  return fc;
}

// Tensor-core rows pass (rows_fista_tc_kernel): persistent CTAs (resident CTAs per SM x SMs),
// shared memory = band tile + forward transpose + staged twiddles + A tiles + B tiles.
template <int KP, int MO, bool MOM, bool TRACE>
static int launch_tc_shape(const bccb_plan_s* p, const Geo& G, const AxisT<float2>& ax, const RowsIO<float2>& io,
                           const EpiFista& epi, unsigned* fl, cudaStream_t st) {
  using TS = TileShape<KP, 128, MO, tc_threads(KP)>;
  using TSH = TcShape<KP, MO, TS::TR>;
  // resident CTAs per SM the register budget targets: the KP-point register DFT dominates
  constexpr int MINB = (KP == 8 ? 4 : (KP == 16 ? 3 : 2)) * (256 / tc_threads(KP));
  auto k = rows_fista_tc_kernel<KP, MO, MOM, MINB, TRACE>;
  size_t smem = (size_t)(TS::TR * TS::XP + TS::TR * TS::SP) * sizeof(float2);
  if (TS::STAGE_TW) smem += (size_t)(KP + MO) * 128 * sizeof(float2);
  smem = ((smem + 127) & ~(size_t)127) + TSH::A_BYTES + TSH::B_BYTES;
  // resident CTAs per SM: the register budget of __launch_bounds__ (MINB), capped by shared
  // memory (228 KB per SM, 1 KB reserved per CTA) and TMEM (512 columns per SM).  The shared-
  // memory carveout is pinned to its maximum so the driver does not pick a smaller split (the
  // occupancy API's default-carveout answer gave one CTA per SM: profiles/r2/r2b_*).
  static int o = 0;                      // per instantiation
  if (!o) {
    int rc = prep_smem(k, smem);
    if (rc) return rc;
    CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  (int)cudaSharedmemCarveoutMaxShared));
    cudaFuncAttributes fa;
    CUDA_TRY(cudaFuncGetAttributes(&fa, k));
    const size_t per_cta = smem + fa.sharedSizeBytes + 1024;       // dynamic + static + reserved
    o = std::min<int>(MINB, (int)((228 * 1024) / per_cta));
    o = std::min(o, 512 / TSH::COLS);
    if (o < 1) return fail(BCCB_ERR_UNSUPPORTED, "tensor-core rows pass does not fit one SM");
    // The kernel spills a few loop-carried scalars (128-register budget): leave the L1 as much
    // room as the resident CTAs allow instead of the maximum shared-memory split (the spill
    // reloads were L2 round trips with a 28 KB L1, profiles/r2/r2j_*).  Keep the smaller split
    // only if the occupancy API confirms the same number of resident CTAs.
    if (!(debug_env() & 4)) {      // BCCB_DEBUG bit 4: keep the maximum shared-memory split (A/B)
      const int want_kb = (int)((o * per_cta + 1023) / 1024);
      const int pct = std::min(100, (want_kb * 100 + 227) / 228 + 1);
      if (cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct) == cudaSuccess) {
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, TS::NT, smem) != cudaSuccess || n < o)
          CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        (int)cudaSharedmemCarveoutMaxShared));
      }
      (void)cudaGetLastError();
    }
  }
  const int ntiles = (int)((G.rows + TS::TR - 1) / TS::TR);
  const unsigned grid = (unsigned)std::min<long long>(ntiles, (long long)o * num_sms());
  LaunchShape sh;
  sh.threads = TS::NT;
  sh.TR = TS::TR;
  sh.smem = smem;
  return launch_pass<float2>(k, KIND_ROWS, grid, sh, st, G, ax, io, epi, fl, ntiles);
}

static int launch_rows_fista_tc(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                                const EpiFista& epi, cudaStream_t st) {
  LaunchShape sh;
  sh.threads = tc_threads(p->ax1.t.KP);
  sh.TR = sh.threads / 128;
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO<float2> io{(const float2*)w.V, (float2*)w.U};
  const AxisT<float2> ax = p->ax1.dev_t();
  unsigned* fl = (unsigned*)w.flags;
  const bool mom = epi.momentum != 0;
#define TC_CASE(KP_, MO_)                                                                          \
  if (ax.KP == KP_ && ax.Mo == MO_) {                                                              \
    if (epi.trace)                                                                                 \
      return mom ? launch_tc_shape<KP_, MO_, true, true>(p, G, ax, io, epi, fl, st)                \
                 : launch_tc_shape<KP_, MO_, false, true>(p, G, ax, io, epi, fl, st);              \
    return mom ? launch_tc_shape<KP_, MO_, true, false>(p, G, ax, io, epi, fl, st)                 \
               : launch_tc_shape<KP_, MO_, false, false>(p, G, ax, io, epi, fl, st);               \
  }
  TC_SHAPES(TC_CASE)
#undef TC_CASE
  return fail(BCCB_ERR_UNSUPPORTED, "no tensor-core rows specialisation (KP %d, Mo %d)", ax.KP, ax.Mo);
}

static int launch_rows_fista_fast(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                                  const EpiFista& epi, bool zs, cudaStream_t st, const FusedCols* fused = nullptr) {
  if (!zs) return fail(BCCB_ERR_UNSUPPORTED, "the specialised rows pass runs with zero-segment skipping");
  LaunchShape sh = fast_shape(p);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO<float2> io{(const float2*)w.V, (float2*)w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<float2> ax = p->ax1.dev<float2>();
  const bool mom = epi.momentum != 0;
  unsigned* fl = (unsigned*)w.flags;
  const int key = fast_key(p->ax1.f);
  if (fused && zs) {
    const AxisPrec& c = p->ax2.s;
    const int pitch2 = (c.R % 2 == 1) ? c.R : c.R + 1;
    const size_t need = ((size_t)fused->TRc * (p->ax2.K + 1) + (size_t)fused->TRc * c.KP * pitch2) * sizeof(float2);
    sh.smem = std::max(sh.smem, need);
    const AxisT<float2> axr = rows_use_kp16(p->ax1) ? p->ax1.dev_s() : p->ax1.dev<float2>();
    const int keyr = fast_key(rows_axis(p->ax1));
#define FUSED_CASE(KP_, R_, MO_, KP2_, MINB_)                                                               \
  if (keyr == KP_ * 100000 + R_ * 10 + MO_ && c.KP == KP2_ && (MINB_ == 2 || MINB_ == fused_minb()))                                               \
    return mom ? launch_pass<float2>(rows_fista_fast_kernel<KP_, R_, MO_, true, true, KP2_, MINB_>, KIND_ROWS, grid, \
                                     sh, st, G, axr, io, epi, fl, *fused)                                   \
               : launch_pass<float2>(rows_fista_fast_kernel<KP_, R_, MO_, false, true, KP2_, MINB_>, KIND_ROWS, grid, \
                                     sh, st, G, axr, io, epi, fl, *fused);
    FUSED_SHAPES(FUSED_CASE)
#undef FUSED_CASE
    return fail(BCCB_ERR_UNSUPPORTED, "no fused specialisation for this line shape");
  }
  if (rows_use_kp16(p->ax1)) {
    const AxisT<float2> axs = p->ax1.dev_s();
    const FusedCols nofc16{};
    const int k16 = fast_key(p->ax1.s);
#define K16_CASE(R_, MO_)                                                                                \
  if (k16 == 16 * 100000 + R_ * 10 + MO_) {                                                              \
    if (epi.trace)                                                                                       \
      return mom ? launch_pass<float2>(rows_fista_fast_kernel<16, R_, MO_, true, true, 0, 3, true>, KIND_ROWS, grid, \
                                       sh, st, G, axs, io, epi, fl, nofc16)                              \
                 : launch_pass<float2>(rows_fista_fast_kernel<16, R_, MO_, false, true, 0, 3, true>, KIND_ROWS,    \
                                       grid, sh, st, G, axs, io, epi, fl, nofc16);                       \
    return mom ? launch_pass<float2>(rows_fista_fast_kernel<16, R_, MO_, true, true, 0, 3>, KIND_ROWS, grid, sh, \
                                     st, G, axs, io, epi, fl, nofc16)                                    \
               : launch_pass<float2>(rows_fista_fast_kernel<16, R_, MO_, false, true, 0, 3>, KIND_ROWS, grid, sh, \
                                     st, G, axs, io, epi, fl, nofc16);                                   \
  }
    K16_CASE(16, 2) K16_CASE(64, 4)
#undef K16_CASE
  }
  const FusedCols nofc{};
  if (epi.trace) {   // traced variants exist for the config-5 line shape only (trace_supported)
    if (zs && key == 32 * 100000 + 128 * 10 + 4)
      return mom ? launch_pass<float2>(rows_fista_fast_kernel<32, 128, 4, true, true, 0, 2, true>, KIND_ROWS, grid,
                                       sh, st, G, ax, io, epi, fl, nofc)
                 : launch_pass<float2>(rows_fista_fast_kernel<32, 128, 4, false, true, 0, 2, true>, KIND_ROWS, grid,
                                       sh, st, G, ax, io, epi, fl, nofc);
    return fail(BCCB_ERR_UNSUPPORTED, "no traced rows specialisation for this line shape");
  }
#define FAST_CASE(KP_, R_, MO_)                                                                              \
  if (key == KP_ * 100000 + R_ * 10 + MO_)                                                                   \
    return mom ? launch_pass<float2>(rows_fista_fast_kernel<KP_, R_, MO_, true, true>, KIND_ROWS, grid, sh, st,   \
                                     G, ax, io, epi, fl, nofc)                                               \
               : launch_pass<float2>(rows_fista_fast_kernel<KP_, R_, MO_, false, true>, KIND_ROWS, grid, sh, st,  \
                                     G, ax, io, epi, fl, nofc);
  FAST_SHAPES(FAST_CASE)
#undef FAST_CASE
  return fail(BCCB_ERR_UNSUPPORTED, "no specialisation for this line shape");
}

// Specialised line shapes of the ADMM rows pass (complex128 axis, KP <= 16).
#define ADMM_SHAPES(X)                                   \
  X(16, 4, 1)    /* L1 = 64,   band 16 */                \
  X(16, 16, 2)   /* L1 = 256,  band 32 */                \
  X(16, 32, 4)   /* L1 = 512,  band 64  (config 3) */    \
  X(16, 64, 4)   /* L1 = 1024, band 64 */                \
  X(16, 256, 8)  /* L1 = 4096, band 128 */

static bool admm_fast_supported(const bccb_plan_s* p, int batch, const void* extra) {
  if (extra || rows_variant() != 0) return false;
  const AxisPrec& a = p->ax1.d;
  const int tr = std::max(256, a.R) / a.R;
  if ((long long)batch * p->L2 >= (1LL << 31) || p->L2 % tr != 0) return false;
  const int key = fast_key(a);
#define ADMM_KEY(KP_, R_, MO_) \
  if (key == KP_ * 100000 + R_ * 10 + MO_) return true;
  ADMM_SHAPES(ADMM_KEY)
#undef ADMM_KEY
  return false;
}

static LaunchShape admm_shape(const bccb_plan_s* p) {
  const AxisPrec& a = p->ax1.d;
  LaunchShape sh;
  sh.threads = std::max(256, a.R);
  sh.TR = sh.threads / a.R;
  const int pitch = (a.R % 2 == 1) ? a.R : a.R + 1;
  sh.smem = ((size_t)sh.TR * (p->ax1.K + 1) + (size_t)sh.TR * a.KP * pitch) * sizeof(double2);
  return sh;
}

static int launch_rows_admm_fast(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                                 const EpiAdmm& epi, cudaStream_t st) {
  const LaunchShape sh = admm_shape(p);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO<double2> io{(const double2*)w.V, (double2*)w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<double2> ax = p->ax1.dev<double2>();
  unsigned* fl = (unsigned*)w.flags;
  const int key = fast_key(p->ax1.d);
#define ADMM_CASE(KP_, R_, MO_)                                                                          \
  if (key == KP_ * 100000 + R_ * 10 + MO_)                                                               \
    return launch_pass<double2>(rows_admm_fast_kernel<KP_, R_, MO_, true>, KIND_ROWS, grid, sh, st, G, ax, io, \
                                epi, fl);
  ADMM_SHAPES(ADMM_CASE)
#undef ADMM_CASE
  return fail(BCCB_ERR_UNSUPPORTED, "no ADMM specialisation for this line shape");
}

static int launch_zero_segments_z(const bccb_plan_s* p, int batch, const Workspace& w, double2* z, cudaStream_t st) {
  LaunchShape sh = admm_shape(p);
  const Geo G = rows_geo(p, batch, sh, false, false);
  sh.smem = 0;
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const int key = fast_key(p->ax1.d);
  const unsigned* fl = (const unsigned*)w.flags;
#define ZZ_CASE(KP_, R_, MO_)                                                                             \
  if (key == KP_ * 100000 + R_ * 10 + MO_)                                                                \
    return launch_pass<double2>(zero_segments_z_kernel<KP_, R_>, KIND_OTHER, grid, sh, st, G, z, fl);
  ADMM_SHAPES(ZZ_CASE)
#undef ZZ_CASE
  return fail(BCCB_ERR_UNSUPPORTED, "no ADMM specialisation for this line shape");
}

template <typename T2>
static int launch_zero_segments(const bccb_plan_s* p, int batch, const Workspace& w, double2* c, T2* d,
                                cudaStream_t st, bool tc = false) {
  LaunchShape sh = fast_shape(p);
  if (tc) {
    sh.threads = tc_threads(p->ax1.t.KP);
    sh.TR = sh.threads / 128;
  }
  const Geo G = rows_geo(p, batch, sh, false, false);
  sh.smem = 0;
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const unsigned* fl = (const unsigned*)w.flags;
  if (tc) {
    const int kp = p->ax1.t.KP;
    if (kp == 8)
      return launch_pass<float2>(zero_segments_kernel<8, 128, T2, tc_threads(8)>, KIND_OTHER, grid, sh, st, G, c, d, fl);
    if (kp == 16)
      return launch_pass<float2>(zero_segments_kernel<16, 128, T2, tc_threads(16)>, KIND_OTHER, grid, sh, st, G, c, d, fl);
    if (kp == 32)
      return launch_pass<float2>(zero_segments_kernel<32, 128, T2, tc_threads(32)>, KIND_OTHER, grid, sh, st, G, c, d, fl);
    return fail(BCCB_ERR_UNSUPPORTED, "no tensor-core zero-segment specialisation");
  }
  if (rows_use_kp16(p->ax1)) {
    if (p->ax1.s.R == 16) return launch_pass<float2>(zero_segments_kernel<16, 16, T2>, KIND_OTHER, grid, sh, st, G, c, d, fl);
    if (p->ax1.s.R == 64) return launch_pass<float2>(zero_segments_kernel<16, 64, T2>, KIND_OTHER, grid, sh, st, G, c, d, fl);
  }
  const int key = fast_key(p->ax1.f);
#define ZERO_CASE(KP_, R_, MO_)                                                                           \
  if (key == KP_ * 100000 + R_ * 10 + MO_)                                                                \
    return launch_pass<float2>(zero_segments_kernel<KP_, R_, T2>, KIND_OTHER, grid, sh, st, G, c, d, fl);
  FAST_SHAPES(ZERO_CASE)
#undef ZERO_CASE
  return fail(BCCB_ERR_UNSUPPORTED, "no specialisation for this line shape");
}

// Generic rows pass (runtime line shape): register-pipelined kernel.
static int launch_rows_fista(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                             const EpiFista& epi, cudaStream_t st) {
  const LaunchShape sh = shape_for<float2>(p->ax1);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO<float2> io{(const float2*)w.V, (float2*)w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<float2> ax = p->ax1.dev<float2>();
  KP_DISPATCH_F(ax.KP, {
    constexpr int CH = KPC < 2 ? KPC : 2;
    return launch_pass<float2>(rows_fista_kernel<KPC, CH, 2>, KIND_ROWS, grid, sh, st, G, ax, io, epi);
  });
  return BCCB_OK;
}

static int launch_rows_admm(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                            const EpiAdmm& epi, cudaStream_t st) {
  const LaunchShape sh = shape_for<double2>(p->ax1);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO<double2> io{(const double2*)w.V, (double2*)w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<double2> ax = p->ax1.dev<double2>();
  KP_DISPATCH_D(ax.KP, {
    constexpr int CH = KPC < 4 ? KPC : 4;
    return launch_pass<double2>(rows_admm_kernel<KPC, CH>, KIND_ROWS, grid, sh, st, G, ax, io, epi);
  });
  return BCCB_OK;
}

// Complex64 column passes run the streaming axis (KP <= 16), or its KP <= 8 variant when the
// launch has so few threads that latency dominates (config 2: 1024 lines x 16 threads;
// measured 153 -> 160 G gpi/s; the larger configs lose with KP 8).
static bool cols_narrow(const bccb_plan_s* p, int batch) {
  const long long threads = (long long)batch * p->ax1.K * p->ax2.s.R;
  return p->ax2.s8.KP < p->ax2.s.KP && threads < 65536;
}

// Warp-per-line column pass (cols_warp_kernel): lines of R = 32 threads with a band of 32
// (KP = 8 or 16): config 2's L2 = 256 (193 -> 205 G gpi/s), config 4's L2 = 512 (288 -> 297 G).
// A band of 64 (config 3's split ADMM, NSET = 2) measured neutral (299 vs 298 G) and keeps the
// shared-memory pass.  BCCB_COLS_WARP=0 keeps the shared-memory column pass everywhere.
static bool cols_warp_supported(const bccb_plan_s* p, const AxisPrec& a) {
  static const int env = [] {
    const char* e = getenv("BCCB_COLS_WARP");
    return e ? atoi(e) : 1;
  }();
  if (!env || a.R != 32) return false;
  const int K = p->ax2.K;
  return K == 32 && (a.KP == 8 || a.KP == 16);
}

template <typename Op, typename... Args>
static int launch_cols_warp(const bccb_plan_s* p, const AxisPrec& a, const Geo& G, cudaStream_t st,
                            Args... args) {
  LaunchShape shw;
  shw.TR = 8;
  shw.threads = 256;
  shw.smem = 0;
  const unsigned gw = (unsigned)((G.rows + 7) / 8);
  const int K = p->ax2.K;
  if (K == 32 && a.KP == 8) return launch_pass<float2>(cols_warp_kernel<8, 1, Op>, KIND_COLS, gw, shw, st, G, args...);
  if (K == 32 && a.KP == 16) return launch_pass<float2>(cols_warp_kernel<16, 1, Op>, KIND_COLS, gw, shw, st, G, args...);
  return fail(BCCB_ERR_UNSUPPORTED, "no warp column pass for this shape");
}

template <typename C>
static int launch_cols(const bccb_plan_s* p, int batch, bool fwd, bool inv, const Workspace& w,
                       const C* D, const C* P, const float2* Bh, C* box_out, cudaStream_t st,
                       const ObjBox* ob = nullptr) {
  const bool stream_axis = std::is_same<C, float2>::value;
  const bool narrow = stream_axis && cols_narrow(p, batch);
  const LaunchShape sh = stream_axis ? shape_for_prec(p->ax2, narrow ? p->ax2.s8 : p->ax2.s, sizeof(C),
                                                      (long long)batch * p->ax1.K)
                                     : shape_for<C>(p->ax2, (long long)batch * p->ax1.K);
  Geo G;
  G.L1 = p->L1;
  G.L2 = p->L2;
  G.rows = (long long)batch * p->ax1.K;
  G.TR = sh.TR;
  G.do_fwd = fwd ? 1 : 0;
  G.do_inv = inv ? 1 : 0;
  G.dbg = debug_env();
  ColsIO<C> io{};
  io.U = (const C*)w.U;
  io.V = (C*)w.V;
  io.D = D;
  io.P = P;
  io.Bh = Bh;
  io.box_out = box_out;
  io.K1 = p->ax1.K;
  if (ob) io.ob = *ob;
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  // room for the split level-2 forward sums of cols_kernel ([NP][TR*K], NP <= 4) when a CTA
  // has at least twice as many threads as band outputs
  LaunchShape shs = sh;
  if (fwd && sh.threads >= 2 * sh.TR * p->ax2.K)
    shs.smem += (size_t)std::min(4, sh.threads / (sh.TR * p->ax2.K)) * sh.TR * p->ax2.K * sizeof(C);
  if constexpr (std::is_same<C, float2>::value) {
    const AxisT<C> ax = p->ax2.dev_s(narrow);
    const AxisPrec& ap = narrow ? p->ax2.s8 : p->ax2.s;
    if (cols_warp_supported(p, ap)) return launch_cols_warp<BandMulAdd>(p, ap, G, st, ax, io, BandMulAdd{});
    KP_DISPATCH_F(ax.KP, return launch_pass<C>(cols_kernel<KPC, C>, KIND_COLS, grid, shs, st, G, ax, io));
  } else {
    const AxisT<C> ax = p->ax2.dev<C>();
    KP_DISPATCH_D(ax.KP, return launch_pass<C>(cols_kernel<KPC, C>, KIND_COLS, grid, shs, st, G, ax, io));
  }
  return BCCB_OK;
}

// D / P boxes for one operation ([K1][K2], complex64 or complex128), from the complex128
// eigenvalue box (1/L of the unnormalised inverse folded in):
//   mode 0 (matvec):  D = (lam - lam_out) / L
//   mode 1 (ISTA):    D = -mu (lam - lam_out) / L,           P = mu / L
//   mode 2 (ADMM):    D = (rho/(lam+rho) - a) / L,           P = 1 / ((lam + rho) L)
template <typename C>
__global__ void coef_kernel(const double2* __restrict__ lam, int n, int mode, double s1,
                            double lam_out, double a, double invL, C* D, C* P) {
  using R = decltype(C::x);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lr = lam[i].x, li = lam[i].y;
  if (mode == 0) {
    D[i] = C{(R)((lr - lam_out) * invL), (R)(li * invL)};
  } else if (mode == 1) {
    D[i] = C{(R)(-s1 * (lr - lam_out) * invL), (R)(-s1 * li * invL)};
    P[i] = C{(R)(s1 * invL), (R)0};
  } else if (mode == 2) {
    // q = 1/(lam + rho) ; D = rho*q - a
    const double dr = lr + s1, di = li;
    const double den = dr * dr + di * di;
    const double qr = dr / den, qi = -di / den;
    D[i] = C{(R)((s1 * qr - a) * invL), (R)(s1 * qi * invL)};
    P[i] = C{(R)(qr * invL), (R)(qi * invL)};
  }
}

template <typename C>
static int launch_coef(const bccb_plan_s* p, int mode, double s1, double a, const Workspace& w,
                       cudaStream_t st) {
  const int n = p->ax1.K * p->ax2.K;
  const double invL = 1.0 / ((double)p->L1 * (double)p->L2);
  ProfEvent* pe;
  prof_before(KIND_OTHER, st, &pe);
  coef_kernel<C><<<(n + 255) / 256, 256, 0, st>>>(p->lam_box_dev, n, mode, s1, p->lam_out.real(), a,
                                                   invL, (C*)w.D, (C*)w.P);
  prof_after(pe, st);
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
template <typename C>
static int matvec_impl(bccb_plan_t p, int batch, const void* x, void* y, void* workspace, void* stream) {
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!x || !y) return fail(BCCB_ERR_INVALID, "x / y is NULL");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  using R = decltype(C::x);
  if ((rc = launch_coef<C>(p, 0, 0.0, 0.0, w, st))) return rc;
  EpiVector<C> e{(const C*)x, nullptr, nullptr, R(0), R(1)};
  if ((rc = launch_rows_vector<C>(p, batch, false, true, w, e, st))) return rc;
  if ((rc = launch_cols<C>(p, batch, true, true, w, (const C*)w.D, nullptr, nullptr, nullptr, st))) return rc;
  EpiVector<C> e2{(const C*)x, (C*)y, nullptr, (R)p->lam_out.real(), R(1)};
  return launch_rows_vector<C>(p, batch, true, false, w, e2, st);
}

extern "C" int bccb_matvec(bccb_plan_t p, int batch, const void* x, void* y, void* workspace,
                           void* stream) {
  EntryScope entry_scope_("bccb_matvec");
  return matvec_impl<float2>(p, batch, x, y, workspace, stream);
}

extern "C" int bccb_matvec_z(bccb_plan_t p, int batch, const void* x, void* y, void* workspace,
                             void* stream) {
  EntryScope entry_scope_("bccb_matvec_z");
  return matvec_impl<double2>(p, batch, x, y, workspace, stream);
}

extern "C" int bccb_spectrum_box(bccb_plan_t p, int batch, const void* x, void* out_box,
                                 void* workspace, void* stream) {
  EntryScope entry_scope_("bccb_spectrum_box");
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!x || !out_box) return fail(BCCB_ERR_INVALID, "x / out_box is NULL");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  EpiVector<float2> e{(const float2*)x, nullptr, nullptr, 0.f, 1.f};
  if ((rc = launch_rows_vector<float2>(p, batch, false, true, w, e, st))) return rc;
  return launch_cols<float2>(p, batch, true, false, w, nullptr, nullptr, nullptr, (float2*)out_box, st);
}

extern "C" int bccb_synthesize(bccb_plan_t p, int batch, const void* box, float scale, const void* x,
                               float alpha, void* out, float* maxabs, void* workspace,
                               void* stream) {
  EntryScope entry_scope_("bccb_synthesize");
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!box) return fail(BCCB_ERR_INVALID, "box is NULL");
  if (alpha != 0.f && !x) return fail(BCCB_ERR_INVALID, "x is NULL with alpha != 0");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  if ((rc = launch_cols<float2>(p, batch, false, true, w, nullptr, nullptr, (const float2*)box, nullptr, st)))
    return rc;
  EpiVector<float2> e{(const float2*)x, (float2*)out, maxabs, alpha, scale};
  return launch_rows_vector<float2>(p, batch, true, false, w, e, st);
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
  EntryScope entry_scope_("bccb_adjoint");
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
  ProfEvent* pe;
  prof_before(KIND_OTHER, st, &pe);
  adjoint_scatter_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      (const float2*)y, p->occ_dev, p->M, K1, K2, total, L, p->occ_alias, (float2*)bhat_box);
  prof_after(pe, st);
  LAUNCH_CHECK();
  if (maxabs) CUDA_TRY(cudaMemsetAsync(maxabs, 0, (size_t)batch * sizeof(float), st));
  if (!b && !maxabs) return BCCB_OK;
  const float invL = (float)(1.0 / ((double)p->L1 * (double)p->L2));
  if ((rc = launch_cols<float2>(p, batch, false, true, w, nullptr, nullptr, (const float2*)bhat_box,
                                nullptr, st)))
    return rc;
  EpiVector<float2> e{nullptr, (float2*)b, maxabs, 0.f, invL};
  return launch_rows_vector<float2>(p, batch, true, false, w, e, st);
}

// ------------------------------------------------------------------ solvers
__global__ void fill_int_kernel(int* p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

static int reset_first_bad(int* first_bad, int batch, cudaStream_t st) {
  ProfEvent* pe;
  prof_before(KIND_OTHER, st, &pe);
  fill_int_kernel<<<(batch + 255) / 256, 256, 0, st>>>(first_bad, batch, INT_MAX);
  prof_after(pe, st);
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

// Sub-batch split into n streams (BCCB_SUBSTREAMS / bccb_set_substreams; 1 disables): only
// while each part still fills the GPU (>= 2048 lines).
static std::atomic<int> g_substreams{-1};

extern "C" int bccb_set_substreams(int n) {
  if (n < 0 || n > bccb_plan_s::MAX_SUB) return fail(BCCB_ERR_INVALID, "substreams must be in [0, %d]", bccb_plan_s::MAX_SUB);
  g_substreams.store(n == 0 ? -1 : n);
  return BCCB_OK;
}

static int sub_batches(const bccb_plan_s* p, int batch) {
  int n = g_substreams.load();
  if (n < 0) {
    const char* e = getenv("BCCB_SUBSTREAMS");
    // short lines (L1 <= 256) are latency-bound: four sub-batches (config 2 with PDL mode 2:
    // 3: 204.2, 4: 204.9 G gpi/s); longer lines keep three (config 4: 297.4 vs 296.9, config 3
    // ADMM: 299.6 vs 298.3; profiles/ab/r1_substreams_pdl2.txt).  Earlier (PDL mode 1):
    n = e ? atoi(e) : (p->L1 <= 256 ? 4 : 3);   // measured at config 2 (2: 171, 3: 186, 4: 177 G gpi/s;
                          // with the warp column pass 2: 202.1, 3: 202.5, 4: 196.5, 5: 179.4)
  }
  n = std::max(1, std::min(n, bccb_plan_s::MAX_SUB));
  // BCCB_SUB_MIN_LINES lowers the per-part floor so small test batches exercise the split
  static const long long min_lines = [] {
    const char* e = getenv("BCCB_SUB_MIN_LINES");
    return e ? std::max(1LL, atoll(e)) : 2048LL;
  }();
  while (n > 1 && (batch < n || (long long)(batch / n) * p->L2 < min_lines)) --n;
  return n;
}

extern "C" int bccb_substreams_for(bccb_plan_t p, int batch) {
  if (!p || batch < 1) return 1;
  return sub_batches(p, batch);
}

// Sub-batch streams and fork/join events: per calling thread and device, so concurrent solves
// on one plan from different threads never share an event (created lazily, reused).
struct SubStreams {
  cudaStream_t aux[bccb_plan_s::MAX_SUB - 1] = {};
  cudaEvent_t fork = nullptr, join[bccb_plan_s::MAX_SUB - 1] = {};
};
static thread_local SubStreams t_sub[64];

static int ensure_aux_streams(const bccb_plan_s* p, int n, SubStreams** out) {
  SubStreams& ss = t_sub[p->device & 63];
  if (!ss.fork) CUDA_TRY(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
  for (int i = 0; i < n - 1; ++i) {
    if (ss.aux[i]) continue;
    CUDA_TRY(cudaStreamCreateWithFlags(&ss.aux[i], cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ss.join[i], cudaEventDisableTiming));
  }
  *out = &ss;
  return BCCB_OK;
}

// ---- small-grid persistent solver (whole snapshot state in shared memory, all iterations in
// one launch, one CTA per snapshot)
static size_t small_smem(const bccb_plan_s* p, bool mom, int* trc_out) {
  const AxisPrec& r = p->ax1.f;
  const AxisPrec& c = p->ax2.s;
  const size_t L = (size_t)p->L1 * p->L2;
  const int nthr = std::max(p->L2 * r.R, 256);
  const int trc = std::min(nthr / c.R, p->ax1.K);
  if (trc_out) *trc_out = trc;
  const int p1 = (r.R % 2 == 1) ? r.R : r.R + 1, p2 = (c.R % 2 == 1) ? c.R : c.R + 1;
  const size_t rows_scr = (size_t)p->L2 * (p->ax1.K + 1) + (size_t)p->L2 * r.KP * p1;
  const size_t cols_scr = (size_t)trc * (p->ax2.K + 1) + (size_t)trc * c.KP * p2;
  return L * 16 + (mom ? L * 8 : 0) + 2 * (size_t)p->ax1.K * p->L2 * 8 + std::max(rows_scr, cols_scr) * 8;
}

static bool small_supported(const bccb_plan_s* p, const void* extra, bool mom) {
  static const int env = [] {
    const char* e = getenv("BCCB_SMALL_GRID");
    return e ? atoi(e) : 1;
  }();
  if (!env || extra || rows_variant() != 0) return false;
  const AxisPrec& r = p->ax1.f;
  const AxisPrec& c = p->ax2.s;
  if ((long long)p->L2 * r.R > 1024) return false;
  int trc = 0;
  if (small_smem(p, mom, &trc) > 220 * 1024) return false;
  if (trc < 1 || p->ax1.K % trc != 0) return false;
  const int key = r.KP * 100 + c.KP;
  return key == 1616 || key == 3216 || key == 1608 || key == 808 || key == 3208;
}

// momentum coefficients beta_t, t <= t_end, in a plan-owned device table (persistent solvers)
// FISTA momentum table beta[0..t_end] of the persistent small-grid / cluster solvers
// (beta_t = (alpha_{t-1} - 1) / alpha_t, solvers.py:294-337).  The sequence does not depend on
// the call, so one process-wide table per device serves every plan and thread; it only grows
// (filled synchronously before its pointer is published) and retired tables are kept, so a
// kernel still reading an older one stays valid.
static std::mutex g_beta_mu;
struct BetaTable {
  double* dev = nullptr;
  size_t cap = 0;
  std::vector<double*> retired;
};
static BetaTable g_beta[64];

static int beta_table(const bccb_plan_s* p, int t_end, const double** out) {
  std::lock_guard<std::mutex> lk(g_beta_mu);
  BetaTable& bt = g_beta[p->device & 63];
  if (bt.cap < (size_t)t_end + 1) {
    const size_t cap = std::max<size_t>({(size_t)t_end + 1, 2 * bt.cap, 1024});
    std::vector<double> host(cap, 0.0);
    double alpha = 1.0;
    for (size_t t = 1; t < cap; ++t) {
      const double an = 0.5 * (std::sqrt(1.0 + 4.0 * alpha * alpha) + 1.0);
      host[t] = (alpha - 1.0) / an;
      alpha = an;
    }
    double* dev = nullptr;
    CUDA_TRY(cudaMalloc(&dev, cap * sizeof(double)));
    CUDA_TRY(cudaMemcpy(dev, host.data(), cap * sizeof(double), cudaMemcpyHostToDevice));
    if (bt.dev) bt.retired.push_back(bt.dev);
    bt.dev = dev;
    bt.cap = cap;
  }
  *out = bt.dev;
  return BCCB_OK;
}

// ---- 64 x 64 cluster solver (8-CTA cluster per snapshot, distributed shared memory)
static bool cluster_supported(const bccb_plan_s* p, const void* extra) {
  static const int env = [] {
    const char* e = getenv("BCCB_CLUSTER");
    return e ? atoi(e) : 1;
  }();
  if (!env || extra || rows_variant() != 0) return false;
  const int K1 = p->ax1.K, K2 = p->ax2.K;
  return p->L1 == 64 && p->L2 == 64 && K1 % 8 == 0 && K2 % 8 == 0 && K1 <= 16 && K2 <= 16;
}

static int launch_cluster64(bccb_plan_s* p, int batch, int first, int iters, const EpiFista& e, const float2* D,
                            const float2* P, const float2* Bh, cudaStream_t st) {
  const double* beta_dev = nullptr;
  int rc = beta_table(p, first + iters, &beta_dev);
  if (rc) return rc;
  ClusterArgs A;
  A.D = D;
  A.P = P;
  A.Bh = Bh;
  A.epi = e;
  A.beta = beta_dev;
  A.K1 = p->ax1.K;
  A.K2 = p->ax2.K;
  A.iterations = iters;
  A.first_iteration = first;
  LaunchShape sh;
  sh.threads = 256;
  sh.TR = 1;
  sh.smem = 0;
  const unsigned grid = (unsigned)batch * 8u;
  return e.momentum ? launch_pass<float2>(cluster64_fista_kernel<true>, KIND_ROWS, grid, sh, st, A)
                    : launch_pass<float2>(cluster64_fista_kernel<false>, KIND_ROWS, grid, sh, st, A);
}

static int launch_small(bccb_plan_s* p, int batch, int first, int iters, const EpiFista& e, const float2* D,
                        const float2* P, const float2* Bh, cudaStream_t st) {
  const bool mom = e.momentum != 0;
  const double* beta_dev = nullptr;
  int rc0 = beta_table(p, first + iters, &beta_dev);
  if (rc0) return rc0;
  SmallArgs A;
  A.ax1 = p->ax1.dev<float2>();
  A.ax2 = p->ax2.dev_s();
  A.cio = ColsIO<float2>{};
  A.cio.D = D;
  A.cio.P = P;
  A.cio.Bh = Bh;
  A.cio.K1 = p->ax1.K;
  A.epi = e;
  A.beta = beta_dev;
  A.L1 = p->L1;
  A.L2 = p->L2;
  A.K1 = p->ax1.K;
  A.K2 = p->ax2.K;
  A.iterations = iters;
  A.first_iteration = first;
  LaunchShape sh;
  sh.smem = small_smem(p, mom, &A.TRc);
  sh.threads = std::max(p->L2 * p->ax1.f.R, 256);
  sh.TR = 1;
  const int key = p->ax1.f.KP * 100 + p->ax2.s.KP;
#define SMALL_CASE(KP1_, KP2_)                                                                         \
  if (key == KP1_ * 100 + KP2_)                                                                        \
    return mom ? launch_pass<float2>(small_fista_kernel<KP1_, KP2_, true>, KIND_ROWS, (unsigned)batch, sh, st, A) \
               : launch_pass<float2>(small_fista_kernel<KP1_, KP2_, false>, KIND_ROWS, (unsigned)batch, sh, st, A);
  SMALL_CASE(16, 16) SMALL_CASE(32, 16) SMALL_CASE(16, 8) SMALL_CASE(8, 8) SMALL_CASE(32, 8)
#undef SMALL_CASE
  return fail(BCCB_ERR_UNSUPPORTED, "no small-grid specialisation");
}

static int fista_run_impl(bccb_plan_t p, int batch, int first_iteration, int iterations, double mu,
                          const double* tau, const void* bhat_box, const void* extra, void* c, void* d,
                          int* first_bad, void* workspace, void* stream, double* trace);

extern "C" int bccb_fista_run(bccb_plan_t p, int batch, int first_iteration, int iterations,
                              double mu, const double* tau,
                              const void* bhat_box, const void* extra, void* c, void* d,
                              int* first_bad, void* workspace, void* stream) {
  EntryScope entry_scope_("bccb_fista_run");
  return fista_run_impl(p, batch, first_iteration, iterations, mu, tau, bhat_box, extra, c, d, first_bad,
                        workspace, stream, nullptr);
}

extern "C" int bccb_fista_run_traced(bccb_plan_t p, int batch, int iterations, double mu, const double* tau,
                                     const void* bhat_box, void* c, void* d, int* first_bad, double* trace,
                                     void* workspace, void* stream) {
  EntryScope entry_scope_("bccb_fista_run_traced");
  if (!trace) return fail(BCCB_ERR_INVALID, "NULL trace");
  return fista_run_impl(p, batch, 0, iterations, mu, tau, bhat_box, nullptr, c, d, first_bad, workspace, stream,
                        trace);
}

static int fista_run_impl(bccb_plan_t p, int batch, int first_iteration, int iterations, double mu,
                          const double* tau, const void* bhat_box, const void* extra, void* c, void* d,
                          int* first_bad, void* workspace, void* stream, double* trace) {
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
  if ((rc = launch_coef<float2>(p, 1, mu, 0.0, w, st))) return rc;
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
  e.trace = nullptr;
  e.trace_stride = 0;
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
  // fused objective trace: the per-pass kernels with zero-segment skipping, a Gram-type
  // spectrum (zero outside the box) and the right-hand side on the box
  if (trace) {
    // traced rows variants: the tensor-core engine, the KP16 engine and the config-5 KP32 shape
    const bool traced_shape = rows_use_tc(p->ax1) || rows_use_kp16(p->ax1) ||
                              fast_key(p->ax1.f) == 32 * 100000 + 128 * 10 + 4;
    if (first_iteration != 0 || extra || p->lam_out != std::complex<double>(0.0, 0.0) ||
        !fast_supported(p, batch, extra) || !traced_shape)
      return fail(BCCB_ERR_UNSUPPORTED, "fused objective trace needs a Gram operator on a specialised grid");
    CUDA_TRY(cudaMemsetAsync(trace, 0, (size_t)batch * iterations * sizeof(double), st));
  }
  // 64 x 64 grids: one 8-CTA cluster per snapshot runs the whole solve (distributed shared memory)
  if (!trace && cluster_supported(p, extra))
    return launch_cluster64(p, batch, first_iteration, iterations, e, (const float2*)w.D, (const float2*)w.P,
                            (const float2*)bhat_box, st);
  // small grids: the whole solve in one persistent launch per snapshot (shared-memory state)
  if (!trace && small_supported(p, extra, e.momentum != 0))
    return launch_small(p, batch, first_iteration, iterations, e, (const float2*)w.D, (const float2*)w.P,
                        (const float2*)bhat_box, st);
  // specialised shapes use zero-segment skipping: flags start all-ones (read everything) and
  // the skipped zeros are written back by one final pass
  const bool zs = fast_supported(p, batch, extra);
  const bool tcr = zs && rows_use_tc(p->ax1);   // tensor-core rows engine (its own tiling)
  if (zs) CUDA_TRY(cudaMemsetAsync(w.flags, 0xff, zs_flag_bytes(p, batch, tcr), st));

  // Sub-batch split: two halves of the batch run on two streams, so one half's (latency-bound)
  // column pass and kernel tails overlap the other half's rows pass.  Snapshots are
  // independent, so the arithmetic is identical to one stream (bitwise).
  const int nsub = sub_batches(p, batch);
  SubStreams* ss = nullptr;
  if (nsub > 1 && (rc = ensure_aux_streams(p, nsub, &ss))) return rc;
  struct Sub {
    int b0, nb;
    cudaStream_t st;
    Workspace w;
    EpiFista e;
  } sub[bccb_plan_s::MAX_SUB];
  for (int q = 0; q < nsub; ++q) {
    Sub& u = sub[q];
    u.b0 = (int)((long long)batch * q / nsub);
    u.nb = (int)((long long)batch * (q + 1) / nsub) - u.b0;
    u.st = q == 0 ? st : ss->aux[q - 1];
    u.w = w;
    const long long inter = (long long)u.b0 * p->ax1.K * p->L2;
    u.w.U = (float2*)w.U + inter;
    u.w.V = (float2*)w.V + inter;
    if (zs) u.w.flags = w.flags + zs_flag_bytes(p, u.b0, tcr);
    u.e = e;
    const long long off = (long long)u.b0 * p->L1 * p->L2;
    u.e.c = e.c + off;
    u.e.d = e.d ? e.d + off : nullptr;
    u.e.extra = e.extra ? e.extra + off : nullptr;
    u.e.tau = e.tau + u.b0;
    u.e.first_bad = e.first_bad + u.b0;
    u.e.it = first_iteration;
    u.e.beta_cur = u.e.momentum ? beta[first_iteration] : 0.0;
    u.e.beta_next = 0.0;
    if (trace) {
      u.e.trace = trace + (long long)u.b0 * iterations;
      u.e.trace_stride = iterations;
    }
  }
  // objective box terms of the column pass of iteration t (X = FFT2(x_t)): C_t from X_t and
  // C_{t-1} (workspace cb, float64), quadratic part into trace column t - 1
  auto obj_box = [&](int q, int t) {
    ObjBox ob{};
    const Sub& u = sub[q];
    const long long boxo = (long long)u.b0 * p->ax1.K * p->ax2.K;
    ob.chat = (double2*)w.cb + boxo;
    ob.lam = p->lam_box_dev;
    ob.bh = (const float2*)bhat_box + boxo;
    ob.trace = t >= 1 ? u.e.trace : nullptr;
    ob.stride = iterations;
    ob.col = t - 1;
    ob.beta = (u.e.momentum && t >= 1) ? beta[t] : 0.0;
    ob.inv_L = 1.0 / ((double)p->L1 * p->L2);
    ob.K2 = p->ax2.K;
    return ob;
  };
  const float2* bh = (const float2*)bhat_box;
  const bool fuse = zs && !tcr && !trace && fused_supported(p);
  FusedCols fcs[bccb_plan_s::MAX_SUB];
  for (int q = 0; q < nsub && fuse; ++q)
    fcs[q] = make_fused(p, sub[q].nb, sub[q].w, (const float2*)w.D, (const float2*)w.P,
                        bh + (long long)sub[q].b0 * p->ax1.K * p->ax2.K);
  if (fuse) {
    for (int q = 0; q < nsub; ++q) fcs[q].counter = w.counters + sub[q].b0;
    CUDA_TRY(cudaMemsetAsync(w.counters, 0, (size_t)batch * sizeof(int), st));
  }
  auto rows = [&](int q, bool inv, bool fwd) {
    Sub& u = sub[q];
    if (tcr) return launch_rows_fista_tc(p, u.nb, inv, fwd, u.w, u.e, u.st);
    return zs ? launch_rows_fista_fast(p, u.nb, inv, fwd, u.w, u.e, true, u.st, fuse ? &fcs[q] : nullptr)
              : launch_rows_fista(p, u.nb, inv, fwd, u.w, u.e, u.st);
  };
  if (nsub > 1) {
    CUDA_TRY(cudaEventRecord(ss->fork, st));
    for (int q = 1; q < nsub; ++q) CUDA_TRY(cudaStreamWaitEvent(ss->aux[q - 1], ss->fork, 0));
  }
  for (int q = 0; q < nsub; ++q)
    if ((rc = rows(q, false, true))) return rc;
  for (int t = first_iteration; t < t_end; ++t) {
    for (int q = 0; q < nsub; ++q) {
      Sub& u = sub[q];
      const ObjBox ob = trace ? obj_box(q, t) : ObjBox{};
      if (!fuse &&
          (rc = launch_cols<float2>(p, u.nb, true, true, u.w, (const float2*)w.D, (const float2*)w.P,
                                    bh + (long long)u.b0 * p->ax1.K * p->ax2.K, nullptr, u.st,
                                    trace ? &ob : nullptr)))
        return rc;
      u.e.it = t;
      u.e.beta_cur = u.e.momentum ? beta[t] : 0.0;
      u.e.beta_next = u.e.momentum ? beta[t + 1] : 0.0;
      if ((rc = rows(q, true, t + 1 < t_end || trace))) return rc;
    }
  }
  // objective of the last iterate: forward-only column pass on FFT2(x_{t_end}) (no V output)
  for (int q = 0; q < nsub && trace; ++q) {
    Sub& u = sub[q];
    const ObjBox ob = obj_box(q, t_end);
    if ((rc = launch_cols<float2>(p, u.nb, true, false, u.w, (const float2*)w.D, (const float2*)w.P,
                                  bh + (long long)u.b0 * p->ax1.K * p->ax2.K, nullptr, u.st, &ob)))
      return rc;
  }
  for (int q = 0; q < nsub; ++q)
    if (zs && (rc = launch_zero_segments(p, sub[q].nb, sub[q].w, sub[q].e.c, sub[q].e.d, sub[q].st, tcr))) return rc;
  for (int q = 1; q < nsub; ++q) {
    CUDA_TRY(cudaEventRecord(ss->join[q - 1], ss->aux[q - 1]));
    CUDA_TRY(cudaStreamWaitEvent(st, ss->join[q - 1], 0));
  }
  return BCCB_OK;
}

// ---- ADMM with the spectral dual split (complex64 band engine; see EpiAdmmSplit)
static bool admm_split_supported(const bccb_plan_s* p, int batch, const void* extra) {
  static const int env = [] {
    const char* e = getenv("BCCB_ADMM_SPLIT");
    return e ? atoi(e) : 1;
  }();
  return env && fast_supported(p, batch, extra);
}

static int launch_rows_admm_split(const bccb_plan_s* p, int batch, bool inv, bool fwd, const Workspace& w,
                                  const EpiAdmmSplit& e, cudaStream_t st) {
  const LaunchShape sh = fast_shape(p);
  const Geo G = rows_geo(p, batch, sh, inv, fwd);
  RowsIO<float2> io{(const float2*)w.V, (float2*)w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  unsigned* fl = (unsigned*)w.flags;
  if (rows_use_kp16(p->ax1)) {
    const AxisT<float2> axs = p->ax1.dev_s();
    const int k16 = fast_key(p->ax1.s);
    if (k16 == 16 * 100000 + 16 * 10 + 2)
      return launch_pass<float2>(rows_admm_split_kernel<16, 16, 2, 3>, KIND_ROWS, grid, sh, st, G, axs, io, e, fl);
    if (k16 == 16 * 100000 + 64 * 10 + 4)
      return launch_pass<float2>(rows_admm_split_kernel<16, 64, 4, 3>, KIND_ROWS, grid, sh, st, G, axs, io, e, fl);
  }
  const AxisT<float2> ax = p->ax1.dev<float2>();
  const int key = fast_key(p->ax1.f);
#define SPLIT_CASE(KP_, R_, MO_)                                                                             \
  if (key == KP_ * 100000 + R_ * 10 + MO_)                                                                  \
    return launch_pass<float2>(rows_admm_split_kernel<KP_, R_, MO_>, KIND_ROWS, grid, sh, st, G, ax, io, e, fl);
  FAST_SHAPES(SPLIT_CASE)
#undef SPLIT_CASE
  return fail(BCCB_ERR_UNSUPPORTED, "no specialisation for this line shape");
}

static Geo cols_geo(const bccb_plan_s* p, int batch, const LaunchShape& sh, bool fwd, bool inv) {
  Geo G;
  G.L1 = p->L1;
  G.L2 = p->L2;
  G.rows = (long long)batch * p->ax1.K;
  G.TR = sh.TR;
  G.do_fwd = fwd ? 1 : 0;
  G.do_inv = inv ? 1 : 0;
  return G;
}

static int launch_cols_admm_split(const bccb_plan_s* p, int batch, const Workspace& w, const AdmmSplitBand& op,
                                  cudaStream_t st) {
  const bool narrow = cols_narrow(p, batch);
  const LaunchShape sh = shape_for_prec(p->ax2, narrow ? p->ax2.s8 : p->ax2.s, sizeof(float2),
                                        (long long)batch * p->ax1.K);
  const Geo G = cols_geo(p, batch, sh, true, true);
  ColsIO<float2> io{};
  io.U = (const float2*)w.U;
  io.V = (float2*)w.V;
  io.K1 = p->ax1.K;
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<float2> ax = p->ax2.dev_s(narrow);
  const AxisPrec& ap = narrow ? p->ax2.s8 : p->ax2.s;
  if (cols_warp_supported(p, ap)) return launch_cols_warp<AdmmSplitBand>(p, ap, G, st, ax, io, op);
  KP_DISPATCH_F(ax.KP, return launch_pass<float2>(cols_admm_split_kernel<KPC>, KIND_COLS, grid, sh, st, G, ax, io, op));
  return BCCB_OK;
}

// complex128 synthesis of a box: V = IFFT_col(box) (first half of IFFT2u(box))
static int launch_cols_box_z(const bccb_plan_s* p, int batch, const Workspace& w, const double2* box,
                             cudaStream_t st) {
  const LaunchShape sh = shape_for<double2>(p->ax2, (long long)batch * p->ax1.K);
  const Geo G = cols_geo(p, batch, sh, false, true);
  ColsIO<double2> io{};
  io.V = (double2*)w.V;
  io.K1 = p->ax1.K;
  const BoxIn<double2> op{box, p->ax2.K};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<double2> ax = p->ax2.dev<double2>();
  KP_DISPATCH_D(ax.KP, return launch_pass<double2>(cols_box_kernel<KPC, double2>, KIND_COLS, grid, sh, st, G, ax, io, op));
  return BCCB_OK;
}

// out = alpha (x1 - x2) + IFFT_row(V)  (complex128 engine)
static int launch_rows_combine_z(const bccb_plan_s* p, int batch, const Workspace& w, const EpiCombine& e,
                                 cudaStream_t st) {
  const LaunchShape sh = shape_for<double2>(p->ax1);
  const Geo G = rows_geo(p, batch, sh, true, false);
  RowsIO<double2> io{(const double2*)w.V, (double2*)w.U};
  const unsigned grid = (unsigned)((G.rows + sh.TR - 1) / sh.TR);
  const AxisT<double2> ax = p->ax1.dev<double2>();
  KP_DISPATCH_D(ax.KP, return launch_pass<double2>(rows_vector_kernel<KPC, double2, EpiCombine>, KIND_ROWS, grid, sh, st,
                                                   G, ax, io, e));
  return BCCB_OK;
}

// The split iteration (EpiAdmmSplit): the dual v is held as r (spatial, in the caller's v
// buffer) + IFFT2u(vs) (box, workspace).  On entry r = v, vs = 0; on exit v = r + IFFT2u(vs)
// and, when requested, c of the last iteration = a (z - r) + IFFT2u(Cb) from the pre-update
// state.  Arithmetic of the rows / column passes: complex64 band FFTs, float64 state and box.
static int admm_run_split(bccb_plan_s* p, int batch, int first_iteration, int iterations, double rho, double a,
                          const double* tau, const float2* bhat, double2* z, double2* v, double2* c_last,
                          int* first_bad, const Workspace& w, cudaStream_t st) {
  int rc;
  const size_t box_bytes = (size_t)batch * p->ax1.K * p->ax2.K * sizeof(double2);
  CUDA_TRY(cudaMemsetAsync(w.vs, 0, box_bytes, st));
  CUDA_TRY(cudaMemsetAsync(w.flags, 0xff, zs_flag_bytes(p, batch), st));
  EpiAdmmSplit e;
  e.z = z;
  e.r = v;
  e.tau = tau;
  e.first_bad = first_bad;
  e.a = a;
  e.kscale = rho;
  e.it = first_iteration;
  AdmmSplitBand op;
  op.D = (const double2*)w.D;
  op.P = (const double2*)w.P;
  op.Bh = bhat;
  op.vs = (double2*)w.vs;
  op.cb_out = nullptr;
  op.rhoL = rho * (double)p->L1 * (double)p->L2;
  op.K1 = p->ax1.K;
  op.K2 = p->ax2.K;
  // sub-batch split over streams, as in bccb_fista_run (independent snapshots: bitwise equal).
  // Not with c_last: its complex128 synthesis borrows the whole U region mid-iteration, which a
  // concurrent part's column pass still reads.
  const int nsub = c_last ? 1 : sub_batches(p, batch);
  SubStreams* ss = nullptr;
  if (nsub > 1 && (rc = ensure_aux_streams(p, nsub, &ss))) return rc;
  struct Sub {
    int b0, nb;
    cudaStream_t st;
    Workspace w;
    EpiAdmmSplit e;
    AdmmSplitBand op;
    double2 *z, *v, *c_last;
  } sub[bccb_plan_s::MAX_SUB];
  for (int q = 0; q < nsub; ++q) {
    Sub& u = sub[q];
    u.b0 = (int)((long long)batch * q / nsub);
    u.nb = (int)((long long)batch * (q + 1) / nsub) - u.b0;
    u.st = q == 0 ? st : ss->aux[q - 1];
    const long long inter = (long long)u.b0 * p->ax1.K * p->L2;
    const long long boxo = (long long)u.b0 * p->ax1.K * p->ax2.K;
    const long long off = (long long)u.b0 * p->L1 * p->L2;
    u.w = w;
    u.w.U = (float2*)w.U + inter;
    u.w.V = (float2*)w.V + inter;
    u.w.vs = (double2*)w.vs + boxo;
    u.w.cb = (double2*)w.cb + boxo;
    u.w.flags = w.flags + zs_flag_bytes(p, u.b0);
    u.z = z + off;
    u.v = v + off;
    u.c_last = c_last ? c_last + off : nullptr;
    u.e = e;
    u.e.z = u.z;
    u.e.r = u.v;
    u.e.tau = tau + u.b0;
    u.e.first_bad = first_bad + u.b0;
    u.op = op;
    u.op.Bh = bhat + boxo;
    u.op.vs = (double2*)u.w.vs;
  }
  if (nsub > 1) {
    CUDA_TRY(cudaEventRecord(ss->fork, st));
    for (int q = 1; q < nsub; ++q) CUDA_TRY(cudaStreamWaitEvent(ss->aux[q - 1], ss->fork, 0));
  }
  const int t_end = first_iteration + iterations;
  for (int q = 0; q < nsub; ++q)
    if ((rc = launch_rows_admm_split(p, sub[q].nb, false, true, sub[q].w, sub[q].e, sub[q].st))) return rc;
  for (int t = first_iteration; t < t_end; ++t) {
    const bool last = t + 1 == t_end;
    for (int q = 0; q < nsub; ++q) {
      Sub& u = sub[q];
      u.op.cb_out = (last && c_last) ? (double2*)u.w.cb : nullptr;
      if ((rc = launch_cols_admm_split(p, u.nb, u.w, u.op, u.st))) return rc;
      if (last && c_last) {
        // c = a (z - r) + IFFT2u(Cb) from the state before the last update; the complex128
        // synthesis runs through U (free: the last rows pass has no forward half)
        if ((rc = launch_zero_segments(p, u.nb, u.w, u.z, u.v, u.st))) return rc;
        Workspace wu = u.w;
        wu.V = u.w.U;
        if ((rc = launch_cols_box_z(p, u.nb, wu, (const double2*)u.w.cb, u.st))) return rc;
        const EpiCombine ec{u.z, u.v, u.c_last, a};
        if ((rc = launch_rows_combine_z(p, u.nb, wu, ec, u.st))) return rc;
      }
      u.e.it = t;
      if ((rc = launch_rows_admm_split(p, u.nb, true, !last, u.w, u.e, u.st))) return rc;
    }
  }
  for (int q = 0; q < nsub; ++q)
    if ((rc = launch_zero_segments(p, sub[q].nb, sub[q].w, sub[q].z, sub[q].v, sub[q].st))) return rc;
  for (int q = 1; q < nsub; ++q) {
    CUDA_TRY(cudaEventRecord(ss->join[q - 1], ss->aux[q - 1]));
    CUDA_TRY(cudaStreamWaitEvent(st, ss->join[q - 1], 0));
  }
  // v = r + IFFT2u(vs)
  if ((rc = launch_cols_box_z(p, batch, w, (const double2*)w.vs, st))) return rc;
  const EpiCombine ev{v, nullptr, v, 1.0};
  return launch_rows_combine_z(p, batch, w, ev, st);
}

extern "C" int bccb_admm_run(bccb_plan_t p, int batch, int first_iteration, int iterations,
                             double rho, const double* tau,
                             const void* bhat_box, const void* extra, void* z, void* v, void* c_last,
                             int* first_bad, void* workspace, void* stream) {
  EntryScope entry_scope_("bccb_admm_run");
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
  if ((rc = launch_coef<double2>(p, 2, rho, a, w, st))) return rc;
  if (first_iteration == 0 && (rc = reset_first_bad(first_bad, batch, st))) return rc;
  EpiAdmm e;
  e.z = (double2*)z;
  e.v = (double2*)v;
  e.c_out = nullptr;
  e.extra = (const float2*)extra;
  e.tau = tau;
  e.first_bad = first_bad;
  e.a = a;
  e.kscale = rho;
  e.extra_scale = 1.0 / (lo + rho);
  e.it = first_iteration;
  const int t_end = first_iteration + iterations;
  if (admm_split_supported(p, batch, extra))
    return admm_run_split(p, batch, first_iteration, iterations, rho, a, tau, (const float2*)bhat_box, (double2*)z,
                          (double2*)v, (double2*)c_last, first_bad, w, st);
  // specialised shapes: zero-segment skipping on the sparse z (dual v is dense)
  const bool zs = admm_fast_supported(p, batch, extra);
  if (zs) CUDA_TRY(cudaMemsetAsync(w.flags, 0xff, zs_flag_bytes_d(p, batch), st));
  auto rows = [&](bool inv, bool fwd) {
    return zs ? launch_rows_admm_fast(p, batch, inv, fwd, w, e, st) : launch_rows_admm(p, batch, inv, fwd, w, e, st);
  };
  if ((rc = rows(false, true))) return rc;
  for (int t = first_iteration; t < t_end; ++t) {
    if ((rc = launch_cols<double2>(p, batch, true, true, w, (const double2*)w.D, (const double2*)w.P,
                                   (const float2*)bhat_box, nullptr, st)))
      return rc;
    e.it = t;
    e.c_out = (t + 1 == t_end) ? (double2*)c_last : nullptr;
    if ((rc = rows(true, t + 1 < t_end))) return rc;
  }
  if (zs && (rc = launch_zero_segments_z(p, batch, w, (double2*)z, st))) return rc;
  return BCCB_OK;
}

// ------------------------------------------------------------------ top-k
extern "C" size_t bccb_topk_workspace_bytes(int batch, long long length, int k) {
  if (batch < 1 || length < 1 || k < 1) return 0;
  const int nchunk = topk_chunks(batch, length);
  return (size_t)batch * nchunk * pow2_ceil(k) * sizeof(TKey) + 256;
}

extern "C" int bccb_topk(int batch, long long length, const void* values, int is_double, int k,
                         int* idx, float* mag, void* workspace, void* stream) {
  EntryScope entry_scope_("bccb_topk");
  if (batch < 1 || length < 1) return fail(BCCB_ERR_INVALID, "empty input");
  if (k < 1 || k > 64) return fail(BCCB_ERR_INVALID, "k must lie in [1, 64]");
  if (k > length) return fail(BCCB_ERR_INVALID, "k exceeds the vector length");
  if (length > 0xFFFFFFFFLL) return fail(BCCB_ERR_UNSUPPORTED, "vector longer than 2^32");
  if (!values || !idx || !workspace) return fail(BCCB_ERR_INVALID, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int nchunk = topk_chunks(batch, length);
  TKey* cand = (TKey*)workspace;
  const int kt = std::max(4, pow2_ceil(k));
#define TOPK_CASE(KT)                                                                            \
  case KT:                                                                                       \
    g_launches.fetch_add(2, std::memory_order_relaxed);                                          \
    topk_partial_kernel<KT><<<dim3(nchunk, batch), 256, 0, st>>>(values, is_double, length, k,   \
                                                                 nchunk, cand);                  \
    topk_merge_kernel<<<batch, 256, 0, st>>>(cand, nchunk * k, k, idx, mag);                     \
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

// ------------------------------------------------------------------ complex128 spectrum / synthesis
// fft2 restricted to the box and the inverse synthesis on the complex128 band engine: the
// float64 paths of bccb_from_first_column / bccb_first_column (bccb.py:93-105, 151-153), pinned
// at rtol 1e-11 by the reference's pkg/tests/test_bccb.py:99-107.
extern "C" int bccb_spectrum_box_z(bccb_plan_t p, int batch, const void* x, void* out_box, void* workspace,
                                   void* stream) {
  EntryScope entry_scope_("bccb_spectrum_box_z");
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!x || !out_box) return fail(BCCB_ERR_INVALID, "x / out_box is NULL");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  EpiVector<double2> e{(const double2*)x, nullptr, nullptr, 0.0, 1.0};
  if ((rc = launch_rows_vector<double2>(p, batch, false, true, w, e, st))) return rc;
  return launch_cols<double2>(p, batch, true, false, w, nullptr, nullptr, nullptr, (double2*)out_box, st);
}

extern "C" int bccb_synthesize_z(bccb_plan_t p, int batch, const void* box, double scale, void* out,
                                 void* workspace, void* stream) {
  EntryScope entry_scope_("bccb_synthesize_z");
  int rc = check_common(p, batch, workspace);
  if (rc) return rc;
  if (!box || !out) return fail(BCCB_ERR_INVALID, "box / out is NULL");
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w = carve(p, batch, workspace);
  if ((rc = launch_cols_box_z(p, batch, w, (const double2*)box, st))) return rc;
  EpiVector<double2> e{nullptr, (double2*)out, nullptr, 0.0, scale};
  return launch_rows_vector<double2>(p, batch, true, false, w, e, st);
}
