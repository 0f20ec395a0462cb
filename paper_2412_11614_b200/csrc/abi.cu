// C ABI + host planner (rows a1 and b) of the ISRS EGN hot path.  See include/isrs_egn.h.
//
// Planner (row a1): validation, canonicalisation (reading C5: offsets from the occupied-band
// midpoint f_c, B_tot edge-to-edge, P_tot = sum P_i; K_s = ceil(L_s/dz)), span classes
// (spans with equal L, alpha, C_r share envelope tables), the region work list of every COI
// (Eq. 16, generalised to arbitrary channel plans: a region (kappa, k1, k2) is listed
// when the f3 range of its bin centres overlaps some band) split into D-only and coherent
// (E/F/G/H-carrying, reading C8) lists.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/isrs_egn.h"
#include "internal.h"

using namespace isrs;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// Device allocations come from the device's default stream-ordered memory pool with the release
// threshold raised, so repeated create / destroy (the one-shot isrs_egn_eta_host path) and work-list
// rebuilds reuse pool memory instead of mapping and unmapping it through the driver each time.
// Every allocation and free is stream-ordered (cudaMallocAsync / cudaFreeAsync on a given stream):
// create() uses the legacy default stream and then synchronises it (create is synchronous by
// contract); a work-list rebuild inside isrs_egn_nli allocates, uploads and frees on the caller's
// stream after that stream has been ordered behind the handle's previous call, so nli never
// synchronises the host or the device.
static void tune_pool(int dev) {
  static std::mutex mu;
  static std::set<int> tuned;
  std::lock_guard<std::mutex> lk(mu);
  if (tuned.count(dev)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  tuned.insert(dev);
}

static cudaError_t dev_alloc_on(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  tune_pool(dev);
  return cudaMallocAsync(p, bytes, st);
}

// Stream-ordered free: `st` must already be ordered after every use of p.
static void dev_free_on(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

// RAII: make `dev` current for the duration of an API call and restore the caller's device after
// (a process may hold handles on several GPUs; torch's current device must not move).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// NVTX ranges around the public entry points (visible in nsys / ncu --nvtx)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void borrow(T* q, size_t cnt) {   // buffers live inside an Arena (one allocation for many)
    p = q;
    n = cnt;
  }
  void clear() {
    p = nullptr;
    n = 0;
  }
};

// One device allocation holding many small buffers (fewer allocations on the create / plan path).
struct Arena {
  char* base = nullptr;
  cudaStream_t st = nullptr;   // stream the allocation was made on (its free follows in that order)
};

// Pinned host staging for work-list uploads issued while the caller's stream is busy.  A pageable-
// source cudaMemcpyAsync returns only once its data sits in the driver's staging buffer, and that
// buffer stays occupied until the stream reaches the copy: the second upload behind a running kernel
// blocked the host for the kernel's whole duration (tools/async_probe.py, profiles/r02zt_*).  From a
// pinned source the copy is a plain stream-ordered DMA; the buffer is reused once the event recorded
// behind its copy has completed, and buffers are only released by destroy (cudaFreeHost may
// synchronise).  An idle stream takes the pageable path (no pinned allocation on the one-shot path).
struct PinPool {
  struct Buf {
    char* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool inflight = false;
  };
  std::vector<Buf> bufs;
  bool busy() {   // some earlier upload from pinned memory has not completed yet
    for (auto& b : bufs)
      if (b.inflight) {
        if (cudaEventQuery(b.ev) == cudaSuccess) b.inflight = false;
        else { cudaGetLastError(); return true; }   // cudaErrorNotReady is not sticky; clear it
      }
    return false;
  }
  Buf* acquire(size_t bytes) {
    for (auto& b : bufs) {
      if (b.inflight && cudaEventQuery(b.ev) == cudaSuccess) b.inflight = false;
      if (!b.inflight && b.cap >= bytes) return &b;
    }
    cudaGetLastError();
    Buf b;
    size_t cap = 1 << 16;
    while (cap < bytes) cap <<= 1;
    if (cudaHostAlloc((void**)&b.p, cap, cudaHostAllocDefault) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    if (cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      cudaFreeHost(b.p);
      return nullptr;
    }
    b.cap = cap;
    bufs.push_back(b);
    return &bufs.back();
  }
  void release_all() {   // destroy only (the device is synchronised first)
    for (auto& b : bufs) {
      if (b.ev) cudaEventDestroy(b.ev);
      if (b.p) cudaFreeHost(b.p);
    }
    bufs.clear();
  }
};

class Packer {
  struct E {
    std::function<void(char*)> bind;
    const void* src;
    size_t bytes, off;
  };
  std::vector<E> init_, dev_;
  static size_t up(size_t b) { return (std::max<size_t>(b, 1) + 255) & ~(size_t)255; }

 public:
  template <class T>
  void add(DevBuf<T>* d, const std::vector<T>& v) {
    const size_t cnt = v.size();
    init_.push_back({[d, cnt](char* q) { d->borrow(reinterpret_cast<T*>(q), cnt); }, v.data(),
                     cnt * sizeof(T), 0});
  }
  template <class T>
  void reserve(DevBuf<T>* d, size_t cnt) {   // device-only, uninitialised
    dev_.push_back({[d, cnt](char* q) { d->borrow(reinterpret_cast<T*>(q), cnt); }, nullptr,
                    cnt * sizeof(T), 0});
  }
  // Allocate one block on `st` and upload the staged host data (stream-ordered; a pageable-source
  // cudaMemcpyAsync returns once the data is staged, so the host vectors may die on return).  Only
  // when both succeed is the old arena freed (on `st`, which the caller has ordered after its last
  // use) and are the DevBufs rebound: on failure the handle keeps its previous, valid buffers.
  // `pins` (the nli path): when `st` still has work in flight the upload is staged in pinned memory
  // so that the call returns without waiting for that work.
  cudaError_t commit(Arena* a, cudaStream_t st, PinPool* pins = nullptr) {
    size_t off = 0;
    for (auto& e : init_) { e.off = off; off += up(e.bytes); }
    const size_t init_bytes = off;
    for (auto& e : dev_) { e.off = off; off += up(e.bytes); }
    void* q = nullptr;
    cudaError_t ce = dev_alloc_on(&q, std::max<size_t>(off, 256), st);
    if (ce != cudaSuccess) return ce;
    if (init_bytes) {
      PinPool::Buf* pb = nullptr;
      if (pins) {
        bool stream_busy = pins->busy();
        if (!stream_busy && cudaStreamQuery(st) != cudaSuccess) {
          cudaGetLastError();
          stream_busy = true;
        }
        if (stream_busy) pb = pins->acquire(init_bytes);   // NULL (no pinned memory): pageable path
      }
      std::vector<char> stage(pb ? 0 : init_bytes);
      char* src = pb ? pb->p : stage.data();
      for (auto& e : init_)
        if (e.bytes) std::memcpy(src + e.off, e.src, e.bytes);
      ce = cudaMemcpyAsync(q, src, init_bytes, cudaMemcpyHostToDevice, st);
      if (ce == cudaSuccess && pb) {
        ce = cudaEventRecord(pb->ev, st);
        if (ce == cudaSuccess) pb->inflight = true;
        else cudaStreamSynchronize(st);   // cannot track the copy: wait for it before the buffer is reused
      }
      if (ce != cudaSuccess) {
        dev_free_on(q, st);
        return ce;
      }
    }
    if (a->base) dev_free_on(a->base, st);
    a->base = static_cast<char*>(q);
    a->st = st;
    for (auto& e : init_) e.bind(a->base + e.off);
    for (auto& e : dev_) e.bind(a->base + e.off);
    return cudaSuccess;
  }
};

struct WorkList {
  std::vector<long long> cost;   // in-support points per region (canonical order)
  std::vector<int> coi;
  std::vector<double> fv;   // NLI frequency of each (COI, f sample)
  std::vector<RegionDesc> desc;
  std::vector<int> mirror;   // ISRS_EGN_FLAG_MIRROR: id of (kappa, k2, k1) written by region id, or -1
  std::vector<long long> coi_off;
  std::vector<int> list_d, list_c;
};

}  // namespace

struct isrs_egn {
  int device = 0;
  isrs_egn_numerics num{};
  int n_ch = 0, n_span = 0, n_cls = 0, N = 0;
  // host canonical data
  std::vector<double> lo, hi, f, G, R, P, phi, psi, delta;
  std::vector<long long> rate;
  double f_c = 0, b_tot = 0, p_tot = 0;
  // device data (views into the arenas)
  DevBuf<double> d_lo, d_hi, d_f, d_G, d_R, d_P, d_phi, d_psi, d_delta;
  DevBuf<long long> d_rate;
  DevBuf<double> d_A2, d_A3, d_Eh, d_ah, d_gh, d_macc, d_aL;
  DevBuf<int> d_K, d_cls, d_Kc, d_chain_s0, d_chain_g, d_grp_c0;
  DevBuf<double> d_lnc_L, d_zeta_L, d_lgA, d_lgB, d_lgC, d_lgD;
  DevBuf<double> d_Ls, d_alpha, d_gamma, d_pcr;
  double gl_x[12], gl_w[12];
  int n_chain = 0, n_grp = 0;
  std::vector<int> chain_g, k_s, cls_of_span, grp_c0;
  DevBuf<double> d_lnA, d_zeta;
  int kstride = 0, tstride = 0, tw = 0;
  // work list cache (last call)
  WorkList wl;
  bool have_wl = false;
  DevBuf<RegionDesc> d_desc;
  DevBuf<long long> d_coi_off;
  DevBuf<int> d_coi, d_list_d, d_list_c, d_mirror;
  DevBuf<double> d_fv;
  // regions launched by the last call (the whole list, or one shard of it)
  // regions launched by the last call: the work list's own launch lists, or the current shard's
  const std::vector<int>* act_d = nullptr;
  const std::vector<int>* act_c = nullptr;
  std::vector<int> sh_act_d, sh_act_c;   // the regions of the current shard (rank, world)
  int sh_rank = -1, sh_world = -1;
  long long sh_lo = 0, sh_hi = 0;
  DevBuf<int> d_sh_d, d_sh_c;
  DevBuf<double> d_partials, d_npts;
  Arena arena_create, arena_plan, arena_shard;
  PinPool pins;   // pinned staging of work-list / shard-list uploads behind in-flight work
  cudaStream_t last_stream = nullptr;
  bool have_result = false;   // the partials hold the last call's values
  bool ordered = false;       // ev[3] marks the end of the handle's last direct call (on last_stream)
  int last_launches = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // coherent-region integrand on a side stream, concurrent with the D-only launch (fills its tail)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, evc[2] = {nullptr, nullptr};
  // fork / join events used only while the caller's stream is being captured into a CUDA graph
  // (the timing and ordering events above are never recorded inside a capture)
  cudaEvent_t cap_fork = nullptr, cap_join = nullptr;
  bool launched[2] = {false, false};
  ~isrs_egn() {   // isrs_egn_destroy synchronises the device first
    for (Arena* a : {&arena_plan, &arena_shard, &arena_create})
      if (a->base) cudaFreeAsync(a->base, 0);
    pins.release_all();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : evc)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {ev_fork, ev_join, cap_fork, cap_join})
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
  }
};

static bool is_fin(double x) { return std::isfinite(x); }

static int validate(const isrs_egn_problem* p, const isrs_egn_numerics* n) {
  if (!p || !n) return fail(ISRS_EGN_EINVAL, "problem/numerics is NULL");
  if (p->n_ch < 1) return fail(ISRS_EGN_EINVAL, "n_ch < 1");
  if (p->n_span < 1) return fail(ISRS_EGN_EINVAL, "n_span < 1");
  if (!p->f_center_hz || !p->symbol_rate_hz || !p->launch_power_w || !p->excess_kurtosis)
    return fail(ISRS_EGN_EINVAL, "channel array is NULL");
  if (!p->length_m || !p->alpha_per_m || !p->beta2_s2_per_m || !p->beta3_s3_per_m ||
      !p->gamma_per_w_m || !p->cr_per_w_m_hz)
    return fail(ISRS_EGN_EINVAL, "span array is NULL");
  if (n->grid_n < 2 || (n->grid_n & 1)) return fail(ISRS_EGN_EINVAL, "grid_n must be even and >= 2");
  if (n->grid_n > 4096) return fail(ISRS_EGN_EINVAL, "grid_n > 4096");
  if (!is_fin(n->delta_z_m) || n->delta_z_m <= 0) return fail(ISRS_EGN_EINVAL, "delta_z_m <= 0");
  if (n->precision != 64 && n->precision != 32 && n->precision != 0)
    return fail(ISRS_EGN_EUNSUPPORTED, "precision must be 64 or 32");
  if (n->precision == 32 && n->mu_mode != ISRS_EGN_MU_SEGMENT)
    return fail(ISRS_EGN_EUNSUPPORTED, "precision 32 (row a8) is a variant of the segment mode only");
  if ((n->flags & ISRS_EGN_FLAG_LITERAL_GAIN) &&
      (n->mu_mode != ISRS_EGN_MU_SEGMENT || n->precision == 32 || (n->flags & ISRS_EGN_FLAG_DEDUP)))
    return fail(ISRS_EGN_EUNSUPPORTED, "LITERAL_GAIN is an fp64 segment-mode variant (no DEDUP)");
  if ((n->flags & ISRS_EGN_FLAG_SPLIT) &&
      (n->mu_mode != ISRS_EGN_MU_SEGMENT || n->precision == 32 ||
       (n->flags & (ISRS_EGN_FLAG_DEDUP | ISRS_EGN_FLAG_LITERAL_GAIN | ISRS_EGN_FLAG_MIRROR | ISRS_EGN_FLAG_UNIT_LINK))))
    return fail(ISRS_EGN_EUNSUPPORTED, "SPLIT is an fp64 segment-mode option (no DEDUP, LITERAL_GAIN, MIRROR, UNIT_LINK)");
  if (n->f_samples < 0 || n->f_samples > 4096) return fail(ISRS_EGN_EINVAL, "f_samples must be in [0, 4096]");
  if (n->mu_mode != ISRS_EGN_MU_SEGMENT && n->mu_mode != ISRS_EGN_MU_MACLAURIN &&
      n->mu_mode != ISRS_EGN_MU_INTEGRAL)
    return fail(ISRS_EGN_EUNSUPPORTED, "unknown mu_mode");
  const double lim = 4.0e15;  // |values| < 2^52: integer-Hz arithmetic exact
  for (int i = 0; i < p->n_ch; ++i) {
    const double F = p->f_center_hz[i], R = p->symbol_rate_hz[i], P = p->launch_power_w[i];
    const std::string at = "[" + std::to_string(i) + "]";
    if (!is_fin(F) || F <= 0 || F > lim || F != std::floor(F))
      return fail(ISRS_EGN_EINVAL, "f_center_hz" + at + " must be a positive integer number of Hz");
    if (!is_fin(R) || R <= 0 || R > 1e14 || R != std::floor(R))
      return fail(ISRS_EGN_EINVAL, "symbol_rate_hz" + at + " must be a positive integer number of Hz");
    const double half = R / (2.0 * n->grid_n);
    if (half != std::floor(half))
      return fail(ISRS_EGN_EINVAL, "symbol_rate_hz" + at + " / (2 grid_n) must be an integer (C10)");
    if (n->f_samples > 0) {
      const double hf = R / (2.0 * n->f_samples);
      if (hf != std::floor(hf))
        return fail(ISRS_EGN_EINVAL, "symbol_rate_hz" + at + " / (2 f_samples) must be an integer (R3)");
    }
    if (!is_fin(P) || P <= 0) return fail(ISRS_EGN_EINVAL, "launch_power_w" + at + " must be > 0");
    if (!is_fin(p->excess_kurtosis[i])) return fail(ISRS_EGN_EINVAL, "excess_kurtosis" + at);
    if (p->psi && !is_fin(p->psi[i])) return fail(ISRS_EGN_EINVAL, "psi" + at);
    if (i > 0 && !(F > p->f_center_hz[i - 1]))
      return fail(ISRS_EGN_EINVAL, "f_center_hz" + at + " not strictly increasing");
    if (i > 0 && F - R / 2 < p->f_center_hz[i - 1] + p->symbol_rate_hz[i - 1] / 2)
      return fail(ISRS_EGN_EOVERLAP, "bands of channels " + std::to_string(i - 1) + " and " +
                                         std::to_string(i) + " overlap");
  }
  // the integrand walks the lattice lines a m1 + b m2 = j of every channel pair (a:b = R1:R2 in
  // lowest terms, (a + b)(N - 1) + 1 lines): rate ratios must be small rationals
  {
    std::vector<long long> rates;
    for (int i = 0; i < p->n_ch; ++i) rates.push_back((long long)p->symbol_rate_hz[i]);
    std::sort(rates.begin(), rates.end());
    rates.erase(std::unique(rates.begin(), rates.end()), rates.end());
    for (size_t i = 0; i < rates.size(); ++i)
      for (size_t j = i + 1; j < rates.size(); ++j) {
        long long x = rates[i], y = rates[j];
        while (y) { const long long t = x % y; x = y; y = t; }
        if ((rates[i] + rates[j]) / x > RATIO_MAX)
          return fail(ISRS_EGN_EUNSUPPORTED,
                      "symbol rates " + std::to_string(rates[i]) + " and " + std::to_string(rates[j]) +
                          " Hz: ratio a:b in lowest terms has a + b > " + std::to_string(RATIO_MAX) +
                          " (lattice line scan); use rates with a small common divisor ratio");
      }
  }
  for (int s = 0; s < p->n_span; ++s) {
    const std::string at = "[" + std::to_string(s) + "]";
    if (!is_fin(p->length_m[s]) || p->length_m[s] <= 0) return fail(ISRS_EGN_EINVAL, "length_m" + at + " <= 0");
    if (!is_fin(p->alpha_per_m[s]) || p->alpha_per_m[s] <= 0)
      return fail(ISRS_EGN_EINVAL, "alpha_per_m" + at + " must be > 0 (Eq. 9 divides by i chi - alpha)");
    if (!is_fin(p->beta2_s2_per_m[s])) return fail(ISRS_EGN_EINVAL, "beta2_s2_per_m" + at);
    if (!is_fin(p->beta3_s3_per_m[s])) return fail(ISRS_EGN_EINVAL, "beta3_s3_per_m" + at);
    if (!is_fin(p->gamma_per_w_m[s]) || p->gamma_per_w_m[s] < 0) return fail(ISRS_EGN_EINVAL, "gamma_per_w_m" + at + " < 0");
    if (!is_fin(p->cr_per_w_m_hz[s]) || p->cr_per_w_m_hz[s] < 0) return fail(ISRS_EGN_EINVAL, "cr_per_w_m_hz" + at + " < 0");
    const double K = std::ceil(p->length_m[s] / n->delta_z_m);
    if (K > (1 << 20)) return fail(ISRS_EGN_ERANGE, "K_s = ceil(L/dz) > 2^20 for span" + at);
  }
  return ISRS_EGN_OK;
}

static int cuda_fail(cudaError_t e, const char* what) {
  return fail(ISRS_EGN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// 12-point Gauss-Legendre rule on [-1, 1] (integral form, reading C12): roots of P_12 by Newton
// iteration from the Chebyshev-like guesses cos(pi (i + 3/4) / (n + 1/2)); w = 2 / ((1 - x^2) P'_12^2).
static void gauss_legendre12(double* x, double* w) {
  const int n = 12;
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;                    // Bonnet recurrence
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (t * p1 - p0) / (t * t - 1.0);
      const double dt = p1 / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-17) break;
    }
    x[n - 1 - i] = t;                              // ascending order
    w[n - 1 - i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
}

// Host-side canonicalisation of the channel plan (reading C5): offsets from the occupied-band
// midpoint f_c, B_tot edge-to-edge, P_tot = sum P_i, G_i = P_i / R_i, delta_i = R_i / N.
static void canon_channels(isrs_egn* h, const isrs_egn_problem* p, const isrs_egn_numerics& num) {
  h->num = num;
  h->n_ch = p->n_ch;
  h->n_span = p->n_span;
  h->N = num.grid_n;
  const int nc = p->n_ch, N = num.grid_n;
  double lo_min = 1e300, hi_max = -1e300;
  for (int i = 0; i < nc; ++i) {
    lo_min = std::min(lo_min, p->f_center_hz[i] - p->symbol_rate_hz[i] / 2);
    hi_max = std::max(hi_max, p->f_center_hz[i] + p->symbol_rate_hz[i] / 2);
  }
  h->f_c = (lo_min + hi_max) / 2;
  h->b_tot = hi_max - lo_min;
  h->p_tot = 0;
  for (int i = 0; i < nc; ++i) {
    const double F = p->f_center_hz[i] - h->f_c, R = p->symbol_rate_hz[i];
    h->f.push_back(F);
    h->R.push_back(R);
    h->lo.push_back(F - R / 2);
    h->hi.push_back(F + R / 2);
    h->P.push_back(p->launch_power_w[i]);
    h->G.push_back(p->launch_power_w[i] / R);
    h->phi.push_back(p->excess_kurtosis[i]);
    h->psi.push_back(p->psi ? p->psi[i] : 0.0);
    h->delta.push_back(R / N);
    h->rate.push_back((long long)R);
    h->p_tot += p->launch_power_w[i];
  }
}

extern "C" int isrs_egn_create(const isrs_egn_problem* p, const isrs_egn_numerics* n, int device,
                               isrs_egn_t** out) {
  if (!out) return fail(ISRS_EGN_EINVAL, "out is NULL");
  *out = nullptr;
  isrs_egn_numerics num = n ? *n : isrs_egn_numerics{};
  if (num.precision == 0) num.precision = 64;
  NvtxRange nv("isrs_egn_create");
  int rc = validate(p, &num);
  if (rc) return rc;
  DeviceGuard dg(device);
  cudaError_t ce = dg.err;
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaSetDevice");

  auto* h = new isrs_egn();
  h->device = device;
  canon_channels(h, p, num);
  const int N = num.grid_n;
  // ---- spans and classes
  std::map<std::tuple<double, double, double>, int> cls_of;
  std::vector<double> cL, cA, cC;
  std::vector<int> cK;
  std::vector<double> A2, A3, Eh, ah, gh, macc, aL;
  std::vector<int> K, cls;
  for (int s = 0; s < p->n_span; ++s) {
    const double L = p->length_m[s], a = p->alpha_per_m[s], cr = p->cr_per_w_m_hz[s];
    const int Ks = (int)std::ceil(L / num.delta_z_m);
    const double hs = L / Ks;
    auto key = std::make_tuple(L, a, cr);
    auto it = cls_of.find(key);
    int c;
    if (it == cls_of.end()) {
      c = (int)cL.size();
      cls_of[key] = c;
      cL.push_back(L);
      cA.push_back(a);
      cC.push_back(cr);
      cK.push_back(Ks);
      const double x = h->b_tot * h->p_tot * cr * (-std::expm1(-a * L) / a);
      if (x > 1400.0) {
        delete h;
        return fail(ISRS_EGN_ERANGE, "B_tot P_tot C_r L_eff too large (sinh overflow) for span " +
                                         std::to_string(s));
      }
    } else {
      c = it->second;
    }
    cls.push_back(c);
    K.push_back(Ks);
    A2.push_back(4.0 * M_PI * p->beta2_s2_per_m[s] * hs);
    A3.push_back(4.0 * M_PI * M_PI * p->beta3_s3_per_m[s] * hs);
    Eh.push_back(std::exp(-a * hs));
    ah.push_back(a * hs);
    gh.push_back(p->gamma_per_w_m[s] * hs);
    macc.push_back(h->p_tot * cr / a);
    aL.push_back(a * L);
  }
  h->n_cls = (int)cL.size();
  // ---- span chains (reading R9): identical consecutive spans (same L, alpha, beta2, beta3,
  // gamma, C_r, hence the same z = e^{i chi h} and envelope table) with an even K_s share one
  // recurrence over G * K_s segments, G * K_s <= CHAIN_MAX.  Segment mode only.
  std::vector<int> ch_s0, ch_g;
  // precision 32 (row a8): runs of identical spans share z, I_0 and the per-span phase step
  // (common subexpressions), but every span keeps its own K-segment recurrence; cap 1024 spans
  const bool chain_ok = num.mu_mode == ISRS_EGN_MU_SEGMENT &&
                        !(num.flags & (ISRS_EGN_FLAG_NO_CHAIN | ISRS_EGN_FLAG_UNIT_LINK));
  const bool dedup = (num.flags & ISRS_EGN_FLAG_DEDUP) && num.precision == 64;
  const long long chain_cap = (num.precision == 32 || dedup) ? 1024LL * 1000000 : CHAIN_MAX;
  for (int s = 0; s < p->n_span; ++s) {
    const bool same = s > 0 && chain_ok && (num.precision == 32 || K[s] % 2 == 0) &&
                      p->length_m[s] == p->length_m[s - 1] &&
                      p->alpha_per_m[s] == p->alpha_per_m[s - 1] &&
                      p->beta2_s2_per_m[s] == p->beta2_s2_per_m[s - 1] &&
                      p->beta3_s3_per_m[s] == p->beta3_s3_per_m[s - 1] &&
                      p->gamma_per_w_m[s] == p->gamma_per_w_m[s - 1] &&
                      p->cr_per_w_m_hz[s] == p->cr_per_w_m_hz[s - 1] &&
                      (long long)(ch_g.back() + 1) * ((num.precision == 32 || dedup) ? 1000000 : K[s]) <= chain_cap;
    if (same) {
      ch_g.back() += 1;
    } else {
      ch_s0.push_back(s);
      ch_g.push_back(1);
    }
  }
  h->n_chain = (int)ch_s0.size();
  // chain groups (fp64 segment mode with chaining): consecutive chains whose spans are identical,
  // every chain but the group's last of the same length G (the cap split)
  std::vector<int> grp_c0;
  const bool group_ok = chain_ok && num.precision == 64 &&
                        !(num.flags & (ISRS_EGN_FLAG_DEDUP | ISRS_EGN_FLAG_LITERAL_GAIN));
  for (int c = 0; c < h->n_chain; ++c) {
    bool join = false;
    if (group_ok && c > 0) {
      const int s = ch_s0[c], r = ch_s0[c - 1];
      join = p->length_m[s] == p->length_m[r] && p->alpha_per_m[s] == p->alpha_per_m[r] &&
             p->beta2_s2_per_m[s] == p->beta2_s2_per_m[r] && p->beta3_s3_per_m[s] == p->beta3_s3_per_m[r] &&
             p->gamma_per_w_m[s] == p->gamma_per_w_m[r] && p->cr_per_w_m_hz[s] == p->cr_per_w_m_hz[r] &&
             ch_g[c - 1] == ch_g[grp_c0.back()];
    }
    if (!join) grp_c0.push_back(c);
  }
  h->n_grp = (int)grp_c0.size();
  grp_c0.push_back(h->n_chain);
  h->grp_c0 = grp_c0;
  // ---- literal gain products (NEXT-4b): SRS gain at each span end, prefix / suffix sums
  const int ns = p->n_span;
  std::vector<double> lncL(ns), zL(ns), lgA(ns, 0.0), lgB(ns, 0.0), lgC(ns, 0.0), lgD(ns, 0.0);
  for (int s = 0; s < ns; ++s) {
    const double a = p->alpha_per_m[s], L = p->length_m[s];
    zL[s] = h->p_tot * p->cr_per_w_m_hz[s] * (-std::expm1(-a * L) / a);   // Eq. 2 at z = L
    const double x = h->b_tot * zL[s];
    lncL[s] = (x == 0.0) ? 0.0 : std::log(x / (2.0 * std::sinh(0.5 * x)));   // Eq. 14
  }
  std::vector<double> vL(ns), vA(ns), vG(ns), vP(ns);
  for (int s = 0; s < ns; ++s) {
    vL[s] = p->length_m[s];
    vA[s] = p->alpha_per_m[s];
    vG[s] = p->gamma_per_w_m[s];
    vP[s] = h->p_tot * p->cr_per_w_m_hz[s];
  }
  gauss_legendre12(h->gl_x, h->gl_w);
  for (int s = 1; s < ns; ++s) {
    lgA[s] = lgA[s - 1] + 3.0 * lncL[s - 1];
    lgB[s] = lgB[s - 1] + zL[s - 1];
  }
  for (int s = ns - 2; s >= 0; --s) {
    lgC[s] = lgC[s + 1] + lncL[s + 1];
    lgD[s] = lgD[s + 1] + zL[s + 1];
  }
  h->chain_g = ch_g;
  h->k_s = K;
  h->cls_of_span = cls;
  int kmax = *std::max_element(cK.begin(), cK.end());
  int kpad = (kmax + 1) & ~1;
  h->kstride = kpad;
  h->tstride = kpad + 2;
  const size_t t_budget = T_BYTES;
  h->tw = (int)std::min<size_t>(TW_MAX, t_budget / ((size_t)h->tstride * 8));
  if (h->tw < 2) {
    delete h;
    return fail(ISRS_EGN_ERANGE, "K_s too large for the shared-memory envelope table (reduce K or raise dz)");
  }
  const size_t smem = integrand_smem_bytes(h->tstride, h->tw, N, true, true);
  if (smem > 220 * 1024) {
    delete h;
    return fail(ISRS_EGN_ERANGE, "grid_n / K_s exceed the shared-memory budget");
  }
  DevBuf<double> dL, dA, dC;
  Packer pk;
  pk.add(&h->d_lo, h->lo); pk.add(&h->d_hi, h->hi); pk.add(&h->d_f, h->f); pk.add(&h->d_G, h->G);
  pk.add(&h->d_R, h->R); pk.add(&h->d_P, h->P); pk.add(&h->d_phi, h->phi); pk.add(&h->d_psi, h->psi);
  pk.add(&h->d_delta, h->delta); pk.add(&h->d_rate, h->rate); pk.add(&h->d_A2, A2);
  pk.add(&h->d_A3, A3); pk.add(&h->d_Eh, Eh); pk.add(&h->d_ah, ah); pk.add(&h->d_gh, gh);
  pk.add(&h->d_macc, macc); pk.add(&h->d_aL, aL); pk.add(&h->d_K, K); pk.add(&h->d_cls, cls);
  pk.add(&h->d_Kc, cK); pk.add(&h->d_chain_s0, ch_s0); pk.add(&h->d_chain_g, ch_g);
  pk.add(&h->d_grp_c0, grp_c0);
  pk.add(&h->d_lnc_L, lncL); pk.add(&h->d_zeta_L, zL); pk.add(&h->d_lgA, lgA); pk.add(&h->d_lgB, lgB);
  pk.add(&h->d_lgC, lgC); pk.add(&h->d_lgD, lgD); pk.add(&h->d_Ls, vL); pk.add(&h->d_alpha, vA);
  pk.add(&h->d_gamma, vG); pk.add(&h->d_pcr, vP); pk.add(&dL, cL); pk.add(&dA, cA); pk.add(&dC, cC);
  pk.reserve(&h->d_lnA, (size_t)h->n_cls * h->kstride);
  pk.reserve(&h->d_zeta, (size_t)h->n_cls * h->kstride);
  // create is synchronous: upload and precompute on the legacy default stream, then wait for it
  ce = pk.commit(&h->arena_create, nullptr);
  if (ce != cudaSuccess) {
    cudaStreamSynchronize(nullptr);
    delete h;
    return fail(ISRS_EGN_ENOMEM, std::string("device allocation/upload failed: ") + cudaGetErrorString(ce));
  }
  PParams pp{dL.p, dA.p, dC.p, h->d_Kc.p, h->n_cls, h->kstride, h->p_tot, h->b_tot, h->d_lnA.p, h->d_zeta.p};
  const int lrc = launch_precompute(pp, nullptr);
  ce = cudaStreamSynchronize(nullptr);
  if (lrc != 0 || ce != cudaSuccess) {
    delete h;
    return cuda_fail(lrc != 0 ? cudaGetLastError() : ce, "precompute");
  }
  *out = h;
  return ISRS_EGN_OK;
}

// sum_{i=0}^{n-1} floor((a i + b) / m) for n, m >= 1, a, b >= 0 (Euclid-like reduction, O(log)).
static long long floor_sum(long long n, long long m, long long a, long long b) {
  long long ans = 0;
  while (true) {
    if (a >= m) { ans += (n - 1) * n / 2 * (a / m); a %= m; }
    if (b >= m) { ans += n * (b / m); b %= m; }
    const long long y_max = a * n + b;
    if (y_max < m) break;
    n = y_max / m;
    b = y_max % m;
    std::swap(m, a);
  }
  return ans;
}

// Grid points of a region on lattice lines j' <= j, i.e. #{(m1, m2) in [0, N)^2 : a m1 + b m2 <= j}
// = sum over m1 <= j/a of min(N, floor((j - a m1)/b) + 1): the m1 with j - a m1 >= b (N - 1) give N
// each, the others a floor sum.
static long long lattice_cum(int N, int a, int b, long long j) {
  if (j < 0) return 0;
  const long long m_hi = std::min<long long>(N - 1, j / a);           // last m1 with j - a m1 >= 0
  const long long full = j - (long long)b * (N - 1);                  // j - a m1 >= b (N-1) <=> m1 <= full / a
  const long long m_full = full < 0 ? -1 : std::min(m_hi, full / a);  // m1 in [0, m_full]: N points
  long long tot = (m_full + 1) * N;
  const long long cnt = m_hi - m_full;                               // m1 in (m_full, m_hi]
  if (cnt > 0) {
    // i = m_hi - m1 in [0, cnt): floor((j - a m_hi + a i) / b) + 1
    tot += floor_sum(cnt, b, a, j - (long long)a * m_hi) + cnt;
  }
  return tot;
}

static long long floor_div(long long x, long long y) { return x / y - ((x % y != 0) && ((x < 0) != (y < 0))); }
static long long ceil_div(long long x, long long y) { return -floor_div(-x, y); }

// Exact number of in-support grid points of region (f, k1, k2) -- the integrand kernel's cost of the
// region and the work metric.  On a lattice line j = a m1 + b m2 (a:b = R1:R2 in lowest terms) f3 =
// C + g j is constant; the lines whose f3 lies in some closed band [lo_c, hi_c] (reading C10: an edge
// tie is in support, counted once even when two bands touch there) form a union of j-intervals, one
// per band, merged where touching bands share an edge line; the points on lines j0..j1 are
// lattice_cum(j1) - lattice_cum(j0 - 1).  All frequencies are multiples of 1/4 Hz (integer-Hz inputs,
// f_c the midpoint of half-integer edges), so the interval ends are computed in exact integers.
// O(bands x (1 or N)) per region instead of a walk over every point.
// `filter` (ISRS_EGN_FLAG_SPLIT): 0 every band, K3_IN only the bands kappa, k1, k2, K3_OUT only the others.
static long long region_points(const isrs_egn* h, double f, int k1, int k2, int kappa = -1, int filter = 0) {
  const int N = h->N, nc = h->n_ch;
  const long long r1 = h->rate[k1], r2 = h->rate[k2];
  long long x = r1, y = r2;
  while (y) { const long long t = x % y; x = y; y = t; }
  const int a = (int)(r1 / x), b = (int)(r2 / x);
  const double d1 = h->delta[k1], d2 = h->delta[k2];
  const double g = d1 / a;
  const double C = h->lo[k1] + h->lo[k2] - f + (0.5 * d1 + 0.5 * d2);
  const long long J = (long long)(a + b) * (N - 1) + 1;
  auto q4 = [](double v) { return (long long)std::llround(4.0 * v); };
  const long long C4 = q4(C), g4 = q4(g);
  const double f3max = C + g * (double)(J - 1);
  long long cnt = 0, cur0 = 0, cur1 = -2;     // current merged interval [cur0, cur1]
  for (int c = (int)(std::lower_bound(h->hi.begin(), h->hi.end(), C) - h->hi.begin());
       c < nc && h->lo[c] <= f3max; ++c) {
    if (filter) {
      const bool in = (c == kappa || c == k1 || c == k2);
      if ((filter == K3_IN) != in) continue;
    }
    const long long j0 = std::max(0LL, ceil_div(q4(h->lo[c]) - C4, g4));
    const long long j1 = std::min(J - 1, floor_div(q4(h->hi[c]) - C4, g4));
    if (j0 > j1) continue;
    if (j0 <= cur1) {                         // touching bands share the edge line
      cur1 = std::max(cur1, j1);
      continue;
    }
    if (cur1 >= cur0) cnt += lattice_cum(N, a, b, cur1) - lattice_cum(N, a, b, cur0 - 1);
    cur0 = j0;
    cur1 = j1;
  }
  if (cur1 >= cur0) cnt += lattice_cum(N, a, b, cur1) - lattice_cum(N, a, b, cur0 - 1);
  return cnt;
}

// Region enumeration for the given COIs (canonical order: COI, then k1, then k2).  The launch
// lists are ordered by decreasing region cost (stable), the partials stay indexed canonically.
static void build_worklist(const isrs_egn* h, const std::vector<int>& coi, WorkList* w) {
  w->coi = coi;
  w->fv.clear();
  w->desc.clear();
  w->coi_off.assign(1, 0);
  w->list_d.clear();
  w->list_c.clear();
  w->mirror.clear();
  std::vector<long long>& cost = w->cost;
  cost.clear();
  const int nc = h->n_ch;
  const bool mirror = (h->num.flags & ISRS_EGN_FLAG_MIRROR) != 0;
  const bool split = (h->num.flags & ISRS_EGN_FLAG_SPLIT) != 0;
  std::vector<int> idmap;
  const int fs = h->num.f_samples, nfs = std::max(1, fs);
  for (int kappa : coi) {
   for (int m = 0; m < nfs; ++m) {
    // NLI frequency: the COI centre (C1), or the 3-D midpoint sample f_m (exact: R/(2 fs) in Z)
    const double f = (fs == 0) ? h->f[kappa]
                               : h->lo[kappa] + (2.0 * m + 1.0) * (h->R[kappa] / (2.0 * fs));
    const int fvi = (int)w->fv.size();
    w->fv.push_back(f);
    const size_t first = w->desc.size();
    if (mirror) idmap.assign((size_t)nc * nc, -1);
    for (int k1 = 0; k1 < nc; ++k1) {
      for (int k2 = 0; k2 < nc; ++k2) {
        const double lo3 = h->lo[k1] + h->lo[k2] - f + (h->delta[k1] + h->delta[k2]) / 2;
        const double hi3 = h->hi[k1] + h->hi[k2] - f - (h->delta[k1] + h->delta[k2]) / 2;
        // first band with hi >= lo3
        int i = (int)(std::lower_bound(h->hi.begin(), h->hi.end(), lo3) - h->hi.begin());
        if (i >= nc || h->lo[i] > hi3) continue;
        auto overlaps = [&](int c) { return h->hi[c] >= lo3 && h->lo[c] <= hi3; };
        int flags = 0;
        if (h->phi[k1] != 0.0 && overlaps(k1)) flags |= NEED_E;
        if (h->phi[k2] != 0.0 && overlaps(k2)) flags |= NEED_F;
        if (h->phi[k1] != 0.0 && k1 == k2) flags |= NEED_G;
        if (h->psi[k1] != 0.0 && k1 == k2 && overlaps(k1)) flags |= NEED_H;
        if (split && (k1 == kappa || k2 == kappa || k1 == k2)) {
          // SCI / XCI / MCI: at most one interfering channel among (k1, k2), so the class of an
          // island depends on whether k3 is one of {kappa, k1, k2}: one entry per class, each over its
          // own lattice lines (E, F, H tie k3 to k1 / k2, so they live in the K3_IN entry; G follows D)
          const long long pin = region_points(h, f, k1, k2, kappa, K3_IN);
          const long long pout = region_points(h, f, k1, k2, kappa, K3_OUT);
          if (pin > 0 || pout == 0) {
            (flags ? w->list_c : w->list_d).push_back((int)w->desc.size());
            w->desc.push_back(RegionDesc{kappa, k1, k2, flags | K3_IN | (fvi << FV_SHIFT)});
            cost.push_back(pin);
          }
          if (pout > 0) {
            const int fo = flags & NEED_G;
            (fo ? w->list_c : w->list_d).push_back((int)w->desc.size());
            w->desc.push_back(RegionDesc{kappa, k1, k2, fo | K3_OUT | (fvi << FV_SHIFT)});
            cost.push_back(pout);
          }
          continue;
        }
        const int id = (int)w->desc.size();
        w->desc.push_back(RegionDesc{kappa, k1, k2, flags | (fvi << FV_SHIFT)});
        cost.push_back(region_points(h, f, k1, k2));
        if (mirror) {
          idmap[(size_t)k1 * nc + k2] = id;
          w->mirror.push_back(-1);
        } else {
          (flags ? w->list_c : w->list_d).push_back(id);
        }
      }
    }
    if (mirror) {
      // f1 <-> f2 symmetry: region (kappa, k1, k2), k1 < k2, also yields (kappa, k2, k1) (the region
      // filter is symmetric, so both are listed or neither); diagonal regions are computed as usual
      for (size_t id = first; id < w->desc.size(); ++id) {
        const RegionDesc& rd = w->desc[id];
        if (rd.k1 > rd.k2) continue;
        if (rd.k1 < rd.k2) w->mirror[id] = idmap[(size_t)rd.k2 * nc + rd.k1];
        ((rd.flags & (NEED_E | NEED_F | NEED_G | NEED_H)) ? w->list_c : w->list_d).push_back((int)id);
      }
    }
   }
    w->coi_off.push_back((long long)w->desc.size());
  }
  auto by_cost = [&](int x, int y) { return cost[x] > cost[y]; };
  std::stable_sort(w->list_d.begin(), w->list_d.end(), by_cost);
  std::stable_sort(w->list_c.begin(), w->list_c.end(), by_cost);
}

static int coi_list(const isrs_egn* h, int32_t n_coi, const int32_t* coi, std::vector<int>* c) {
  c->clear();
  if (!coi) {
    if (n_coi != h->n_ch) return fail(ISRS_EGN_EINVAL, "coi == NULL requires n_coi == n_ch");
    for (int i = 0; i < h->n_ch; ++i) c->push_back(i);
    return ISRS_EGN_OK;
  }
  if (n_coi < 1) return fail(ISRS_EGN_EINVAL, "n_coi < 1");
  for (int i = 0; i < n_coi; ++i) {
    if (coi[i] < 0 || coi[i] >= h->n_ch)
      return fail(ISRS_EGN_EINVAL, "coi[" + std::to_string(i) + "] out of range");
    c->push_back(coi[i]);
  }
  return ISRS_EGN_OK;
}

// Shard `rank` of `world`: the contiguous canonical region range whose cumulative
// cost (points) lies in [rank, rank + 1) * total / world.  world = 1 -> everything.
static void shard_range(const WorkList& w, int rank, int world, long long* lo, long long* hi) {
  const long long n = (long long)w.cost.size();
  if (world <= 1) {
    *lo = 0;
    *hi = n;
    return;
  }
  long double tot = 0;
  for (long long v : w.cost) tot += (long double)v + 1;   // +1: empty regions still cost a CTA
  const long double a = tot * rank / world, b = tot * (rank + 1) / world;
  long double acc = 0;
  long long i = 0;
  while (i < n && acc + 0.5L * ((long double)w.cost[i] + 1) < a) acc += (long double)w.cost[i++] + 1;
  *lo = i;
  while (i < n && acc + 0.5L * ((long double)w.cost[i] + 1) < b) acc += (long double)w.cost[i++] + 1;
  *hi = (rank == world - 1) ? n : i;
}

// The hot path: integrand over the regions of shard (rank, world) of the COI set, then either the
// per-COI assembly into eta (part_out == NULL; world must be 1) or the raw per-COI sums.
// Asynchronous on `st`: a new COI set (or shard) rebuilds the work list on the host and allocates,
// uploads and frees its device copy stream-ordered on `st` -- no host or device synchronisation.
// Every check that can fail (work-list limits, allocation, kernel attributes, pending errors) runs
// before the first kernel is enqueued; a failure after that point is a CUDA launch error (ECUDA).
// While `st` is being captured into a CUDA graph the call only enqueues kernels (no allocation: the
// work list must exist already, no timing or ordering events; fork / join use capture-only events).
static int run_nli(isrs_egn* h, const std::vector<int>& c, int rank, int world, double* eta_dev,
                   double* terms_dev, double* part_out, cudaStream_t st, double* split_dev = nullptr) {
  DeviceGuard dg(h->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) return cuda_fail(ce, "pending CUDA error");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  ce = cudaStreamIsCapturing(st, &cap);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamIsCapturing");
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  const bool rebuild = !h->have_wl || h->wl.coi != c;
  const bool reshard = world > 1 && (rebuild || h->sh_rank != rank || h->sh_world != world);
  if (capturing && (rebuild || reshard))
    return fail(ISRS_EGN_EINVAL, "stream capture: call isrs_egn_nli once with this COI set (and shard) "
                                 "on a non-capturing stream first, so that nothing is allocated inside the capture");
  if (rebuild) {
    // region ids are int32 and the f-sample index lives in 23 flag bits
    // (FLAG_SPLIT lists the < 3 n_ch regions with at most one interfering channel twice)
    const double nreg_max = (double)c.size() * std::max(1, h->num.f_samples) * h->n_ch * ((double)h->n_ch + 3);
    if (nreg_max > 2147483647.0 || (double)c.size() * std::max(1, h->num.f_samples) >= 8388608.0)
      return fail(ISRS_EGN_ERANGE, "n_coi x f_samples x n_ch^2 regions exceed the 2^31 work-list limit");
  }
  if (!h->ev[0]) {
    for (auto& e : h->ev)
      if (cudaEventCreate(&e) != cudaSuccess) return cuda_fail(cudaGetLastError(), "cudaEventCreate");
  }
  if (!h->side) {
    if (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->cap_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->cap_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreate(&h->evc[0]) != cudaSuccess || cudaEventCreate(&h->evc[1]) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "side stream / events");
  }
  const int mode = (h->num.flags & ISRS_EGN_FLAG_UNIT_LINK) ? MODE_UNIT
                   : (h->num.mu_mode == ISRS_EGN_MU_INTEGRAL ? MODE_QUAD
                   : (h->num.mu_mode == ISRS_EGN_MU_MACLAURIN ? MODE_MACLAURIN
                      : (h->num.precision == 32 ? MODE_SEG32
                         : ((h->num.flags & ISRS_EGN_FLAG_DEDUP)
                            ? (*std::max_element(h->chain_g.begin(), h->chain_g.end()) > 32 ? MODE_SEGDDL : MODE_SEGDD)
                            : ((h->num.flags & ISRS_EGN_FLAG_LITERAL_GAIN) ? MODE_SEGLG
                               : ((h->num.flags & ISRS_EGN_FLAG_SPLIT)
                                  ? (h->n_grp < h->n_chain ? MODE_SEGGRPSPL : MODE_SEGSPL)
                                  : (h->n_grp < h->n_chain ? MODE_SEGGRP : MODE_SEGMENT)))))));
  if (integrand_prepare(mode, h->tstride, h->tw, h->N) != 0)
    return cuda_fail(cudaGetLastError(), "integrand kernel attributes");
  // calls on one handle share its partials (and a rebuild frees the previous work list): a call on
  // another stream than the previous one waits (on the device) for the previous call's end
  if (!capturing && h->ordered && st != h->last_stream) cudaStreamWaitEvent(st, h->ev[3], 0);
  if (rebuild) {
    WorkList wl;
    build_worklist(h, c, &wl);
    Packer pk;
    DevBuf<RegionDesc> desc;
    DevBuf<long long> coi_off;
    DevBuf<int> coi_d, list_d, list_c;
    DevBuf<double> fv, partials, npts;
    DevBuf<int> mir;
    if (!wl.mirror.empty()) pk.add(&mir, wl.mirror);
    pk.add(&desc, wl.desc); pk.add(&coi_off, wl.coi_off); pk.add(&coi_d, wl.coi);
    pk.add(&list_d, wl.list_d); pk.add(&list_c, wl.list_c); pk.add(&fv, wl.fv);
    pk.reserve(&partials, wl.desc.size() * 6);
    pk.reserve(&npts, c.size());
    ce = pk.commit(&h->arena_plan, st, &h->pins);      // on failure the handle keeps its previous work list
    if (ce != cudaSuccess) return fail(ISRS_EGN_ENOMEM, std::string("work-list allocation failed: ") + cudaGetErrorString(ce));
    h->d_desc = desc; h->d_coi_off = coi_off; h->d_coi = coi_d; h->d_list_d = list_d;
    h->d_list_c = list_c; h->d_fv = fv; h->d_partials = partials; h->d_npts = npts;
    h->d_mirror = mir;
    h->wl = std::move(wl);
    h->have_wl = true;
    h->have_result = false;   // the new partials hold nothing until this call's kernels ran
    cudaEventRecord(h->ev[3], st);   // later calls on other streams order behind this rebuild
    h->ordered = true;
    h->last_stream = st;
    h->sh_rank = h->sh_world = -1;
  }
  const int* dl_d = h->d_list_d.p;
  const int* dl_c = h->d_list_c.p;
  long long r_lo = 0, r_hi = (long long)h->wl.desc.size();
  std::vector<int> act_d, act_c;
  if (world > 1) {
    if (reshard) {
      long long lo, hi;
      shard_range(h->wl, rank, world, &lo, &hi);
      for (int id : h->wl.list_d)
        if (id >= lo && id < hi) act_d.push_back(id);
      for (int id : h->wl.list_c)
        if (id >= lo && id < hi) act_c.push_back(id);
      Packer pk;
      DevBuf<int> sd, sc;
      pk.add(&sd, act_d);
      pk.add(&sc, act_c);
      ce = pk.commit(&h->arena_shard, st, &h->pins);
      if (ce != cudaSuccess) return fail(ISRS_EGN_ENOMEM, std::string("shard list allocation failed: ") + cudaGetErrorString(ce));
      h->d_sh_d = sd;
      h->d_sh_c = sc;
      h->sh_lo = lo;
      h->sh_hi = hi;
      h->sh_rank = rank;
      h->sh_world = world;
      h->sh_act_d = std::move(act_d);
      h->sh_act_c = std::move(act_c);
      cudaEventRecord(h->ev[3], st);   // later calls on other streams order behind this upload
      h->ordered = true;
      h->last_stream = st;
    }
    h->act_d = &h->sh_act_d;
    h->act_c = &h->sh_act_c;
    dl_d = h->d_sh_d.p;
    dl_c = h->d_sh_c.p;
    r_lo = h->sh_lo;
    r_hi = h->sh_hi;
  } else {
    h->act_d = &h->wl.list_d;
    h->act_c = &h->wl.list_c;
  }
  KParams kp{};
  kp.lo = h->d_lo.p; kp.hi = h->d_hi.p; kp.f = h->d_f.p; kp.G = h->d_G.p; kp.R = h->d_R.p;
  kp.P = h->d_P.p; kp.phi = h->d_phi.p; kp.psi = h->d_psi.p; kp.delta = h->d_delta.p;
  kp.rate = h->d_rate.p; kp.n_ch = h->n_ch;
  kp.A2 = h->d_A2.p; kp.A3 = h->d_A3.p; kp.Eh = h->d_Eh.p; kp.ah = h->d_ah.p; kp.gh = h->d_gh.p;
  kp.mac_c = h->d_macc.p; kp.aL = h->d_aL.p; kp.K = h->d_K.p; kp.cls = h->d_cls.p;
  kp.n_span = h->n_span;
  kp.chain_s0 = h->d_chain_s0.p; kp.chain_g = h->d_chain_g.p; kp.n_chain = h->n_chain;
  kp.grp_c0 = h->d_grp_c0.p; kp.n_grp = h->n_grp;
  kp.lnc_L = h->d_lnc_L.p; kp.zeta_L = h->d_zeta_L.p; kp.lgA = h->d_lgA.p; kp.lgB = h->d_lgB.p;
  kp.lgC = h->d_lgC.p; kp.lgD = h->d_lgD.p;
  kp.Ls = h->d_Ls.p; kp.alpha = h->d_alpha.p; kp.gamma = h->d_gamma.p; kp.pcr = h->d_pcr.p;
  kp.b_tot = h->b_tot;
  for (int i = 0; i < 12; ++i) { kp.gl_x[i] = h->gl_x[i]; kp.gl_w[i] = h->gl_w[i]; }
  kp.lnA = h->d_lnA.p; kp.zeta = h->d_zeta.p; kp.Kc = h->d_Kc.p; kp.n_cls = h->n_cls;
  kp.kstride = h->kstride; kp.tstride = h->tstride; kp.tw = h->tw; kp.N = h->N;
  kp.fv = h->d_fv.p; kp.desc = h->d_desc.p; kp.partials = h->d_partials.p;
  kp.mirror = (h->num.flags & ISRS_EGN_FLAG_MIRROR) ? h->d_mirror.p : nullptr;
  kp.mode = mode;
  int launches = 0;
#ifdef ISRS_PROF
  static unsigned long long* d_prof = nullptr;
  if (!d_prof) cudaMalloc(&d_prof, 16 * sizeof(unsigned long long));
  cudaMemsetAsync(d_prof, 0, 16 * sizeof(unsigned long long), st);
  kp.prof = d_prof;
#endif
  // fork: the coherent regions run on the side stream while the D-only regions run on `st`;
  // join before the per-COI reduce.  ev[0] -> ev[2] brackets the whole integrand phase.
  cudaEvent_t fork = capturing ? h->cap_fork : h->ev_fork, join = capturing ? h->cap_join : h->ev_join;
  if (!capturing) cudaEventRecord(h->ev[0], st);
  cudaEventRecord(fork, st);
  cudaStreamWaitEvent(h->side, fork, 0);
  if (!capturing) cudaEventRecord(h->evc[0], h->side);
  if (launch_integrand(kp, dl_c, (long long)h->act_c->size(), true, h->side, &launches) != 0)
    return cuda_fail(cudaGetLastError(), "integrand launch (coherent regions)");
  if (!capturing) cudaEventRecord(h->evc[1], h->side);
  cudaEventRecord(join, h->side);
  if (launch_integrand(kp, dl_d, (long long)h->act_d->size(), false, st, &launches) != 0)
    return cuda_fail(cudaGetLastError(), "integrand launch (D-only regions)");
  if (!capturing) cudaEventRecord(h->ev[1], st);
  cudaStreamWaitEvent(st, join, 0);
  if (!capturing) cudaEventRecord(h->ev[2], st);
  RParams rp{h->d_desc.p, h->d_partials.p, h->d_coi_off.p, h->d_coi.p, h->d_G.p, h->d_R.p,
             h->d_P.p, h->d_phi.p, h->d_psi.p, (int)c.size(),
             1.0 / std::max(1, h->num.f_samples), eta_dev, terms_dev, h->d_npts.p, r_lo, r_hi,
             part_out};
  if (launch_reduce(rp, st) != 0) return cuda_fail(cudaGetLastError(), "reduce launch");
  launches += 1;
  if (split_dev) {   // SCI / XCI / MCI parts from the same partials (ISRS_EGN_FLAG_SPLIT work list)
    if (launch_reduce_split(rp, split_dev, st) != 0) return cuda_fail(cudaGetLastError(), "split reduce launch");
    launches += 1;
  }
  if (capturing) return ISRS_EGN_OK;     // the handle's timing / ordering state describes direct calls
  cudaEventRecord(h->ev[3], st);
  h->ordered = true;
  h->launched[0] = !h->act_d->empty();
  h->launched[1] = !h->act_c->empty();
#ifdef ISRS_PROF
  {
    unsigned long long hp[16];
    cudaMemcpyAsync(hp, d_prof, sizeof(hp), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double tot = 0;
    for (int i = 0; i < 7; ++i) tot += (double)hp[i];
    const char* nm[7] = {"prologue", "line scan", "chunk setup", "table build", "span math",
                         "accumulate", "epilogue"};
    fprintf(stderr, "ISRS_PROF warp-cycles:");
    for (int i = 0; i < 7; ++i) fprintf(stderr, " %s %.2f%%", nm[i], 100.0 * hp[i] / tot);
    fprintf(stderr, " (total %.3e)\n", tot);
    fprintf(stderr, "ISRS_PROF table builds %llu, mean rows %.2f; chunks %llu, mean slots %.1f, mean lines %.2f\n",
            hp[8], hp[8] ? (double)hp[9] / hp[8] : 0.0, hp[10], hp[10] ? (double)hp[11] / hp[10] : 0.0,
            hp[10] ? (double)hp[12] / hp[10] : 0.0);
  }
#endif
  h->last_launches = launches;
  h->last_stream = st;
  h->have_result = true;
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_nli(isrs_egn_t* h, int32_t n_coi, const int32_t* coi, double* eta_dev,
                            double* terms_dev, void* cuda_stream) {
  if (!h) return fail(ISRS_EGN_EINVAL, "handle is NULL");
  if (!eta_dev) return fail(ISRS_EGN_EINVAL, "eta_dev is NULL");
  NvtxRange nv("isrs_egn_nli");
  std::vector<int> c;
  int rc = coi_list(h, n_coi, coi, &c);
  if (rc) return rc;
  return run_nli(h, c, 0, 1, eta_dev, terms_dev, nullptr, (cudaStream_t)cuda_stream);
}

extern "C" int isrs_egn_nli_split(isrs_egn_t* h, int32_t n_coi, const int32_t* coi, double* eta_dev,
                                  double* terms_dev, double* split_dev, void* cuda_stream) {
  if (!h) return fail(ISRS_EGN_EINVAL, "handle is NULL");
  if (!eta_dev || !split_dev) return fail(ISRS_EGN_EINVAL, "eta_dev / split_dev is NULL");
  if (!(h->num.flags & ISRS_EGN_FLAG_SPLIT))
    return fail(ISRS_EGN_EINVAL, "isrs_egn_nli_split needs a handle created with ISRS_EGN_FLAG_SPLIT");
  NvtxRange nv("isrs_egn_nli_split");
  std::vector<int> c;
  int rc = coi_list(h, n_coi, coi, &c);
  if (rc) return rc;
  return run_nli(h, c, 0, 1, eta_dev, terms_dev, nullptr, (cudaStream_t)cuda_stream, split_dev);
}

extern "C" int isrs_egn_nli_shard(isrs_egn_t* h, int32_t n_coi, const int32_t* coi, int32_t rank,
                                  int32_t world, double* coi_sums_dev, void* cuda_stream) {
  if (!h) return fail(ISRS_EGN_EINVAL, "handle is NULL");
  if (!coi_sums_dev) return fail(ISRS_EGN_EINVAL, "coi_sums_dev is NULL");
  NvtxRange nv("isrs_egn_nli_shard");
  if (world < 1 || rank < 0 || rank >= world) return fail(ISRS_EGN_EINVAL, "rank/world out of range");
  if (h->num.flags & ISRS_EGN_FLAG_MIRROR)
    return fail(ISRS_EGN_EUNSUPPORTED, "FLAG_MIRROR writes partner regions across the region list: no shards");
  if (h->num.flags & ISRS_EGN_FLAG_SPLIT)
    return fail(ISRS_EGN_EUNSUPPORTED, "FLAG_SPLIT: the SCI / XCI / MCI parts are not sharded");
  std::vector<int> c;
  int rc = coi_list(h, n_coi, coi, &c);
  if (rc) return rc;
  return run_nli(h, c, rank, world, nullptr, nullptr, coi_sums_dev, (cudaStream_t)cuda_stream);
}

extern "C" int isrs_egn_combine(isrs_egn_t* h, int32_t n_coi, const int32_t* coi, int32_t world,
                                const double* gathered_dev, double* eta_dev, double* terms_dev,
                                void* cuda_stream) {
  if (!h) return fail(ISRS_EGN_EINVAL, "handle is NULL");
  if (!gathered_dev || !eta_dev) return fail(ISRS_EGN_EINVAL, "gathered_dev / eta_dev is NULL");
  if (world < 1) return fail(ISRS_EGN_EINVAL, "world < 1");
  std::vector<int> c;
  int rc = coi_list(h, n_coi, coi, &c);
  if (rc) return rc;
  DeviceGuard dg(h->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  if (!h->have_wl || h->wl.coi != c || !h->d_coi.p)
    return fail(ISRS_EGN_EINVAL, "combine: COI set differs from the last shard call");
  CParams cp{gathered_dev, world, h->d_coi.p, h->d_R.p, h->d_P.p, (int)c.size(),
             1.0 / std::max(1, h->num.f_samples), eta_dev, terms_dev, nullptr};
  if (launch_combine(cp, cuda_stream) != 0) return cuda_fail(cudaGetLastError(), "combine launch");
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_plan_shards(const isrs_egn_problem* p, const isrs_egn_numerics* n, int32_t n_coi,
                                    const int32_t* coi, int32_t world, int64_t* regions_out,
                                    int64_t* points_out, int64_t* first_region_out) {
  isrs_egn_numerics num = n ? *n : isrs_egn_numerics{};
  if (num.precision == 0) num.precision = 64;
  int rc = validate(p, &num);
  if (rc) return rc;
  if (world < 1) return fail(ISRS_EGN_EINVAL, "world < 1");
  isrs_egn h;                       // host-only: no device memory is touched
  canon_channels(&h, p, num);
  std::vector<int> c;
  rc = coi_list(&h, n_coi, coi, &c);
  if (rc) return rc;
  WorkList w;
  build_worklist(&h, c, &w);
  for (int r = 0; r < world; ++r) {
    long long lo, hi;
    shard_range(w, r, world, &lo, &hi);
    long long pts = 0;
    for (long long i = lo; i < hi; ++i) pts += w.cost[i];
    if (regions_out) regions_out[r] = hi - lo;
    if (points_out) points_out[r] = pts;
    if (first_region_out) first_region_out[r] = lo;
  }
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_region_partials(isrs_egn_t* h, int32_t n, const int32_t* kappa,
                                        const int32_t* k1, const int32_t* k2, double* out_host) {
  if (!h || !out_host || n < 0 || (n > 0 && (!kappa || !k1 || !k2)))
    return fail(ISRS_EGN_EINVAL, "bad argument");
  if (!h->have_result) return fail(ISRS_EGN_EINVAL, "no isrs_egn_nli() result yet");
  DeviceGuard dg(h->device);
  cudaError_t ce = cudaEventSynchronize(h->ev[3]);
  if (ce != cudaSuccess) return cuda_fail(ce, "event sync");
  const auto& w = h->wl;
  for (int q = 0; q < n; ++q) {
    double* o = out_host + 6 * (size_t)q;
    for (int k = 0; k < 5; ++k) o[k] = 0.0;
    o[5] = -1.0;
    auto itc = std::find(w.coi.begin(), w.coi.end(), kappa[q]);
    if (itc == w.coi.end()) continue;
    const size_t ci = itc - w.coi.begin();
    bool found = false;
    for (long long r = w.coi_off[ci]; r < w.coi_off[ci + 1]; ++r) {
      if (w.desc[r].k1 == k1[q] && w.desc[r].k2 == k2[q]) {
        double v[6];
        ce = cudaMemcpy(v, h->d_partials.p + r * 6, 6 * sizeof(double), cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) return cuda_fail(ce, "partials copy");
        for (int k = 0; k < 6; ++k) o[k] = found ? o[k] + v[k] : v[k];
        found = true;
        if (!(h->num.flags & ISRS_EGN_FLAG_SPLIT)) break;   // SPLIT: a region may have two entries
      }
    }
  }
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_work(const isrs_egn_t* h, int32_t n_coi, const int32_t* coi, int64_t* points,
                             int64_t* point_spans, int64_t* regions) {
  if (!h) return fail(ISRS_EGN_EINVAL, "handle is NULL");
  std::vector<int> c;
  int rc = coi_list(h, n_coi, coi, &c);
  if (rc) return rc;
  WorkList w;
  build_worklist(h, c, &w);   // host planner only: exact in-support point counts per region
  long long tot = 0;
  for (long long v : w.cost) tot += v;
  if (points) *points = tot;
  if (point_spans) *point_spans = tot * h->n_span;
  if (regions) *regions = (long long)w.desc.size();
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_last_work(isrs_egn_t* h, int64_t* points, int64_t* point_spans, int64_t* regions) {
  if (!h) return fail(ISRS_EGN_EINVAL, "handle is NULL");
  if (!h->have_result) return fail(ISRS_EGN_EINVAL, "no isrs_egn_nli() result yet");
  DeviceGuard dg(h->device);
  cudaError_t ce = cudaEventSynchronize(h->ev[3]);
  if (ce != cudaSuccess) return cuda_fail(ce, "event sync");
  const size_t nr = h->wl.desc.size();
  std::vector<double> np(nr);
  ce = cudaMemcpy2D(np.data(), sizeof(double), h->d_partials.p + 5, 6 * sizeof(double), sizeof(double), nr,
                    cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_fail(ce, "npts copy");
  long long tot = 0;
  for (int id : *h->act_d) tot += (long long)np[id];
  for (int id : *h->act_c) tot += (long long)np[id];
  if (points) *points = tot;
  if (point_spans) *point_spans = tot * h->n_span;
  if (regions) *regions = (long long)(h->act_d->size() + h->act_c->size());
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_last_kernel_ms(isrs_egn_t* h, double* ms_out, double* point_spans_out) {
  if (!h || !ms_out) return fail(ISRS_EGN_EINVAL, "bad argument");
  if (!h->have_result) return fail(ISRS_EGN_EINVAL, "no isrs_egn_nli() result yet");
  DeviceGuard dg(h->device);
  cudaError_t ce = cudaEventSynchronize(h->ev[3]);
  if (ce != cudaSuccess) return cuda_fail(ce, "event sync");
  // [0] D-only launch (start of the integrand phase -> its end on st), [1] coherent launch (side
  // stream, concurrent), [2] the per-COI reduce; [3] = the whole integrand phase (both launches)
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
  ms_out[0] = h->launched[0] ? (double)ms : 0.0;
  cudaEventElapsedTime(&ms, h->evc[0], h->evc[1]);
  ms_out[1] = h->launched[1] ? (double)ms : 0.0;
  cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]);
  ms_out[2] = (double)ms;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[2]);
  ms_out[3] = (double)ms;
  if (point_spans_out) {
    const size_t nr = h->wl.desc.size();
    std::vector<double> np(nr);
    ce = cudaMemcpy2D(np.data(), sizeof(double), h->d_partials.p + 5, 6 * sizeof(double),
                      sizeof(double), nr, cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) return cuda_fail(ce, "npts copy");
    double a = 0, b = 0;
    for (int id : *h->act_d) a += np[id];
    for (int id : *h->act_c) b += np[id];
    point_spans_out[0] = a * h->n_span;
    point_spans_out[1] = b * h->n_span;
    point_spans_out[2] = (a + b) * h->n_span;
  }
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_span_chains(const isrs_egn_t* h, int32_t* n_chain, int32_t* chain_g, int32_t* k_s) {
  if (!h || !n_chain) return fail(ISRS_EGN_EINVAL, "bad argument");
  *n_chain = h->n_chain;
  if (chain_g)
    for (int c = 0; c < h->n_chain; ++c) chain_g[c] = h->chain_g[c];
  if (k_s)
    for (int s = 0; s < h->n_span; ++s) k_s[s] = h->k_s[s];
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_profile_tables(isrs_egn_t* h, int32_t span, int32_t* k_out, double* ln_a_out,
                                       double* zeta_out) {
  if (!h || !k_out) return fail(ISRS_EGN_EINVAL, "bad argument");
  if (span < 0 || span >= h->n_span) return fail(ISRS_EGN_EINVAL, "span out of range");
  const int K = h->k_s[span];
  *k_out = K;
  if (!ln_a_out && !zeta_out) return ISRS_EGN_OK;
  DeviceGuard dg(h->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  const size_t off = (size_t)h->cls_of_span[span] * h->kstride;
  cudaError_t ce = cudaSuccess;
  if (ln_a_out) ce = cudaMemcpy(ln_a_out, h->d_lnA.p + off, sizeof(double) * K, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess && zeta_out)
    ce = cudaMemcpy(zeta_out, h->d_zeta.p + off, sizeof(double) * K, cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_fail(ce, "table copy");
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_chain_groups(const isrs_egn_t* h, int32_t* n_grp, int32_t* grp_c0) {
  if (!h || !n_grp) return fail(ISRS_EGN_EINVAL, "bad argument");
  *n_grp = h->n_grp;
  if (grp_c0)
    for (int g = 0; g <= h->n_grp; ++g) grp_c0[g] = h->grp_c0[g];
  return ISRS_EGN_OK;
}

extern "C" int isrs_egn_last_launch_count(const isrs_egn_t* h) { return h ? h->last_launches : 0; }

extern "C" int isrs_egn_eta_host(const isrs_egn_problem* p, const isrs_egn_numerics* n, int device,
                                 int32_t n_coi, const int32_t* coi, double* eta_host, double* terms_host) {
  if (!eta_host) return fail(ISRS_EGN_EINVAL, "eta_host is NULL");
  NvtxRange nv("isrs_egn_eta_host");
  isrs_egn_t* h = nullptr;
  int rc = isrs_egn_create(p, n, device, &h);
  if (rc) return rc;
  DeviceGuard dg(device);
  const int nco = coi ? n_coi : p->n_ch;
  double* d = nullptr;
  cudaError_t ce = dev_alloc_on(reinterpret_cast<void**>(&d), sizeof(double) * (size_t)nco * 6, nullptr);
  if (ce != cudaSuccess) {
    isrs_egn_destroy(h);
    return cuda_fail(ce, "device allocation");
  }
  rc = isrs_egn_nli(h, nco, coi, d, terms_host ? d + nco : nullptr, nullptr);
  if (rc == 0) {
    ce = cudaMemcpy(eta_host, d, sizeof(double) * nco, cudaMemcpyDeviceToHost);
    if (ce == cudaSuccess && terms_host)
      ce = cudaMemcpy(terms_host, d + nco, sizeof(double) * nco * 5, cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) rc = cuda_fail(ce, "result copy");
  }
  cudaStreamSynchronize(nullptr);
  dev_free_on(d, nullptr);
  isrs_egn_destroy(h);
  return rc;
}

extern "C" void isrs_egn_destroy(isrs_egn_t* h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  cudaDeviceSynchronize();
  delete h;
}

extern "C" const char* isrs_egn_strerror(int code) {
  switch (code) {
    case ISRS_EGN_OK: return "ok";
    case ISRS_EGN_EINVAL: return "invalid argument";
    case ISRS_EGN_EOVERLAP: return "channel bands overlap";
    case ISRS_EGN_ERANGE: return "value out of supported range";
    case ISRS_EGN_ENOMEM: return "out of memory";
    case ISRS_EGN_ECUDA: return "CUDA error";
    case ISRS_EGN_EUNSUPPORTED: return "unsupported option";
    default: return "unknown status";
  }
}

extern "C" const char* isrs_egn_last_error(void) { return g_err.c_str(); }
