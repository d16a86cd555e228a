// kk_host.cpp — libkkrx.so host side: the C ABI of include/kkrx.h.
//
// kk_init validates the configuration and computes every constant of the chain once, in fp64:
//   * RRC taps h[j], j = −512..512 (unit energy, β = rolloff, span 256 at 4 sps)
//     and the MF spectrum H[k] = Σ_j h[j]·cos(2πkj/4096) / 4096 (real: h is symmetric; R6);
//   * LO table exp(−2πiσq/lo_den), q < lo_den (R9: the LO is indexed by the global sample, no accumulator);
//   * the tap count L = 2⌈τ_max/(T/2)⌉ + 7 and the CD-inverse init taps w_cd by least
//     squares over 2001 frequencies of the data band (modified Gram–Schmidt QR, fp64);
//   * FFT twiddle tables W_N^{r·k} in the [r][k] layouts the kernels read;
// then allocates scratch for max_samples_per_call. kk_process_frames enqueues K1 → K2 → K3 on the caller's
// stream with no host synchronisation.
#include <cfloat>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <array>
#include <algorithm>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: host-side ranges for nsys / ncu --nvtx timelines

#include "../../include/kkrx.h"

namespace {
// NVTX range around a library call or one of its kernel launches (SURVEY §5 tracing); no-op cost without a tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace
#include "kk_params.h"

namespace kk {
size_t k3_smem_bytes(int K);
}

using cd = std::complex<double>;

struct kk_ctx {
  kk_config cfg;
  int device = 0, num_sms = 148;
  int L = 0, K = 0;
  bool ddlms = false;   // eq_mode == KK_EQ_DDLMS
  int Ky = 0;           // 2-sps margin of y around the core: K (block LS) or 2·warmup + 2 (DDLMS)
  std::vector<uint8_t> schedule;
  std::vector<cd> w_cd;
  // device constants
  float* d_H = nullptr;
  float2* d_Hc = nullptr;   // complex static filter RRC × CD inverse (DDLMS mode)
  float2* d_lo = nullptr;
  float2* d_wcd = nullptr;
  float2 *d_tw1024 = nullptr, *d_tw256 = nullptr, *d_twN = nullptr, *d_twI = nullptr;
  int mfN = 4096, mfKeep = 1536;   // MF overlap-save grid: FFT size, kept 2-sps outputs per tile
  float2* d_tw2048u = nullptr;   // K1U twiddles W₂₀₄₈^{t·k1}, [k1·64 + t] (k1 < 32, t < 64)
  int64_t halo = 0;              // kk_halo: kHalo, or kHaloUp with upsample = 2
  double hb_odd[8] = {0};        // odd half-band taps f[1], f[3], …, f[15] (upsample = 2)
  uint8_t* d_sched = nullptr;
  uint32_t ref_key = 0;          // ref_prbs: key of the transmitter's label hash (kk::ref_prbs_key(ref_seed))
  uint8_t* d_refgen = nullptr;   // ref_prbs: generated reference labels of a device-buffer call
  // scratch
  int64_t nmax = 0;
  float2* d_E = nullptr;
  float2* d_part = nullptr;
  int* d_clamp = nullptr;
  float2* d_y = nullptr;
  CUtensorMap ymaps[2];   // K3's tensor-TMA views of d_y (K ≤ 4)
  double* d_k3rec = nullptr;   // K3a → K3s per-frame records
  float2* d_k3th = nullptr;    // K3s → K3c per-frame θ₁ records
  float2* d_z = nullptr;
  float* d_segpow = nullptr;     // DDLMS mode: K2's per-64-symbol power sums (K3′ AGC)
  unsigned long long* d_counters = nullptr;
  // host-buffer path staging (lazy)
  void* d_in[2] = {nullptr, nullptr};
  uint8_t* d_ref[2] = {nullptr, nullptr};
  uint8_t* d_dec[2] = {nullptr, nullptr};
  cudaStream_t hs[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t entry_ev[2] = {nullptr, nullptr};   // host path: order after the legacy stream and the last caller stream
  // last call
  bool have_call = false;
  int64_t last_first = 0, last_n = 0;
  bool last_z = false;
  cudaStream_t last_stream = nullptr;
  bool have_stream = false;                         // last_stream holds a call's stream (nullptr = legacy stream)
  cudaEvent_t order_ev = nullptr;                   // cross-stream ordering of consecutive calls (order_after_last)
  std::string err;
  // debug_guard: canary-padded allocations {name, base, user bytes}
  struct GuardRec { const char* name; unsigned char* base; size_t bytes; };
  std::vector<GuardRec> guards;
  // per-kernel timing (kk_enable_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::array<cudaEvent_t, 4>> ev_pending;
  double k_ms[3] = {0, 0, 0};
  int64_t k_launches[3] = {0, 0, 0};
};

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kC = 299792458.0;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

kk_status fail(kk_ctx* c, kk_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

// ---------------------------------------------------------------- fp64 constants
std::vector<double> rrc_taps(double beta, int span, int sps) {
  const int half = span * sps / 2;
  std::vector<double> h(2 * half + 1);
  double e = 0.0;
  for (int idx = 0; idx <= 2 * half; ++idx) {
    const double t = (double)(idx - half) / sps;   // symbol periods
    double v;
    if (t == 0.0) {
      v = 1.0 - beta + 4.0 * beta / kPi;
    } else if (std::fabs(4.0 * beta * std::fabs(t) - 1.0) < 1e-12) {
      v = beta / std::sqrt(2.0) *
          ((1.0 + 2.0 / kPi) * std::sin(kPi / (4.0 * beta)) + (1.0 - 2.0 / kPi) * std::cos(kPi / (4.0 * beta)));
    } else {
      v = (std::sin(kPi * t * (1.0 - beta)) + 4.0 * beta * t * std::cos(kPi * t * (1.0 + beta))) /
          (kPi * t * (1.0 - (4.0 * beta * t) * (4.0 * beta * t)));
    }
    h[idx] = v;
    e += v * v;
  }
  const double s = 1.0 / std::sqrt(e);
  for (auto& v : h) v *= s;
  return h;
}

double beta2L(const kk_config& c) {
  const double dl_si = c.dispersion_ps_per_nm * 1e-3;   // ps/nm → s/m
  return -dl_si * c.lambda_m * c.lambda_m / (2.0 * kPi * kC);
}

int tap_rule(const kk_config& c) {
  if (c.eq_taps) return c.eq_taps;
  const double fc = c.fs_hz * (double)c.lo_num / (double)c.lo_den;
  const double tau = std::fabs(beta2L(c)) * 2.0 * kPi * (fc + (1.0 + c.rolloff) * c.baud_hz / 2.0);
  const double half_T = 0.5 / c.baud_hz;
  return 2 * (int)std::ceil(tau / half_T - 1e-12) + 7;
}

// least squares min ||A w − b|| via modified Gram–Schmidt QR (A: m×n complex, column-major)
std::vector<cd> lstsq_mgs(std::vector<cd> A, std::vector<cd> b, int m, int n) {
  std::vector<cd> R((size_t)n * n, cd(0, 0));
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < j; ++i) {
      cd r(0, 0);
      for (int k = 0; k < m; ++k) r += std::conj(A[(size_t)i * m + k]) * A[(size_t)j * m + k];
      R[(size_t)i * n + j] = r;
      for (int k = 0; k < m; ++k) A[(size_t)j * m + k] -= r * A[(size_t)i * m + k];
    }
    // re-orthogonalise once (MGS2) for the ill-conditioned band-limited Vandermonde columns
    for (int i = 0; i < j; ++i) {
      cd r(0, 0);
      for (int k = 0; k < m; ++k) r += std::conj(A[(size_t)i * m + k]) * A[(size_t)j * m + k];
      R[(size_t)i * n + j] += r;
      for (int k = 0; k < m; ++k) A[(size_t)j * m + k] -= r * A[(size_t)i * m + k];
    }
    double nr = 0.0;
    for (int k = 0; k < m; ++k) nr += std::norm(A[(size_t)j * m + k]);
    nr = std::sqrt(nr);
    R[(size_t)j * n + j] = nr;
    for (int k = 0; k < m; ++k) A[(size_t)j * m + k] /= nr;
  }
  std::vector<cd> qb(n);
  for (int j = 0; j < n; ++j) {
    cd s(0, 0);
    for (int k = 0; k < m; ++k) s += std::conj(A[(size_t)j * m + k]) * b[k];
    qb[j] = s;
  }
  std::vector<cd> w(n);
  for (int j = n - 1; j >= 0; --j) {
    cd s = qb[j];
    for (int i = j + 1; i < n; ++i) s -= R[(size_t)j * n + i] * w[i];
    w[j] = s / R[(size_t)j * n + j];
  }
  return w;
}

std::vector<cd> cd_init_taps(const kk_config& c, int L) {
  const int K = (L - 1) / 2;
  const int m = 2001;
  const double fc = c.fs_hz * (double)c.lo_num / (double)c.lo_den;
  const double edge = (1.0 + c.rolloff) * c.baud_hz / 2.0;
  const double b2 = beta2L(c);
  std::vector<cd> A((size_t)m * L), b(m);
  for (int k = 0; k < m; ++k) {
    const double nu = -edge + 2.0 * edge * (double)k / (double)(m - 1);
    for (int j = -K; j <= K; ++j) {
      const double ph = -2.0 * kPi * nu * (double)j / (2.0 * c.baud_hz);
      A[(size_t)(j + K) * m + k] = cd(std::cos(ph), std::sin(ph));
    }
    const double w = 2.0 * kPi * (nu + (double)c.sideband * fc);
    const double ph = -(b2 / 2.0) * w * w;
    b[k] = cd(std::cos(ph), std::sin(ph));
  }
  return lstsq_mgs(A, b, m, L);
}

std::vector<float2> twiddles(int N, int R, int Ns) {   // [r][k] = exp(−2πi r k /(Ns R)), k < Ns
  std::vector<float2> t((size_t)R * Ns);
  for (int r = 0; r < R; ++r)
    for (int k = 0; k < Ns; ++k) {
      const double a = -2.0 * kPi * (double)((int64_t)r * k % (Ns * R)) / (double)(Ns * R);
      t[(size_t)r * Ns + k] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  (void)N;
  return t;
}

constexpr size_t kGuardBytes = 64 * 1024;
constexpr unsigned char kGuardByte = 0xA5;

// Scratch allocation; with cfg.debug_guard the buffer sits between two kGuardBytes canary zones.
template <typename T>
cudaError_t dalloc(kk_ctx* c, const char* name, T** dst, size_t bytes) {
  if (!c->cfg.debug_guard) return cudaMalloc((void**)dst, bytes);
  unsigned char* base = nullptr;
  cudaError_t e = cudaMalloc((void**)&base, bytes + 2 * kGuardBytes);
  if (e != cudaSuccess) return e;
  e = cudaMemset(base, kGuardByte, bytes + 2 * kGuardBytes);
  if (e != cudaSuccess) { cudaFree(base); return e; }
  c->guards.push_back({name, base, bytes});
  *dst = reinterpret_cast<T*>(base + kGuardBytes);
  return cudaSuccess;
}

void dfree(kk_ctx* c, void* p) {
  if (!p) return;
  for (auto& g : c->guards)
    if (g.base + kGuardBytes == p) { cudaFree(g.base); return; }
  cudaFree(p);
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc((void**)dst, v.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// Odd taps of the 31-tap half-band filter (DESIGN.md §3 "KK upsampling"): f[k] = ½·sinc(k/2)·kaiser₁₀(k),
// k = 2i − 1, rescaled so that Σ_{k odd} f[k] = ½ (unit DC gain). Kaiser: I0(β√(1 − (k/15)²)) / I0(β).
void halfband_odd(double out[8]) {
  constexpr double beta = 10.0;
  auto i0 = [](double x) {
    double sum = 1.0, term = 1.0;
    for (int m = 1; m < 200; ++m) {
      term *= (x / (2.0 * m)) * (x / (2.0 * m));
      sum += term;
      if (term < 1e-18 * sum) break;
    }
    return sum;
  };
  double acc = 0.0;
  for (int i = 1; i <= 8; ++i) {
    const double k = 2.0 * i - 1.0;
    const double w = i0(beta * std::sqrt(1.0 - (k / 15.0) * (k / 15.0))) / i0(beta);
    const double sinc = std::sin(kPi * k / 2.0) / (kPi * k / 2.0);
    out[i - 1] = 0.5 * sinc * w;
    acc += out[i - 1];
  }
  for (int i = 0; i < 8; ++i) out[i] *= 0.25 / acc;   // 2·Σ_i f = ½
}

kk_status validate(const kk_config& c, std::string& why) {
  auto bad = [&](const char* m) { why = m; return KK_ERR_CONFIG; };
  if (!(c.fs_hz > 0) || !(c.baud_hz > 0) || std::fabs(c.fs_hz / c.baud_hz - 4.0) > 1e-9) return bad("fs/baud must be 4");
  if (c.debug_guard != 0 && c.debug_guard != 1) return bad("debug_guard must be 0 or 1");
  if (c.upsample != 1 && c.upsample != 2) return bad("upsample must be 1 or 2");
  if (c.ref_prbs < 0 || c.ref_prbs > 2) return bad("ref_prbs must be 0, 1 (transmitter hash) or 2 (PRBS-31)");
  if (c.lo_den <= 0 || c.lo_den > 4096 || c.lo_num < 0 || c.lo_num >= c.lo_den) return bad("lo_num/lo_den out of range");
  if (c.sideband != 1 && c.sideband != -1) return bad("sideband must be +1 or -1");
  if (!(c.rolloff > 0 && c.rolloff <= 1)) return bad("rolloff must be in (0,1]");
  if (!is_pow2(c.hilbert_n) || c.hilbert_hop < 1 || c.hilbert_hop > c.hilbert_n) return bad("hilbert_n must be pow2, hop in [1,n]");
  if (c.hilbert_n != kk::kHilbertN || c.hilbert_hop != kk::kHilbertHop) return bad("kernels are built for hilbert 1024/512");
  if (!((c.mf_fft_n == 4096 && c.mf_hop == 3072) || (c.mf_fft_n == 8192 && c.mf_hop == 7168)))
    return bad("kernels are built for MF 4096/3072 and 8192/7168");
  if (c.rrc_span_sym < 8 || c.rrc_span_sym * 4 > c.mf_fft_n - c.mf_hop) return bad("rrc span: taps-1 must fit the MF overlap");
  if (c.frame_symbols != kk::kFrameSym) return bad("kernels are built for 4096-symbol frames");
  if (c.eq_taps != 0 && (c.eq_taps < 3 || c.eq_taps > 2 * kk::kMaxK + 1 || (c.eq_taps % 2) == 0)) return bad("eq_taps must be 0 or odd in [3,15]");
  if (c.cpr_window != 256 && c.cpr_window != 512 && c.cpr_window != 1024 && c.cpr_window != 2048 && c.cpr_window != 4096)
    return bad("cpr_window must be one of 256,512,1024,2048,4096");
  if (!(c.eq_ridge >= 0)) return bad("eq_ridge must be >= 0");
  if (c.input_dtype != KK_IN_INT16 && c.input_dtype != KK_IN_FLOAT32 && c.input_dtype != KK_IN_UINT8) return bad("input_dtype");
  if (!(c.ref_intensity > 0) || !(c.clamp_rel >= FLT_MIN))
    return bad("ref_intensity must be > 0 and clamp_rel a normal float >= FLT_MIN");
  if (c.max_samples_per_call < kk::kFrameSamp || c.max_samples_per_call % kk::kFrameSamp) return bad("max_samples_per_call must be a positive multiple of 16384");
  auto okM = [](int M) { return M == 4 || M == 8 || M == 16 || M == 32 || M == 64; };
  if (c.format_schedule) {
    if (c.n_segments <= 0 || c.segment_frames <= 0) return bad("schedule needs n_segments > 0 and segment_frames > 0");
    for (int i = 0; i < c.n_segments; ++i) if (!okM(c.format_schedule[i])) return bad("unsupported QAM order in schedule");
  } else if (!okM(c.default_format)) {
    return bad("unsupported QAM order (default_format)");
  }
  if (!(c.lambda_m > 0)) return bad("lambda_m must be > 0");
  if (c.eq_mode != KK_EQ_BLOCK_LS && c.eq_mode != KK_EQ_DDLMS) return bad("eq_mode");
  if (c.static_cd != 0 && c.static_cd != 1) return bad("static_cd must be 0 or 1");
  if (c.eq_mode == KK_EQ_DDLMS) {
    if (c.ddlms_block < 256 || c.ddlms_block > kk::kFrameSym || !is_pow2(c.ddlms_block)) return bad("ddlms_block must be a power of two in [256, 4096]");
    // K2's outermost tiles must read E inside core ± one frame: with Ky = 2·W + 2 (2-sps margin) and
    // keep = mf_fft_n/2 − 512, 2·Ky + 2·keep − 2 + 512 ≤ kFrameSamp (both ends)
    // ⇒ W ≤ 3136 on the 4096/3072 grid, W ≤ 2112 on the 8192/7168 grid
    const int keep = c.mf_fft_n / 2 - 512;
    if (c.ddlms_warmup < 0 || c.ddlms_warmup % 64 ||
        2 * (2 * c.ddlms_warmup + 2) + 2 * keep - 2 + 512 > kk::kFrameSamp)
      return bad("ddlms_warmup must be a multiple of 64 in [0, 3136] (MF 4096) or [0, 2112] (MF 8192)");
    if (!(c.ddlms_mu_warm >= 0) || !(c.ddlms_mu >= 0) || !(c.ddlms_mu_mid >= 0)) return bad("ddlms step sizes must be >= 0");
  }
  return KK_OK;
}

cudaEvent_t take_event(kk_ctx* c) {
  if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// resolve (synchronise + accumulate) the oldest `count` pending timing records
void resolve_timing(kk_ctx* c, size_t count) {
  count = std::min(count, c->ev_pending.size());
  for (size_t i = 0; i < count; ++i) {
    auto& r = c->ev_pending[i];
    cudaEventSynchronize(r[3]);
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, r[k], r[k + 1]) == cudaSuccess) { c->k_ms[k] += ms; c->k_launches[k] += 1; }
    }
    for (auto e : r) c->ev_pool.push_back(e);
  }
  c->ev_pending.erase(c->ev_pending.begin(), c->ev_pending.begin() + count);
}

void free_all(kk_ctx* c) {
  void* ptrs[] = {c->d_H, c->d_Hc, c->d_lo, c->d_wcd, c->d_tw1024, c->d_tw256, c->d_twN, c->d_twI, c->d_tw2048u, c->d_sched,
                  c->d_E, c->d_part, c->d_clamp, c->d_y, c->d_z, c->d_segpow, c->d_counters, c->d_k3rec, c->d_k3th,
                  c->d_in[0], c->d_in[1], c->d_ref[0], c->d_ref[1], c->d_dec[0], c->d_dec[1]};
  for (void* p : ptrs) dfree(c, p);
  c->guards.clear();
  for (auto& r : c->ev_pending) for (auto e : r) cudaEventDestroy(e);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  c->ev_pending.clear();
  c->ev_pool.clear();
  for (int i = 0; i < 2; ++i) {
    if (c->hs[i]) cudaStreamDestroy(c->hs[i]);
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    if (c->entry_ev[i]) cudaEventDestroy(c->entry_ev[i]);
  }
  if (c->order_ev) cudaEventDestroy(c->order_ev);
}

}  // namespace

extern "C" {

void kk_config_default(kk_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->fs_hz = 4e9;
  c->baud_hz = 1e9;
  c->lo_num = 129;
  c->lo_den = 1000;
  c->sideband = 1;
  c->rrc_span_sym = 256;
  c->rolloff = 0.01;
  c->hilbert_n = 1024;
  c->hilbert_hop = 512;
  c->mf_fft_n = 4096;
  c->mf_hop = 3072;
  c->frame_symbols = 4096;
  c->eq_taps = 0;
  c->eq_widely_linear = 1;
  c->cpr_window = 256;
  c->eq_ridge = 1e-3;
  c->dispersion_ps_per_nm = 0.0;
  c->lambda_m = 1550.51e-9;
  c->input_dtype = KK_IN_INT16;
  c->adc_scale = 1.0f;
  c->adc_offset = 0.0f;
  c->ref_intensity = 1.0f;
  c->clamp_rel = 1e-12f;
  c->format_schedule = nullptr;
  c->n_segments = 0;
  c->default_format = 4;
  c->segment_frames = 1;
  c->max_samples_per_call = (int64_t)1 << 24;
  c->device = 0;
  c->keep_intermediate = 0;
  c->eq_mode = KK_EQ_BLOCK_LS;
  c->ddlms_block = 512;
  c->ddlms_warmup = 1024;
  c->debug_guard = 0;
  c->ddlms_mu_warm = 2e-3;
  c->ddlms_mu = 2.5e-4;
  c->ddlms_mu_mid = 5e-4;
  c->static_cd = 0;
  c->upsample = 1;
  c->ref_prbs = 0;
  c->ref_seed = 0;
  c->reserved2 = 0;
}

size_t kk_config_sizeof(void) { return sizeof(kk_config); }
size_t kk_stats_sizeof(void) { return sizeof(kk_stats_t); }

kk_status kk_init(const kk_config* cfg, kk_ctx** out) {
  if (!cfg || !out) return KK_ERR_NULL;
  *out = nullptr;
  std::string why;
  if (validate(*cfg, why) != KK_OK) {
    std::fprintf(stderr, "kk_init: %s\n", why.c_str());
    return KK_ERR_CONFIG;
  }
  const bool ddlms = cfg->eq_mode == KK_EQ_DDLMS;
  const bool scd = !ddlms && cfg->static_cd;  // block LS after the static CD inverse (NEXT-2 arrangement)
  const int L = ddlms ? 3 : scd ? (cfg->eq_taps ? cfg->eq_taps : 5) : tap_rule(*cfg);   // (DDLMS: LS taps unused)
  if (L < 3 || L > 2 * kk::kMaxK + 1 || (L % 2) == 0) {
    std::fprintf(stderr, "kk_init: tap-count rule gives L=%d outside [3,15]\n", L);
    return KK_ERR_CONFIG;
  }
  kk_ctx* c = new kk_ctx();
  c->cfg = *cfg;
  c->device = cfg->device;
  c->L = ddlms ? 4 : L;
  c->K = (L - 1) / 2;
  c->ddlms = ddlms;
  c->Ky = ddlms ? 2 * cfg->ddlms_warmup + 2 : c->K;
  c->mfN = cfg->mf_fft_n;
  c->mfKeep = cfg->mf_fft_n / 2 - 512;
  c->halo = cfg->upsample == 2 ? kk::kHaloUp : kk::kHalo;
  if (cfg->upsample == 2) halfband_odd(c->hb_odd);
  if (cfg->format_schedule) {
    c->schedule.assign(cfg->format_schedule, cfg->format_schedule + cfg->n_segments);
  } else {
    c->schedule.assign(1, (uint8_t)cfg->default_format);
    c->cfg.segment_frames = 1;
  }
  c->cfg.format_schedule = nullptr;   // never keep the caller's pointer
  c->cfg.n_segments = (int)c->schedule.size();

  DeviceGuard g(c->device);
  cudaError_t e = cudaSetDevice(c->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "kk_init: %s\n", cudaGetErrorString(e));
    delete c;
    return KK_ERR_CUDA;
  }

  // ---- fp64 constants
  const std::vector<double> h = rrc_taps(cfg->rolloff, cfg->rrc_span_sym, 4);
  const int half = (int)(h.size() - 1) / 2;
  const int NM = cfg->mf_fft_n;                 // MF grid (4096 or 8192)
  std::vector<float> H(NM);
  for (int k = 0; k < NM; ++k) {
    double s = h[half];
    for (int j = 1; j <= half; ++j) s += 2.0 * h[half + j] * std::cos(2.0 * kPi * (double)((int64_t)k * j % NM) / NM);
    H[k] = (float)(s / NM);
  }
  std::vector<float2> lo(cfg->lo_den);
  for (int q = 0; q < cfg->lo_den; ++q) {
    const double a = -2.0 * kPi * (double)cfg->sideband * (double)q / (double)cfg->lo_den;
    lo[q] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  // paper arrangement: complex static filter H_cd = DFT_NM of h_cd, h_cd = IDFT4096(H_rrc·C) truncated to
  // j = −512..512 (the same definition as oracle.receiver.static_filter_taps: the taps live on the 4096 grid
  // whatever the MF grid), ×1/NM folded in
  std::vector<float2> Hc;
  if (ddlms || scd) {
    const int N = 4096;
    std::vector<double> Hr(N);
    for (int k = 0; k < N; ++k) {
      double s = h[half];
      for (int j = 1; j <= half; ++j) s += 2.0 * h[half + j] * std::cos(2.0 * kPi * (double)((int64_t)k * j % N) / N);
      Hr[k] = s;
    }
    std::vector<double> ct(N), st(N);
    for (int m = 0; m < N; ++m) { ct[m] = std::cos(2.0 * kPi * m / N); st[m] = std::sin(2.0 * kPi * m / N); }
    const double fc = cfg->fs_hz * (double)cfg->lo_num / (double)cfg->lo_den, b2 = beta2L(*cfg);
    std::vector<cd> HC(N);
    for (int k = 0; k < N; ++k) {
      const double nu = (k < N / 2 ? (double)k : (double)(k - N)) * cfg->fs_hz / N;
      const double w = 2.0 * kPi * (nu + (double)cfg->sideband * fc);
      const double ph = -(b2 / 2.0) * w * w;
      HC[k] = Hr[k] * cd(std::cos(ph), std::sin(ph));
    }
    std::vector<cd> hcd(2 * half + 1);
    for (int j = -half; j <= half; ++j) {
      cd acc(0, 0);
      for (int k = 0; k < N; ++k) {
        const int m = (int)(((int64_t)k * (j + N)) % N);
        acc += HC[k] * cd(ct[m], st[m]);
      }
      hcd[j + half] = acc / (double)N;
    }
    Hc.resize(NM);
    for (int k = 0; k < NM; ++k) {
      cd acc(0, 0);
      for (int j = -half; j <= half; ++j) {
        const double a = -2.0 * kPi * (double)(((int64_t)k * (j + NM)) % NM) / (double)NM;
        acc += hcd[j + half] * cd(std::cos(a), std::sin(a));
      }
      acc /= (double)NM;
      Hc[k] = make_float2((float)acc.real(), (float)acc.imag());
    }
  }
  {   // θ₀: the CD-inverse fit referenced to the carrier — the centre spike when K2 already inverts CD
    kk_config c0 = *cfg;
    if (scd) c0.dispersion_ps_per_nm = 0.0;
    c->w_cd = cd_init_taps(c0, L);
  }
  std::vector<float2> wcd(L);
  for (int i = 0; i < L; ++i) wcd[i] = make_float2((float)c->w_cd[i].real(), (float)c->w_cd[i].imag());

  e = cudaSuccess;
  auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  chk(upload(&c->d_H, H));
  if (ddlms || scd) chk(upload(&c->d_Hc, Hc));
  chk(upload(&c->d_lo, lo));
  chk(upload(&c->d_wcd, wcd));
  chk(upload(&c->d_tw1024, twiddles(1024, 32, 32)));
  chk(upload(&c->d_tw256, twiddles(256, 16, 16)));
  // K2 last-pass twiddles: forward W_NM^{r·k} (radix NM/256), inverse W_{NM/2}^{r·k} (radix NM/512), k < 256
  chk(upload(&c->d_twN, twiddles(c->mfN, c->mfN / 256, 256)));
  chk(upload(&c->d_twI, twiddles(c->mfN / 2, c->mfN / 512, 256)));
  if (cfg->upsample == 2) {
    std::vector<float2> t(2048);
    for (int k1 = 0; k1 < 32; ++k1)
      for (int l = 0; l < 64; ++l) {
        const double a = -2.0 * kPi * (double)(l * k1) / 2048.0;
        t[(size_t)k1 * 64 + l] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
    chk(upload(&c->d_tw2048u, t));
  }
  chk(upload(&c->d_sched, c->schedule));

  // ---- scratch
  const int64_t n = cfg->max_samples_per_call;
  c->nmax = n;
  const int64_t nE = n + 2 * kk::kFrameSamp;
  chk(dalloc(c, "E", &c->d_E, (size_t)nE * sizeof(float2)));
  chk(dalloc(c, "part", &c->d_part, (size_t)(nE / kk::kHilbertHop) * sizeof(float2)));
  chk(dalloc(c, "clamp", &c->d_clamp, (size_t)(nE / kk::kHilbertHop) * sizeof(int)));
  chk(dalloc(c, "y", &c->d_y, (size_t)(n / 2 + 2 * c->Ky + 2) * sizeof(float2)));
  if (c->d_y && !kk::k3_encode_ymaps(c->d_y, n / 2 + 2 * c->Ky + 2, c->ymaps) && e == cudaSuccess) e = cudaErrorNotSupported;
  if (cfg->keep_intermediate) chk(dalloc(c, "z", &c->d_z, (size_t)(n / 4) * sizeof(float2)));
  if (!ddlms) {
    chk(dalloc(c, "k3rec", &c->d_k3rec, (size_t)(n / kk::kFrameSamp) * kk::k3_rec_bytes(c->K)));
    chk(dalloc(c, "k3th", &c->d_k3th, (size_t)(n / kk::kFrameSamp) * kk::k3_threc_bytes(c->K)));
  }
  if (ddlms) chk(dalloc(c, "segpow", &c->d_segpow, (size_t)((n / 2 + 2 * c->Ky) / 512 + 2 * (c->mfKeep / 512) + 16) * sizeof(float)));
  chk(dalloc(c, "counters", &c->d_counters, 32 * sizeof(unsigned long long)));
  if (cfg->ref_prbs) {
    chk(dalloc(c, "refgen", &c->d_refgen, (size_t)(n / 4)));
    c->ref_key = cfg->ref_prbs == 2 ? kk::ref_prbs31_w0(cfg->ref_seed) : kk::ref_prbs_key(cfg->ref_seed);
    if (cfg->ref_prbs == 2) chk(kk::ref_prbs31_init());
  }
  chk(cudaMemset(c->d_counters, 0, 32 * sizeof(unsigned long long)));
  if (e == cudaSuccess) {
    const size_t k3 = kk::k3_smem_bytes(c->K);
    if (k3 > 227 * 1024) { std::fprintf(stderr, "kk_init: K3 shared memory too large\n"); free_all(c); delete c; return KK_ERR_CONFIG; }
  }
  if (e != cudaSuccess) {
    std::fprintf(stderr, "kk_init: %s\n", cudaGetErrorString(e));
    const kk_status s = (e == cudaErrorMemoryAllocation) ? KK_ERR_NOMEM : KK_ERR_CUDA;
    free_all(c);
    delete c;
    cudaGetLastError();
    return s;
  }
  *out = c;
  return KK_OK;
}

kk_status kk_halo(const kk_ctx* c, int64_t* left, int64_t* right) {
  if (!c || !left || !right) return KK_ERR_NULL;
  *left = c->halo;
  *right = c->halo;
  return KK_OK;
}

kk_status kk_eq_taps(const kk_ctx* c, int32_t* taps) {
  if (!c || !taps) return KK_ERR_NULL;
  *taps = c->L;
  return KK_OK;
}

// Calls share the context's scratch buffers and counters. A call queued on a different stream than the context's
// previous device call first waits (event) for the work queued there, so callers need not synchronise when they
// switch streams. The host path's staging streams are exempt: it orders its own sub-calls and synchronises both
// streams before it returns.
static void order_after_last(kk_ctx* c, cudaStream_t s) {
  if (!c->have_stream || s == c->last_stream) return;
  if (c->last_stream != nullptr && (c->last_stream == c->hs[0] || c->last_stream == c->hs[1])) return;
  if (!c->order_ev && cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming) != cudaSuccess) return;
  if (cudaEventRecord(c->order_ev, c->last_stream) == cudaSuccess) cudaStreamWaitEvent(s, c->order_ev, 0);
  else (void)cudaGetLastError();   // e.g. the caller destroyed that stream: not an error of this call
}
static void set_last(kk_ctx* c, cudaStream_t s) { c->last_stream = s; c->have_stream = true; }

kk_status kk_process_frames(kk_ctx* c, const void* d_adc, int64_t first, int64_t n, const uint8_t* d_ref,
                            uint8_t* d_dec, kk_stream_t stream) {
  return kk_process_frames_ex(c, d_adc, first, n, d_ref, d_dec, nullptr, stream);
}

kk_status kk_process_frames_ex(kk_ctx* c, const void* d_adc, int64_t first, int64_t n, const uint8_t* d_ref,
                               uint8_t* d_dec, uint32_t* d_ferr, kk_stream_t stream) {
  NvtxRange call_("kk_process_frames");
  if (!c || !d_adc) return fail(c, KK_ERR_NULL, "kk_process_frames: NULL ctx or input");
  if (n < kk::kFrameSamp) return fail(c, KK_ERR_SHORT, "kk_process_frames: n_samples < one frame");
  if (first < 0 || first % kk::kFrameSamp || n % kk::kFrameSamp)
    return fail(c, KK_ERR_ALIGN, "kk_process_frames: first_sample/n_samples not multiples of 16384");
  if (n > c->nmax) return fail(c, KK_ERR_CONFIG, "kk_process_frames: n_samples > max_samples_per_call");
  if (reinterpret_cast<uintptr_t>(d_adc) % 16) return fail(c, KK_ERR_ALIGN, "kk_process_frames: input not 16-B aligned");
  DeviceGuard g(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  order_after_last(c, s);
  const kk_config& cf = c->cfg;
  const size_t esz = cf.input_dtype == KK_IN_FLOAT32 ? 4 : cf.input_dtype == KK_IN_UINT8 ? 1 : 2;
  const int F = kk::kFrameSamp;
  if (!d_ref && cf.ref_prbs) {                   // the transmitter's known labels, generated on the device
    NvtxRange r_("kk::ref_prbs");
    if (cf.ref_prbs == 2)
      kk::launch_ref_prbs31(c->d_refgen, first / 4, n / 4, c->ref_key, c->d_sched, cf.n_segments, cf.segment_frames, s);
    else
      kk::launch_ref_prbs(c->d_refgen, first / 4, n / 4, c->ref_key, c->d_sched, cf.n_segments, cf.segment_frames, s);
    d_ref = c->d_refgen;
  }

  // K1 over blocks [ (first − F)/512, (first + n + F)/512 )
  const int64_t jb0 = (first - F) / kk::kHilbertHop;
  const int64_t nblk = (n + 2 * F) / kk::kHilbertHop;
  kk::K1Params p1;
  p1.adc_scale = cf.adc_scale;
  p1.adc_offset = cf.adc_offset;
  p1.inv_iref = 1.0f / cf.ref_intensity;
  p1.clamp_rel = cf.clamp_rel;
  p1.half_ln_iref = (float)(0.5 * std::log((double)cf.ref_intensity));
  p1.sideband = (float)cf.sideband;
  const char* adc0 = static_cast<const char*>(d_adc) - (int64_t)kk::kHalo * (int64_t)esz;
  kk::K1UParams pu;
  if (cf.upsample == 2) {
    pu.adc_scale = p1.adc_scale;
    pu.adc_offset = p1.adc_offset;
    pu.inv_iref = p1.inv_iref;
    pu.clamp_rel = p1.clamp_rel;
    pu.half_ln_iref = p1.half_ln_iref;
    pu.sideband = p1.sideband;
    for (int i = 0; i < 8; ++i) { pu.c[i] = (float)c->hb_odd[i]; pu.c2[i] = (float)(2.0 * c->hb_odd[i]); }
  }
  std::array<cudaEvent_t, 4> tev{};
  if (c->timing) {
    if (c->ev_pending.size() >= 512) resolve_timing(c, 256);
    for (auto& e : tev) e = take_event(c);
    cudaEventRecord(tev[0], s);
  }
  if (cf.upsample == 2) {
    NvtxRange r_("kk::K1U KK front end + Hilbert (8 sps)");
    kk::launch_k1u(static_cast<const char*>(d_adc) - (int64_t)kk::kHaloUp * (int64_t)esz, cf.input_dtype, nblk,
                   c->d_E, c->d_part, c->d_clamp, c->d_tw2048u, pu, s);
  } else {
    NvtxRange r_("kk::K1 KK front end + Hilbert");
    kk::launch_k1(adc0, cf.input_dtype, nblk / 2, c->d_E, c->d_part, c->d_clamp, c->d_tw1024, p1, s);
  }

  // K2 over the MF tiles covering y[first/2 − K, (first + n)/2 + K)
  const int64_t y_first = first / 2 - c->Ky;
  const int64_t y_count = n / 2 + 2 * c->Ky;
  auto fdiv = [](int64_t a, int64_t b) { int64_t q = a / b; return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q; };
  const int64_t t_lo = fdiv(y_first, c->mfKeep);
  const int64_t t_hi = fdiv(y_first + y_count - 1, c->mfKeep);
  if (c->timing) cudaEventRecord(tev[1], s);
  kk::K2Params p2{};
  p2.lo_num = cf.lo_num;
  p2.lo_den = cf.lo_den;
  p2.seg_pow = c->d_segpow;
  p2.seg_first = t_lo * (c->mfKeep / 512);
  {
    // ρ^r = LO[(r·stepJ) mod lo_den], stepJ = (NF/16)·lo_num: the LO advance between a pass-1 thread's samples
    // (the same fp64 formula as the LO table, so ρ^r equals the table entry)
    const int64_t stepJ = ((int64_t)(c->mfN / 16) * cf.lo_num) % cf.lo_den;
    for (int r = 0; r < 16; ++r) {
      const int64_t q = ((int64_t)r * stepJ) % cf.lo_den;
      const double a = -2.0 * kPi * (double)cf.sideband * (double)q / (double)cf.lo_den;
      p2.rho[r] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  }
  {
    NvtxRange r2_("kk::K2 carrier removal + mixer + MF + decimation");
    kk::launch_k2(c->mfN, c->d_E, first - F, c->d_part, c->d_clamp, jb0, t_lo, t_hi - t_lo + 1, c->d_y, y_first,
                  y_count, c->d_H, c->d_Hc, c->d_lo, c->d_tw256, c->d_twN, c->d_twI, p2, c->num_sms, s);
  }

  if (c->timing) cudaEventRecord(tev[2], s);
  // K3 one CTA per frame
  kk::K3Params p3;
  p3.schedule = c->d_sched;
  p3.n_segments = cf.n_segments;
  p3.segment_frames = cf.segment_frames;
  p3.ridge = (float)cf.eq_ridge;
  p3.widely_linear = cf.eq_widely_linear;
  p3.cpr_window = cf.cpr_window;
  p3.p0_min = (float)(1e-20 * cf.ref_intensity);
  p3.frame_err = d_ref ? d_ferr : nullptr;
  for (int i = 0; i < 15; ++i)
    p3.w_cd[i] = (i < (int)c->w_cd.size()) ? make_float2((float)c->w_cd[i].real(), (float)c->w_cd[i].imag())
                                           : make_float2(0.f, 0.f);
  const int64_t nfr = n / F;
  if (c->ddlms) {
    kk::K3DParams pd;
    pd.seg_pow = c->d_segpow;
    pd.seg_first = p2.seg_first;
    pd.schedule = c->d_sched;
    pd.n_segments = cf.n_segments;
    pd.segment_frames = cf.segment_frames;
    pd.mu_warm = (float)cf.ddlms_mu_warm;
    pd.mu = (float)cf.ddlms_mu;
    pd.mu_mid = (float)cf.ddlms_mu_mid;
    pd.widely_linear = cf.eq_widely_linear;
    pd.frame_err = d_ref ? d_ferr : nullptr;
    if (pd.frame_err) cudaMemsetAsync(pd.frame_err, 0, (size_t)(n / F) * 2 * sizeof(uint32_t), s);
    NvtxRange r3_("kk::K3' DDLMS");
    kk::launch_k3_ddlms(c->d_y, c->Ky, first / 4, n / 4 / cf.ddlms_block, cf.ddlms_block, cf.ddlms_warmup,
                        c->d_clamp, (int64_t)F / kk::kHilbertHop, d_ref, d_dec,
                        cf.keep_intermediate ? c->d_z : nullptr, c->d_counters, pd, s);
  } else {
    NvtxRange r3_("kk::K3 block-LS EQ + CPR + decisions");
    kk::launch_k3(c->d_y, first / F, nfr, c->K, c->d_wcd, c->d_clamp, (int64_t)F / kk::kHilbertHop /*skip frame −1*/,
                  d_ref, d_dec, cf.keep_intermediate ? c->d_z : nullptr, c->d_counters, p3, c->ymaps, c->d_k3rec,
                  c->d_k3th, c->num_sms, s);
  }
  if (c->timing) {
    cudaEventRecord(tev[3], s);
    c->ev_pending.push_back(tev);
  }
  cudaError_t e = cudaGetLastError();
  c->have_call = true;
  c->last_first = first;
  c->last_n = n;
  c->last_z = cf.keep_intermediate != 0;
  set_last(c, s);
  if (e != cudaSuccess) return fail(c, KK_ERR_CUDA, std::string("kk_process_frames: launch: ") + cudaGetErrorString(e));
  return KK_OK;
}

kk_status kk_process_frames_host(kk_ctx* c, const void* h_adc, int64_t first, int64_t n, const uint8_t* h_ref,
                                 uint8_t* h_dec) {
  NvtxRange call_("kk_process_frames_host");
  if (!c || !h_adc) return fail(c, KK_ERR_NULL, "kk_process_frames_host: NULL ctx or input");
  if (n < kk::kFrameSamp) return fail(c, KK_ERR_SHORT, "kk_process_frames_host: n_samples < one frame");
  if (first < 0 || first % kk::kFrameSamp || n % kk::kFrameSamp)
    return fail(c, KK_ERR_ALIGN, "kk_process_frames_host: first_sample/n_samples not multiples of 16384");
  DeviceGuard g(c->device);
  const size_t esz = c->cfg.input_dtype == KK_IN_FLOAT32 ? 4 : c->cfg.input_dtype == KK_IN_UINT8 ? 1 : 2;
  const int64_t H = c->halo;
  // staging granularity: ≤ 2^26 samples per transfer so that copies and kernels of consecutive sub-calls
  // overlap on the two streams even when the context was sized for much larger device calls
  const int64_t hc = std::min<int64_t>(c->nmax, (int64_t)1 << 26);
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  for (int i = 0; i < 2; ++i) {
    if (!c->d_in[i]) chk(dalloc(c, "host_in", &c->d_in[i], (size_t)(hc + 2 * H) * esz));
    if (!c->d_ref[i]) chk(dalloc(c, "host_ref", &c->d_ref[i], (size_t)(hc / 4)));
    if (!c->d_dec[i]) chk(dalloc(c, "host_dec", &c->d_dec[i], (size_t)(hc / 4)));
    if (!c->hs[i]) chk(cudaStreamCreateWithFlags(&c->hs[i], cudaStreamNonBlocking));
    if (!c->ev[i]) chk(cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
    if (!c->entry_ev[i]) chk(cudaEventCreateWithFlags(&c->entry_ev[i], cudaEventDisableTiming));
  }
  if (e != cudaSuccess) return fail(c, e == cudaErrorMemoryAllocation ? KK_ERR_NOMEM : KK_ERR_CUDA, cudaGetErrorString(e));
  // The staging streams are non-blocking: order them after work still in flight on the legacy default stream
  // (e.g. kk_reset_stats(ctx, NULL)) and on the stream of the context's last device call (kk_process_frames /
  // kk_reset_stats on a caller stream), which share the scratch buffers and the counters with this call.
  chk(cudaEventRecord(c->entry_ev[0], cudaStreamLegacy));
  const bool own_last = c->last_stream == nullptr || c->last_stream == c->hs[0] || c->last_stream == c->hs[1];
  if (!own_last) chk(cudaEventRecord(c->entry_ev[1], c->last_stream));
  for (int i = 0; i < 2; ++i) {
    chk(cudaStreamWaitEvent(c->hs[i], c->entry_ev[0], 0));
    if (!own_last) chk(cudaStreamWaitEvent(c->hs[i], c->entry_ev[1], 0));
  }
  const char* src = static_cast<const char*>(h_adc);
  int64_t done = 0;
  int k = 0;
  while (done < n && e == cudaSuccess) {
    const int64_t nc = std::min<int64_t>(hc, n - done);
    const int b = k & 1;
    cudaStream_t s = c->hs[b];
    chk(cudaMemcpyAsync(c->d_in[b], src + (done - H) * (int64_t)esz, (size_t)(nc + 2 * H) * esz, cudaMemcpyHostToDevice, s));
    if (h_ref) chk(cudaMemcpyAsync(c->d_ref[b], h_ref + done / 4, (size_t)(nc / 4), cudaMemcpyHostToDevice, s));
    if (k > 0) chk(cudaStreamWaitEvent(s, c->ev[b ^ 1], 0));   // scratch is shared: kernels in order
    const kk_status st = kk_process_frames(c, static_cast<char*>(c->d_in[b]) + H * (int64_t)esz, first + done, nc,
                                           h_ref ? c->d_ref[b] : nullptr, c->d_dec[b], s);
    if (st != KK_OK) return st;
    chk(cudaEventRecord(c->ev[b], s));
    if (h_dec) chk(cudaMemcpyAsync(h_dec + done / 4, c->d_dec[b], (size_t)(nc / 4), cudaMemcpyDeviceToHost, s));
    done += nc;
    ++k;
  }
  chk(cudaStreamSynchronize(c->hs[0]));
  chk(cudaStreamSynchronize(c->hs[1]));
  set_last(c, c->hs[(k - 1) & 1]);
  if (e != cudaSuccess) return fail(c, KK_ERR_CUDA, std::string("kk_process_frames_host: ") + cudaGetErrorString(e));
  return KK_OK;
}

kk_status kk_stats(kk_ctx* c, kk_stats_t* out) {
  if (!c || !out) return KK_ERR_NULL;
  DeviceGuard g(c->device);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long buf[32];
  if (e == cudaSuccess) e = cudaMemcpy(buf, c->d_counters, sizeof(buf), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(c, KK_ERR_CUDA, std::string("kk_stats: ") + cudaGetErrorString(e));
  static_assert(sizeof(kk_stats_t) == KK_STATS_WORDS * 8, "kk_stats_t layout");
  std::memcpy(out, buf, sizeof(kk_stats_t));
  return KK_OK;
}

kk_status kk_stats_device(kk_ctx* c, uint64_t* d_out, kk_stream_t stream) {
  if (!c || !d_out) return KK_ERR_NULL;
  DeviceGuard g(c->device);
  order_after_last(c, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaMemcpyAsync(d_out, c->d_counters, KK_STATS_WORDS * 8, cudaMemcpyDeviceToDevice,
                                  static_cast<cudaStream_t>(stream));
  set_last(c, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KK_OK : fail(c, KK_ERR_CUDA, cudaGetErrorString(e));
}

kk_status kk_reset_stats(kk_ctx* c, kk_stream_t stream) {
  if (!c) return KK_ERR_NULL;
  DeviceGuard g(c->device);
  order_after_last(c, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaMemsetAsync(c->d_counters, 0, 32 * sizeof(unsigned long long), static_cast<cudaStream_t>(stream));
  set_last(c, static_cast<cudaStream_t>(stream));               // later calls (and the host path) order after it
  return e == cudaSuccess ? KK_OK : fail(c, KK_ERR_CUDA, cudaGetErrorString(e));
}

kk_status kk_intermediate_range(const kk_ctx* c, int stage, int64_t* first_index, int64_t* count) {
  if (!c || !first_index || !count) return KK_ERR_NULL;
  if (!c->have_call) return KK_ERR_STATE;
  const int64_t f = c->last_first, n = c->last_n;
  switch (stage) {
    case KK_STAGE_FIELD: *first_index = f - kk::kFrameSamp; *count = n + 2 * kk::kFrameSamp; return KK_OK;
    case KK_STAGE_MF: *first_index = f / 2 - c->Ky; *count = n / 2 + 2 * c->Ky; return KK_OK;
    case KK_STAGE_EQ:
      if (!c->last_z) return KK_ERR_STATE;
      *first_index = f / 4; *count = n / 4; return KK_OK;
    default: return KK_ERR_CONFIG;
  }
}

kk_status kk_get_intermediate(kk_ctx* c, int stage, void* d_dst, size_t bytes, kk_stream_t stream) {
  if (!c || !d_dst) return KK_ERR_NULL;
  int64_t first = 0, count = 0;
  kk_status st = kk_intermediate_range(c, stage, &first, &count);
  if (st != KK_OK) return st;
  if (bytes < (size_t)count * 8) return fail(c, KK_ERR_CONFIG, "kk_get_intermediate: destination too small");
  const void* src = stage == KK_STAGE_FIELD ? (const void*)c->d_E : stage == KK_STAGE_MF ? (const void*)c->d_y : (const void*)c->d_z;
  DeviceGuard g(c->device);
  order_after_last(c, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaMemcpyAsync(d_dst, src, (size_t)count * 8, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
  set_last(c, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KK_OK : fail(c, KK_ERR_CUDA, cudaGetErrorString(e));
}

kk_status kk_enable_timing(kk_ctx* c, int enable) {
  if (!c) return KK_ERR_NULL;
  c->timing = enable != 0;
  return KK_OK;
}

kk_status kk_kernel_times(kk_ctx* c, double ms_out[3], int64_t launches_out[3], int reset) {
  if (!c || !ms_out || !launches_out) return KK_ERR_NULL;
  DeviceGuard g(c->device);
  resolve_timing(c, c->ev_pending.size());
  for (int k = 0; k < 3; ++k) { ms_out[k] = c->k_ms[k]; launches_out[k] = c->k_launches[k]; }
  if (reset) for (int k = 0; k < 3; ++k) { c->k_ms[k] = 0; c->k_launches[k] = 0; }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? KK_OK : fail(c, KK_ERR_CUDA, cudaGetErrorString(e));
}

kk_status kk_q_from_ber(double ber, double* q_db) {
  if (!q_db) return KK_ERR_NULL;
  if (!(ber > 0.0 && ber < 0.5)) return KK_ERR_DOMAIN;
  // erfcinv(2·BER) by Newton on erfc(x) = 2·BER (erfc is monotone, convex on x > 0)
  const double target = 2.0 * ber;
  double x = 0.5;
  for (int it = 0; it < 200; ++it) {
    const double f = std::erfc(x) - target;
    const double df = -2.0 / std::sqrt(kPi) * std::exp(-x * x);
    const double step = f / df;
    x -= step;
    if (std::fabs(step) < 1e-15 * std::fabs(x)) break;
  }
  *q_db = 20.0 * std::log10(std::sqrt(2.0) * x);
  return KK_OK;
}

void kk_destroy(kk_ctx* c) {
  if (!c) return;
  {
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    free_all(c);
  }
  delete c;
}

kk_status kk_check_guards(kk_ctx* c, int32_t* n_checked) {
  if (!c) return KK_ERR_NULL;
  if (n_checked) *n_checked = 0;
  if (!c->cfg.debug_guard) return KK_OK;
  DeviceGuard g(c->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(c, KK_ERR_CUDA, std::string("kk_check_guards: ") + cudaGetErrorString(e));
  std::vector<unsigned char> h(kGuardBytes);
  int32_t n = 0;
  for (const auto& r : c->guards) {
    for (int side = 0; side < 2; ++side) {
      const unsigned char* zone = side ? r.base + kGuardBytes + r.bytes : r.base;
      e = cudaMemcpy(h.data(), zone, kGuardBytes, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return fail(c, KK_ERR_CUDA, std::string("kk_check_guards: ") + cudaGetErrorString(e));
      for (size_t i = 0; i < kGuardBytes; ++i)
        if (h[i] != kGuardByte) {
          // offset of the corrupted byte relative to the buffer start (negative: before it)
          const long long off = side ? (long long)(r.bytes + i) : (long long)i - (long long)kGuardBytes;
          return fail(c, KK_ERR_STATE, std::string("kk_check_guards: out-of-bounds write into buffer '") + r.name +
                                           "' at byte offset " + std::to_string(off) + " (size " +
                                           std::to_string(r.bytes) + ")");
        }
    }
    ++n;
  }
  if (n_checked) *n_checked = n;
  return KK_OK;
}

const char* kk_strerror(kk_status s) {
  switch (s) {
    case KK_OK: return "ok";
    case KK_ERR_CONFIG: return "invalid or unsupported configuration";
    case KK_ERR_ALIGN: return "misaligned sample range or pointer";
    case KK_ERR_SHORT: return "fewer samples than one frame";
    case KK_ERR_NULL: return "null pointer";
    case KK_ERR_NOMEM: return "device allocation failed";
    case KK_ERR_CUDA: return "CUDA error";
    case KK_ERR_DOMAIN: return "BER outside (0, 0.5): Q undefined";
    case KK_ERR_STATE: return "call out of order";
    default: return "unknown status";
  }
}

const char* kk_last_error(const kk_ctx* c) { return c ? c->err.c_str() : ""; }

}  // extern "C"
