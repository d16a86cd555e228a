// kk_params.h — plain-old-data launch parameters and launch wrappers shared by the host library and
// the kernels (no torch, no CUDA types beyond cudaStream_t / float2).
#pragma once
#include <cstdint>
#include <cuda.h>             // CUtensorMap (K3's swizzled frame loads)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

namespace kk {

constexpr int kHilbertN = 1024;      // PAPER.md:82 "1024-point"
constexpr int kHilbertHop = 512;     // R1: 100 % overlap of the hop, central 512 kept
constexpr int kHilbertLead = 256;    // (N − hop)/2 discarded at each block end
constexpr int kFrameSym = 4096;      // R23
constexpr int kFrameSamp = 16384;
constexpr int kMfN = 4096;           // R6: FFT4096 → ×H → fold → IFFT2048
constexpr int kMfHop = 3072;
constexpr int kMfLead = 512;         // input of tile t starts at 3072 t − 512
constexpr int kMfKeep0 = 256;        // IFFT2048 outputs kept: [256, 1792)
constexpr int kMfKeep = 1536;
constexpr int kHalo = kFrameSamp + kHilbertLead;   // 16640
constexpr int kK1uPad = kHilbertLead + 16;   // K1U staging lead: half window + half-band reach (16-B aligned)
constexpr int kHaloUp = kFrameSamp + kK1uPad;  // 16656 (upsample = 2)
constexpr int kMaxK = 7;             // L = 2K + 1 ≤ 15 (one real-system row per lane: 2L ≤ 32)
constexpr int kNumCounters = 24;     // kk_stats_t layout

struct K1Params {
  float adc_scale, adc_offset;       // I = scale·(code − offset)
  float inv_iref;                    // 1/I_ref
  float clamp_rel;                   // ε / I_ref
  float half_ln_iref;                // ½·ln I_ref
  float sideband;                    // ±1
};

struct K1UParams {                  // K1 + 2× upsampling (DESIGN.md §3 "KK upsampling")
  float adc_scale, adc_offset;
  float inv_iref;
  float clamp_rel;
  float half_ln_iref;
  float sideband;
  float c[8];                        // odd half-band taps f[1], f[3], …, f[15] (decimation)
  float c2[8];                       // 2·c (interpolation)
};

struct K2Params {
  int lo_num, lo_den;
  float2 rho[16];                    // LO step between a pass-1 thread's samples r and 0: LO[(r·(NF/16)·lo_num) mod lo_den]
  float* seg_pow;                    // DDLMS mode (CH): Σ|y[2n]|² per 256-symbol segment (global y/512 grid)
  int64_t seg_first;                 // global segment index of seg_pow[0]
};

struct K3Params {
  const uint8_t* schedule;           // device, n_segments entries
  int n_segments;
  int64_t segment_frames;
  float ridge;
  int widely_linear;
  int cpr_window;                    // symbols
  float p0_min;                      // AGC power at or below which a frame is silent (bad; z = 0): 1e-20·I_ref
  unsigned* frame_err;               // nullable: [2f] symbol errors, [2f+1] bit errors per local frame
  float2 w_cd[15];                   // θ₀'s CD taps by value (kernel-parameter space: uniform operands, no registers)
};

struct K3DParams {
  const float* seg_pow;              // from K2: Σ|y[2n]|² per 256-symbol segment
  int64_t seg_first;                 // global segment index of seg_pow[0]
  const uint8_t* schedule;
  int n_segments;
  int64_t segment_frames;
  float mu_warm, mu, mu_mid;         // μ: first half of the warm-up, kept symbols, second half of the warm-up
  int widely_linear;
  unsigned* frame_err;               // nullable, zeroed by the host before the launch
};

// K1: KK front end + Hilbert + field; one warp per pair of 512-blocks, 8 warps per CTA.
void launch_k1(const void* adc_cta0, int input_dtype, int64_t n_pairs, float2* E, float2* part, int* clampcnt,
               const float2* tw1024, const K1Params& p, cudaStream_t s);
// K1U: K1 with 2× KK upsampling; one warp per pair of 512-blocks, 4 warps per CTA (n_blocks % 8 == 0).
void launch_k1u(const void* adc_cta0, int input_dtype, int64_t n_blocks, float2* E, float2* part, int* clampcnt,
                const float2* tw2048u, const K1UParams& p, cudaStream_t s);
// K2: carrier removal + mixer + RRC MF + decimation by 2 on the global tile grid (nf = 4096 or 8192:
// FFT size; hop nf − 1024, nf/2 − 512 kept 2-sps outputs per tile). twN: W_nf^{r·k} [r][k < 256];
// twI: W_{nf/2}^{r·k} [r][k < 256].
void launch_k2(int nf, const float2* E, int64_t E_first, const float2* part, const int* clampcnt, int64_t jb0,
               int64_t tile0, int64_t n_tiles, float2* y, int64_t y_first, int64_t y_count, const float* Hs,
               const float2* Hc, const float2* lo_tab, const float2* tw256, const float2* twN,
               const float2* twI, const K2Params& p, int num_sms, cudaStream_t s);
// K3: per-frame widely-linear DD-LS equalizer, CPR, decisions, counters — three launches (K3a sums, K3s batched
// solves, K3c pass 2 / CPR / decisions). ymaps: the two tensor maps of y from k3_encode_ymaps (used for K ≤ 4);
// rec / threc: n_frames records of k3_rec_bytes(K) / k3_threc_bytes(K) bytes (scratch).
void launch_k3(const float2* y, int64_t frame0, int64_t n_frames, int K, const float2* w_cd, const int* clampcnt,
               int64_t clamp_frame_off, const uint8_t* ref, uint8_t* dec, float2* z, unsigned long long* counters,
               const K3Params& p, const CUtensorMap* ymaps, double* rec, float2* threc, int num_sms, cudaStream_t s);
size_t k3_rec_bytes(int K);
size_t k3_threc_bytes(int K);
bool k3_encode_ymaps(const float2* y, int64_t n_float2, CUtensorMap* maps);

// Reference labels of the synthetic transmitter for global symbols [sym0, sym0 + n_sym) (kk_config.ref_prbs).
uint32_t ref_prbs_key(uint32_t seed);
void launch_ref_prbs(uint8_t* out, int64_t sym0, int64_t n_sym, uint32_t key, const uint8_t* schedule,
                     int n_segments, int64_t segment_frames, cudaStream_t s);
// ITU-T O.150 PRBS-31 labels (kk_config.ref_prbs = 2): init once (constant-memory jump matrices), then launch.
uint32_t ref_prbs31_w0(uint32_t seed);
cudaError_t ref_prbs31_init();
void launch_ref_prbs31(uint8_t* out, int64_t sym0, int64_t n_sym, uint32_t w0, const uint8_t* schedule,
                       int n_segments, int64_t segment_frames, cudaStream_t s);

// K3 (paper arrangement): 4-tap T/2-spaced widely-linear DDLMS, one thread per restart block.
void launch_k3_ddlms(const float2* y, int64_t y_base, int64_t sym_first, int64_t n_blocks, int B, int W,
                     const int* clampcnt, int64_t clamp_frame_off, const uint8_t* ref, uint8_t* dec, float2* z,
                     unsigned long long* counters, const K3DParams& p, cudaStream_t s);

}  // namespace kk
