/*
 * kkrx.h — C ABI of libkkrx.so, the B200 (sm_100a) Kramers-Kronig receive chain.
 *
 * What the library computes (§2 "DSP chain", Fig. 1b; BASELINE.json north_star;
 * readings R1–R27 of SURVEY.md §8(c), restated in DESIGN.md §3): from int16 ADC codes of a
 * minimum-phase KK photocurrent sampled at 4 GS/s it recovers
 *     a = ½ ln max(I, ε)            sqrt/log front end
 *     φ = σ·H[a]                     1024-pt 50 %-hop overlap-save Hilbert FFT pair (R1, R2)
 *     E = √max(I,ε)·e^{iφ}           field reconstruction
 *     b = (E − A_f)·e^{−2πiσ f_c n/f_s}   carrier removal + downshift (north_star; R8, R9)
 *     y[m] = Σ h[j] b[2m−j]          RRC 1 % matched filter at 2 sps via FFT4096/fold/IFFT2048 (R4–R6)
 *     per 4096-symbol frame: widely-linear block-adaptive FIR absorbing CD (DD least squares),
 *     carrier-phase recovery, QAM decision, bit/symbol error counting (north_star; R10–R27)
 * Q = 20·log10(√2·erfcinv(2·BER)) is computed on the host by kk_q_from_ber.
 *
 * Conventions
 *  - Global indices: sample n (int64, 4 GS/s), symbol k = n/4 (sample 4k is the centre of symbol k),
 *    frame f = samples [16384 f, 16384 f + 16384). All block/tile/frame grids are anchored at n = 0,
 *    so any chunking or sharding of a stream gives bit-identical decisions.
 *  - Device pointers are plain CUDA device addresses (e.g. torch.Tensor.data_ptr()). The caller owns
 *    every buffer passed in; the context owns its constants, scratch and counters. The library never
 *    frees caller memory. Buffers must stay valid until the stream passes the call.
 *  - Every call returns a kk_status; nothing throws across the ABI. Asynchronous kernel faults are
 *    reported at the next synchronising call (kk_stats) as KK_ERR_CUDA.
 *  - Calls on one context are not re-entrant (one host thread at a time). They may be queued on different
 *    streams without synchronisation: a call on another stream than the context's previous device call first
 *    waits (CUDA event) for the work queued there, since the calls share the context's scratch and counters
 *    (a caller that destroys that stream first must synchronise it: its pending work can no longer be waited on).
 */
#ifndef KKRX_H
#define KKRX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kk_ctx kk_ctx;          /* opaque */
typedef void* kk_stream_t;             /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  KK_OK = 0,
  KK_ERR_CONFIG = -1,   /* invalid or unsupported configuration            */
  KK_ERR_ALIGN = -2,    /* first_sample / n_samples not on the frame grid, or pointer not 16-B aligned */
  KK_ERR_SHORT = -3,    /* n_samples < one frame (SPEC.md:307 analogue)                               */
  KK_ERR_NULL = -4,     /* required pointer is NULL                                                   */
  KK_ERR_NOMEM = -5,    /* device allocation failed                                                   */
  KK_ERR_CUDA = -6,     /* CUDA launch / runtime error (sticky errors surface at kk_stats)            */
  KK_ERR_DOMAIN = -7,   /* kk_q_from_ber outside 0 < BER < 0.5                           */
  KK_ERR_STATE = -8     /* call out of order (e.g. intermediate not kept / no call yet)               */
} kk_status;

enum { KK_IN_INT16 = 0, KK_IN_FLOAT32 = 1, KK_IN_UINT8 = 2 };  /* input_dtype */
enum { KK_EQ_BLOCK_LS = 0, KK_EQ_DDLMS = 1 };                 /* eq_mode */
enum { KK_STAGE_FIELD = 0, KK_STAGE_MF = 1, KK_STAGE_EQ = 2 }; /* kk_get_intermediate stages */

/* Receiver configuration. kk_config_default() fills the paper's values; fields marked [fixed] must
 * keep them (the kernels are specialised for them) or kk_init returns KK_ERR_CONFIG. */
typedef struct kk_config {
  double  fs_hz;                 /* 4e9  ADC rate; fs/baud must be 4 [fixed]              */
  double  baud_hz;               /* 1e9  symbol rate                                       */
  int32_t lo_num, lo_den;        /* f_c/f_s as a reduced rational: 129/1000 = 0.516 GHz / 4 GS/s; den ≤ 4096 */
  int32_t sideband;              /* +1: data above the tone (φ = +H[a]); −1 mirrors φ and the LO (R2)   */
  int32_t rrc_span_sym;          /* 256 → 1025 taps (R4); span·4 ≤ mf_fft_n − mf_hop                    */
  double  rolloff;               /* 0.01 ("1% roll-off")                                     */
  int32_t hilbert_n, hilbert_hop;/* 1024, 512 [fixed] ("1024-point 100% overlap-save"; R1)  */
  int32_t mf_fft_n, mf_hop;      /* 4096, 3072 (default: FFT4096 → fold → IFFT2048; R6) or 8192, 7168 (same exact
                                  * convolution on a larger overlap-save grid; DDLMS warm-up ≤ 2112)      */
  int32_t frame_symbols;         /* 4096 [fixed] (R23)                                                   */
  int32_t eq_taps;               /* 0 = tap-count rule of SURVEY §8(a); else odd L in [3, 15]           */
  int32_t eq_widely_linear;      /* 1 = widely linear ("widely-linear"), 0 = linear only    */
  int32_t cpr_window;            /* 256 symbols; one of 256, 512, 1024, 2048, 4096 (R12; whole 256-blocks)   */
  double  eq_ridge;              /* 1e-3: λ = ridge·tr(R)/(2L) (R10)                                     */
  double  dispersion_ps_per_nm;  /* accumulated D·L, e.g. 200000 for 10,000 km at 20 ps/nm/km          */
  double  lambda_m;              /* 1550.51e-9                                             */
  int32_t input_dtype;           /* KK_IN_INT16 / KK_IN_UINT8 (ADC codes) | KK_IN_FLOAT32 (intensities) */
  float   adc_scale, adc_offset; /* I = adc_scale·(code − adc_offset)                                    */
  float   ref_intensity;         /* I_ref > 0; ε = clamp_rel·I_ref (R7)                                  */
  float   clamp_rel;             /* 1e-12; a normal float (>= FLT_MIN), else kk_init fails               */
  const uint8_t* format_schedule;/* host array of n_segments QAM orders in {4,8,16,32,64}; NULL → default_format */
  int32_t n_segments;            /* entries in format_schedule (copied at kk_init)                       */
  int32_t default_format;        /* M when format_schedule is NULL                                       */
  int64_t segment_frames;        /* frames per schedule entry; format(f) = schedule[(f/segment_frames) mod n_segments] (R26) */
  int64_t max_samples_per_call;  /* sizes the scratch; multiple of 16384                                 */
  int32_t device;                /* CUDA device ordinal the context lives on                             */
  int32_t keep_intermediate;     /* 1: K3 also stores z (EQ stage) for kk_get_intermediate               */
  /* Equalizer mode. KK_EQ_BLOCK_LS (default, BASELINE north star): RRC static filter + per-frame widely-linear
   * block-adaptive FIR absorbing CD + CPR. KK_EQ_DDLMS (the paper's arrangement):
   * static filter = RRC × CD inverse (the "offline-optimized filter"), then the 4-tap T/2-spaced widely-linear
   * DDLMS, restarted every ddlms_block symbols after ddlms_warmup warm-up symbols (global grid). */
  int32_t eq_mode;
  int32_t ddlms_block;           /* 256 … 4096, power of two (kept symbols per restart; default 512)     */
  int32_t ddlms_warmup;          /* 0 … 3136, multiple of 64 (default 1024): warm-up from the centre spike */
  int32_t debug_guard;           /* 1: surround every device scratch buffer with 64 KiB canaries (kk_check_guards) */
  double  ddlms_mu_warm;         /* 2e-3 step size over the first half of the warm-up (then ddlms_mu_mid) */
  double  ddlms_mu;              /* 2.5e-4 step size on kept symbols                                     */
  /* KK upsampling (SPEC S:277 upsample_factor; DESIGN.md §3 "KK upsampling"):
   * 1 = the paper's chain (KK at the ADC rate); 2 = interpolate I to 8 sps with a 31-tap half-band filter,
   * sqrt/log + 2048-point OLS Hilbert at 8 sps, half-band decimation back to 4 sps. Halo grows to 16,656. */
  int32_t upsample;
  /* Reference labels for the error counters (BER counted against the transmitted sequence, which
   * the real-time receiver knows). A non-NULL d_ref / h_ref argument always wins. With ref_prbs = 1 and a NULL
   * ref argument the library generates the transmitter's known label sequence on the device instead of reading
   * it — no host→device label transfer on the host path: label(k) = H(ref_seed, k) & (M(k) − 1) for global symbol
   * k, M(k) the QAM order of k's frame (R26 schedule) and H the synthetic transmitter's counter-based 32-bit hash
   * (kkgen.hash_u32(seed, 1, k): murmur3 fmix32 rounds keyed by the seed). With ref_prbs = 2 the
   * known sequence is the standard ITU-T O.150 PRBS-31 (x^31 + x^28 + 1) bit stream that real transmitters send:
   * b[n] = b[n−28] ⊕ b[n−31], b[0..30] = bits of W0 = (ref_seed·0x9E3779B1 mod 2^32) >> 1 (1 if zero), symbol k's
   * label = (bits 6k … 6k+5 of the stream, LSB first) & (M(k) − 1) (kkgen LinkConfig.label_source = "prbs31").
   * ref_prbs = 0 (default): a NULL ref argument means no error counting. */
  int32_t ref_prbs;
  uint32_t ref_seed;
  int32_t reserved2;
  double  ddlms_mu_mid;          /* 5e-4 step size over the second half of the warm-up     */
  /* KK_EQ_BLOCK_LS only: 1 = the paper's static arrangement for the dispersion ("offline-optimized
   * filter"): K2's static filter is RRC × CD inverse (as in KK_EQ_DDLMS) and the block-adaptive widely-linear
   * FIR only trims the residual: θ₀ = the centre spike, L = eq_taps or 5 by default. */
  int32_t static_cd;
  int32_t reserved3;
} kk_config;

/* Counters (all uint64, summed over calls until kk_reset_stats; index i = log2(M) − 2 for M = 4..64).
 * Layout is fixed: 24 consecutive uint64 — the same layout kk_stats_device writes. */
typedef struct kk_stats_t {
  uint64_t sym[5], sym_err[5], bits[5], bit_err[5];
  uint64_t clamped;       /* core samples with I < ε (R7)                                   */
  uint64_t frames;        /* frames processed                                               */
  uint64_t dead_frames;   /* frames whose 16384 samples are all clamped (signal loss)        */
  uint64_t bad_frames;    /* frames whose LS solve failed (fell back to the CD-init taps)    */
} kk_stats_t;
#define KK_STATS_WORDS 24

/* Fill *cfg with the paper's defaults (4 GS/s, 1 GBaud, 0.516 GHz tone, 1 % RRC span 256, 1024/512 Hilbert,
 * 4096/3072 MF, 4096-symbol frames, rule-based L, widely linear, W = 256, λ = 1e-3, 4-QAM, 0 ps/nm). */
void kk_config_default(kk_config* cfg);
/* sizeof(kk_config) and sizeof(kk_stats_t) as compiled into the library (lets bindings check their layout). */
size_t kk_config_sizeof(void);
size_t kk_stats_sizeof(void);

/* Validate cfg, compute the fp64 constants (RRC taps → MF spectrum, LO table, CD-inverse LS taps, tap
 * count, FFT twiddles), upload them and allocate scratch + counters on cfg->device. No kernel runs.
 * Errors: KK_ERR_NULL, KK_ERR_CONFIG, KK_ERR_NOMEM, KK_ERR_CUDA. On error *out is NULL. */
kk_status kk_init(const kk_config* cfg, kk_ctx** out);

/* Samples that must be readable before (left) and after (right) the core of every call:
 * one neighbour frame (its carrier estimate A_f and MF support) + half a Hilbert block = 16640. */
kk_status kk_halo(const kk_ctx* ctx, int64_t* left, int64_t* right);

/* Equalizer taps L actually used (rule or override; 4 in DDLMS mode). */
kk_status kk_eq_taps(const kk_ctx* ctx, int32_t* taps);

/* Process the core [first_sample, first_sample + n_samples) of the stream; asynchronous on `stream`.
 *   d_adc       device pointer to the CORE start (global sample first_sample); the range
 *               [d_adc − left, d_adc + n_samples + right) must be readable (kk_halo). int16 or float32
 *               int16, uint8 or float32 per cfg.input_dtype; must be 16-byte aligned.
 *   first_sample global index, multiple of 16384 (frame grid), ≥ 0.
 *   n_samples   multiple of 16384, 16384 ≤ n_samples ≤ max_samples_per_call.
 *   d_ref       nullable device uint8[n_samples/4]: transmitted labels; if given, error counters update. NULL
 *               with kk_config.ref_prbs = 1: the transmitter's known labels are generated on the device instead.
 *               Any alignment; 16-byte aligned enables K3's TMA staging (byte loads otherwise, ~15 % slower K3).
 *   d_decisions nullable device uint8[n_samples/4]: decided labels out.
 * Symbol/bit/frame/clamp counters always update. Errors: KK_ERR_NULL, KK_ERR_ALIGN, KK_ERR_SHORT,
 * KK_ERR_CONFIG (n_samples too large), KK_ERR_CUDA (launch failure). */
kk_status kk_process_frames(kk_ctx* ctx, const void* d_adc, int64_t first_sample, int64_t n_samples,
                            const uint8_t* d_ref, uint8_t* d_decisions, kk_stream_t stream);

/* As kk_process_frames, plus per-frame error counts for binned Q traces ("Q-factors were
 * estimated from BER in bins of 21 ms"): d_frame_errors (nullable device uint32[2·n/16384])
 * receives, for local frame f of the call, [2f] = symbol errors and [2f+1] = bit errors (needs d_ref).
 * The caller bins frames into ≈21 ms (5127-frame) bins and maps BER → Q with kk_q_from_ber. */
kk_status kk_process_frames_ex(kk_ctx* ctx, const void* d_adc, int64_t first_sample, int64_t n_samples,
                               const uint8_t* d_ref, uint8_t* d_decisions, uint32_t* d_frame_errors,
                               kk_stream_t stream);

/* End-to-end variant with HOST buffers (pinned recommended): copies [h_adc − left, h_adc + n + right)
 * host→device, runs kk_process_frames, copies decisions device→host, in chunks of ≤ min(max_samples_per_call, 2^26)
 * with two internal streams so the copies of chunk i+1 overlap the kernels of chunk i. Blocks until done.
 * h_ref / h_decisions nullable host uint8[n_samples/4] (h_ref NULL with ref_prbs = 1: generated labels, so only
 * the samples cross PCIe). Same constraints/errors as kk_process_frames,
 * except n_samples may exceed max_samples_per_call (it must be a multiple of 16384). Ordering: the internal
 * streams first wait for work already queued on the legacy default stream and on the stream of the context's
 * last kk_process_frames / kk_reset_stats call, so no caller synchronisation is needed before it. */
kk_status kk_process_frames_host(kk_ctx* ctx, const void* h_adc, int64_t first_sample, int64_t n_samples,
                                 const uint8_t* h_ref, uint8_t* h_decisions);

/* Synchronise the context's last stream and copy the counters to *host_out. KK_ERR_CUDA on sticky error. */
kk_status kk_stats(kk_ctx* ctx, kk_stats_t* host_out);
/* Asynchronously copy the 24 counters (kk_stats_t layout) to device memory d_out (e.g. for NCCL allreduce). */
kk_status kk_stats_device(kk_ctx* ctx, uint64_t* d_out, kk_stream_t stream);
/* Zero the counters (asynchronous on stream). */
kk_status kk_reset_stats(kk_ctx* ctx, kk_stream_t stream);

/* Describe / copy the last call's intermediate of a stage (device→device, async on stream):
 *   KK_STAGE_FIELD: E (complex64 interleaved) for samples [first − 16384, first + n + 16384)
 *   KK_STAGE_MF   : y (complex64) for 2-sps indices [first/2 − K, (first + n)/2 + K), K = (L−1)/2
 *                   (DDLMS mode: K = 2·ddlms_warmup + 2)
 *   KK_STAGE_EQ   : z (complex64) for symbols [first/4, (first + n)/4); needs keep_intermediate
 * kk_intermediate_range gives (first global index, count) of the stage. KK_ERR_STATE if no call yet /
 * not kept; KK_ERR_CONFIG if bytes < count·8. */
kk_status kk_intermediate_range(const kk_ctx* ctx, int stage, int64_t* first_index, int64_t* count);
kk_status kk_get_intermediate(kk_ctx* ctx, int stage, void* d_dst, size_t bytes, kk_stream_t stream);

/* Per-kernel timing (measurement support). When enabled, kk_process_frames records CUDA
 * events around each of its kernel launches (K1 KK, K2 MF, K3 EQ) on the call's stream. kk_kernel_times
 * synchronises those events and returns, per kernel, the summed device time in ms and the launch count
 * since the last reset (reset = 1 clears them after reading). */
kk_status kk_enable_timing(kk_ctx* ctx, int enable);
kk_status kk_kernel_times(kk_ctx* ctx, double ms_out[3], int64_t launches_out[3], int reset);

/* Q = 20·log10(√2·erfcinv(2·BER)) in dB; KK_ERR_DOMAIN unless 0 < ber < 0.5. */
kk_status kk_q_from_ber(double ber, double* q_db);

/* Free everything the context owns (synchronises its device first). NULL is a no-op. */
void kk_destroy(kk_ctx* ctx);

/* Debug aid (needs debug_guard = 1 at kk_init; a bounds check the library does on itself, since device
 * sanitizers are not always available): synchronizes the context's device, then checks that the 64 KiB
 * canary zones (byte 0xA5) before and after every scratch buffer — field E, ΣE partials, clamp counts, y,
 * z, counters and the host-path staging buffers — are intact. KK_OK if they are (or debug_guard = 0 and
 * nothing was checked: *n_checked = 0); KK_ERR_STATE if a kernel wrote out of bounds, with kk_last_error
 * naming the buffer and the first corrupted byte offset. n_checked (may be NULL) receives the number of
 * buffers checked. */
kk_status kk_check_guards(kk_ctx* ctx, int32_t* n_checked);

const char* kk_strerror(kk_status status);
/* Last error message of the context, with (stage, frame) where known; "" if none. */
const char* kk_last_error(const kk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* KKRX_H */
