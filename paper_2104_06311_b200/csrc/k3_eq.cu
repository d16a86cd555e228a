// k3_eq.cu — K3: per-frame block-adaptive widely-linear FIR equalizer (absorbs CD), carrier-phase
// recovery, QAM decision and error counting.
//
// PAPER.md:82 (§2): "the signal is further filtered by a four-tap adaptive time-domain DDLMS widely-linear
// equalizer. The decisions made by the equalizer are demapped"; "equalization, which
// automatically handles dispersion compensation"; PAPER.md:112 BER → Q. BASELINE.json north_star replaces
// the sequential DDLMS by a "block-adaptive FIR equalizer absorbing chromatic dispersion" and adds
// "carrier-phase recovery". SURVEY §8(a) a7–a9 with readings R10 (T/2-spaced, L taps, WL, DD-LS with
// ridge λ = ridge·tr(R)/(2L) toward θ₀), R12 (CPR per W-symbol window), R25 (AGC), R27 (gain unbias):
//   per frame f (4096 symbols k, regressor φ̃_k = [y[2k − j]]_{j=−K..K} ‖ conj(·)):
//   (1) y⁰ = φ̃ᵀθ₀, θ₀ = [w_cd; 0];  g = (mean|y⁰|²)^{−½};  θ₀ ← gθ₀          (AGC)
//   (2) d_k = D(g·y⁰_k)
//   (3) R = Σ conj(φ̃)φ̃ᵀ, p = Σ conj(φ̃)d;  θ₁ = (R + λI)⁻¹(p + λθ₀)
//   (4) y¹ = φ̃ᵀθ₁;  γ = Σ y¹·conj(D(y¹)) / Σ|D(y¹)|²;  u = y¹/|γ|           (unbias)
//   (5) per window b: c_b = Σ u·conj(D(u)),  z = u·conj(c_b)/|c_b|           (CPR: e^{−i·arg c_b})
//   (6) label = D(z); counts vs reference labels.
//
// Three launches per call ("the batched per-frame equalizer", BASELINE north_star):
//   K3a k3a_kernel  — steps (1)–(3)'s sums: persistent CTAs (2 per SM), one frame at a time: sweep A (lag sums,
//                     pass 1, power), AGC, sweep B (training decisions, p, remaining lags), fixed-order fp64
//                     reduction → one record per frame (the sums, g, flags) in global memory;
//   K3s k3s_kernel  — step (3)'s solve for every frame at once: one small CTA per frame assembles the real system
//                     from the sums and the frame's edge samples and eliminates it (fp64 Gauss–Jordan) → θ₁;
//                     thousands of independent solves in flight hide their serial latency (inside K3a/K3c they
//                     idled the CTA: the solve phase cost 11 % of the former single kernel);
//   K3c k3c_kernel  — steps (4)–(6): persistent CTAs, θ₁ arrives by TMA with the frame: sweep C (pass 2, unbias
//                     sums), CPR, decisions, counters.
// The frame is loaded twice (K3a and K3c): 64 KiB per frame from HBM each time, far below K3's compute time.
//
// Structure used (exact identities):
//  * R from lag sums: with a_j = y[2k − j],  S(i,d) = Σ_k conj(a_i)·a_{i+d},  T(i,d) = Σ_k a_i·a_{i+d}.
//    Only the bases i = −K, −K+1 are accumulated (4L complex MACs per symbol); every other S(i,d), T(i,d)
//    follows from the exact sliding-window recurrence S(i+2,d) = S(i,d) + term_i(k0−1) − term_i(k1−1).
//  * Real form of the widely-linear normal equations: with x_k = [Re a; Im a] ∈ R^{2L}, the complex
//    augmented ridge system (R + λI)θ = p + λθ₀ is the same problem as two real systems
//    (G + λ/2·I)m_r = q_r + λ/2·m_r0 (r = 1, 2; G = Σ x xᵀ, q_1 = Σ x·Re d, q_2 = Σ x·Im d) with
//    m_1 = [w_r + v_r; v_i − w_i], m_2 = [w_i + v_i; w_r − v_r]. G and q are read off S, T and p.
//    Linear-only mode solves the real 2L form [[Re R, −Im R],[Im R, Re R]] of the Hermitian system.
//    Both are solved in fp64 (Gauss–Jordan with 2×2 pivots, no pivoting on an SPD matrix; failure ⇒ fall back
//    to θ₀ and count a bad frame).
//
// Mapping (K3a, K3c): 256 threads per frame; warp w owns symbols [512w, 512w + 512). K ≤ 4: each lane works on
// groups of 4 consecutive symbols, the frame's 2-sps samples (64 KiB) arriving by 2-D tensor TMA with the 64-B
// swizzle (a group's K + 4 16-byte window pairs serve its 4 symbols; conflict-free); K ≥ 5: one symbol at a time
// from a plain bulk copy. Reductions: in-warp transpose-reduce (31 shuffles per 32 values), then fp64 over the
// 8 warps in fixed order (deterministic).
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {

constexpr int K3_THREADS = 256;
constexpr int K3_WARPS = 8;
constexpr int K3_SPT = kFrameSym / K3_THREADS;   // 16 symbols per thread
constexpr int kGJWarpN = 18;                     // largest real system solved by one warp (2N fp64 registers/lane)

// In-warp transpose-reduce of 32 floats: afterwards lane l holds the warp sum of element l.
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const float send = up ? v[i] : v[i + off];
      const float keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

__host__ __device__ constexpr int pow2_ceil(int n) { return n <= 1 ? 1 : 2 * pow2_ceil((n + 1) / 2); }

// Write this warp's sums of acc[0..N) to red_w[base + i] (red_w = this warp's slice of the reduction buffer).
// Whole groups of 32 values: in-warp transpose-reduce. A remainder of R < 32 values (padded to P = 2^⌈log2 R⌉):
// plain butterflies over the lane bits ≥ P (every lane keeps all P values), then the transpose-reduce over the
// low log2 P bits — about half the instructions of a zero-padded 32-value transpose for R = 4 or 8.
// Two segments (N1 < N): values [0, N1) go to red_w[base + i], values [N1, N) to red_w[base2 + i − N1] — one
// reduction for two arrays (a single remainder instead of two).
template <int N, int N1 = N>
__device__ __forceinline__ void warp_partials(const float (&acc)[N], float* red_w, int base, int lane, int base2 = 0) {
  constexpr int NF = N / 32, R = N % 32, P = pow2_ceil(R);
  auto out = [&](int i) { return (N1 >= N || i < N1) ? base + i : base2 + (i - N1); };
#pragma unroll
  for (int b = 0; b < NF; ++b) {
    float t[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) t[i] = acc[b * 32 + i];
    const float r = warp_transpose_reduce(t, lane);
    red_w[out(b * 32 + lane)] = r;
  }
  if constexpr (R > 0) {
    float t[P];
#pragma unroll
    for (int i = 0; i < P; ++i) t[i] = (i < R) ? acc[NF * 32 + i] : 0.f;
#pragma unroll
    for (int off = 16; off >= P; off >>= 1) {
#pragma unroll
      for (int i = 0; i < P; ++i) t[i] += __shfl_xor_sync(0xffffffffu, t[i], off);
    }
#pragma unroll
    for (int off = P / 2; off >= 1; off >>= 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < off; ++i) {
        const float send = up ? t[i] : t[i + off];
        const float keep = up ? t[i + off] : t[i];
        t[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    if (lane < R) red_w[out(NF * 32 + lane)] = t[0];   // lane l (< P) holds element l
  }
}

template <int K>
struct K3Layout {
  static constexpr int L = 2 * K + 1;
  static constexpr int ND = 2 * K + 1;             // lags 0..2K for base i = −K (ρ = 0); 0..2K−1 for ρ = 1
  // Every lane works on groups of GS consecutive symbols (a group's K + GS window pairs serve its GS symbols'
  // windows) on a frame buffer written by tensor TMA with the 64-B swizzle (conflict-free group loads). K ≤ 4:
  // GS = 4, lags [0, LA) in sweep A (with pass 1), [LA, ND) in sweep B (with p). K ≥ 5 (L ≥ 11): GS = 2 (register
  // budget), lags [0, 7) with pass 1 and [7, ND) in two passes of sweep A, sweep B carries p only.
  static constexpr int GS = (K <= 4) ? 4 : 2;
  static constexpr int LA = (K <= 4) ? (K + 2 < ND ? K + 2 : ND) : ND;   // lags of sweep A
  static constexpr int LA1 = (K <= 4) ? LA : 7;                         // … of its first pass (with pass 1)
  static constexpr int LB = ND - LA;
  static constexpr int N = 2 * L;                  // real system size
  static constexpr int NP = 4 * L;                 // p floats: p1, p2 complex
  static constexpr int RG = (K <= 4) ? ND : 8;     // lags per R sweep (register budget)
  static constexpr int NRG = (ND + RG - 1) / RG;   // R sweeps
  static constexpr int NR = 8 * RG * NRG;          // S0,T0,S1,T1 per lag (padded to whole groups)
  static constexpr int NRED = ((NP + NR + 1 + 31) / 32) * 32;   // + frame power
  static constexpr int IPOW = NP + NR;             // index of the frame power in the reduction
  static constexpr int YS = 2 * kFrameSym + 2 * K; // float2 used per frame (y_s[0 .. 8191 + 2K])
  static constexpr int YB = (1024 + 8) * 64;        // frame buffer bytes: 8 × 128 + 8 rows of 64 B (tensor TMA)
  static constexpr int WS = N + 3;                 // odd row stride (doubles) of the real system [A | q1 q2]
  static constexpr int RED_B = K3_WARPS * NRED * 4;
  static constexpr int MAT_B = N * WS * 8;
  // two label buffers (the next frame's labels land while this frame's are read) when two CTAs per SM still
  // fit in the SM's 228 KB with them (1 KB reserved per CTA): K ≤ 6
  static constexpr int TOTAL1 = YB + kFrameSym + kFrameSym * 8 + (RED_B > MAT_B ? RED_B : MAT_B) +
                                (NRED > 128 ? NRED : 128) * 8 + 2 * L * 8 + 16 * 8 + 32 * 4 + 16 + 64 * 4;
  static constexpr int NREFB = (2 * (TOTAL1 + kFrameSym + 1024) <= 228 * 1024) ? 2 : 1;
  // shared memory (bytes)
  static constexpr int Y = 0;                      // frame samples; reused for the CPR products after pass 2
  static constexpr int REF = Y + YB;               // NREFB × 4096 labels
  static constexpr int US = REF + NREFB * kFrameSym;   // y⁰ (pass 1), then y¹ (pass 2) per symbol (float2 × 4096)
  static constexpr int RED = US + kFrameSym * 8;   // warp partial sums; the solve's matrix aliases it
  static constexpr int MAT = RED;
  static constexpr int DRES = RED + (RED_B > MAT_B ? RED_B : MAT_B);
  static constexpr int TH = DRES + (NRED > 128 ? NRED : 128) * 8;   // (dres doubles as the GJ pivot rows)
  static constexpr int ROT = TH + 2 * L * 8;       // (spare: 16 float2)
  static constexpr int CC = ROT + 16 * 8;          // the frame's 32 per-block clamp counts (TMA, with the samples)
  static constexpr int BAR = CC + 32 * 4;          // mbarrier
  static constexpr int MISC = BAR + 16;
  static constexpr int TOTAL = MISC + 64 * 4;
  static_assert(TOTAL == TOTAL1 + (NREFB - 1) * kFrameSym, "layout size");
  static_assert(N <= 32, "one matrix row per lane");
  static_assert((2 * ND - 1) * (K + 1) <= K3_THREADS, "one thread per chain point");
  static_assert(2 * (K + 1) * 8 <= 2 * L * 8, "trace terms fit in th");
  static_assert((YS * 8) % 16 == 0 && YB >= YS * 8, "TMA size");
};

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// 2-D tensor TMA (tile mode) into shared memory, completion on the mbarrier (the tensor map carries the swizzle)
__device__ __forceinline__ void tma_tensor_2d(void* dst_smem, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst_smem)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}


// per-frame records between the launches: K3a → K3s: the fp64 sums (NRED), g, flags; K3s → K3c: θ₁ (w, v), flags
template <int K> struct K3Rec {
  static constexpr int REC = K3Layout<K>::NRED + 2;   // doubles: [0, NRED) sums, [NRED] g, [NRED + 1] flags
  static constexpr int TREC = 2 * K3Layout<K>::L + 2; // float2: [0, L) cr = (wr + vr, wi + vi), [L, 2L) ci = (vi − wi, wr − vr) (θ₁ in pass 2's real form), [2L].x = flags (int bits)
};
constexpr int kFlagDead = 1, kFlagSilent = 2, kFlagFail = 4;

template <int K, int PH>
__global__ void __launch_bounds__(K3_THREADS, 2)
k3_frame_kernel(const float2* __restrict__ y, int64_t frame0, int n_frames, const float2* __restrict__ w_cd,
                const int* __restrict__ clampcnt, int64_t clamp_frame_off, const uint8_t* __restrict__ ref,
                uint8_t* __restrict__ dec, float2* __restrict__ zout, unsigned long long* __restrict__ counters,
                K3Params p, double* __restrict__ rec, const float2* __restrict__ threc,
                const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap ymap_tail) {
  using Lay = K3Layout<K>;
  constexpr int L = Lay::L, ND = Lay::ND, N = Lay::N, NRED = Lay::NRED;
  constexpr int GS = Lay::GS, NG = K3_SPT / GS, NW = K + GS, LA = Lay::LA, LB = Lay::LB;
  extern __shared__ __align__(1024) unsigned char smem[];
  float2* ys = reinterpret_cast<float2*>(smem + Lay::Y);
  const float4* ys4 = reinterpret_cast<const float4*>(smem + Lay::Y);
  uint8_t* ref_s = smem + Lay::REF;
  float2* us = reinterpret_cast<float2*>(smem + Lay::US);
  float* red = reinterpret_cast<float*>(smem + Lay::RED);
  float2* th = reinterpret_cast<float2*>(smem + Lay::TH);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::BAR);
  const int* cc_s = reinterpret_cast<const int*>(smem + Lay::CC);
  int* misc = reinterpret_cast<int*>(smem + Lay::MISC);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool wl = p.widely_linear != 0;
  float* red_w = red + warp * NRED;
  const bool ref_tma = (PH == 1) && ref && ((reinterpret_cast<uintptr_t>(ref) & 15) == 0);
  constexpr uint32_t TBYTES = (PH == 1) ? (uint32_t)(K3Rec<K>::TREC * 8) : 0u;   // θ record (K3c)
  // double-buffered labels: frame `it` of this CTA reads buffer it & 1; the next frame's labels are requested
  // as soon as this frame's copies have landed (its own buffer was last read before the previous frame's
  // closing barrier), so the frame start no longer waits for a label copy issued at the end of the frame
  const bool dbl = (Lay::NREFB == 2) && ref_tma;
  auto ref_buf = [&](int b) { return ref_s + (dbl ? (b & 1) * kFrameSym : 0); };
  constexpr uint32_t YBYTES = Lay::YB;

  // thread 0: TMA the frame samples (and, separately, its labels) into shared memory. One arrival with the
  // total byte count; the copies may be issued at different times (the phase completes when all land). The
  // arrival comes with the first copy of the frame: the samples' (single label buffer) or the labels' (dbl).
  auto issue_y = [&](int fl) {
    fence_proxy_async_smem();                     // the frame buffer was written by generic stores (CPR products)
    if (!dbl) mbar_arrive_expect_tx(bar, YBYTES + 128u + TBYTES + (ref_tma ? (uint32_t)kFrameSym : 0u));
    {                           // 8 boxes of 128 rows + one of 8 rows (64-B rows of 8 float2)
#pragma unroll
      for (int b = 0; b < 8; ++b) tma_tensor_2d(smem + Lay::Y + b * 8192, &ymap, 0, fl * 1024 + 128 * b, bar);
      tma_tensor_2d(smem + Lay::Y + 65536, &ymap_tail, 0, fl * 1024 + 1024, bar);
    }
    tma_bulk_g2s(smem + Lay::CC, clampcnt + clamp_frame_off + (int64_t)fl * 32, 128u, bar);
    if constexpr (PH == 1) tma_bulk_g2s(th, threc + (int64_t)fl * K3Rec<K>::TREC, TBYTES, bar);
  };
  auto issue_ref = [&](int fl, int b) {
    if (!ref_tma) return;
    fence_proxy_async_smem();
    if (dbl) mbar_arrive_expect_tx(bar, YBYTES + 128u + TBYTES + (uint32_t)kFrameSym);
    tma_bulk_g2s(ref_buf(b), ref + (int64_t)fl * kFrameSym, kFrameSym, bar);
  };
  auto prefetch = [&](int fl) {
    prefetch_l2(y + (int64_t)fl * (2 * kFrameSym), Lay::YS * 8);
    if (ref_tma) prefetch_l2(ref + (int64_t)fl * kFrameSym, kFrameSym);
  };
  auto frame_order = [&](int64_t f) -> int {     // QAM order of global frame f (R26)
    return (int)p.schedule[(int)(((f / p.segment_frames) % p.n_segments + p.n_segments) % p.n_segments)];
  };
  if (tid == 0) mbar_init(bar, 1);
  uint8_t* lut32 = reinterpret_cast<uint8_t*>(misc + 32);   // 32-cross label table (36 bytes)
  cross32_lut_fill(lut32, tid, K3_THREADS);
  __syncthreads();
  if (tid == 0 && (int)blockIdx.x < n_frames) {
    if (dbl) { issue_ref(blockIdx.x, 0); issue_y(blockIdx.x); }
    else { issue_y(blockIdx.x); issue_ref(blockIdx.x, 0); }
    if ((int)blockIdx.x + (int)gridDim.x < n_frames) prefetch(blockIdx.x + gridDim.x);
  }
  // θ₀'s taps w_cd[a], a = j + K (tap j ↔ window index e), read from the kernel parameters where they are used
  static_assert(L <= 15, "K3Params::w_cd holds 15 taps");

  // tap window of local symbol kl: w[e] = y_s[2kl + 2K − e] = y[2k − (e − K)], e = 0..2K, i.e. the K+1 16-B pairs
  // (y_s[2kl + 2m], y_s[2kl + 2m + 1]) = (w[2K − 2m], w[2K − 2m − 1]). Symbol ownership: warp w owns the 512
  // consecutive symbols [512w, 512w + 512) — a 256-symbol CPR window is one half of a warp — in groups of GS
  // consecutive symbols per lane: the lane's group g starts at symbol G0(g); 32·GS symbols per warp step
  auto G0 = [&](int g) { return 512 * warp + 32 * GS * g + GS * lane; };
  // frame buffer: float4 i (samples 2i, 2i + 1) lives at swz(i) — TMA SWIZZLE_64B XORs the 16-B chunk bits 4–5 of
  // the address with bits 7–8 (the buffer is 1024-B aligned); a group window is NW consecutive float4 from G0(g),
  // at the same lane-relative offsets for every g (32·GS·g float4 is a multiple of 4 rows of 128 B)
  auto swz = [](int i) { return i ^ ((i >> 3) & 3); };
  auto ysw = [&](int e) -> float2 { const int q = e >> 1; return ys[2 * swz(q) + (e & 1)]; };   // sample e
  // shared-memory byte address of the lane's window float4 t in group 0 (formed at the start of each sweep, so
  // that it is not live across the solve); group g adds 512·GS·g bytes
  auto make_wadr = [&](uint32_t (&wadr)[NW]) {
#pragma unroll
    for (int t = 0; t < NW; ++t) wadr[t] = smem_u32(ys4 + 512 * warp + swz(GS * lane + t));
  };
  auto load_group = [&](const uint32_t (&wadr)[NW], int g, float4 (&F)[NW]) {
    const uint32_t go = (uint32_t)(512 * GS * g);
#pragma unroll
    for (int t = 0; t < NW; ++t)
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(F[t].x), "=f"(F[t].y), "=f"(F[t].z), "=f"(F[t].w) : "r"(wadr[t] + go));
  };
  // window of the group's symbol j from the group's float4 (compile-time indices after unrolling)
  auto win = [&](const float4 (&F)[NW], int j, float2 (&w)[L]) {
#pragma unroll
    for (int m = 0; m <= K; ++m) {
      w[2 * K - 2 * m] = make_float2(F[j + m].x, F[j + m].y);
      if (m < K) w[2 * K - 2 * m - 1] = make_float2(F[j + m].z, F[j + m].w);
    }
  };
  // per-symbol values (y⁰, then y¹) in groups: float4 q = symbols (2q, 2q + 1) at uswz(q) (conflict-free 16-B
  // accesses at the 32-B lane stride of 4-symbol groups)
  float4* us4 = reinterpret_cast<float4*>(smem + Lay::US);
  auto uswz = [](int q) { return q ^ ((q >> 3) & 1); };
  auto uget = [&](int kl) -> float2 { const int q = kl >> 1; return us[2 * uswz(q) + (kl & 1)]; };
  auto ustore = [&](int g, const float2 (&v)[GS]) {        // the group's GS per-symbol values, 16 B at a time
    const int q = G0(g) >> 1;
#pragma unroll
    for (int h = 0; h < GS / 2; ++h) us4[uswz(q + h)] = make_float4(v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y);
  };
  auto uload = [&](int g, float2 (&v)[GS]) {
    const int q = G0(g) >> 1;
#pragma unroll
    for (int h = 0; h < GS / 2; ++h) {
      const float4 a = us4[uswz(q + h)];
      v[2 * h] = make_float2(a.x, a.y);
      v[2 * h + 1] = make_float2(a.z, a.w);
    }
  };

  int it = 0;
  for (int fl = blockIdx.x; fl < n_frames; fl += gridDim.x, ++it) {
    bool early = false;                                // thread 0: next frame's samples already requested
    const int64_t sym0 = (int64_t)fl * kFrameSym;
    // the frame's QAM order (R26): one 64-bit division per frame by one thread, broadcast through shared memory;
    // computed here for the CTA's first frame, later ones during the previous frame and published at its end
    if (it == 0 && tid == 32) misc[2] = frame_order(frame0 + fl);
    mbar_wait(bar, it & 1);
    // dbl: arm the next frame's phase now and request its labels into the other buffer (the phase cannot
    // complete before its samples are requested after the CPR sums, when every thread is past this wait)
    if (dbl && tid == 0 && fl + (int)gridDim.x < n_frames) issue_ref(fl + (int)gridDim.x, it + 1);
    const uint8_t* ref_cur = ref_buf(it);
    // the previous frame's closing barrier already ordered misc[] (the QAM order) and every read of the buffers;
    // the TMA data is visible through the mbarrier — only the CTA's first frame needs a barrier here
    if (it == 0) __syncthreads();
    const int M = misc[2];
    const int bi = (M == 4) ? 0 : (M == 8) ? 1 : (M == 16) ? 2 : (M == 32) ? 3 : 4;
    Slicer sl;
    sl.init(M);
    sl.lut = lut32;
    // frame clamp count (K1's 32 per-block counts, landed with the samples) → dead-frame rule; every warp sums
    // them itself (fixed order), so no extra barrier
    int ccount = cc_s[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ccount += __shfl_xor_sync(0xffffffffu, ccount, o);
    const int fn = fl + (int)gridDim.x;
    const int m_next = (tid == 32 && fn < n_frames) ? frame_order(frame0 + fn) : 0;
    const bool dead = (ccount >= kFrameSamp);
    if constexpr (PH == 0) {
      // ======== K3a: sums of steps (1)–(3) → the frame's record
      int flags = dead ? kFlagDead : 0;
      double* rg = rec + (int64_t)fl * K3Rec<K>::REC;
      if (!dead) {
      // ---- sweep A: lag sums for bases ρ = 0 (i = −K, w[0]) and ρ = 1 (i = −K+1, w[1]) + pass-1 power
      //      S_ρ(d) = Σ conj(w[ρ])·w[ρ + d],  T_ρ(d) = Σ w[ρ]·w[ρ + d];  y⁰ = Σ_e w_cd[e]·w[e]
      //      conj(a)·b and a·b share the four real products: accumulate Σ ar·br, Σ ai·bi, Σ ar·bi, Σ ai·br
      //      (4 FMA for both); S = (A1 + A2, A3 − A4), T = (A1 − A2, A3 + A4) after the fp64 reduction;
      //      packed: (A1, A3) += ar·(br, bi), (A4, A2) += ai·(br, bi) — 2 FFMA2
      // red layout: [0, NP) {B1, B3, B4, B2} per tap; [NP + 8·d + {A1, A3, A4, A2} (ρ = 0), + 4 + {…} (ρ = 1)];
      // [IPOW] power  (A1 = Σ ar·br, A2 = Σ ai·bi, A3 = Σ ar·bi, A4 = Σ ai·br; B likewise with d)
      auto lag_acc = [&](float* acc, const float2 (&w)[L], int d0, int nd) {
#pragma unroll
        for (int gg = 0; gg < nd; ++gg) {
          const int d = d0 + gg;
          if (d < ND) {
            ffma2s(acc[8 * gg], acc[8 * gg + 1], w[0].x, w[d]);
            ffma2s(acc[8 * gg + 2], acc[8 * gg + 3], w[0].y, w[d]);
            if (d < ND - 1) {
              ffma2s(acc[8 * gg + 4], acc[8 * gg + 5], w[1].x, w[1 + d]);
              ffma2s(acc[8 * gg + 6], acc[8 * gg + 7], w[1].y, w[1 + d]);
            }
          }
        }
      };
      auto pass1 = [&](const float2 (&w)[L]) {   // w_cd·a = wr·a + wi·(i·a), the cmul form (taps stay scalars)
        float2 y0 = make_float2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < L; ++e) cmac2(y0, w[e], p.w_cd[e]);
        return y0;
      };
      {
        constexpr int LA1 = Lay::LA1;
        float acc[8 * LA1];
#pragma unroll
        for (int i = 0; i < 8 * LA1; ++i) acc[i] = 0.f;
        float pw = 0.f;
uint32_t wadr[NW];
        make_wadr(wadr);
#pragma unroll 1
        for (int g = 0; g < NG; ++g) {
          float4 F[NW];
          load_group(wadr, g, F);
          float2 y0[GS];
#pragma unroll
          for (int j = 0; j < GS; ++j) {
            float2 w[L];
            win(F, j, w);
            lag_acc(acc, w, 0, LA1);
            y0[j] = pass1(w);
            pw = fmaf(y0[j].x, y0[j].x, fmaf(y0[j].y, y0[j].y, pw));
          }
          ustore(g, y0);                           // y⁰ of the group (kept in us until sweep B)
        }
        warp_partials<8 * LA1>(acc, red_w, Lay::NP, lane);
        pw = warp_sum(pw);
        if (lane == 0) red_w[Lay::IPOW] = pw;
        if constexpr (LA > LA1) {                  // second pass: lags [LA1, LA)
          float acc2[8 * (LA - LA1)];
#pragma unroll
          for (int i = 0; i < 8 * (LA - LA1); ++i) acc2[i] = 0.f;
          uint32_t wadr2[NW];
          make_wadr(wadr2);
#pragma unroll 1
          for (int g = 0; g < NG; ++g) {
            float4 F[NW];
            load_group(wadr2, g, F);
#pragma unroll
            for (int j = 0; j < GS; ++j) {
              float2 w[L];
              win(F, j, w);
              lag_acc(acc2, w, LA1, LA - LA1);
            }
          }
          warp_partials<8 * (LA - LA1)>(acc2, red_w, Lay::NP + 8 * LA1, lane);
        }
      }
      __syncthreads();
      double P0 = 0.0;
#pragma unroll
      for (int w8 = 0; w8 < K3_WARPS; ++w8) P0 += (double)red[w8 * NRED + Lay::IPOW];
      P0 /= (double)kFrameSym;
      // AGC (R25). A frame without signal power (P0 ≤ p0_min = 1e-20·I_ref, or not finite: e.g. the tone
      // without modulation) cannot be trained: it is a bad frame with z = 0 and decisions D(0)
      const bool p0ok = (P0 > (double)p.p0_min) && isfinite(P0);
      const float g_agc = p0ok ? (float)rsqrt(P0) : 1.0f;
      if (!p0ok) flags |= kFlagSilent;
      if (p0ok) {
      // ---- sweep B: decisions on g·y⁰ and p1[e] = Σ conj(a_j)·d, p2[e] = Σ a_j·d  (a_j = w[e]);
      //      (plus the lags [LA, ND) of the lag sums when K ≤ 4)
      auto p_acc = [&](float* acc, const float2 (&w)[L], float2 d) {
#pragma unroll
        for (int e = 0; e < L; ++e) {       // (B1, B3) += ar·(dr, di), (B4, B2) += ai·(dr, di): p1, p2 later
          ffma2s(acc[4 * e], acc[4 * e + 1], w[e].x, d);
          ffma2s(acc[4 * e + 2], acc[4 * e + 3], w[e].y, d);
        }
      };
      {
        constexpr int NB = Lay::NP + 8 * LB;        // p sums, then the lags [LA, ND): one reduction
        float acc[NB];
        float* accl = acc + Lay::NP;
#pragma unroll
        for (int i = 0; i < NB; ++i) acc[i] = 0.f;
uint32_t wadr[NW];
        make_wadr(wadr);
#pragma unroll 1
        for (int g = 0; g < NG; ++g) {
          float4 F[NW];
          load_group(wadr, g, F);
          float2 y0[GS];
          uload(g, y0);
#pragma unroll
          for (int j = 0; j < GS; ++j) {
            float2 w[L];
            win(F, j, w);
            p_acc(acc, w, sl.point(cscale(y0[j], g_agc)));
            if constexpr (LB > 0) lag_acc(accl, w, LA, LB);
          }
        }
        __syncthreads();   // every read of the frame buffer is done: request the next frame (overlaps the reductions)
        if (tid == 0 && fn < n_frames) { issue_y(fn); early = true; }
        warp_partials<NB, Lay::NP>(acc, red_w, 0, lane, Lay::NP + 8 * LA);
      }
      }
      __syncthreads();
      if (!p0ok && tid == 0 && fn < n_frames) { issue_y(fn); early = true; }   // silent: sweep A was the last reader
      if (p0ok) {        // fp64 sums over the 8 warp partials, fixed order → the record
        for (int v = tid; v < NRED; v += K3_THREADS) {
          double s = 0.0;
#pragma unroll
          for (int w8 = 0; w8 < K3_WARPS; ++w8) s += (double)red[w8 * NRED + v];
          rg[v] = s;
        }
      }
      if (tid == 0) rg[NRED] = (double)g_agc;
      }
      if (tid == 0) rg[NRED + 1] = (double)flags;
      if (tid == 32) misc[2] = m_next;                 // publish the next frame's QAM order
      __syncthreads();   // all reads of ys / red / misc for this frame are done
      if (tid == 0 && fn < n_frames) {
        if (!early) issue_y(fn);
        if (fn + (int)gridDim.x < n_frames) prefetch(fn + gridDim.x);
      }
    } else {
      // ======== K3c: steps (4)–(6) with θ₁ from K3s (arrived with the frame)
      const int fflags = __float_as_int(th[2 * L].x);
      int bad = (fflags & (kFlagSilent | kFlagFail)) ? 1 : 0;   // silent frame or solve failure (θ₀ used)
      const bool zero = dead || (fflags & kFlagSilent);    // z = 0, decisions D(0): dead or silent frame
      float2 rA = make_float2(0.f, 0.f), rB = make_float2(0.f, 0.f);   // CPR rotations (× unbias) of the halves
      if (!zero) {
      // ---- sweep C: pass 2 y¹ = Σ_e w_e·a + v_e·conj(a) → us, and the gain-unbias sums (R27)
      float2 gacc = make_float2(0.f, 0.f), gdd = make_float2(0.f, 0.f);   // Σ y¹·conj(D), Σ (D.x², D.y²)
      {
        // w·a + v·conj(a) = (ar·(wr + vr) + ai·(vi − wi), ar·(wi + vi) + ai·(wr − vr)): 4 FMA per tap; K3s
        // delivers the taps in this form: th[e] = cr = (wr + vr, wi + vi), th[L + e] = ci = (vi − wi, wr − vr)
        float2 cr[L], ci[L];
#pragma unroll
        for (int e = 0; e < L; ++e) { cr[e] = th[e]; ci[e] = th[L + e]; }
        auto pass2 = [&](const float2 (&w)[L]) {
          float2 o = make_float2(0.f, 0.f);
#pragma unroll
          for (int e = 0; e < L; ++e) {         // o += ar·(c1, c3) + ai·(c2, c4)
            ffma2s(o, w[e].x, cr[e]);
            ffma2s(o, w[e].y, ci[e]);
          }
          const float2 dd = sl.point(o);        // γ = Σ y¹·conj(D(y¹)) / Σ|D(y¹)|²
          cmacc2(gacc, o, dd);
          ffma2(gdd, dd, dd);
          return o;
        };
        {
uint32_t wadr[NW];
          make_wadr(wadr);
#pragma unroll 1
          for (int g = 0; g < NG; ++g) {
            float4 F[NW];
            load_group(wadr, g, F);
            float2 o[GS];
#pragma unroll
            for (int j = 0; j < GS; ++j) {
              float2 w[L];
              win(F, j, w);
              o[j] = pass2(w);
            }
            ustore(g, o);
          }
        }
      }
      {
        const float gr = warp_sum(gacc.x), gi = warp_sum(gacc.y), gd = warp_sum(gdd.x + gdd.y);
        if (lane == 0) { red_w[0] = gr; red_w[1] = gi; red_w[2] = gd; }
      }
      __syncthreads();
      // the frame buffer is dead now (every thread is past sweep C): start the next frame's sample copy so that it
      // overlaps the CPR and the decisions (its labels: already requested (dbl), else at the end of the frame,
      // after the single label buffer is read)
      if (tid == 0) {
        const int nf = fl + (int)gridDim.x;
        if (nf < n_frames) { issue_y(nf); early = true; }
      }
      float sc = 1.0f;
      {
        // fp64 sums over the 8 warps' (gr, gi, gd), lane-parallel: lane 3·w8 + c holds warp w8's component c;
        // a fixed tree over w8 (offsets 12, 6, 3 — the same in every warp) leaves component c in lane c
        double gv = (lane < 3 * K3_WARPS) ? (double)red[(lane / 3) * NRED + lane % 3] : 0.0;
#pragma unroll
        for (int o = 12; o >= 3; o >>= 1) gv += __shfl_down_sync(0xffffffffu, gv, o);
        const double Gr = __shfl_sync(0xffffffffu, gv, 0), Gi = __shfl_sync(0xffffffffu, gv, 1),
                     Gd = __shfl_sync(0xffffffffu, gv, 2);
        const double isc = Gd * rsqrt(Gr * Gr + Gi * Gi);          // 1/|γ| = Σ|D|² / |Σ y¹·conj(D)|
        if (isc > 0.0 && isfinite(isc)) sc = (float)isc; else bad = 1;
      }
      // ---- CPR (R12): c_b = Σ_{k∈b} u_k·conj(D(u_k)) with u = sc·y¹; rotation conj(c_b)/|c_b| (none if c_b = 0).
      //      The warp owns 512 consecutive symbols (two 256-symbol halves, s < 8 and s ≥ 8): W = 256 / 512 windows
      //      are summed inside the warp (fixed order: s ascending, then lane butterflies); larger windows add
      //      the warps' sums in warp order through shared memory.
      {
        float2 c0 = make_float2(0.f, 0.f), c1 = make_float2(0.f, 0.f);
        {
          auto grp = [&](int g, float2& c) {
            float2 v[GS];
            uload(g, v);
#pragma unroll
            for (int j = 0; j < GS; ++j) {
              const float2 uu = cscale(v[j], sc);
              cmacc2(c, uu, sl.point(uu));
            }
          };
#pragma unroll 1
          for (int g = 0; g < NG / 2; ++g) grp(g, c0);
#pragma unroll 1
          for (int g = NG / 2; g < NG; ++g) grp(g, c1);
        }
        float cr0 = c0.x, ci0 = c0.y, cr1 = c1.x, ci1 = c1.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          cr0 += __shfl_xor_sync(0xffffffffu, cr0, o);
          ci0 += __shfl_xor_sync(0xffffffffu, ci0, o);
          cr1 += __shfl_xor_sync(0xffffffffu, cr1, o);
          ci1 += __shfl_xor_sync(0xffffffffu, ci1, o);
        }
        if (p.cpr_window != 256) { cr0 += cr1; ci0 += ci1; }          // the warp's 512 symbols
        if (p.cpr_window > 512) {                                      // kernel-uniform: windows of W/512 warps
          float* cw = red + K3_WARPS * NRED - 2 * K3_WARPS;            // (past the γ partials of every warp)
          if (lane == 0) { cw[2 * warp] = cr0; cw[2 * warp + 1] = ci0; }
          __syncthreads();
          const int per = p.cpr_window / 512, w0 = (warp / per) * per;
          cr0 = 0.f; ci0 = 0.f;
          for (int q = 0; q < per; ++q) { cr0 += cw[2 * (w0 + q)]; ci0 += cw[2 * (w0 + q) + 1]; }
        }
        if (p.cpr_window != 256) { cr1 = cr0; ci1 = ci0; }
        auto rotation = [&](float cr, float ci) {                      // z = y¹·(sc·conj(c)/|c|)
          const float m2 = cr * cr + ci * ci;
          const float rs = (m2 > 0.f && isfinite(m2)) ? rsqrtf(m2) : 0.f;
          const float rsc = rs * sc;
          return (rs > 0.f) ? make_float2(cr * rsc, -ci * rsc) : make_float2(sc, 0.f);
        };
        rA = rotation(cr0, ci0);
        rB = rotation(cr1, ci1);
      }
      }


    // ---- decisions, counts, outputs: z = u·e^{−iϑ_b} (dead or silent frame: z = 0); rotation rA for the warp's
    //      first 256 symbols (s < 8), rB for the second
    int serr = 0, berr = 0;
    if (!zero && ref_tma && dec && ((reinterpret_cast<uintptr_t>(dec) & 3) == 0) && !zout) {
      // the common case (labels from shared memory, no z output): a lane's 4 consecutive symbols — one 16-B pair of
      // us loads, one 32-bit label word, one 32-bit decision store per group (the 32-cross labels from the table)
      auto groups = [&](auto lab_of) {
#pragma unroll 2
        for (int g = 0; g < NG; ++g) {
          const int kl = G0(g);
          const float2 r = (g < NG / 2) ? rA : rB;
          float2 v[GS];
          uload(g, v);
          const uint32_t rw = (GS == 4) ? *reinterpret_cast<const uint32_t*>(ref_cur + kl)
                                        : (uint32_t)*reinterpret_cast<const uint16_t*>(ref_cur + kl);
          uint32_t lw = 0u;
#pragma unroll
          for (int j = 0; j < GS; ++j) lw |= (uint32_t)lab_of(cmul(v[j], r)) << (8 * j);
          // per-byte compares: symbol errors = nonzero bytes of lw ^ rw, bit errors = popc(lw ^ rw)
          const uint32_t x = lw ^ rw;
          serr += __popc(__vcmpne4(x, 0u)) >> 3;
          berr += __popc(x);
          if constexpr (GS == 4) *reinterpret_cast<uint32_t*>(dec + sym0 + kl) = lw;
          else *reinterpret_cast<uint16_t*>(dec + sym0 + kl) = (uint16_t)lw;
        }
      };
      if (sl.cross) groups([&](float2 z) { return sl.label(z); });
      else groups([&](float2 z) { return sl.label_sq(z); });
    } else {
#pragma unroll 4
      for (int s = 0; s < K3_SPT; ++s) {
        const int kl = G0(s / GS) + (s % GS);
        const float2 zz = zero ? make_float2(0.f, 0.f) : cmul(uget(kl), s < K3_SPT / 2 ? rA : rB);
        const int lab = sl.label(zz);
        if (ref) {
          const int r = ref_tma ? (int)ref_cur[kl] : (int)__ldg(&ref[sym0 + kl]);
          serr += (lab != r);
          berr += __popc(lab ^ r);
        }
        if (dec) dec[sym0 + kl] = (uint8_t)lab;
        if (zout) zout[sym0 + kl] = zz;
      }
    }
    if (ref) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        serr += __shfl_xor_sync(0xffffffffu, serr, o);
        berr += __shfl_xor_sync(0xffffffffu, berr, o);
      }
      if (lane == 0) { misc[8 + warp] = serr; misc[16 + warp] = berr; }
    }
    if (tid == 32) misc[2] = m_next;                   // publish the next frame's QAM order
    __syncthreads();   // all reads of ys / ref_s / misc for this frame are done
    if (tid == 0) {
      const int nf = fl + (int)gridDim.x;
      if (nf < n_frames) {
        // from L2 (prefetched one frame ago); dbl: the labels were requested at the frame start
        if (!early) issue_y(nf);
        if (!dbl) issue_ref(nf, 0);
        if (nf + (int)gridDim.x < n_frames) prefetch(nf + gridDim.x);
      }
      if (ref) {
        long long se = 0, be = 0;
        for (int w8 = 0; w8 < K3_WARPS; ++w8) { se += misc[8 + w8]; be += misc[16 + w8]; }
        if (se) atomicAdd(&counters[5 + bi], (unsigned long long)se);
        if (be) atomicAdd(&counters[15 + bi], (unsigned long long)be);
        if (p.frame_err) { p.frame_err[2 * fl] = (unsigned)se; p.frame_err[2 * fl + 1] = (unsigned)be; }
      }
      atomicAdd(&counters[bi], (unsigned long long)kFrameSym);
      atomicAdd(&counters[10 + bi], (unsigned long long)kFrameSym * (bi + 2));
      if (ccount) atomicAdd(&counters[20], (unsigned long long)ccount);
      atomicAdd(&counters[21], 1ull);
      if (dead) atomicAdd(&counters[22], 1ull);
      if (!dead && bad) atomicAdd(&counters[23], 1ull);
    }
    }
  }
}

// ======== K3s: one CTA per frame: the real normal equations from the frame's sums and edge samples, eliminated in
// fp64 (warp 0: Gauss–Jordan with 2×2 pivots and lanes holding columns, N ≤ 18; the CTA for larger N) → θ₁
template <int K> struct K3S { static constexpr int THREADS = (K3Layout<K>::N <= kGJWarpN) ? 32 : 256; };

template <int K>
// one-warp CTAs: 32 resident per SM (64 registers; the solve is latency-bound, −0.35 % of K3 despite 16 B of spill)
__global__ void __launch_bounds__(K3S<K>::THREADS, (K3S<K>::THREADS == 32 ? 32 : 1))
k3s_kernel(const double* __restrict__ rec, const float2* __restrict__ y, const float2* __restrict__ w_cd,
           float2* __restrict__ threc, K3Params p) {
  using Lay = K3Layout<K>;
  constexpr int L = Lay::L, ND = Lay::ND, N = Lay::N, NRED = Lay::NRED, THREADS = K3S<K>::THREADS;
  constexpr int K3_WARPS_S = THREADS / 32;
  (void)K3_WARPS_S;
  __shared__ __align__(16) double dres[NRED > 128 ? NRED : 128];
  __shared__ __align__(16) double mat[N * Lay::WS];
  __shared__ __align__(16) double tl[2 * (K + 1)];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fl = blockIdx.x;
  const bool wl = p.widely_linear != 0;
  const double* rg = rec + (int64_t)fl * K3Rec<K>::REC;
  float2* tr = threc + (int64_t)fl * K3Rec<K>::TREC;
  const int flags = (int)rg[NRED + 1];
  if (flags & (kFlagDead | kFlagSilent)) {             // no solve: K3c outputs z = 0 for this frame
    if (tid == 0) tr[2 * L] = make_float2(__int_as_float(flags), 0.f);
    return;
  }
  for (int v = tid; v < NRED; v += THREADS) dres[v] = rg[v];
  const float g = (float)rg[NRED];
  // the chains read only the frame's edge samples: y_s[0, 2K] and y_s[8190 − 2K, 8190 + 2K] — one load per
  // thread into shared memory (a single global round trip instead of one per chain step)
  constexpr int NE_LO = 2 * K + 1, NE_HI = 4 * K + 1, HI0 = 8190 - 2 * K;
  __shared__ float2 edge[NE_LO + NE_HI];
  const float2* yf = y + (int64_t)fl * (2 * kFrameSym);
  for (int v = tid; v < NE_LO + NE_HI; v += THREADS) edge[v] = __ldg(&yf[v < NE_LO ? v : HI0 + (v - NE_LO)]);
  auto ysw = [&](int e) -> float2 { return edge[e < NE_LO ? e : NE_LO + (e - HI0)]; };   // edge sample e
  __syncthreads();
  {
      {
        double* A = mat;   // row-major N × WS: [G + λI | q1 q2]
        constexpr int W = Lay::WS;
        for (int pt = tid; pt < (2 * ND - 1) * (K + 1); pt += THREADS) {
          const int c = pt / (K + 1), m = pt % (K + 1);
          const int rho = c / ND, d = c % ND;
          const int npts = (2 * K - d - rho) / 2 + 1;  // chain points
          if (m < npts) {
            const double A1 = dres[Lay::NP + 8 * d + 4 * rho], A3 = dres[Lay::NP + 8 * d + 4 * rho + 1];
            const double A4 = dres[Lay::NP + 8 * d + 4 * rho + 2], A2 = dres[Lay::NP + 8 * d + 4 * rho + 3];
            double sr = A1 + A2, si = A3 - A4, tr_ = A1 - A2, ti = A3 + A4;   // S = Σ conj(a)·b, T = Σ a·b
#pragma unroll
            for (int mm = 0; mm < K; ++mm) {
              if (mm < m) {
                // fp32 edge increments: O(|y|²) terms added to fp64 sums of 4096 such terms
                const int i = -K + rho + 2 * mm;
                const float2 a1 = ysw(K - 2 - i), a2 = ysw(K - 2 - i - d), b1 = ysw(8190 + K - i), b2 = ysw(8190 + K - i - d);
                const float i0 = fmaf(a1.x, a2.x, a1.y * a2.y) - fmaf(b1.x, b2.x, b1.y * b2.y);
                const float i1 = fmaf(a1.x, a2.y, -a1.y * a2.x) - fmaf(b1.x, b2.y, -b1.y * b2.x);
                const float i2 = fmaf(a1.x, a2.x, -a1.y * a2.y) - fmaf(b1.x, b2.x, -b1.y * b2.y);
                const float i3 = fmaf(a1.x, a2.y, a1.y * a2.x) - fmaf(b1.x, b2.y, b1.y * b2.x);
                sr += (double)i0; si += (double)i1; tr_ += (double)i2; ti += (double)i3;
              }
            }
            const int i = -K + rho + 2 * m;
            const int r = i + K, q = i + d + K;     // S(r, q) = Σ conj(a_r)·a_q, T(r, q) = Σ a_r·a_q
            if (wl) {
              // G = [[Σ ar arᵀ, Σ ar aiᵀ], [Σ ai arᵀ, Σ ai aiᵀ]] from S and T (both orders of (r, q))
              const double rr = 0.5 * (sr + tr_), ii = 0.5 * (sr - tr_);
              const double ri = 0.5 * (si + ti), ir = 0.5 * (ti - si);   // Σ ar_r·ai_q, Σ ai_r·ar_q
              A[r * W + q] = rr;             A[q * W + r] = rr;
              A[(L + r) * W + (L + q)] = ii; A[(L + q) * W + (L + r)] = ii;
              A[r * W + (L + q)] = ri;       A[(L + q) * W + r] = ri;
              A[(L + r) * W + q] = ir;       A[q * W + (L + r)] = ir;
              if (d == 0) tl[rho * (K + 1) + m] = rr + ii;
            } else {
              // real form of the Hermitian R11: [[Re R, −Im R], [Im R, Re R]], R[r][q] = S, R[q][r] = conj(S)
              A[r * W + q] = sr;             A[q * W + r] = sr;
              A[(L + r) * W + (L + q)] = sr; A[(L + q) * W + (L + r)] = sr;
              A[(L + r) * W + q] = si;       A[(L + q) * W + r] = -si;
              A[r * W + (L + q)] = -si;      A[q * W + (L + r)] = si;
              if (d == 0) tl[rho * (K + 1) + m] = sr + sr;
            }
          }
        }
      }
  }
  __syncthreads();
      int fail = 0;
      if (warp == 0) {
        double* A = mat;
        constexpr int W = Lay::WS;
        // ridge (R10): λ_c = ridge·tr(R)/n_c. WL: real form uses λ_c/2 and tr(R) = 2·tr(G). Linear: tr(M) = 2·tr(R11)
        // tr(G): the d = 0 terms in chain order (ρ = 0: K + 1 points, ρ = 1: K points)
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int m = 0; m <= K; ++m) t0 += tl[m];
#pragma unroll
        for (int m = 0; m < K; ++m) t1 += tl[K + 1 + m];
        const double trG = t0 + t1;
        // (the factor ridge/n_c does not wait for the trace)
        const double lam = trG * (wl ? (double)p.ridge / (double)N : (double)p.ridge * 0.5 / (double)L);
        if (lane < L) {
          const int e = lane;
          const double B1 = dres[4 * e], B3 = dres[4 * e + 1], B4 = dres[4 * e + 2], B2 = dres[4 * e + 3];
          const double p1r = B1 + B2, p1i = B3 - B4, p2r = B1 - B2, p2i = B3 + B4;   // p1 = Σ conj(a)·d, p2 = Σ a·d
          const float2 w0 = __ldg(&w_cd[e]);
          const double w0r = (double)g * (double)w0.x, w0i = (double)g * (double)w0.y;
          if (wl) {
            // q1 = [Σ ar·dr; Σ ai·dr], q2 = [Σ ar·di; Σ ai·di];  m1₀ = [w0r; −w0i], m2₀ = [w0i; w0r]
            A[e * W + N] = 0.5 * (p1r + p2r) + lam * w0r;
            A[(L + e) * W + N] = 0.5 * (p2i - p1i) - lam * w0i;
            A[e * W + N + 1] = 0.5 * (p1i + p2i) + lam * w0i;
            A[(L + e) * W + N + 1] = 0.5 * (p1r - p2r) + lam * w0r;
          } else {
            A[e * W + N] = p1r + lam * w0r;
            A[(L + e) * W + N] = p1i + lam * w0i;
            A[e * W + N + 1] = 0.0;
            A[(L + e) * W + N + 1] = 0.0;
          }
        }
        if (lane < N) A[lane * W + lane] += lam;
        if constexpr (N <= kGJWarpN) {
        __syncwarp();
          // ---- Gauss–Jordan on [G + λI | q1 q2] by warp 0 with 2×2 pivot blocks (SPD ⇒ every leading 2×2 block
        //      is SPD, no pivoting; N = 4K + 2 is even). Lane c holds column c in registers (a[i] = A[i][c]); per
        //      step the two pivot lanes publish their columns as (A[i][k], A[i][k+1]) pairs in a double-buffered
        //      shared strip (dres is consumed) that every lane reads with broadcast 16-B loads — no CTA barriers
        //      and no shuffles (warp 0 runs this alone: shuffles in that branch would compile to collectives).
        //      Division-free form: the pivot rows become s·adj(P)·[row k; row k+1] and every other row
        //      row_i ← s·det(P)·row_i − A[i][k]·u0 − A[i][k+1]·u1, with s a power of two (≈ 1/pa², exact scaling
        //      that keeps the rows bounded). The matrix ends as diag(D) with D = s·det·(later factors) per pivot
        //      block, so x_i = rhs_i / D_i — one reciprocal per row at the end instead of one per step on the
        //      serial path (each step's chain is ~5 dependent fp64 operations instead of ~11 + a conversion round
        //      trip through MUFU.RCP).
        double a[N];
#pragma unroll
        for (int i = 0; i < N; ++i) a[i] = (lane < N + 2) ? A[i * W + lane] : 0.0;
#pragma unroll
        for (int k = 0; k < N; k += 2) {
          double* col = dres + ((k >> 1) & 1) * (2 * N);
          if (lane == k || lane == k + 1) {
#pragma unroll
            for (int i = 0; i < N; ++i) col[2 * i + (lane - k)] = a[i];
          }
          __syncwarp();
          const double2 pk = reinterpret_cast<const double2*>(col)[k];       // (A[k][k], A[k][k+1])
          const double2 pk1 = reinterpret_cast<const double2*>(col)[k + 1];  // (A[k+1][k], A[k+1][k+1])
          const double pa = pk.x, pb = pk.y, pc = pk1.x, pd = pk1.y;
          const double det = pa * pd - pb * pc;
          fail |= !(pa > 0.0) || !(det > 0.0) || !isfinite(det);
          // s = 2^(−2e), e = unbiased exponent of pa (clamped so that s stays a normal double)
          const int e = min(max((int)((__double_as_longlong(pa) >> 52) & 0x7ff) - 1023, -500), 500);
          const double sc = __longlong_as_double((long long)(1023 - 2 * e) << 52);
          const double r0 = a[k] * sc, r1 = a[k + 1] * sc;
          const double u0 = pd * r0 - pb * r1, u1 = pa * r1 - pc * r0;        // s·adj(P)·[r0; r1]
          const double ds = det * sc;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            if (i == k || i == k + 1) continue;
            const double2 c = reinterpret_cast<const double2*>(col)[i];      // (A[i][k], A[i][k+1])
            a[i] = fma(-c.y, u1, fma(-c.x, u0, a[i] * ds));
          }
          a[k] = u0;
          a[k + 1] = u1;
        }
        {
          // lane c < N owns D_c = a[c]: 1/D_c (fp32 seed + two Newton steps, full double precision) → strip
          double* rD = dres + 4 * N;
          if (lane < N) {
            double dg = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) dg = (i == lane) ? a[i] : dg;
            double rc = (double)__frcp_rn((float)dg);
            rc = rc * fma(-dg, rc, 2.0);
            rc = rc * fma(-dg, rc, 2.0);
            fail |= !(dg > 0.0) || !isfinite(rc) || !((float)dg > 0.f);
            rD[lane] = rc;
          }
          __syncwarp();
          if (lane == N || lane == N + 1) {
#pragma unroll
            for (int i = 0; i < N; ++i) a[i] *= rD[i];
          }
        }
        // solution columns N, N+1 back to shared memory (rows < N)
        if (lane == N || lane == N + 1) {
#pragma unroll
          for (int i = 0; i < N; ++i) A[i * W + lane] = a[i];
        }
        __syncwarp();
        }
      }
      // ---- Gauss–Jordan on [G + λI | q1 q2] by the whole CTA with 2×2 pivot blocks (SPD ⇒ every leading
      //      2×2 block is SPD, no pivoting; N = 4K + 2 is even). The matrix lives in registers: lane = column c,
      //      warp w owns rows w, w+8, w+16, w+24. Per step the pivot columns arrive by warp shuffles and the two
      //      pivot rows through a double-buffered shared row pair — one barrier per step, N/2 steps.
      if constexpr (N > kGJWarpN) {
        __syncthreads();
        constexpr int W = Lay::WS;
        double* A = mat;
        double* prow = dres;                          // 2 buffers × 2 rows × 32 columns (dres is consumed)
        double a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = warp + 8 * q;
          a[q] = (i < N && lane < N + 2) ? A[i * W + lane] : 0.0;
        }
        for (int k = 0, par = 0; k < N; k += 2, par ^= 1) {
          // owners of rows k, k+1 publish them (row k is row w = k % 8 of q = k / 8)
          double* pr = prow + par * 64;
          const int qk = k >> 3;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (q == qk && warp == (k & 7)) pr[lane] = a[q];
            if (q == ((k + 1) >> 3) && warp == ((k + 1) & 7)) pr[32 + lane] = a[q];
          }
          // this warp's rows' pivot-column entries A[i][k], A[i][k+1]
          double ck[4], ck1[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ck[q] = __shfl_sync(0xffffffffu, a[q], k);
            ck1[q] = __shfl_sync(0xffffffffu, a[q], k + 1);
          }
          __syncthreads();
          const double pa = pr[k], pb = pr[k + 1], pc = pr[32 + k], pd = pr[32 + k + 1];
          const double det = pa * pd - pb * pc;
          fail |= !(pa > 0.0) || !(det > 0.0) || !isfinite(det);
          // 1/det: fp32 seed + two Newton steps (relative error ~1e-28 → full double precision; det is the
          // determinant of an SPD 2×2 pivot block ≥ λ² ≫ FLT_MIN, so the seed is finite when det is)
          double idet = (double)__frcp_rn((float)det);
          idet = idet * fma(-det, idet, 2.0);
          idet = idet * fma(-det, idet, 2.0);
          const double r0 = pr[lane], r1 = pr[32 + lane];
          const double R0 = (pd * r0 - pb * r1) * idet, R1 = (pa * r1 - pc * r0) * idet;   // P⁻¹·[r0; r1]
          if (lane >= k + 2) {                        // columns ≤ k+1 are never read again
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int i = warp + 8 * q;
              a[q] = (i == k) ? R0 : (i == k + 1) ? R1 : fma(-ck1[q], R1, fma(-ck[q], R0, a[q]));
            }
          }
        }
        // solution columns N, N+1 back to shared memory (rows < N)
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = warp + 8 * q;
          if (i < N && (lane == N || lane == N + 1)) A[i * W + lane] = a[q];
        }
        __syncthreads();
      }
      // θ₁ from m1 = column N, m2 = column N+1 (rows e and L+e); fallback θ₀ on failure
      if (warp == 0) {
        __syncwarp();
        constexpr int W = Lay::WS;
        const double* A = mat;
          if (lane < N) fail |= !isfinite(A[lane * W + N]) || !isfinite(A[lane * W + N + 1]);
          fail = __any_sync(0xffffffffu, fail) ? 1 : 0;
          // tap e in K3c's real form: w·a + v·conj(a) = ar·cr + ai·ci with cr = (wr + vr, wi + vi),
          // ci = (vi − wi, wr − vr); from the solution columns (w = ((m1 + m2b)/2, (m2 − m1b)/2),
          // v = ((m1 − m2b)/2, (m2 + m1b)/2)) that is cr = (m1, m2), ci = (m1b, m2b) — one rounding each
          if (lane < L) {
            float2 cr, ci;
            if (fail) {                          // θ₀: w = g·w_cd, v = 0
              const float2 w0 = __ldg(&w_cd[lane]);
              cr = make_float2(g * w0.x, g * w0.y);
              ci = make_float2(-cr.y, cr.x);
            } else {
              const double m1 = A[lane * W + N], m2 = A[lane * W + N + 1];
              const double m1b = A[(L + lane) * W + N], m2b = A[(L + lane) * W + N + 1];
              if (wl) {
                cr = make_float2((float)m1, (float)m2);
                ci = make_float2((float)m1b, (float)m2b);
              } else {                           // strictly linear: w = (m1, m1b), v = 0
                cr = make_float2((float)m1, (float)m1b);
                ci = make_float2(-cr.y, cr.x);
              }
            }
            tr[lane] = cr;
            tr[L + lane] = ci;
          }
          if (lane == 0) tr[2 * L] = make_float2(__int_as_float(flags | (fail ? kFlagFail : 0)), 0.f);
          
        }
}
template <int K>
static void launch_k3_t(const float2* y, int64_t frame0, int64_t n_frames, const float2* w_cd, const int* clampcnt,
                        int64_t clamp_frame_off, const uint8_t* ref, uint8_t* dec, float2* z,
                        unsigned long long* counters, const K3Params& p, const CUtensorMap* ymaps, double* rec,
                        float2* threc, int num_sms, cudaStream_t s) {
  constexpr int smem = K3Layout<K>::TOTAL;
  cudaFuncSetAttribute(k3_frame_kernel<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k3_frame_kernel<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int64_t grid = (int64_t)num_sms * 2;
  if (grid > n_frames) grid = n_frames;
  k3_frame_kernel<K, 0><<<(unsigned)grid, K3_THREADS, smem, s>>>(y, frame0, (int)n_frames, w_cd, clampcnt,
                                                                 clamp_frame_off, nullptr, nullptr, nullptr, counters,
                                                                 p, rec, threc, ymaps[0], ymaps[1]);
  k3s_kernel<K><<<(unsigned)n_frames, K3S<K>::THREADS, 0, s>>>(rec, y, w_cd, threc, p);
  k3_frame_kernel<K, 1><<<(unsigned)grid, K3_THREADS, smem, s>>>(y, frame0, (int)n_frames, w_cd, clampcnt,
                                                                 clamp_frame_off, ref, dec, z, counters, p, rec,
                                                                 threc, ymaps[0], ymaps[1]);
}

// Tensor maps of the 2-sps buffer y (n_float2 entries) for the swizzled K ≤ 4 frame loads: a 2-D view of
// 64-B rows (8 float2 as 8-byte elements), boxes of 128 rows (map 0) and 8 rows (map 1), SWIZZLE_64B, OOB rows
// zero-filled. Returns false if the driver entry point is unavailable or the encode fails.
bool k3_encode_ymaps(const float2* y, int64_t n_float2, CUtensorMap* maps) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {8, (cuuint64_t)((n_float2 + 7) / 8)};
  const cuuint64_t strides[1] = {64};
  const cuuint32_t estr[2] = {1, 1};
  const cuuint32_t rows[2] = {128, 8};
  for (int i = 0; i < 2; ++i) {
    const cuuint32_t box[2] = {8, rows[i]};
    if (enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<float2*>(y), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

size_t k3_smem_bytes(int K) {
  switch (K) {
    case 1: return K3Layout<1>::TOTAL;
    case 2: return K3Layout<2>::TOTAL;
    case 3: return K3Layout<3>::TOTAL;
    case 4: return K3Layout<4>::TOTAL;
    case 5: return K3Layout<5>::TOTAL;
    case 6: return K3Layout<6>::TOTAL;
    case 7: return K3Layout<7>::TOTAL;
    default: return 0;
  }
}

// per-frame record sizes (bytes) of the K3a → K3s and K3s → K3c hand-offs
size_t k3_rec_bytes(int K) {
  switch (K) {
#define KK_R(KV) case KV: return (size_t)K3Rec<KV>::REC * 8;
    KK_R(1) KK_R(2) KK_R(3) KK_R(4) KK_R(5) KK_R(6) KK_R(7)
#undef KK_R
    default: return 0;
  }
}
size_t k3_threc_bytes(int K) { return (size_t)(2 * (2 * K + 1) + 2) * 8; }

void launch_k3(const float2* y, int64_t frame0, int64_t n_frames, int K, const float2* w_cd, const int* clampcnt,
               int64_t clamp_frame_off, const uint8_t* ref, uint8_t* dec, float2* z, unsigned long long* counters,
               const K3Params& p, const CUtensorMap* ymaps, double* rec, float2* threc, int num_sms, cudaStream_t s) {
#define KK_K3(KV) case KV: launch_k3_t<KV>(y, frame0, n_frames, w_cd, clampcnt, clamp_frame_off, ref, dec, z, counters, p, ymaps, rec, threc, num_sms, s); break;
  switch (K) {
    KK_K3(1) KK_K3(2) KK_K3(3) KK_K3(4) KK_K3(5) KK_K3(6) KK_K3(7)
    default: break;
  }
#undef KK_K3
}

}  // namespace kk
