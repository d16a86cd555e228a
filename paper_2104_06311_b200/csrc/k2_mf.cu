// k2_mf.cu — K2: carrier removal, downshift to DC, RRC matched filter and 4→2 sps decimation.
//
// PAPER.md:82 (§2): the reconstructed field "is subsequently downshifted to DC for further processing.
// Frequency-domain static equalization and downsampling from 4 to 2 samples-per-symbol is performed by
// multiplication with an offline-optimized filter enabled by another FFT and IFFT pair." With the
// north-star carrier removal and SURVEY readings R4 (RRC 1 %, span 256 = 1025 taps), R5 (static filter =
// RRC MF), R6 (exact decimation by spectral fold), R8 (A_f = per-frame mean of E), R9 (LO indexed by the
// global sample: exp(−2πiσ·((lo_num·n) mod lo_den)/lo_den)):
//     b[n] = (E[n] − A_{f(n)})·LO[n]
//     tile t (global grid, N = 4096 or 8192, hop N − 1024, keep N/2 − 512):
//     x = b[hop·t − 512, hop·t − 512 + N)
//     Y = FFT_N(x)·H   (H = DFT_N of the circularly centred taps, ×1/N folded in)
//     Y2[q] = Y[q] + Y[q + N/2], q < N/2              (fold = decimation by 2 in frequency)
//     y[keep·t − 256 + p] = IFFT_{N/2}(Y2)[p], p ∈ [256, N/2 − 256)   (the alias-free, non-wrapped outputs)
// which equals y[m] = Σ_{j=−512}^{512} h[j]·b[2m − j] exactly (up to fp32 rounding) for either grid.
// The 8192/7168 grid does ≈ 17 % fewer FFT flops and 14 % fewer shared-memory element passes per sample.
//
// Mapping: persistent CTAs of N/32 threads (32 values per thread per radix-16 pass), one tile at a time in
// shared memory (padded 1 float2 per 16 to make the radix-16 Stockham scatter conflict-free); LO table
// resident in shared memory for the CTA's lifetime; H and the twiddles read through the read-only path.
// FFT_N = 16 · 16 · (N/256), IFFT_{N/2} = 16 · 16 · (N/512); the first pass loads E straight from global
// memory, the last forward pass applies ×H and the fold, the last inverse pass stores y.
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {


__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

__host__ __device__ constexpr int hibit16(int r) { return r >= 8 ? 8 : r >= 4 ? 4 : r >= 2 ? 2 : 1; }

// v[r] ·= w^r (DIR < 0) or ·= conj(w)^r (DIR > 0) for r = 1..R−1, R ≤ 16, with tw[r·stride] = w^r. Only the
// entries r = 1, 2, 4, 8 are loaded; every other power is the product of two loaded/formed ones (≤ 3 roundings
// deep). K2 is bound by L1/shared-memory wavefronts, so 11 of 15 twiddle loads move to the FMA pipe (2 packed
// instructions per product).
template <int R, int DIR>
__device__ __forceinline__ void apply_twiddles(float2 (&v)[R], const float2* __restrict__ tw, int stride) {
  float2 w[R];
#pragma unroll
  for (int r = 1; r < R; r <<= 1) w[r] = __ldg(tw + r * stride);
#pragma unroll
  for (int r = 3; r < R; ++r)
    if (r != hibit16(r)) w[r] = cmul(w[hibit16(r)], w[r - hibit16(r)]);
#pragma unroll
  for (int r = 1; r < R; ++r) v[r] = DIR < 0 ? cmul(v[r], w[r]) : cmulc(v[r], w[r]);
}

// One radix-R Stockham pass over an N-point array in shared memory, src → dst (the same buffer: in place, a
// barrier between the reads and the writes; different buffers: no such barrier), closing barrier.
// tw: table of W_{Ns·R}^{r·k} laid out [r][k] (k < Ns), conjugated when DIR = +1.
template <int N, int R, int Ns, int DIR, int T>
__device__ __forceinline__ void stockham_pass(const float2* srcb, float2* buf, const float2* __restrict__ tw, int tid) {
  constexpr int NJ = N / R;
  constexpr int PER = NJ / T;
  static_assert(PER >= 1 && NJ % T == 0, "pass shape");
  static_assert(NJ % 16 == 0 && (Ns == 1 ? R == 16 : Ns % 16 == 0), "padding algebra below");
  float2 v[PER][R];
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int j = tid + it * T;
    const float2* src = srcb + pad16(j);            // pad16(j + r·NJ) = pad16(j) + r·(NJ + NJ/16)
#pragma unroll
    for (int r = 0; r < R; ++r) v[it][r] = src[r * (NJ + NJ / 16)];
  }
  if (srcb == buf) __syncthreads();
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int j = tid + it * T;
    const int k = j & (Ns - 1);
    if (Ns > 1) apply_twiddles<R, DIR>(v[it], tw + k, Ns);
    dft_reg<R, DIR>(v[it]);
    const int idxD = (j / Ns) * Ns * R + k;
    // Ns = 1 (R = 16): pad16(16j + r) = 17j + r;  Ns ≥ 16: pad16(idxD + r·Ns) = pad16(idxD) + r·(Ns + Ns/16)
    float2* dst = buf + (Ns == 1 ? 17 * j : pad16(idxD));
    constexpr int stride = (Ns == 1) ? 1 : (Ns + Ns / 16);
#pragma unroll
    for (int r = 0; r < R; ++r) dst[r * stride] = v[it][r];
  }
  __syncthreads();
}

// ⌊a / kFrameSamp⌋ for any sign: an arithmetic shift (kFrameSamp = 2^14)
static_assert(kFrameSamp == 16384, "frame index by shift");
__device__ __forceinline__ int64_t frame_of(int64_t a) { return a >> 14; }

// CH = false: real H (RRC matched filter, north star). CH = true: complex H_cd = RRC × CD inverse (the paper's
// static filter, eq_mode DDLMS). NF = 4096 or 8192 (the OLS grid).
// Resident CTAs per SM of the persistent grid (register-limited: 65536 / (T · regs)).
#ifndef K2_CTAS_4096
#define K2_CTAS_4096 4
#endif
template <int NF>
constexpr int k2_ctas_per_sm() { return NF == 4096 ? K2_CTAS_4096 : 16384 / NF; }

template <int NF, bool CH, bool SP = CH>
__global__ void __launch_bounds__(NF / 32, k2_ctas_per_sm<NF>())
k2_mf_kernel(const float2* __restrict__ E, int64_t E_first, const float2* __restrict__ part, int64_t jb0,
             int64_t tile0, int64_t n_tiles, float2* __restrict__ y, int64_t y_first, int64_t y_count,
             const float* __restrict__ Hs, const float2* __restrict__ Hc, const float2* __restrict__ lo_tab,
             const float2* __restrict__ tw256, const float2* __restrict__ twN, const float2* __restrict__ twI,
             K2Params p) {
  constexpr int T = NF / 32;                 // threads
  constexpr int NI = NF / 2;                 // inverse size
  constexpr int NJ1 = NF / 16;               // pass-1 stride (= 2T)
  constexpr int R3 = NF / 256;               // last forward radix (16 / 32)
  constexpr int RI3 = NI / 256;              // last inverse radix (8 / 16)
  constexpr int HOP = NF - 1024, KEEP = NI - 512, LEAD = 512, KEEP0 = 256;
  constexpr int PER3 = 256 / T;              // last-pass DFTs per thread (2 / 1)
  extern __shared__ __align__(16) float2 k2_smem[];
  float2* buf = k2_smem;                                   // NF + NF/16 (padded tile)
  __shared__ float2 A_s[2][2];                             // [tile parity][frame fa, fa + 1]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // LO of local sample i = j + NJ1·r of a tile starting at global sample s0 (R9, exponents add mod lo_den):
  //   LO[(lo_num·(s0 + i)) mod lo_den] = φ_t · λ_j · ρ^r,  φ_t = LO[qb_t], qb_t = (lo_num·s0) mod lo_den,
  //   λ_j = LO[(lo_num·j) mod lo_den] (per thread, loaded once), ρ^r = LO[(r·NJ1·lo_num) mod lo_den] (p.rho)
  // — no per-sample table lookups or index arithmetic; qb_t advances by a fixed dq between a CTA's tiles.
  float2 lam[2];
#pragma unroll
  for (int it = 0; it < 2; ++it) lam[it] = __ldg(&lo_tab[(int)(((int64_t)(tid + T * it) * p.lo_num) % p.lo_den)]);
  int qb;
  {
    const int64_t s0f = (tile0 + (n_tiles - 1 - (int64_t)blockIdx.x)) * HOP - LEAD;
    qb = (int)((((s0f % p.lo_den) + p.lo_den) % p.lo_den) * p.lo_num % p.lo_den);
  }
  const int dq = (int)(((p.lo_den - ((int64_t)gridDim.x * HOP) % p.lo_den) % p.lo_den) * p.lo_num % p.lo_den);

  // warps 0, 1: this lane's K1 block sum of the tile's first / second frame (A_f, R5), loaded one tile ahead so
  // that the carrier estimate at a tile's start does not wait for a global load
  auto load_part = [&](int64_t ti_) -> float2 {
    const int64_t s0_ = (tile0 + (n_tiles - 1 - ti_)) * HOP - LEAD;
    const int64_t fa_ = frame_of(s0_);
    float2 a = make_float2(0.f, 0.f);
    if (warp == 0 || s0_ + NF > (fa_ + 1) * kFrameSamp) a = part[(fa_ + warp) * 32 - jb0 + lane];
    return a;
  };
  // the carrier estimates of a tile are formed one tile ahead (warps 0, 1, into A_s[parity]), so that the tile
  // start needs no barrier: the previous tile's closing barrier orders them
  // (the lane's block sum `pa` of the tile after next is loaded one tile earlier still, so no global-load wait)
  auto form_A = [&](float2 a, int par) {
    if (warp < 2) {
      a.x = warp_sum(a.x); a.y = warp_sum(a.y);
      if (lane == 0) A_s[par][warp] = make_float2(a.x * (1.0f / kFrameSamp), a.y * (1.0f / kFrameSamp));
    }
  };
  float2 pa = make_float2(0.f, 0.f);
  if (warp < 2 && (int64_t)blockIdx.x < n_tiles) form_A(load_part(blockIdx.x), 0);
  if (warp < 2 && (int64_t)blockIdx.x + gridDim.x < n_tiles) pa = load_part(blockIdx.x + gridDim.x);
  __syncthreads();
  int par = 0;

  // tiles are visited from the END of the range: K1 wrote E front to back, so its most recent (L2-resident)
  // output is consumed first; K3 then walks y front to back, again reading K2's most recent writes first.
  for (int64_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    const int64_t t = tile0 + (n_tiles - 1 - ti);
    const int64_t s0 = t * HOP - LEAD;                       // global sample of x[0]
    const int64_t fa = frame_of(s0);
    const int64_t fsplit = (fa + 1) * kFrameSamp;            // first sample of frame fa+1 (NF < 16384: ≤ 2 frames)
    // ---- FFT pass 1 (radix 16, Ns = 1) fused with the load: x_i = (E_i − A_f(i))·LO_i, i = j + NJ1·r.
    //      The E loads are issued first so their latency overlaps the carrier estimate below.
    float2 v[2][16];
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int j = tid + T * it;
      const float2* src = E + (s0 - E_first) + j;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[it][r] = __ldg(src + NJ1 * r);
    }
    const float2 phi = __ldg(&lo_tab[qb]);
    qb += dq; qb -= (qb >= p.lo_den) ? p.lo_den : 0;
    // next tile's input (NF·8 bytes of E) → L2 while this tile computes
    if (tid == 0 && ti + gridDim.x < n_tiles) {
      const int64_t s0n = (t - gridDim.x) * HOP - LEAD;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(E + (s0n - E_first)), "r"(NF * 8) : "memory");
    }
    {
      // carrier estimates A_fa, A_fa+1 from K1's per-512-block sums (fixed order → deterministic), formed during
      // the previous tile
      const float2 A0 = A_s[par][0], A1 = A_s[par][1];
      const int isplit = (int)(fsplit - s0);                 // first local sample of frame fa+1
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = tid + T * it;
        const float2 c = cmul(phi, lam[it]);                 // LO of sample j (r = 0)
        if (isplit >= NF) {                                  // tile inside one frame (uniform branch)
#pragma unroll
          for (int r = 0; r < 16; ++r) v[it][r] = cmul(csub(v[it][r], A0), r == 0 ? c : cmul(c, p.rho[r]));
        } else {
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            const float2 A = (j + NJ1 * r < isplit) ? A0 : A1;
            v[it][r] = cmul(csub(v[it][r], A), r == 0 ? c : cmul(c, p.rho[r]));
          }
        }
        dft_reg<16, -1>(v[it]);
        float2* dst = buf + 17 * j;                          // pad16(16j + r) = 17j + r
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r] = v[it][r];
      }
      __syncthreads();
    }
    stockham_pass<NF, 16, 16, -1, T>(buf, buf, tw256, tid);
    // ---- last forward pass (radix R3, Ns = 256) fused with × H and the fold: thread j owns Y[j + 256 r],
    //      r < R3, so Y2[j + 256 r] = Y[j + 256 r]·H[j + 256 r] + Y[j + 256 (r + R3/2)]·H[…], r < R3/2
    {
      float2 v3[PER3][R3];
#pragma unroll
      for (int it = 0; it < PER3; ++it) {
        const int j = tid + T * it;
        const float2* src = buf + pad16(j);
#pragma unroll
        for (int r = 0; r < R3; ++r) v3[it][r] = src[r * (256 + 16)];
      }
      // no barrier: the folded outputs Y2[j + 256 r] (r < R3/2) overwrite only this thread's own inputs
#pragma unroll
      for (int it = 0; it < PER3; ++it) {
        const int j = tid + T * it;
        apply_twiddles<R3, -1>(v3[it], twN + j, 256);
        dft_reg<R3, -1>(v3[it]);
        float2* dst = buf + pad16(j);
#pragma unroll
        for (int r = 0; r < R3 / 2; ++r) {
          const float2 a = v3[it][r], b = v3[it][r + R3 / 2];
          if constexpr (CH) {
            float2 yv = cmul(a, __ldg(&Hc[j + 256 * r]));        // + b·H[…] in the cmul form: 4 packed ops
            cmac2(yv, b, __ldg(&Hc[j + 256 * (r + R3 / 2)]));
            dst[r * (256 + 16)] = yv;
          } else {
            const float ha = __ldg(&Hs[j + 256 * r]), hb = __ldg(&Hs[j + 256 * (r + R3 / 2)]);
            float2 yv = cscale(b, hb);                         // packed: b·hb, then + a·ha (same roundings)
            ffma2s(yv, ha, a);
            dst[r * (256 + 16)] = yv;
          }
        }
      }
      __syncthreads();
    }
    // ---- IFFT_{NI} (radix 16, 16, RI3); the last pass stores the kept outputs straight to y. The NI-point
    //      array needs half the tile buffer, so its first two passes ping-pong between the halves (A → B → A):
    //      no barrier between a pass's reads and its writes (the fold's reads of B ended before its barrier)
    stockham_pass<NI, 16, 1, +1, T>(buf, buf + (NI + NI / 16), nullptr, tid);
    stockham_pass<NI, 16, 16, +1, T>(buf + (NI + NI / 16), buf, tw256, tid);
    {
      const int64_t m_base = t * KEEP - KEEP0;                // y index of IFFT output p: m_base + p
      float2 v3[PER3][RI3];
#pragma unroll
      for (int it = 0; it < PER3; ++it) {
        const int j = tid + T * it;
        const float2* src = buf + pad16(j);
#pragma unroll
        for (int r = 0; r < RI3; ++r) v3[it][r] = src[r * (256 + 16)];
      }
      float pw[PER3][RI3];                                    // DDLMS mode: |y|² of the symbol-centre outputs
#pragma unroll
      for (int it = 0; it < PER3; ++it) {
        const int j = tid + T * it;
        apply_twiddles<RI3, +1>(v3[it], twI + j, 256);
        dft_reg<RI3, +1>(v3[it]);
        const bool inside = (m_base + 256 >= y_first) && (m_base + NI - 256 <= y_first + y_count);   // tile-uniform
#pragma unroll
        for (int r = 1; r < RI3 - 1; ++r) {                  // p = j + 256 r ∈ [256, NI − 256) ⇔ 1 ≤ r ≤ RI3 − 2
          const int64_t m = m_base + j + 256 * r;
          if (inside || (m >= y_first && m < y_first + y_count)) y[m - y_first] = v3[it][r];
          if constexpr (SP) pw[it][r] = (j & 1) ? 0.f : fmaf(v3[it][r].x, v3[it][r].x, v3[it][r].y * v3[it][r].y);
        }
      }
      if constexpr (SP) {                                     // K3′'s AGC segment powers
        // per-256-symbol (512-sample) segment power for K3′'s AGC: output p = j + 256 r lies in tile segment
        // (r − 1)/2 for every j, so each thread sums its values per segment, then warp sums and the warps'
        // partials in fixed order → deterministic. Segment g (global) = m / 512.
        constexpr int NSEG = KEEP / 512;                      // 3 (4096 grid) or 7 (8192 grid)
        constexpr int NW = T / 32;
        float* red = reinterpret_cast<float*>(buf + NF + NF / 16);   // NSEG × NW floats past the tile
#pragma unroll
        for (int sg = 0; sg < NSEG; ++sg) {
          float a = 0.f;
#pragma unroll
          for (int it = 0; it < PER3; ++it) a += pw[it][2 * sg + 1] + pw[it][2 * sg + 2];
          a = warp_sum(a);
          if (lane == 0) red[sg * NW + warp] = a;
        }
        __syncthreads();
        if (tid < NSEG) {
          float a = 0.f;
          for (int w8 = 0; w8 < NW; ++w8) a += red[tid * NW + w8];
          p.seg_pow[t * NSEG + tid - p.seg_first] = a;
        }
      }
      if (ti + gridDim.x < n_tiles) {                         // the next tile's carrier estimates
        form_A(pa, par ^ 1);
        if (warp < 2 && ti + 2 * (int64_t)gridDim.x < n_tiles) pa = load_part(ti + 2 * gridDim.x);
      }
      par ^= 1;
      __syncthreads();                                        // buf is rewritten by the next tile
    }
  }
}

template <int NF, bool CH, bool SP>
static void launch_k2_t(const float2* E, int64_t E_first, const float2* part, int64_t jb0, int64_t tile0,
                        int64_t n_tiles, float2* y, int64_t y_first, int64_t y_count, const float* Hs,
                        const float2* Hc, const float2* lo_tab, const float2* tw256, const float2* twN,
                        const float2* twI, const K2Params& p, int num_sms, cudaStream_t s) {
  constexpr int T = NF / 32;
  int64_t grid = (int64_t)num_sms * k2_ctas_per_sm<NF>();
  if (grid > n_tiles) grid = n_tiles;
  const size_t dyn = (size_t)(NF + NF / 16) * sizeof(float2) +
                     (SP ? (size_t)(NF / 2 - 512) / 512 * (NF / 1024) * sizeof(float) : 0);
  cudaFuncSetAttribute(k2_mf_kernel<NF, CH, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  k2_mf_kernel<NF, CH, SP><<<(unsigned)grid, T, dyn, s>>>(E, E_first, part, jb0, tile0, n_tiles, y, y_first, y_count,
                                                      Hs, Hc, lo_tab, tw256, twN, twI, p);
}

void launch_k2(int nf, const float2* E, int64_t E_first, const float2* part, const int* /*clampcnt*/, int64_t jb0,
               int64_t tile0, int64_t n_tiles, float2* y, int64_t y_first, int64_t y_count, const float* Hs,
               const float2* Hc, const float2* lo_tab, const float2* tw256, const float2* twN,
               const float2* twI, const K2Params& p, int num_sms, cudaStream_t s) {
  // real H (RRC) | complex H (RRC × CD inverse) with K3′'s segment powers (p.seg_pow) | complex H alone (static CD)
#define KK_K2(NFV, CHV, SPV) launch_k2_t<NFV, CHV, SPV>(E, E_first, part, jb0, tile0, n_tiles, y, y_first, y_count, Hs, Hc, lo_tab, tw256, twN, twI, p, num_sms, s)
  if (nf == 8192) {
    if (Hc && p.seg_pow) KK_K2(8192, true, true);
    else if (Hc) KK_K2(8192, true, false);
    else KK_K2(8192, false, false);
  } else {
    if (Hc && p.seg_pow) KK_K2(4096, true, true);
    else if (Hc) KK_K2(4096, true, false);
    else KK_K2(4096, false, false);
  }
#undef KK_K2
}

}  // namespace kk
