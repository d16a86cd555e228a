// k2_mf.cu — K2: carrier removal, downshift to DC, RRC matched filter and 4→2 sps decimation.
//
// PAPER.md:82 (§2): the reconstructed field "is subsequently downshifted to DC for further processing.
// Frequency-domain static equalization and downsampling from 4 to 2 samples-per-symbol is performed by
// multiplication with an offline-optimized filter enabled by another FFT and IFFT pair." With the
// north-star carrier removal and SURVEY readings R4 (RRC 1 %, span 256 = 1025 taps), R5 (static filter =
// RRC MF), R6 (exact decimation by spectral fold), R8 (A_f = per-frame mean of E), R9 (LO indexed by the
// global sample: exp(−2πiσ·((lo_num·n) mod lo_den)/lo_den)):
//     b[n] = (E[n] − A_{f(n)})·LO[n]
//     tile t (global grid): x = b[3072t − 512, 3072t + 3584)
//     Y = FFT4096(x)·H   (H = DFT of the circularly centred taps, real, ×1/4096 folded in)
//     Y2[q] = Y[q] + Y[q + 2048], q < 2048            (fold = decimation by 2 in frequency)
//     y[1536t − 256 + p] = IFFT2048(Y2)[p], p ∈ [256, 1792)   (the alias-free, non-wrapped outputs)
// which equals y[m] = Σ_{j=−512}^{512} h[j]·b[2m − j] exactly (up to fp32 rounding).
//
// Mapping: persistent CTAs of 128 threads, one 4096-point tile at a time in shared memory (34.8 KB,
// padded 1 float2 per 16 to make the radix-16 Stockham scatter conflict-free); LO table resident in
// shared memory for the CTA's lifetime; H and the twiddles read through the read-only path (L1-resident).
// E is read with 16-byte vector loads; the 1536 kept outputs are written coalesced.
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {

constexpr int K2_THREADS = 128;
constexpr int K2_BUF = 4096 + 256;

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

// One radix-R Stockham pass over an N-point array in shared memory (in place, barrier-separated).
// tw: table of W_{Ns·R}^{r·k} laid out [r][k] (k < Ns), conjugated when DIR = +1.
template <int N, int R, int Ns, int DIR>
__device__ __forceinline__ void stockham_pass(float2* buf, const float2* __restrict__ tw, int tid) {
  constexpr int NJ = N / R;
  constexpr int PER = NJ / K2_THREADS;
  static_assert(PER >= 1 && NJ % K2_THREADS == 0, "pass shape");
  static_assert(NJ % 16 == 0 && (Ns == 1 ? R == 16 : Ns % 16 == 0), "padding algebra below");
  float2 v[PER][R];
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int j = tid + it * K2_THREADS;
    const float2* src = buf + pad16(j);             // pad16(j + r·NJ) = pad16(j) + r·(NJ + NJ/16)
#pragma unroll
    for (int r = 0; r < R; ++r) v[it][r] = src[r * (NJ + NJ / 16)];
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int j = tid + it * K2_THREADS;
    const int k = j & (Ns - 1);
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const float2 w = __ldg(&tw[r * Ns + k]);
        v[it][r] = DIR < 0 ? cmul(v[it][r], w) : cmulc(v[it][r], w);
      }
    }
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

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// CH = false: real H (RRC matched filter, north star). CH = true: complex H_cd = RRC × CD inverse (the paper's
// static filter, eq_mode DDLMS).
template <bool CH>
__global__ void __launch_bounds__(K2_THREADS, 4)
k2_mf_kernel(const float2* __restrict__ E, int64_t E_first, const float2* __restrict__ part, int64_t jb0,
             int64_t tile0, int64_t n_tiles, float2* __restrict__ y, int64_t y_first, int64_t y_count,
             const float* __restrict__ Hs, const float2* __restrict__ Hc, const float2* __restrict__ lo_tab,
             const float2* __restrict__ tw256, const float2* __restrict__ tw4096, const float2* __restrict__ tw2048,
             K2Params p) {
  __shared__ __align__(16) float2 buf[K2_BUF];
  __shared__ float2 A_s[2];
  __shared__ int qb_s;
  extern __shared__ float2 lo_s[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < p.lo_den; i += K2_THREADS) lo_s[i] = lo_tab[i];
  const int step256 = (int)(((int64_t)256 * p.lo_num) % p.lo_den);     // LO index step between r and r+1
  // LO index of local sample j of a tile: (lo_num·(s0 + j)) mod lo_den = (qb + offj) mod lo_den with the
  // tile base qb = (lo_num·s0) mod lo_den and the per-thread constant offj = (lo_num·j) mod lo_den
  int offj[2];
#pragma unroll
  for (int it = 0; it < 2; ++it) offj[it] = (int)(((int64_t)(tid + K2_THREADS * it) * p.lo_num) % p.lo_den);

  // tiles are visited from the END of the range: K1 wrote E front to back, so its most recent (L2-resident)
  // output is consumed first; K3 then walks y front to back, again reading K2's most recent writes first.
  for (int64_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    const int64_t t = tile0 + (n_tiles - 1 - ti);
    const int64_t s0 = t * kMfHop - kMfLead;                 // global sample of x[0]
    const int64_t fa = floordiv(s0, kFrameSamp);
    const int64_t fsplit = (fa + 1) * kFrameSamp;            // first sample of frame fa+1
    // ---- FFT4096 pass 1 (radix 16, Ns = 1) fused with the load: x_i = (E_i − A_f(i))·LO_i, i = j + 256 r.
    //      The E loads are issued first so their latency overlaps the carrier estimate below.
    float2 v[2][16];
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int j = tid + K2_THREADS * it;
      const float2* src = E + (s0 - E_first) + j;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[it][r] = __ldg(src + 256 * r);
    }
    // carrier estimates A_fa, A_fa+1 from K1's per-512-block sums (fixed order → deterministic); tile LO base
    if (warp < 2) {
      const int64_t f = fa + warp;
      float2 a = make_float2(0.f, 0.f);
      if (warp == 0 || s0 + kMfN > fsplit) a = part[f * 32 - jb0 + lane];
      a.x = warp_sum(a.x); a.y = warp_sum(a.y);
      if (lane == 0) A_s[warp] = make_float2(a.x * (1.0f / kFrameSamp), a.y * (1.0f / kFrameSamp));
    } else if (tid == 64) {
      const int sm = (int)(((s0 % p.lo_den) + p.lo_den) % p.lo_den);
      qb_s = (sm * p.lo_num) % p.lo_den;                    // < 4096², 32-bit
    }
    __syncthreads();
    // next tile's input (32 KiB of E) → L2 while this tile computes
    if (tid == 0 && ti + gridDim.x < n_tiles) {
      const int64_t s0n = (t - gridDim.x) * kMfHop - kMfLead;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(E + (s0n - E_first)), "r"(kMfN * 8) : "memory");
    }
    {
      const float2 A0 = A_s[0], A1 = A_s[1];
      const int qb = qb_s;
      const int isplit = (int)(fsplit - s0);                 // first local sample of frame fa+1
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = tid + K2_THREADS * it;
        int q = qb + offj[it];
        q -= (q >= p.lo_den) ? p.lo_den : 0;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const float2 A = (j + 256 * r < isplit) ? A0 : A1;
          v[it][r] = cmul(make_float2(v[it][r].x - A.x, v[it][r].y - A.y), lo_s[q]);
          q += step256; q -= (q >= p.lo_den) ? p.lo_den : 0;
        }
        dft_reg<16, -1>(v[it]);
        float2* dst = buf + 17 * j;                          // pad16(16j + r) = 17j + r
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r] = v[it][r];
      }
      __syncthreads();
    }
    stockham_pass<4096, 16, 16, -1>(buf, tw256, tid);
    // ---- FFT4096 pass 3 (Ns = 256) fused with × H and the fold: thread j owns Y[j + 256 r], r < 16, so
    //      Y2[j + 256 r] = Y[j + 256 r]·H[j + 256 r] + Y[j + 256 (r+8)]·H[j + 256 (r+8)], r < 8
    {
      float2 v[2][16];
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = tid + K2_THREADS * it;
        const float2* src = buf + pad16(j);
#pragma unroll
        for (int r = 0; r < 16; ++r) v[it][r] = src[r * (256 + 16)];
      }
      __syncthreads();
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = tid + K2_THREADS * it;
#pragma unroll
        for (int r = 1; r < 16; ++r) v[it][r] = cmul(v[it][r], __ldg(&tw4096[r * 256 + j]));
        dft_reg<16, -1>(v[it]);
        float2* dst = buf + pad16(j);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float2 a = v[it][r], b = v[it][r + 8];
          if constexpr (CH) {
            dst[r * (256 + 16)] = cadd(cmul(a, __ldg(&Hc[j + 256 * r])), cmul(b, __ldg(&Hc[j + 256 * (r + 8)])));
          } else {
            const float ha = __ldg(&Hs[j + 256 * r]), hb = __ldg(&Hs[j + 256 * (r + 8)]);
            dst[r * (256 + 16)] = make_float2(fmaf(a.x, ha, b.x * hb), fmaf(a.y, ha, b.y * hb));
          }
        }
      }
      __syncthreads();
    }
    // ---- IFFT2048 (radix 16, 16, 8); the last pass stores the kept outputs straight to y
    stockham_pass<2048, 16, 1, +1>(buf, nullptr, tid);
    stockham_pass<2048, 16, 16, +1>(buf, tw256, tid);
    {
      const int64_t m_base = t * kMfKeep - kMfKeep0;          // y index of IFFT output p: m_base + p
      float2 v[2][8];
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = tid + K2_THREADS * it;
        const float2* src = buf + pad16(j);
#pragma unroll
        for (int r = 0; r < 8; ++r) v[it][r] = src[r * (256 + 16)];
      }
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = tid + K2_THREADS * it;
#pragma unroll
        for (int r = 1; r < 8; ++r) v[it][r] = cmulc(v[it][r], __ldg(&tw2048[r * 256 + j]));
        dft_reg<8, +1>(v[it]);
#pragma unroll
        for (int r = 1; r < 7; ++r) {                        // p = j + 256 r ∈ [256, 1792) ⇔ 1 ≤ r ≤ 6
          const int64_t m = m_base + j + 256 * r;
          if (m >= y_first && m < y_first + y_count) y[m - y_first] = v[it][r];
        }
      }
      __syncthreads();                                        // buf is rewritten by the next tile
    }
  }
}

void launch_k2(const float2* E, int64_t E_first, const float2* part, const int* /*clampcnt*/, int64_t jb0,
               int64_t tile0, int64_t n_tiles, float2* y, int64_t y_first, int64_t y_count, const float* Hs,
               const float2* Hc, const float2* lo_tab, const float2* tw256, const float2* tw4096,
               const float2* tw2048, const K2Params& p, int num_sms, cudaStream_t s) {
  int per_sm = 4;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > n_tiles) grid = n_tiles;
  const size_t dyn = (size_t)p.lo_den * sizeof(float2);
  if (Hc)
    k2_mf_kernel<true><<<(unsigned)grid, K2_THREADS, dyn, s>>>(E, E_first, part, jb0, tile0, n_tiles, y, y_first,
                                                               y_count, Hs, Hc, lo_tab, tw256, tw4096, tw2048, p);
  else
    k2_mf_kernel<false><<<(unsigned)grid, K2_THREADS, dyn, s>>>(E, E_first, part, jb0, tile0, n_tiles, y, y_first,
                                                                y_count, Hs, Hc, lo_tab, tw256, tw4096, tw2048, p);
}

}  // namespace kk
