// k1u_kk.cu — K1U: K1 with 2× KK upsampling (SPEC S:277 upsample_factor, S:375;
// DESIGN.md §3 "KK upsampling"). Same outputs and layout as K1 (E at 4 sps, per-512-block ΣE partials and
// ADC clamp counts), so K2/K3 are unchanged.
//
// Per 4-sps Hilbert block j (outputs [512j, 512j + 512)) the 8-sps window is P ∈ [1024j − 512, +2048):
//   I₂[2n] = I[n];  I₂[2n+1] = Σ_{i=1..8} 2c_i·(I[n+1−i] + I[n+i])          half-band interpolation
//   a₂ = ½·ln max(I₂/I_ref, ε_rel);  φ₂ = σ·Hilbert₂₀₄₈(a₂)                     O2, O3 at 8 sps
//   E₂ = √I_ref·e^{a₂}·e^{iφ₂};  E[n] = ½E₂[2n] + Σ_i c_i·(E₂[2n−2i+1] + E₂[2n+2i−1])   O4 + decimation
// with c_i = f[2i−1] the odd half-band taps (host-computed in fp64) and E₂ taken from the block's own
// window (positions [497, 1551) of it).
//
// Mapping: 4 warps per CTA, one warp per PAIR of blocks (two real windows packed as re/im of one
// complex 2048-point FFT), CTA = 8 blocks = 4096 outputs. The CTA stages its 4640 ADC samples with one
// TMA bulk copy, converts them to I/I_ref once (ADC clamp counts per block), interpolates and takes the
// log for all 9216 window samples once (a₂ in shared memory, shared by overlapping windows), then each
// warp runs the FFT2048 = 64 × 32 decomposition in registers:
//   radix-2 stage + 2×DFT32 (= DFT64 over r of x[l + 32r], lane l)  → twiddle W₂₀₄₈^{l·k1}
//   → transpose (smem, stride 33, even/odd k1 halves) → 2×DFT32 over l → X[k1 + 64k2]
//   × (−i·sgn q) → the same steps inverted → lane l holds positions l + 32r, l + 1024 + 32r.
// E₂ at the positions the decimation needs goes to the warp's smem scratch split into polyphase arrays
// (even samples Ev, odd samples Od); each lane makes 4 adjacent outputs per step from one 20-sample Od
// window (10 conflict-free 16-B loads, 16-B lane stride) and stores them with 16-B coalesced stores.
// Occupancy: 255 registers (64 complex values per lane) and 90 KB smem → 2 CTAs = 8 warps per SM; the
// next step is splitting each FFT2048 over two warps (≤ 128 registers) for 16 warps per SM.
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {

constexpr int K1U_WARPS = 4;
constexpr int K1U_THREADS = K1U_WARPS * 32;
constexpr int K1U_BLOCKS = 2 * K1U_WARPS;            // 4-sps Hilbert blocks per CTA
constexpr int K1U_OUT = K1U_BLOCKS * kHilbertHop;    // 4096 outputs per CTA
constexpr int K1U_PAD = kK1uPad;                     // 272 staged samples before/after (256 + 16)
constexpr int K1U_IN = K1U_OUT + 2 * K1U_PAD;        // 4640
constexpr int K1U_UP = 2 * K1U_OUT + 1024;           // 9216 window samples at 8 sps
constexpr int K1U_E2 = 1088;                         // E₂ positions kept per block: window [480, 1568)
constexpr int K1U_E2_0 = 480;
constexpr size_t K1U_SMEM = (size_t)K1U_UP * 4 + (size_t)K1U_IN * 4 + (size_t)K1U_WARPS * K1U_E2 * 8 + 16 +
                            K1U_BLOCKS * 4;

template <typename Tin>
__global__ void __launch_bounds__(K1U_THREADS, 2)
k1u_kk_kernel(const Tin* __restrict__ adc0, float2* __restrict__ E, float2* __restrict__ part,
              int* __restrict__ clampcnt, const float2* __restrict__ tw, K1UParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* a2 = reinterpret_cast<float*>(smem);
  float* Ib = a2 + K1U_UP;
  float2* ws = reinterpret_cast<float2*>(Ib + K1U_IN);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ws + K1U_WARPS * K1U_E2);
  int* cblk = reinterpret_cast<int*>(bar + 2);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t cta = blockIdx.x;
  const Tin* src = adc0 + cta * (int64_t)K1U_OUT;
  Tin* stage = reinterpret_cast<Tin*>(ws);            // TMA landing zone (aliases the warp scratch)
  constexpr uint32_t bytes = (uint32_t)(K1U_IN * sizeof(Tin));

  if (tid == 0) mbar_init(bar, 1);
  if (tid < K1U_BLOCKS) cblk[tid] = 0;
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, bytes);
    tma_bulk_g2s(stage, src, bytes, bar);
  }
  mbar_wait(bar, 0);

  // ---- I/I_ref for the staged samples; ADC clamp count per kept 512-block (8-sample groups)
  const float sc_in = p.adc_scale * p.inv_iref, off_in = -p.adc_offset * p.adc_scale * p.inv_iref;
  for (int gi = tid; gi < K1U_IN / 8; gi += K1U_THREADS) {
    float x[8];
    if constexpr (sizeof(Tin) == 2) {
      const int4 raw = reinterpret_cast<const int4*>(stage)[gi];
      const short* h = reinterpret_cast<const short*>(&raw);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fmaf((float)h[j], sc_in, off_in);
    } else if constexpr (sizeof(Tin) == 1) {
      const uint2 raw = reinterpret_cast<const uint2*>(stage)[gi];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fmaf((float)(((j < 4 ? raw.x : raw.y) >> (8 * (j & 3))) & 0xffu), sc_in, off_in);
    } else {
      const float4 r0 = reinterpret_cast<const float4*>(stage)[2 * gi];
      const float4 r1 = reinterpret_cast<const float4*>(stage)[2 * gi + 1];
      const float rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fmaf(rr[j], sc_in, off_in);
    }
    int ncl = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) ncl += !(x[j] >= p.clamp_rel);
    reinterpret_cast<float4*>(Ib)[2 * gi] = make_float4(x[0], x[1], x[2], x[3]);
    reinterpret_cast<float4*>(Ib)[2 * gi + 1] = make_float4(x[4], x[5], x[6], x[7]);
    if (ncl) {
      const int o = 8 * gi - K1U_PAD;
      if (o >= 0 && o < K1U_OUT) atomicAdd(&cblk[o >> 9], ncl);
    }
  }
  __syncthreads();

  // ---- a₂ over the 9216 window samples: window sample P ↔ Ib index P/2 + 16 (P even).
  // 8 consecutive m per step (P = 2m, 2m+1): one 24-float window Ib[8g + 8, 8g + 32) in registers.
  for (int g = tid; g < K1U_UP / 16; g += K1U_THREADS) {
    float w[24];
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float4 q = reinterpret_cast<const float4*>(Ib + 8 * g + 8)[t];
      w[4 * t] = q.x; w[4 * t + 1] = q.y; w[4 * t + 2] = q.z; w[4 * t + 3] = q.w;
    }
    float out[16];
#pragma unroll
    for (int u = 0; u < 8; ++u) {            // m = 8g + u: I[m] = Ib[m + 16] = w[u + 8]
      const float ev = w[u + 8];
      float od = 0.f;
#pragma unroll
      for (int i = 1; i <= 8; ++i) od = fmaf(p.c2[i - 1], w[u + 8 + 1 - i] + w[u + 8 + i], od);
      out[2 * u] = 0.34657359027997264f * __log2f(ev >= p.clamp_rel ? ev : p.clamp_rel);
      out[2 * u + 1] = 0.34657359027997264f * __log2f(od >= p.clamp_rel ? od : p.clamp_rel);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      reinterpret_cast<float4*>(a2 + 16 * g)[t] = make_float4(out[4 * t], out[4 * t + 1], out[4 * t + 2], out[4 * t + 3]);
  }
  __syncthreads();

  // ---- FFT2048 pair per warp
  float2* S = ws + warp * K1U_E2;
  const float* w0 = a2 + (2 * warp) * 1024;          // window of block 2w (local 8-sps start)
  const float* w1 = w0 + 1024;
  float2 va[32], vb[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    va[r] = make_float2(w0[lane + 32 * r], w1[lane + 32 * r]);
    vb[r] = make_float2(w0[lane + 1024 + 32 * r], w1[lane + 1024 + 32 * r]);
  }
  // DFT64 over r of x[lane + 32r] (DIF radix-2 stage, then DFT32 of each half): va[k] = Y[2k], vb[k] = Y[2k+1]
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float2 a = va[i], b = vb[i];
    va[i] = cadd(a, b);
    float2 wv = unit_root64(i);
    wv.y = -wv.y;                                   // W₆₄^{i} = e^{−2πi·i/64}
    vb[i] = cmul(csub(a, b), wv);
  }
  dft_reg<32, -1>(va);
  dft_reg<32, -1>(vb);
  // twiddle W₂₀₄₈^{l·k1}, table tw[k1·32 + l]
#pragma unroll
  for (int k = 1; k < 32; ++k) va[k] = cmul(va[k], __ldg(&tw[(2 * k) * 32 + lane]));
#pragma unroll
  for (int k = 0; k < 32; ++k) vb[k] = cmul(vb[k], __ldg(&tw[(2 * k + 1) * 32 + lane]));
  // transpose: lane m ← Y'[l][2m] (va[l]) and Y'[l][2m+1] (vb[l])
#pragma unroll
  for (int k = 0; k < 32; ++k) S[lane * 33 + k] = va[k];
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) va[l] = S[l * 33 + lane];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) S[lane * 33 + k] = vb[k];
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) vb[l] = S[l * 33 + lane];
  __syncwarp();
  dft_reg<32, -1>(va);                              // X[2m + 64k2], k2 = 0..31
  dft_reg<32, -1>(vb);                              // X[2m + 1 + 64k2]

  // −i·sgn(q), q = k1 + 64k2: k2 < 16 ⇒ 0 < q < 1024 (except q = 0); k2 ≥ 16 ⇒ q > 1024 (except 1024)
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const float2 x = va[r], y = vb[r];
    va[r] = (r < 16) ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
    vb[r] = (r < 16) ? make_float2(y.y, -y.x) : make_float2(-y.y, y.x);
  }
  if (lane == 0) { va[0] = make_float2(0.f, 0.f); va[16] = make_float2(0.f, 0.f); }

  dft_reg<32, +1>(va);                              // Z[2m][l']
  dft_reg<32, +1>(vb);                              // Z[2m+1][l']
#pragma unroll
  for (int k = 0; k < 32; ++k) S[lane * 33 + k] = va[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) va[k] = S[k * 33 + lane];   // lane l': va[k] = Z[2k][l']
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) S[lane * 33 + k] = vb[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) vb[k] = S[k * 33 + lane];   // vb[k] = Z[2k+1][l']
  __syncwarp();
#pragma unroll
  for (int k = 1; k < 32; ++k) va[k] = cmulc(va[k], __ldg(&tw[(2 * k) * 32 + lane]));
#pragma unroll
  for (int k = 0; k < 32; ++k) vb[k] = cmulc(vb[k], __ldg(&tw[(2 * k + 1) * 32 + lane]));
  // inverse DFT64 over k1 (DIT): A = IDFT32(even), B = IDFT32(odd); x[r] = A + W^{−r}… (conj roots)
  dft_reg<32, +1>(va);
  dft_reg<32, +1>(vb);
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const float2 t = cmul(vb[r], unit_root64(r));   // e^{+2πi r/64}
    const float2 a = va[r];
    va[r] = cadd(a, t);                             // window position lane + 32r
    vb[r] = csub(a, t);                             // window position lane + 1024 + 32r
  }

  // ---- E₂ on the window positions the decimation reads → polyphase smem arrays → E, ΣE.
  // Ev[n] = E₂[2n + 512] (n ∈ [0, 512)), Od[m + 8] = E₂[2m + 513] (m ∈ [−8, 520)); then
  // E[n] = ½·Ev[n] + Σ_{i=1..8} c_i·(Od[n + 8 − i] + Od[n + 7 + i])   — 16 consecutive Od per output.
  const float sc = p.sideband * (1.0f / 2048.0f);
  const int64_t blk0 = cta * K1U_BLOCKS + 2 * warp;   // 4-sps block index relative to jb0
  float2* Ev = S;
  float2* Od = S + 512;
  auto put = [&](int pos, float ph, const float* wb) {
    const bool odd = pos & 1;
    const int idx = odd ? ((pos - 513) >> 1) + 8 : (pos - 512) >> 1;
    if (odd ? (idx >= 0 && idx < 528) : (idx >= 0 && idx < 512)) {
      float sn, cs;
      __sincosf(ph * sc, &sn, &cs);
      const float m = __expf(wb[pos] + p.half_ln_iref);
      (odd ? Od : Ev)[idx] = make_float2(m * cs, m * sn);
    }
  };
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const float* wb = b ? w1 : w0;
#pragma unroll
    for (int r = 15; r < 32; ++r) put(lane + 32 * r, b ? va[r].y : va[r].x, wb);          // [480, 1024)
#pragma unroll
    for (int r = 0; r < 17; ++r) put(lane + 1024 + 32 * r, b ? vb[r].y : vb[r].x, wb);   // [1024, 1568)
    __syncwarp();
    float2* Eo = E + (blk0 + b) * kHilbertHop;
    float2 s = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int i = 0; i < 4; ++i) {
      const int n = 4 * lane + 128 * i;             // 4 adjacent outputs n … n+3 share Od[n … n+18]
      float2 o[20];
#pragma unroll
      for (int u = 0; u < 10; ++u) {
        const float4 q = reinterpret_cast<const float4*>(Od + n)[u];
        o[2 * u] = make_float2(q.x, q.y);
        o[2 * u + 1] = make_float2(q.z, q.w);
      }
      const float4 e01 = reinterpret_cast<const float4*>(Ev + n)[0];
      const float4 e23 = reinterpret_cast<const float4*>(Ev + n)[1];
      float2 acc[4] = {make_float2(0.5f * e01.x, 0.5f * e01.y), make_float2(0.5f * e01.z, 0.5f * e01.w),
                       make_float2(0.5f * e23.x, 0.5f * e23.y), make_float2(0.5f * e23.z, 0.5f * e23.w)};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int t = 1; t <= 8; ++t) {
          const float2 u = cadd(o[j + 8 - t], o[j + 7 + t]);
          acc[j].x = fmaf(p.c[t - 1], u.x, acc[j].x);
          acc[j].y = fmaf(p.c[t - 1], u.y, acc[j].y);
        }
      }
      reinterpret_cast<float4*>(Eo + n)[0] = make_float4(acc[0].x, acc[0].y, acc[1].x, acc[1].y);
      reinterpret_cast<float4*>(Eo + n)[1] = make_float4(acc[2].x, acc[2].y, acc[3].x, acc[3].y);
      s = cadd(s, cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3])));
    }
    s.x = warp_sum(s.x);
    s.y = warp_sum(s.y);
    if (lane == 0) part[blk0 + b] = s;
    __syncwarp();
  }
  if (tid < K1U_BLOCKS) clampcnt[cta * K1U_BLOCKS + tid] = cblk[tid];
}

void launch_k1u(const void* adc_cta0, int input_dtype, int64_t n_blocks, float2* E, float2* part, int* clampcnt,
                const float2* tw2048u, const K1UParams& p, cudaStream_t s) {
  const int64_t grid = n_blocks / K1U_BLOCKS;
  if (input_dtype == 2) {   // KK_IN_UINT8
    cudaFuncSetAttribute(k1u_kk_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1U_SMEM);
    k1u_kk_kernel<uint8_t><<<(unsigned)grid, K1U_THREADS, K1U_SMEM, s>>>(static_cast<const uint8_t*>(adc_cta0), E,
                                                                          part, clampcnt, tw2048u, p);
  } else if (input_dtype == 1) {   // KK_IN_FLOAT32
    cudaFuncSetAttribute(k1u_kk_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1U_SMEM);
    k1u_kk_kernel<float><<<(unsigned)grid, K1U_THREADS, K1U_SMEM, s>>>(static_cast<const float*>(adc_cta0), E,
                                                                        part, clampcnt, tw2048u, p);
  } else {
    cudaFuncSetAttribute(k1u_kk_kernel<int16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1U_SMEM);
    k1u_kk_kernel<int16_t><<<(unsigned)grid, K1U_THREADS, K1U_SMEM, s>>>(static_cast<const int16_t*>(adc_cta0), E,
                                                                          part, clampcnt, tw2048u, p);
  }
}

}  // namespace kk
