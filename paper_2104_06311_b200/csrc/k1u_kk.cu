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
// Mapping: 8 warps per CTA = 4 groups of 64 threads; a group handles a PAIR of blocks (two real windows
// packed as re/im of one complex 2048-point FFT), CTA = 8 blocks = 4096 outputs. The CTA stages its 4640
// ADC samples with one TMA bulk copy, converts them to I/I_ref once (ADC clamp counts per block),
// interpolates and takes the log for all 9216 window samples once (a₂ in shared memory, shared by the
// overlapping windows); staging and I alias the FFT scratch. FFT2048 = 64 × 32 over the group, 32 values
// per thread (128 registers → 2 CTAs = 16 warps per SM):
//   thread t: DFT32 over r of x[t + 64r] → twiddle W₂₀₄₈^{t·k1} → transpose (stride 33; the half-warp
//   picks the parity h of t, conflict-free) → thread (k1', h): DFT32 over s of Y'[2s + h][k1'] → radix-2
//   combine with lane ^ 16 (P₀ ± W₆₄^{k2'}·P₁) → X[k1' + 32k2' + 1024h]; × (−i·sgn q); the inverse
//   mirrors it (split with lane ^ 16, IDFT32, transpose, conj twiddle, IDFT32) → x[t + 64r].
// E₂ at the positions the decimation needs goes to group scratch as even/odd polyphase arrays (both
// blocks); each warp then decimates one block, 4 adjacent outputs per lane-step from one 20-sample odd
// window (16-B loads, conflict-free through the chunk swizzle swz2) with 16-B coalesced stores. I, a₂ and the
// polyphase arrays are stored chunk-swizzled (swz4, swz4x, swz2 in kk_device.cuh) so that the 32- and 64-B lane-stride vector accesses
// of the conversion, the interpolation and the decimation are conflict-free (ncu: 36 % excess wavefronts before).
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {

constexpr int K1U_WARPS = 8;
constexpr int K1U_THREADS = K1U_WARPS * 32;
constexpr int K1U_GROUPS = K1U_WARPS / 2;            // FFT groups of 64 threads, one block pair each
constexpr int K1U_BLOCKS = 2 * K1U_GROUPS;           // 4-sps Hilbert blocks per CTA (8)
constexpr int K1U_OUT = K1U_BLOCKS * kHilbertHop;    // 4096 outputs per CTA
constexpr int K1U_PAD = kK1uPad;                     // 272 staged samples before/after (256 + 16)
constexpr int K1U_IN = K1U_OUT + 2 * K1U_PAD;        // 4640
constexpr int K1U_UP = 2 * K1U_OUT + 1024;           // 9216 window samples at 8 sps
constexpr int K1U_GS = 64 * 33;                      // float2 scratch per group (transpose 64 × 33)
constexpr int K1U_POLY = 1040;                       // Ev (512) + Od (528) per block
constexpr size_t K1U_SMEM = (size_t)K1U_UP * 4 + (size_t)K1U_GROUPS * K1U_GS * 8 + 16 + K1U_BLOCKS * 4;
static_assert(2 * K1U_POLY <= K1U_GS, "E2 polyphase arrays of a block pair fit the group scratch");
static_assert((size_t)K1U_IN * 4 * 2 <= (size_t)K1U_GROUPS * K1U_GS * 8, "staging + I alias the scratch");

__device__ __forceinline__ void group_sync(int id) {   // named barrier for the 64 threads of one group
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

template <typename Tin>
__global__ void __launch_bounds__(K1U_THREADS, 2)
k1u_kk_kernel(const Tin* __restrict__ adc0, float2* __restrict__ E, float2* __restrict__ part,
              int* __restrict__ clampcnt, const float2* __restrict__ tw, K1UParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* a2 = reinterpret_cast<float*>(smem);
  float2* ws = reinterpret_cast<float2*>(a2 + K1U_UP);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ws + K1U_GROUPS * K1U_GS);
  int* cblk = reinterpret_cast<int*>(bar + 2);
  Tin* stage = reinterpret_cast<Tin*>(ws);                                   // TMA landing zone
  float* Ib = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(ws) + K1U_IN * 4);   // I/I_ref

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t cta = blockIdx.x;
  const Tin* src = adc0 + cta * (int64_t)K1U_OUT;
  constexpr uint32_t bytes = (uint32_t)(K1U_IN * sizeof(Tin));

  if (tid == 0) mbar_init(bar, 1);
  if (tid < K1U_BLOCKS) cblk[tid] = 0;
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, bytes);
    tma_bulk_g2s(stage, src, bytes, bar);
    // the input of the CTA that follows this one (blockIdx + 2 resident CTAs × SMs) → L2 (as in K1)
    uint32_t nsm;
    asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    if (cta + 2 * (int64_t)nsm < (int64_t)gridDim.x)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + 2 * (int64_t)nsm * K1U_OUT), "r"(bytes)
                   : "memory");
  }
  mbar_wait(bar, 0);

  // ---- I/I_ref for the staged samples; ADC clamp count per kept 512-block (8-sample groups)
  const float sc_in = p.adc_scale * p.inv_iref, off_in = -p.adc_offset * p.adc_scale * p.inv_iref;
  for (int gi = tid; gi < K1U_IN / 8; gi += K1U_THREADS) {
    float x[8];
    if constexpr (sizeof(Tin) == 2) {
      codes8_to_float(reinterpret_cast<const uint4*>(stage)[gi], sc_in, off_in, x);   // no I2F (kk_device.cuh)
    } else if constexpr (sizeof(Tin) == 1) {
      codes8_to_float(reinterpret_cast<const uint2*>(stage)[gi], sc_in, off_in, x);
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
    *reinterpret_cast<float4*>(Ib + swz4(8 * gi)) = make_float4(x[0], x[1], x[2], x[3]);
    *reinterpret_cast<float4*>(Ib + swz4(8 * gi + 4)) = make_float4(x[4], x[5], x[6], x[7]);
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
      const float4 q = *reinterpret_cast<const float4*>(Ib + swz4(8 * g + 8 + 4 * t));
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
      *reinterpret_cast<float4*>(a2 + swz4x(16 * g + 4 * t)) = make_float4(out[4 * t], out[4 * t + 1], out[4 * t + 2], out[4 * t + 3]);
  }
  __syncthreads();

  // ---- FFT2048 pair per 64-thread group: x[t + 64r] (t = group thread, r < 32), 2048 = 64 × 32.
  const int grp = warp >> 1, t = tid & 63, wg = warp & 1;
  const int bid = 1 + grp;                          // named barrier id (0 = __syncthreads)
  float2* S = ws + grp * K1U_GS;
  const int w0i = (2 * grp) * 1024, w1i = w0i + 1024;   // windows of blocks 2·grp, 2·grp + 1 in a2 (swizzled)
  const int k1p = 16 * wg + (lane & 15), h = lane >> 4;   // role after the transpose: (k1', parity of t)
  float2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = make_float2(a2[swz4x(w0i + t + 64 * r)], a2[swz4x(w1i + t + 64 * r)]);
  dft_reg<32, -1>(v);                               // Y[t][k1] = Σ_r x[t + 64r]·W₃₂^{r·k1}
  twiddle32<-1, 64>(v, tw + t);               // × W₂₀₄₈^{t·k1}
#pragma unroll
  for (int k = 0; k < 32; ++k) S[t * 33 + k] = v[k];
  group_sync(bid);
#pragma unroll
  for (int s2 = 0; s2 < 32; ++s2) v[s2] = S[(2 * s2 + h) * 33 + k1p];       // Y'[2s + h][k1']
  dft_reg<32, -1>(v);                               // P_h[k2'] = Σ_s Y'[2s + h][k1']·W₃₂^{s·k2'}
  // radix-2 combine with the partner (lane ^ 16): X[k1' + 32(k2' + 32h)] = P₀ ± W₆₄^{k2'}·P₁
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, v[k].x, 16), __shfl_xor_sync(0xffffffffu, v[k].y, 16));
    float2 wv = unit_root64(k);
    wv.y = -wv.y;                                   // e^{−2πi k/64}
    const float2 a = h ? o : v[k], b = h ? v[k] : o;
    const float2 tb = cmul(b, wv);
    v[k] = h ? csub(a, tb) : cadd(a, tb);
  }
  // −i·sgn(q), q = k1' + 32k2' + 1024h: h = 0 ⇒ 0 ≤ q < 1024, h = 1 ⇒ q ≥ 1024; q ∈ {0, 1024} → 0
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float2 x = v[k];
    v[k] = h ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
  }
  if (k1p == 0) v[0] = make_float2(0.f, 0.f);
  // inverse: A_g[k2'] = (X₀ + (−1)^g X₁)·W₆₄^{−g·k2'}… (conj roots), g = h
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, v[k].x, 16), __shfl_xor_sync(0xffffffffu, v[k].y, 16));
    if (h) {
      v[k] = cmul(csub(o, v[k]), unit_root64(k));  // (X₀ − X₁)·e^{+2πi k/64}
    } else {
      v[k] = cadd(v[k], o);                         // X₀ + X₁
    }
  }
  dft_reg<32, +1>(v);                               // Z[k1'][2s + h], s = 0..31
  group_sync(bid);                                  // every thread finished reading S (forward transpose)
#pragma unroll
  for (int s2 = 0; s2 < 32; ++s2) S[(2 * s2 + h) * 33 + k1p] = v[s2];
  group_sync(bid);
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = S[t * 33 + k];                          // Z[k1][t]
  twiddle32<+1, 64>(v, tw + t);               // × W₂₀₄₈^{−t·k1}
  dft_reg<32, +1>(v);                               // 2048·(φ₀ + iφ₁)[t + 64r]
  group_sync(bid);                                  // S is reused for E₂ below

  // ---- E₂ at the window positions the decimation reads → polyphase arrays per block:
  // Ev[n] = E₂[2n + 512] (n ∈ [0, 512)), Od[m + 8] = E₂[2m + 513] (m ∈ [−8, 520)); then
  // E[n] = ½·Ev[n] + Σ_{i=1..8} c_i·(Od[n + 8 − i] + Od[n + 7 + i]).
  const float sc = p.sideband * (1.0f / 2048.0f);
  const float l2m = p.half_ln_iref * 1.4426950408889634f;   // log2 √I_ref (e^{a + ½ln I_ref} = 2^{a·log2 e + l2m})
  float2* poly0 = S;
  float2* poly1 = S + K1U_POLY;
#pragma unroll
  for (int r = 7; r < 25; ++r) {
    const int pos = t + 64 * r;                     // positions [448, 1600) ⊇ [497, 1551)
    const bool odd = pos & 1;
    const int idx = odd ? 512 + ((pos - 513) >> 1) + 8 : (pos - 512) >> 1;
    const bool need = odd ? (pos >= 497 && pos < 1552) : (pos >= 512 && pos < 1536);
    if (need) {
      float sn, cs;
      __sincosf(v[r].x * sc, &sn, &cs);
      float m = ex2_approx(fmaf(a2[swz4x(w0i + pos)], 1.4426950408889634f, l2m));
      poly0[swz2(idx)] = make_float2(m * cs, m * sn);
      __sincosf(v[r].y * sc, &sn, &cs);
      m = ex2_approx(fmaf(a2[swz4x(w1i + pos)], 1.4426950408889634f, l2m));
      poly1[swz2(idx)] = make_float2(m * cs, m * sn);
    }
  }
  group_sync(bid);
  // decimation: warp wg of the group makes the 512 outputs of block 2·grp + wg, 4 adjacent per lane-step
  const float2* Ev = wg ? poly1 : poly0;             // Ev at [0, 512), Od at [512, 1040) of the swizzled array
  const int64_t blk = cta * K1U_BLOCKS + 2 * grp + wg;   // 4-sps block index relative to jb0
  float2* Eo = E + blk * kHilbertHop;
  float2 s = make_float2(0.f, 0.f);
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    const int n = 4 * lane + 128 * i;               // outputs n … n+3 share Od[n … n+18]
    float2 o[20];
#pragma unroll
    for (int u = 0; u < 10; ++u) {
      const float4 q = *reinterpret_cast<const float4*>(Ev + swz2(512 + n + 2 * u));
      o[2 * u] = make_float2(q.x, q.y);
      o[2 * u + 1] = make_float2(q.z, q.w);
    }
    const float4 e01 = *reinterpret_cast<const float4*>(Ev + swz2(n));
    const float4 e23 = *reinterpret_cast<const float4*>(Ev + swz2(n + 2));
    float2 acc[4] = {make_float2(0.5f * e01.x, 0.5f * e01.y), make_float2(0.5f * e01.z, 0.5f * e01.w),
                     make_float2(0.5f * e23.x, 0.5f * e23.y), make_float2(0.5f * e23.z, 0.5f * e23.w)};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int tt = 1; tt <= 8; ++tt) {
        const float2 u = cadd(o[j + 8 - tt], o[j + 7 + tt]);
        acc[j].x = fmaf(p.c[tt - 1], u.x, acc[j].x);
        acc[j].y = fmaf(p.c[tt - 1], u.y, acc[j].y);
      }
    }
    reinterpret_cast<float4*>(Eo + n)[0] = make_float4(acc[0].x, acc[0].y, acc[1].x, acc[1].y);
    reinterpret_cast<float4*>(Eo + n)[1] = make_float4(acc[2].x, acc[2].y, acc[3].x, acc[3].y);
    s = cadd(s, cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3])));
  }
  s.x = warp_sum(s.x);
  s.y = warp_sum(s.y);
  if (lane == 0) part[blk] = s;
  if (tid < K1U_BLOCKS) clampcnt[cta * K1U_BLOCKS + tid] = cblk[tid];
}

void launch_k1u(const void* adc_cta0, int input_dtype, int64_t n_blocks, float2* E, float2* part, int* clampcnt,
                const float2* tw2048u, const K1UParams& p, cudaStream_t s) {
  const int64_t grid = n_blocks / K1U_BLOCKS;   // n_blocks % 8 == 0 (n is a multiple of 16384)
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
