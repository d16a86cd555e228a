// k1_kk.cu — K1: fused KK front end, 1024-point overlap-save Hilbert transform and field reconstruction.
//
// PAPER.md:82 (§2): "converts the samples to floating point and performs KK front-end consisting of the
// square-root and logarithm operations. The phase ..., obtained through a Hilbert transform enabled by a
// pair of 1024-point 100% overlap-save FFTs, is combined with the amplitude to digitally reconstruct the
// optical field". Readings R1 (hop 512, central 512 kept), R2 (multiplier −i·sgn q, zero at DC/Nyquist,
// φ = σ·H[a]), R7 (ε = clamp_rel·I_ref) of SURVEY §8(c).
//
// Mapping: one warp per PAIR of 512-sample Hilbert blocks (two real blocks packed as re/im of one complex
// 1024-point FFT — exact because the Hilbert multiplier is applied complex-linearly to A₁ + iA₂ and
// maps each real block to a real output). 8 warps per CTA = 16 blocks = 8192 output samples; the CTA
// stages its 8704 input samples with one TMA bulk copy (cp.async.bulk) into shared memory, converts
// them once to a = ½·ln max(I/I_ref, ε_rel) (MUFU lg2), then every warp runs
//   DFT32 (registers) → transpose (smem, stride 33) → twiddle → DFT32      = Stockham FFT1024 radix 32
//   × (−i·sgn q)
//   IDFT32 → transpose → conj twiddle → IDFT32                              = inverse
// and writes E = √I_ref·e^{a}·e^{iσφ} for the central 512 samples of each block with coalesced 256-B
// stores, plus the per-block complex sum ΣE (fixed-order shuffle tree → deterministic) for the
// carrier estimate A_f of K2 and a per-block clamp count.
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {

constexpr int K1_WARPS = 8;
constexpr int K1_THREADS = K1_WARPS * 32;
constexpr int K1_SAMPLES = K1_WARPS * 1024 + 512;   // staged input samples per CTA (8704)
constexpr int K1_TR = 32 * 33;                      // float2 per warp transpose tile
constexpr size_t K1_SMEM = (size_t)K1_SAMPLES * 4 + (size_t)K1_WARPS * K1_TR * 8 + 16 + 2 * K1_WARPS * 4;

template <typename Tin>
__global__ void __launch_bounds__(K1_THREADS, 2)
k1_kk_kernel(const Tin* __restrict__ adc0, float2* __restrict__ E, float2* __restrict__ part,
             int* __restrict__ clampcnt, const float2* __restrict__ tw, K1Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* a_s = reinterpret_cast<float*>(smem);
  float2* tr = reinterpret_cast<float2*>(smem + (size_t)K1_SAMPLES * 4);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)K1_SAMPLES * 4 + (size_t)K1_WARPS * K1_TR * 8);
  int* cblk = reinterpret_cast<int*>(bar + 2);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t cta = blockIdx.x;
  const Tin* src = adc0 + cta * (int64_t)(K1_WARPS * 1024);
  Tin* stage = reinterpret_cast<Tin*>(tr);   // TMA landing zone (aliases the transpose tiles)
  constexpr uint32_t bytes = (uint32_t)(K1_SAMPLES * sizeof(Tin));

  if (tid == 0) mbar_init(bar, 1);
  if (tid < 2 * K1_WARPS) cblk[tid] = 0;
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, bytes);
    tma_bulk_g2s(stage, src, bytes, bar);
    // the input of the CTA that will follow this one on the GPU (blockIdx + 2 resident CTAs × SMs) → L2, so
    // that its copy does not wait on DRAM (a CTA otherwise spends ~14 % of its stall samples in this wait)
    uint32_t nsm;
    asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    if (cta + 2 * (int64_t)nsm < (int64_t)gridDim.x)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + 2 * (int64_t)nsm * (K1_WARPS * 1024)),
                   "r"(bytes) : "memory");
  }
  mbar_wait(bar, 0);

  // ---- a1/a2: int → float, I/I_ref, ε-clamp, b = log2(.) = 2·a/ln 2 with a = ½ ln(.) (one MUFU.LG2 per staged
  //      sample, no denormal fix-up: the operand is ≥ ε, a normal float; the Hilbert transform is linear, so the
  //      constant ½·ln 2 is applied after it, folded into the phase scale and into the magnitude's FFMA)
  // 8 consecutive samples per thread per step: one 16-B (int16) or two 16-B (float) shared loads, two
  // 16-B stores; the group never straddles a 512-block, so its clamp count goes to one block counter.
  const float sc_in = p.adc_scale * p.inv_iref, off_in = -p.adc_offset * p.adc_scale * p.inv_iref;
  for (int gi = tid; gi < K1_SAMPLES / 8; gi += K1_THREADS) {
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
    float av[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool cl = !(x[j] >= p.clamp_rel);
      ncl += cl;
      av[j] = lg2_approx(cl ? p.clamp_rel : x[j]);   // b = log2 x (a = ½·ln 2·b; the ½·ln 2 goes into sc and l2m's FFMA)
    }
    reinterpret_cast<float4*>(a_s)[2 * gi] = make_float4(av[0], av[1], av[2], av[3]);
    reinterpret_cast<float4*>(a_s)[2 * gi + 1] = make_float4(av[4], av[5], av[6], av[7]);
    if (ncl) {
      const int o = 8 * gi - kHilbertLead;        // output position inside the CTA
      if (o >= 0 && o < K1_WARPS * 1024) atomicAdd(&cblk[o >> 9], ncl);
    }
  }
  __syncthreads();

  // ---- a3: Hilbert by FFT1024 pair, two real blocks per complex transform
  float2* S = tr + warp * K1_TR;
  const float* ab0 = a_s + (2 * warp) * kHilbertHop;   // block 2w input: local samples [1024w, +1024)
  const float* ab1 = ab0 + kHilbertHop;
  float2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = make_float2(ab0[lane + 32 * r], ab1[lane + 32 * r]);

  dft_reg<32, -1>(v);                       // Stockham pass 1 (Ns = 1): lane j holds d1[32j + r]
#pragma unroll
  for (int r = 0; r < 32; ++r) S[lane * 33 + r] = v[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = S[r * 33 + lane];
  __syncwarp();
  twiddle32<-1, 32>(v, tw + lane);                // × W_1024^{r·j}
  dft_reg<32, -1>(v);                       // pass 2 (Ns = 32): lane j holds X[j + 32 r]

  // −i·sgn(q), q = j + 32 r: r < 16 ⇒ 0 < q < 512 (except q = 0); r ≥ 16 ⇒ q > 512 (except q = 512)
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    float2 x = v[r];
    v[r] = (r < 16) ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
  }
  if (lane == 0) { v[0] = make_float2(0.f, 0.f); v[16] = make_float2(0.f, 0.f); }

  dft_reg<32, +1>(v);                       // inverse pass 1: lane j holds d1[32j + r]
#pragma unroll
  for (int r = 0; r < 32; ++r) S[lane * 33 + r] = v[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = S[r * 33 + lane];
  twiddle32<+1, 32>(v, tw + lane);                // × W_1024^{−r·j}
  dft_reg<32, +1>(v);                       // lane j holds 1024·(φ₀ + iφ₁)[j + 32 r]

  // ---- a4: E = √I_ref·e^{a}·e^{iσφ} on the central 512 samples; per-block ΣE
  const float sc = p.sideband * (0.34657359027997264f / 1024.0f);   // σ·(½·ln 2)/1024: φ = ½·ln 2·H{b}
  const float l2m = p.half_ln_iref * 1.4426950408889634f;           // log2 √I_ref
  const int64_t blk0 = cta * (2 * K1_WARPS) + 2 * warp;    // block index relative to jb0
  float2* E0 = E + blk0 * kHilbertHop - kHilbertLead;
  float2* E1 = E0 + kHilbertHop;
  float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int r = 8; r < 24; ++r) {
    const int pos = lane + 32 * r;
    float sn0, cs0, sn1, cs1;
    __sincosf(v[r].x * sc, &sn0, &cs0);
    __sincosf(v[r].y * sc, &sn1, &cs1);
    // e^{a + ½ln I_ref} = 2^{b/2 + log2 √I_ref}: one FFMA (immediate form) + MUFU.EX2
    const float m0 = ex2_approx(fmaf(ab0[pos], 0.5f, l2m)), m1 = ex2_approx(fmaf(ab1[pos], 0.5f, l2m));
    const float2 e0 = cscale(make_float2(cs0, sn0), m0), e1 = cscale(make_float2(cs1, sn1), m1);
    E0[pos] = e0;
    E1[pos] = e1;
    s0 = cadd(s0, e0);
    s1 = cadd(s1, e1);
  }
  s0.x = warp_sum(s0.x); s0.y = warp_sum(s0.y);
  s1.x = warp_sum(s1.x); s1.y = warp_sum(s1.y);
  if (lane == 0) { part[blk0] = s0; part[blk0 + 1] = s1; }
  if (tid < 2 * K1_WARPS) clampcnt[cta * (2 * K1_WARPS) + tid] = cblk[tid];
}

void launch_k1(const void* adc_cta0, int input_dtype, int64_t n_pairs, float2* E, float2* part, int* clampcnt,
               const float2* tw1024, const K1Params& p, cudaStream_t s) {
  const int64_t grid = n_pairs / K1_WARPS;
  if (input_dtype == 2) {   // KK_IN_UINT8
    cudaFuncSetAttribute(k1_kk_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1_SMEM);
    k1_kk_kernel<uint8_t><<<(unsigned)grid, K1_THREADS, K1_SMEM, s>>>(static_cast<const uint8_t*>(adc_cta0), E,
                                                                       part, clampcnt, tw1024, p);
  } else if (input_dtype == 1) {   // KK_IN_FLOAT32
    cudaFuncSetAttribute(k1_kk_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1_SMEM);
    k1_kk_kernel<float><<<(unsigned)grid, K1_THREADS, K1_SMEM, s>>>(static_cast<const float*>(adc_cta0), E, part,
                                                                     clampcnt, tw1024, p);
  } else {
    cudaFuncSetAttribute(k1_kk_kernel<int16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1_SMEM);
    k1_kk_kernel<int16_t><<<(unsigned)grid, K1_THREADS, K1_SMEM, s>>>(static_cast<const int16_t*>(adc_cta0), E,
                                                                       part, clampcnt, tw1024, p);
  }
}

}  // namespace kk
