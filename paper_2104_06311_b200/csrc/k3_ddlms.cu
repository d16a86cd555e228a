// k3_ddlms.cu — K3 (paper arrangement, eq_mode = KK_EQ_DDLMS): 4-tap T/2-spaced widely-linear DDLMS.
//
// PAPER.md:82 (§2): "the signal is further filtered by a four-tap adaptive time-domain DDLMS widely-linear
// equalizer. The decisions made by the equalizer are demapped". CD is removed by the static filter in K2
// (RRC × CD inverse, the "offline-optimized filter"), so the 4 adaptive taps only track residual ISI, gain and
// phase:
//   x_n = g·[y[2n+1], y[2n], y[2n−1], y[2n−2]],  g = (mean |y[2n]|²)^(−½) over the block and its warm-up
//   (the power comes from K2's per-64-symbol segment sums)
//   o_n = wᵀx_n + vᵀconj(x_n),  d_n = D(o_n),  e_n = d_n − o_n,  w += μ e conj(x),  v += μ e x
//   w₀ = centre spike on y[2n], v₀ = 0; μ = mu_warm over the first half of the warm-up, mu_mid over the second
//   half (the taps settle toward the small-μ state before the kept symbols), mu over the kept symbols; every symbol
//   is decided in its own frame's QAM order (warm-up symbols in the previous frame in that frame's order).
// The paper carries the equalizer state across 2^22-sample buffers in stream order (events serialise the
// streams). Here the recursion restarts on a global grid of B-symbol blocks, each preceded by W
// warm-up symbols: blocks are independent, so they run in parallel and any sharding gives the
// same decisions; the warm-up (≫ the adaptation time constant) makes the kept outputs those of a converged
// sequential equalizer.
//
// Mapping: one thread per block (B = 1024 ⇒ 65,536 threads per 2^26-sample call); the recursion is
// sequential in registers (4 + 4 complex taps, a 4-sample sliding window refilled with 2 samples per symbol).
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {

constexpr int K3D_THREADS = 64;

// WL = true: the widely-linear recursion in real form — per tap c = (wr + vr, vi − wi, wi + vi, wr − vr), so
// o = (Σ xr·c1 + xi·c2, Σ xr·c3 + xi·c4) and w += μe·conj(x), v += μe·x become c += 2μe ⊗ (xr, xi)
// (4 FMA per tap for each instead of 8). WL = false: linear taps only (v ≡ 0), complex form.
template <bool WL>
// 8 resident CTAs per SM (≤ 128 registers: 16 warps/SM instead of 14 at 140 registers; the recursion is
// latency-bound, K3′ −7 %; 10 CTAs would spill)
__global__ void __launch_bounds__(K3D_THREADS, 8)
k3_ddlms_kernel(const float2* __restrict__ y, int64_t y_base, int64_t sym_first, int n_blocks, int B, int W,
                const int* __restrict__ clampcnt, int64_t clamp_frame_off, const uint8_t* __restrict__ ref,
                uint8_t* __restrict__ dec, float2* __restrict__ zout, unsigned long long* __restrict__ counters,
                K3DParams p) {
  __shared__ uint8_t lut32[36];                              // 32-cross label table
  cross32_lut_fill(lut32, threadIdx.x, K3D_THREADS);
  __syncthreads();
  const int blk = blockIdx.x * K3D_THREADS + threadIdx.x;
  if (blk >= n_blocks) return;
  const int64_t n_keep0 = (int64_t)blk * B;                  // local index of the first kept symbol
  const int fl = (int)(n_keep0 / kFrameSym);                 // local frame
  const int64_t f = sym_first / kFrameSym + fl;
  // QAM order of global frame g: schedule[floor(g / segment_frames) mod n_segments] (floor: g may be < 0)
  auto fmt = [&](int64_t g) {
    int64_t sg = g / p.segment_frames;
    if (g < 0 && sg * p.segment_frames != g) --sg;
    return (int)p.schedule[(int)(((sg % p.n_segments) + p.n_segments) % p.n_segments)];
  };
  const int M = fmt(f);
  const int bi = (M == 4) ? 0 : (M == 8) ? 1 : (M == 16) ? 2 : (M == 32) ? 3 : 4;
  Slicer sl;
  sl.init(M);
  sl.lut = lut32;
  // warm-up symbols before the frame start belong to frame f − 1 and are decided in its format (W < 4096)
  Slicer slp;
  slp.init(fmt(f - 1));
  slp.lut = lut32;
  int ccount = 0;
  for (int q = 0; q < 32; ++q) ccount += __ldg(&clampcnt[clamp_frame_off + (int64_t)fl * 32 + q]);
  const bool dead = (ccount >= kFrameSamp);
  // y index of local 2-sps sample m is y_base + m; symbol n ↔ m = 2n
  const float2* yy = y + y_base;
  const int64_t n0 = n_keep0 - W;
  int serr = 0, berr = 0;
  if (!dead) {
    // AGC over the block and its warm-up (symbol-centre samples): K2 summed |y[2n]|² per 256-symbol segment
    // (global grid); the block's range [n_keep0 − W, n_keep0 + B) is (W mod 256) leading symbols read here plus
    // whole segments — no second pass over the block's samples
    const int Wr = W & 255;
    float pw = 0.f;
    for (int i = 0; i < Wr; ++i) {
      const float2 c = __ldg(&yy[2 * (n0 + i)]);
      pw = fmaf(c.x, c.x, fmaf(c.y, c.y, pw));
    }
    const int64_t g0 = (sym_first + n0 + Wr) >> 8;             // first whole segment
    const float* sp = p.seg_pow + (g0 - p.seg_first);
    for (int q = 0; q < (W - Wr + B) / 256; ++q) pw += __ldg(&sp[q]);
    const float P = pw / (float)(W + B);
    const float g = (P > 0.f) ? rsqrtf(P) : 1.0f;
    float2 w[4] = {make_float2(0.f, 0.f), make_float2(1.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float2 v[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    // real form (WL): cr = (c1, c3) = (wr + vr, wi + vi), ci = (c2, c4) = (vi − wi, wr − vr); centre spike w1 = 1
    float2 cr[4] = {make_float2(0.f, 0.f), make_float2(1.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float2 ci[4] = {make_float2(0.f, 0.f), make_float2(0.f, 1.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    // window x = [u[2n+1], u[2n], u[2n−1], u[2n−2]]
    float2 x[4];
    x[0] = cscale(__ldg(&yy[2 * n0 + 1]), g);
    x[1] = cscale(__ldg(&yy[2 * n0]), g);
    x[2] = cscale(__ldg(&yy[2 * n0 - 1]), g);
    x[3] = cscale(__ldg(&yy[2 * n0 - 2]), g);
    // the new samples y[2n+2], y[2n+3] of the next PF symbols are kept in a register ring (loads issued PF
    // symbols ahead of use, so L2 latency is hidden behind the recursion)
    constexpr int PF = 8;
    float4 ring[PF];
#pragma unroll
    for (int q = 0; q < PF; ++q) ring[q] = __ldg(reinterpret_cast<const float4*>(yy + 2 * (n0 + q) + 2));
    const int total = W + B;                                   // multiple of PF (W multiple of 64, B of 256)
    // labels: 8 per chunk as one 8-byte word (kept chunks start at multiples of 8 symbols), the reference word
    // loaded one chunk ahead; byte accesses when a pointer is not 8-byte aligned
    const bool ref8 = ref && ((reinterpret_cast<uintptr_t>(ref) & 7) == 0);
    const bool dec8 = dec && ((reinterpret_cast<uintptr_t>(dec) & 7) == 0);
    // reference words two chunks ahead of use (ra: this chunk, rb: the next one)
    auto rword = [&](int i) { return __ldg(reinterpret_cast<const uint2*>(ref + (n0 + i))); };
    uint2 ra = make_uint2(0u, 0u), rb = make_uint2(0u, 0u);
    if (ref8 && 0 >= W) ra = rword(0);
    if (ref8 && PF >= W && PF < total) rb = rword(PF);
    const int wprev = (int)((int64_t)fl * kFrameSym - n0);    // warm-up symbols in frame f − 1 (≤ 0: none)
    for (int i0 = 0; i0 < total; i0 += PF) {
      const bool kept = i0 >= W;
      const Slicer sc = (i0 < wprev) ? slp : sl;                 // chunk-uniform (wprev is a multiple of 64)
      const uint2 rcur = ra;
      ra = rb;
      if (ref8 && i0 + 2 * PF >= W && i0 + 2 * PF < total) rb = rword(i0 + 2 * PF);
      uint32_t dlo = 0u, dhi = 0u;
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int i = i0 + q;
        const int64_t n = n0 + i;
        const float4 nx = ring[q];                             // (y[2n+2], y[2n+3])
        if (i + PF < total) ring[q] = __ldg(reinterpret_cast<const float4*>(yy + 2 * (n + PF) + 2));
        // o = Σ_k w_k x_k + v_k conj(x_k) as two independent partial sums (shorter dependency chain)
        float2 o0 = make_float2(0.f, 0.f), o1 = make_float2(0.f, 0.f);
        if constexpr (WL) {
#pragma unroll
          for (int k = 0; k < 4; k += 2) {              // o += xr·(c1, c3) + xi·(c2, c4), packed
            ffma2s(o0, x[k].x, cr[k]);         ffma2s(o0, x[k].y, ci[k]);
            ffma2s(o1, x[k + 1].x, cr[k + 1]); ffma2s(o1, x[k + 1].y, ci[k + 1]);
          }
        } else {
          cmac(o0, w[0], x[0]); cmac(o1, w[1], x[1]);
          cmac(o0, w[2], x[2]); cmac(o1, w[3], x[3]);
        }
        const float2 o = cadd(o0, o1);
        int lab = 0;
        const float2 d = kept ? sl.decide(o, lab) : sc.point(o);   // kept: point and label from one slicing
        const float2 e = csub(d, o);
        const float mu = kept ? p.mu : (i0 < (W >> 1) ? p.mu_warm : p.mu_mid);   // chunk-uniform
        if (kept) {
          const int64_t kl = n;                                // local kept symbol index
          if (ref) {
            const int r = ref8 ? (int)(((q < 4 ? rcur.x : rcur.y) >> (8 * (q & 3))) & 0xffu) : (int)__ldg(&ref[kl]);
            serr += (lab != r);
            berr += __popc(lab ^ r);
          }
          if (q < 4) dlo |= (uint32_t)lab << (8 * q); else dhi |= (uint32_t)lab << (8 * (q - 4));
          if (dec && !dec8) dec[kl] = (uint8_t)lab;
          if (zout) zout[kl] = o;
        }
        if constexpr (WL) {
          const float2 m2 = cscale(e, 2.f * mu);             // c += 2μe ⊗ (xr, xi)
#pragma unroll
          for (int k = 0; k < 4; ++k) {                 // (c1, c3) += xr·m2, (c2, c4) += xi·m2, packed
            ffma2s(cr[k], x[k].x, m2);
            ffma2s(ci[k], x[k].y, m2);
          }
        } else {
          const float2 me = cscale(e, mu);
#pragma unroll
          for (int k = 0; k < 4; ++k) cmac(w[k], me, cconj(x[k]));
        }
        x[3] = x[1]; x[2] = x[0];
        x[1] = cscale(make_float2(nx.x, nx.y), g); x[0] = cscale(make_float2(nx.z, nx.w), g);
      }
      if (kept && dec8) *reinterpret_cast<uint2*>(dec + (n0 + i0)) = make_uint2(dlo, dhi);
    }
  } else {
    const int lab = sl.label(make_float2(0.f, 0.f));
    for (int i = 0; i < B; ++i) {
      const int64_t kl = n_keep0 + i;
      if (ref) {
        const int r = __ldg(&ref[kl]);
        serr += (lab != r);
        berr += __popc(lab ^ r);
      }
      if (dec) dec[kl] = (uint8_t)lab;
      if (zout) zout[kl] = make_float2(0.f, 0.f);
    }
  }
  if (ref) {
    if (serr) atomicAdd(&counters[5 + bi], (unsigned long long)serr);
    if (berr) atomicAdd(&counters[15 + bi], (unsigned long long)berr);
    if (p.frame_err) {
      if (serr) atomicAdd(&p.frame_err[2 * fl], (unsigned)serr);
      if (berr) atomicAdd(&p.frame_err[2 * fl + 1], (unsigned)berr);
    }
  }
  atomicAdd(&counters[bi], (unsigned long long)B);
  atomicAdd(&counters[10 + bi], (unsigned long long)B * (bi + 2));
  if (n_keep0 % kFrameSym == 0) {                            // once per frame
    if (ccount) atomicAdd(&counters[20], (unsigned long long)ccount);
    atomicAdd(&counters[21], 1ull);
    if (dead) atomicAdd(&counters[22], 1ull);
  }
}

void launch_k3_ddlms(const float2* y, int64_t y_base, int64_t sym_first, int64_t n_blocks, int B, int W,
                     const int* clampcnt, int64_t clamp_frame_off, const uint8_t* ref, uint8_t* dec, float2* z,
                     unsigned long long* counters, const K3DParams& p, cudaStream_t s) {
  const unsigned grid = (unsigned)((n_blocks + K3D_THREADS - 1) / K3D_THREADS);
  if (p.widely_linear)
    k3_ddlms_kernel<true><<<grid, K3D_THREADS, 0, s>>>(y, y_base, sym_first, (int)n_blocks, B, W, clampcnt,
                                                       clamp_frame_off, ref, dec, z, counters, p);
  else
    k3_ddlms_kernel<false><<<grid, K3D_THREADS, 0, s>>>(y, y_base, sym_first, (int)n_blocks, B, W, clampcnt,
                                                        clamp_frame_off, ref, dec, z, counters, p);
}

}  // namespace kk
