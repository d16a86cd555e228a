// kk_device.cuh — device helpers shared by the KK kernels (K1, K2, K3): complex arithmetic,
// register-resident radix-2 DFT-R (R = 8/16/32) used by the shared-memory Stockham FFTs,
// the QAM slicers and TMA 1-D bulk-copy / mbarrier wrappers (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kk {

// ------------------------------------------------------------------ complex float2 helpers
// complex add / subtract as one packed FP32x2 instruction (sm_100a FADD2; .rn = the scalar FADD rounding, so
// results are bit-identical to the two scalar adds while taking one issue slot instead of two)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pr;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\t"
      "add.rn.f32x2 pr, pa, pb;\n\tmov.b64 {%0, %1}, pr;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pr;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\t"
      "sub.rn.f32x2 pr, pa, pb;\n\tmov.b64 {%0, %1}, pr;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// (x, y) += s·(b.x, b.y) as one packed FP32x2 FMA (FFMA2 with a scalar-broadcast operand; each lane is the
// scalar fmaf, so results are bit-identical to two FFMAs)
__device__ __forceinline__ void ffma2s(float& x, float& y, float s, float2 b) {
  asm("{\n\t.reg .b64 pa, pb, pc;\n\tmov.b64 pa, {%2, %2};\n\tmov.b64 pb, {%3, %4};\n\tmov.b64 pc, {%0, %1};\n\t"
      "fma.rn.f32x2 pc, pa, pb, pc;\n\tmov.b64 {%0, %1}, pc;\n\t}"
      : "+f"(x), "+f"(y) : "f"(s), "f"(b.x), "f"(b.y));
}
__device__ __forceinline__ void ffma2s(float2& acc, float s, float2 b) { ffma2s(acc.x, acc.y, s, b); }
// complex multiply as two packed FP32x2 instructions: a·b = b.x·a + b.y·(i·a), i·a = (−a.y, a.x). ptxas folds the
// swapped, half-negated operand into FFMA2's operand modifiers (R.F32x2.LO_HI.NP) and b.x, b.y into scalar
// broadcasts, so the product is FMUL2 + FFMA2 (scalar form: 2 FMUL + 2 FFMA). Per lane: re = fma(−a.y, b.y,
// a.x·b.x), im = fma(a.x, b.y, a.y·b.x) — the same accuracy as the scalar form (one product rounded, one fused).
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 pa, ps, pc, pn, pr;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 ps, {%3, %2};\n\t"
      "mov.b64 pc, {%4, %4};\n\tmov.b64 pn, {%5, %6};\n\t"
      "mul.rn.f32x2 pr, pa, pc;\n\tfma.rn.f32x2 pr, ps, pn, pr;\n\tmov.b64 {%0, %1}, pr;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(-b.y), "f"(b.y));
  return r;
}
// a·conj(b) = b.x·a − b.y·(i·a): re = fma(a.y, b.y, a.x·b.x), im = fma(−a.x, b.y, a.y·b.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 pa, ps, pc, pn, pr;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 ps, {%3, %2};\n\t"
      "mov.b64 pc, {%4, %4};\n\tmov.b64 pn, {%5, %6};\n\t"
      "mul.rn.f32x2 pr, pa, pc;\n\tfma.rn.f32x2 pr, ps, pn, pr;\n\tmov.b64 {%0, %1}, pr;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(-b.y));
  return r;
}
// (acc.x, acc.y) += (a.x·b.x, a.y·b.y) as one packed FP32x2 FMA (each lane the scalar fmaf)
__device__ __forceinline__ void ffma2(float2& acc, float2 a, float2 b) {
  asm("{\n\t.reg .b64 pa, pb, pc;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\tmov.b64 pc, {%0, %1};\n\t"
      "fma.rn.f32x2 pc, pa, pb, pc;\n\tmov.b64 {%0, %1}, pc;\n\t}"
      : "+f"(acc.x), "+f"(acc.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
}
// acc += a·conj(b) in the cmul form (FFMA2 + FFMA2): acc += b.x·a − b.y·(i·a)
__device__ __forceinline__ void cmacc2(float2& acc, float2 a, float2 b) {
  asm("{\n\t.reg .b64 pa, ps, pc, pn, pr;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 ps, {%3, %2};\n\t"
      "mov.b64 pc, {%4, %4};\n\tmov.b64 pn, {%5, %6};\n\tmov.b64 pr, {%0, %1};\n\t"
      "fma.rn.f32x2 pr, pa, pc, pr;\n\tfma.rn.f32x2 pr, ps, pn, pr;\n\tmov.b64 {%0, %1}, pr;\n\t}"
      : "+f"(acc.x), "+f"(acc.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(-b.y));
}
// acc += a·b in the cmul form (FFMA2 + FFMA2): acc += b.x·a + b.y·(i·a) — the swap and the half-negation fold into
// FFMA2 operand modifiers, so a tap b held as two scalars (e.g. uniform registers) needs no register pair
__device__ __forceinline__ void cmac2(float2& acc, float2 a, float2 b) {
  asm("{\n\t.reg .b64 pa, ps, pc, pn, pr;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 ps, {%3, %2};\n\t"
      "mov.b64 pc, {%4, %4};\n\tmov.b64 pn, {%5, %6};\n\tmov.b64 pr, {%0, %1};\n\t"
      "fma.rn.f32x2 pr, pa, pc, pr;\n\tfma.rn.f32x2 pr, ps, pn, pr;\n\tmov.b64 {%0, %1}, pr;\n\t}"
      : "+f"(acc.x), "+f"(acc.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(-b.y), "f"(b.y));
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// 2^x by one MUFU.EX2 (flush-to-zero; the same instruction __expf issues after its ×log2 e)
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {   // MUFU.LG2 without the denormal fix-up (x normal or ≥ 1)
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// a·s as one packed FP32x2 multiply with a scalar-broadcast operand (FMUL2; bit-identical to two FMULs)
__device__ __forceinline__ float2 cscale(float2 a, float s) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pr;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %4};\n\t"
      "mul.rn.f32x2 pr, pa, pb;\n\tmov.b64 {%0, %1}, pr;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(s));
  return r;
}
// acc += a * b
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y); acc.y = fmaf(a.y, b.x, acc.y);
}

// ------------------------------------------------------------------ register DFT
// cos(2πk/32) for k = 0..8 (quarter wave); other angles by symmetry. Folded to immediates after unroll.
__device__ __forceinline__ float cos32q(int k) {
  const float q[9] = {1.0f, 0.98078528040323044913f, 0.92387953251128675613f, 0.83146961230254523708f,
                      0.70710678118654752440f, 0.55557023301960222474f, 0.38268343236508977173f,
                      0.19509032201612826785f, 0.0f};
  return q[k];
}
// exp(2πi e/R) for R | 32 (angle in units of 1/32 turn: u = e·32/R)
template <int R>
__device__ __forceinline__ float2 unit_root(int e) {
  int u = (e * (32 / R)) & 31;
  float c, s;
  if (u <= 8) { c = cos32q(u); s = cos32q(8 - u); }
  else if (u <= 16) { c = -cos32q(16 - u); s = cos32q(u - 8); }
  else if (u <= 24) { c = -cos32q(u - 16); s = -cos32q(24 - u); }
  else { c = cos32q(32 - u); s = -cos32q(u - 24); }
  return make_float2(c, s);
}
// exp(2πi u/64) for u = 0..63 (K1U's 64-point radix-2 stage); folded to immediates after unroll.
__device__ __forceinline__ float cos64q(int u) {   // cos(2πu/64), u = 0..16
  const float q[17] = {1.0f, 0.99518472667219688624f, 0.98078528040323044913f, 0.95694033573220886494f,
                       0.92387953251128675613f, 0.88192126434835502971f, 0.83146961230254523708f,
                       0.77301045336273696081f, 0.70710678118654752440f, 0.63439328416364549822f,
                       0.55557023301960222474f, 0.47139673682599764856f, 0.38268343236508977173f,
                       0.29028467725446236764f, 0.19509032201612826785f, 0.09801714032956060199f, 0.0f};
  return q[u];
}
__device__ __forceinline__ float2 unit_root64(int u) {
  u &= 63;
  float c, s;
  if (u <= 16) { c = cos64q(u); s = cos64q(16 - u); }
  else if (u <= 32) { c = -cos64q(32 - u); s = cos64q(u - 16); }
  else if (u <= 48) { c = -cos64q(u - 32); s = -cos64q(48 - u); }
  else { c = cos64q(64 - u); s = -cos64q(u - 48); }
  return make_float2(c, s);
}
__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }
// non-recursive so that it folds to a constant after loop unrolling (recursion would block inlining)
__host__ __device__ __forceinline__ constexpr int bitrevc(int x, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1) << (bits - 1 - b);
  return r;
}

// x · W_R^{e} for DIR = −1 (W = e^{−2πi/R}), x · conj(W_R^{e}) for DIR = +1; e is a compile-time constant after
// unrolling, so the trivial angles (0, ±i, −1) fold to moves/negations.
template <int R, int DIR>
__device__ __forceinline__ float2 twiddle(float2 x, int e) {
  e &= R - 1;
  if (e == 0) return x;
  if (2 * e == R) return make_float2(-x.x, -x.y);
  if (4 * e == R) return DIR < 0 ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
  if (4 * e == 3 * R) return DIR < 0 ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
  float2 w = unit_root<R>(e);
  if (DIR < 0) w.y = -w.y;
  return cmul(x, w);
}

// In-register DFT of length R (power of two ≤ 32), natural order in and out, unnormalised.
// DIR = −1: X[k] = Σ x[n] e^{−2πi nk/R} (forward);  DIR = +1: inverse (no 1/R).
// Decimation in frequency, two radix-2 stages fused into one radix-4 butterfly where possible: for
// a = v[s+j], b = v[s+j+q], c = v[s+j+2q], d = v[s+j+3q] (q = R/2^{st+2}, j < q, u = 2^st):
//   v[s+j]    = (a + c) + (b + d)
//   v[s+j+q]  = ((a + c) − (b + d))·W^{2ju}
//   v[s+j+2q] = ((a − c) ∓ i(b − d))·W^{ju}
//   v[s+j+3q] = ((a − c) ± i(b − d))·W^{3ju}
// — exactly the two radix-2 stages (same output positions, so the final bit reversal is unchanged) with the
// (j + q) twiddle W^{ju}·(∓i) folded into the butterfly: 3 twiddle multiplies per group instead of 4.
template <int R, int DIR>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
  constexpr int LOGR = ilog2c(R);
#pragma unroll
  for (int st = 0; st < LOGR; st += 2) {
    if (st + 1 < LOGR) {
      const int q = R >> (st + 2);
#pragma unroll
      for (int i = 0; i < R / 4; ++i) {
        const int j = i & (q - 1);
        const int s = (i - j) * 4;
        const float2 a = v[s + j], b = v[s + j + q], c = v[s + j + 2 * q], d = v[s + j + 3 * q];
        const float2 apc = cadd(a, c), amc = csub(a, c), bpd = cadd(b, d), bmd = csub(b, d);
        // ∓i·(b − d): forward −i, inverse +i
        const float2 ibmd = DIR < 0 ? make_float2(bmd.y, -bmd.x) : make_float2(-bmd.y, bmd.x);
        const int u = 1 << st;
        v[s + j] = cadd(apc, bpd);
        v[s + j + q] = twiddle<R, DIR>(csub(apc, bpd), 2 * j * u);
        v[s + j + 2 * q] = twiddle<R, DIR>(cadd(amc, ibmd), j * u);
        v[s + j + 3 * q] = twiddle<R, DIR>(csub(amc, ibmd), 3 * j * u);
      }
    } else {
      const int half = R >> (st + 1);
#pragma unroll
      for (int i = 0; i < R / 2; ++i) {
        const int j = i & (half - 1);
        const int s = (i - j) * 2;
        const float2 a = v[s + j], b = v[s + j + half];
        v[s + j] = cadd(a, b);
        v[s + j + half] = twiddle<R, DIR>(csub(a, b), j << st);
      }
    }
  }
  // DIF leaves bit-reversed order: permute back (compile-time renaming)
  float2 t[R];
#pragma unroll
  for (int i = 0; i < R; ++i) t[i] = v[bitrevc(i, LOGR)];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = t[i];
}

// v[r] ·= w^r (DIR < 0) or conj(w)^r (DIR > 0), r = 1..31, tw[S·r] = w^r (K1: W_1024^{r·j}, S = 32; K1U:
// W_2048^{r·t}, S = 64): loads w^1..w^3 and w^{4a} (10 of the 31 table entries — the twiddle loads were a quarter
// of K1's L1 wavefronts) and forms w^{4a+b} = w^{4a}·w^b (one product: every twiddle ≤ two roundings from exact)
template <int DIR, int S>
__device__ __forceinline__ void twiddle32(float2 (&v)[32], const float2* __restrict__ tw) {
  const float2 w1 = __ldg(tw + S), w2 = __ldg(tw + 2 * S), w3 = __ldg(tw + 3 * S);
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const float2 base = a ? __ldg(tw + 4 * S * a) : make_float2(1.f, 0.f);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * a + b;
      if (r == 0) continue;
      const float2 wb = (b == 1) ? w1 : (b == 2) ? w2 : w3;
      const float2 w = (b == 0) ? base : (a == 0) ? wb : cmul(base, wb);
      v[r] = DIR < 0 ? cmul(v[r], w) : cmulc(v[r], w);
    }
  }
}

// 16-B chunk XOR swizzles within 128-B rows (K1U's shared arrays). A quarter-warp's eight 16-B accesses are
// conflict-free iff they hit eight distinct chunk positions of their rows; scalar accesses to 32 consecutive floats
// (one row) stay conflict-free under any chunk permutation of the row.
//   swz4x: float index, chunk bits ^= row bits (3) — for 64-B lane strides (4 chunks per lane);
//   swz4 / swz2: float / float2 index, chunk bit 0 ^= row bit 0 — for 32-B lane strides (2 chunks per lane).
__device__ __forceinline__ int swz4x(int m) { return m ^ (((m >> 5) & 7) << 2); }
__device__ __forceinline__ int swz4(int m) { return m ^ (((m >> 5) & 1) << 2); }
__device__ __forceinline__ int swz2(int m) { return m ^ (((m >> 4) & 1) << 1); }

// ------------------------------------------------------------------ ADC codes → float (K1, K1U)
// x_j = fmaf((float)c_j, sc, off) for 8 consecutive codes, without I2F: code c (biased to u = c + 32768 ≥ 0 for
// int16) becomes the low mantissa bits of 2²³ by one byte permute (bits 0x4B00_0000 | u = 2²³ + u exactly), one
// packed subtraction of 2²³ (+ 32768) recovers (float)c exactly (all values are integers < 2²⁴), then a packed
// FMA per pair (each lane the scalar fmaf) — bit-identical to the I2F form.
__device__ __forceinline__ void codes8_to_float(uint4 raw, float sc, float off, float (&x)[8]) {   // int16
  const unsigned w[4] = {raw.x ^ 0x80008000u, raw.y ^ 0x80008000u, raw.z ^ 0x80008000u, raw.w ^ 0x80008000u};
  constexpr float kBias = 8388608.0f + 32768.0f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float2 f = make_float2(__uint_as_float(__byte_perm(w[q], 0x4B000000u, 0x7410)),
                           __uint_as_float(__byte_perm(w[q], 0x4B000000u, 0x7432)));
    f = csub(f, make_float2(kBias, kBias));
    float2 o = make_float2(off, off);
    ffma2s(o, sc, f);
    x[2 * q] = o.x; x[2 * q + 1] = o.y;
  }
}
__device__ __forceinline__ void codes8_to_float(uint2 raw, float sc, float off, float (&x)[8]) {   // uint8
  constexpr float kBias = 8388608.0f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const unsigned wq = (q < 2) ? raw.x : raw.y;
    const unsigned b0 = 2u * (unsigned)(q & 1);
    float2 f = make_float2(__uint_as_float(__byte_perm(wq, 0x4B000000u, 0x7440u | b0)),
                           __uint_as_float(__byte_perm(wq, 0x4B000000u, 0x7440u | (b0 + 1u))));
    f = csub(f, make_float2(kBias, kBias));
    float2 o = make_float2(off, off);
    ffma2s(o, sc, f);
    x[2 * q] = o.x; x[2 * q + 1] = o.y;
  }
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ QAM slicer
// Decision regions: per axis, a value exactly on a boundary goes to the lower level; the 32-cross
// corner cells go to the nearer of the two adjacent points (ties to the lower label).
__device__ __forceinline__ int gray(int i) { return i ^ (i >> 1); }
// 32-cross label of grid cell (iI, iQ) (level index 0 = −5); corners unused.
// rows iQ = 0..5 (Q = −5..+5), 5 bits per column iI = 0..5.
__device__ __forceinline__ int cross32_label(int iI, int iQ) {
  const unsigned long long rows[6] = {
      (0ull) | (0ull << 5) | (1ull << 10) | (17ull << 15) | (16ull << 20) | (0ull << 25),
      (4ull) | (12ull << 5) | (8ull << 10) | (24ull << 15) | (28ull << 20) | (20ull << 25),
      (5ull) | (13ull << 5) | (9ull << 10) | (25ull << 15) | (29ull << 20) | (21ull << 25),
      (7ull) | (15ull << 5) | (11ull << 10) | (27ull << 15) | (31ull << 20) | (23ull << 25),
      (6ull) | (14ull << 5) | (10ull << 10) | (26ull << 15) | (30ull << 20) | (22ull << 25),
      (0ull) | (3ull << 5) | (2ull << 10) | (18ull << 15) | (19ull << 20) | (0ull << 25)};
  unsigned long long r = rows[0];
#pragma unroll
  for (int q = 1; q < 6; ++q) r = (iQ == q) ? rows[q] : r;
  return (int)((r >> (5 * iI)) & 31ull);
}

// runtime-uniform QAM slicer parameters (CTA-uniform: one format per frame, R26)
//
// Per axis with m levels at the odd integers −(m−1)..(m−1) (grid units x·s): the decided level is 2r − 1 with
// r = ceil(x·s/2) clamped to [−(m−2)/2, m/2] — a value exactly on a boundary (x·s/2 an integer) goes to the lower
// level. r is formed on the FMA pipe: t = kSliceMagic + x·(s/2) rounded toward +∞ (one FFMA2.RP for both axes;
// kSliceMagic = 1.5·2²³ has ulp 1, so t − kSliceMagic = ceil(x·s/2) exactly for |x·s/2| < 2²²), clamped in the
// biased domain; the level index r + (m−2)/2 is then an integer subtraction on the bits of t, and the decided
// point (2r − 1)/s one FADD2 + one FFMA2 (the same value as the former FRND.CEIL / F2I path, which rounded x·s
// first; both are exact ceil semantics, they can differ only within one fp32 ulp of a boundary). A NaN input
// clamps to the lowest level on both paths.
constexpr float kSliceMagic = 12582912.0f;   // 1.5·2^23
// 32-cross labels as a 36-entry table (cell iI + 6·iQ), for a shared-memory copy (one LDS per label)
__device__ __forceinline__ void cross32_lut_fill(uint8_t* lut, int tid, int nthreads) {
  for (int c = tid; c < 36; c += nthreads) lut[c] = (uint8_t)cross32_label(c % 6, c / 6);
}
struct Slicer {
  int mI, mQ, hb, cross;
  float s, inv_s;
  float sh, loI, hiI, loQ, hiQ;   // s/2; clamp bounds of t per axis
  int offI, offQ;                 // level index = bits(t) − off
  const uint8_t* lut = nullptr;   // 32-cross label table in shared memory (nullptr: cross32_label)
  __device__ __forceinline__ int xlabel(int iI, int iQ) const {
    return lut ? (int)lut[iI + 6 * iQ] : cross32_label(iI, iQ);
  }
  // 32-cross: a corner cell (level 0 or 5 on both axes) goes to the nearer of its two inner neighbours (exact
  // tie: the lower label) — done on t (one level = ±1.0 exactly), so the point keeps the FMA-pipe form below
  __device__ __forceinline__ float2 cross_fix(float2 t, float2 z) const {
    const int iI = __float_as_int(t.x) - offI, iQ = __float_as_int(t.y) - offQ;
    if (__builtin_expect((0x21u >> iI) & (0x21u >> iQ) & 1u, 0)) {
      const float ax = fabsf(z.x * s), ay = fabsf(z.y * s);
      const int dQ = (iQ == 0) ? 1 : -1, dI = (iI == 0) ? 1 : -1;
      bool moveQ = ax > ay;
      if (__builtin_expect(ax == ay, 0)) moveQ = xlabel(iI, iQ + dQ) < xlabel(iI + dI, iQ);
      if (moveQ) t.y += (float)dQ; else t.x += (float)dI;
    }
    return t;
  }
  __device__ __forceinline__ void init(int M) {
    cross = (M == 32);
    if (M == 8) { mI = 4; mQ = 2; hb = 1; s = 2.44948974278317810f; }
    else if (M == 32) { mI = 6; mQ = 6; hb = 0; s = 4.47213595499957940f; }
    else {
      mI = mQ = (M == 4) ? 2 : (M == 16) ? 4 : 8;
      hb = (M == 4) ? 1 : (M == 16) ? 2 : 3;
      s = (M == 4) ? 1.41421356237309505f : (M == 16) ? 3.16227766016837933f : 6.48074069840786023f;
    }
    inv_s = 1.0f / s;
    sh = 0.5f * s;
    loI = kSliceMagic - (float)((mI - 2) / 2); hiI = kSliceMagic + (float)(mI / 2);
    loQ = kSliceMagic - (float)((mQ - 2) / 2); hiQ = kSliceMagic + (float)(mQ / 2);
    offI = __float_as_int(kSliceMagic) - (mI - 2) / 2;
    offQ = __float_as_int(kSliceMagic) - (mQ - 2) / 2;
  }
  // biased, clamped per-axis ceil: t = kSliceMagic + clamp(ceil(z·s/2))
  __device__ __forceinline__ float2 tq(float2 z) const {
    float tx, ty;
    asm("{\n\t.reg .b64 pa, pb, pc;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %4};\n\tmov.b64 pc, {%5, %5};\n\t"
        "fma.rp.f32x2 pa, pa, pb, pc;\n\tmov.b64 {%0, %1}, pa;\n\t}"
        : "=f"(tx), "=f"(ty) : "f"(z.x), "f"(z.y), "f"(sh), "f"(kSliceMagic));
    return make_float2(fminf(fmaxf(tx, loI), hiI), fminf(fmaxf(ty, loQ), hiQ));
  }
  // point (2r − 1)/s from t: (t − kSliceMagic)·(2/s) − 1/s, each lane one exact subtraction + one rounding
  __device__ __forceinline__ float2 point_t(float2 t) const {
    float px, py;
    asm("{\n\t.reg .b64 pa, pb, pc;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %4};\n\t"
        "sub.rn.f32x2 pa, pa, pb;\n\tmov.b64 pb, {%5, %5};\n\tmov.b64 pc, {%6, %6};\n\t"
        "fma.rn.f32x2 pa, pa, pb, pc;\n\tmov.b64 {%0, %1}, pa;\n\t}"
        : "=f"(px), "=f"(py) : "f"(t.x), "f"(t.y), "f"(kSliceMagic), "f"(2.0f * inv_s), "f"(-inv_s));
    return make_float2(px, py);
  }
  __device__ __forceinline__ void levels(float2 z, int& iI, int& iQ) const {
    const float2 t = tq(z);
    iI = __float_as_int(t.x) - offI;
    iQ = __float_as_int(t.y) - offQ;
    if (cross) {                                        // uniform: one format per frame / block
      // 32-cross corner cell → the nearer of the two adjacent points (rare); an exact tie (measure zero)
      // goes to the lower label
      if (__builtin_expect((iI == 0 || iI == 5) && (iQ == 0 || iQ == 5), 0)) {
        const float ax = fabsf(z.x * s), ay = fabsf(z.y * s);
        const int iQa = (iQ == 0) ? 1 : 4, iIb = (iI == 0) ? 1 : 4;
        if (ax > ay) iQ = iQa;
        else if (ay > ax) iI = iIb;
        else if (__builtin_expect(cross32_label(iI, iQa) < cross32_label(iIb, iQ), 0)) iQ = iQa;
        else iI = iIb;
      }
    }
  }
  __device__ __forceinline__ float2 point_i(int iI, int iQ) const {
    return make_float2((float)(2 * iI - (mI - 1)) * inv_s, (float)(2 * iQ - (mQ - 1)) * inv_s);
  }
  // decided point (the 32-cross corner rule on t; point_t(t) = point_i of t's levels, bit for bit: both round the
  // exact (2r − 1)/s once)
  __device__ __forceinline__ float2 point(float2 z) const {
    const float2 t = tq(z);
    return point_t(cross ? cross_fix(t, z) : t);
  }
  __device__ __forceinline__ int label_i(int iI, int iQ) const {
    return cross ? cross32_label(iI, iQ) : ((gray(iI) << hb) | gray(iQ));
  }
  // square / rectangular grids only (no 32-cross corner logic): gray(iI) << hb | gray(iQ)
  __device__ __forceinline__ int label_sq(float2 z) const {
    const float2 t = tq(z);
    return (gray(__float_as_int(t.x) - offI) << hb) | gray(__float_as_int(t.y) - offQ);
  }
  __device__ __forceinline__ int label(float2 z) const {
    float2 t = tq(z);
    if (cross) t = cross_fix(t, z);
    const int iI = __float_as_int(t.x) - offI, iQ = __float_as_int(t.y) - offQ;
    return cross ? xlabel(iI, iQ) : ((gray(iI) << hb) | gray(iQ));
  }
  // point and label of one decision from a single slicing (same values as point() / label())
  __device__ __forceinline__ float2 decide(float2 z, int& lab) const {
    if (!cross) {
      const float2 t = tq(z);
      lab = (gray(__float_as_int(t.x) - offI) << hb) | gray(__float_as_int(t.y) - offQ);
      return point_t(t);
    }
    const float2 t = cross_fix(tq(z), z);
    lab = xlabel(__float_as_int(t.x) - offI, __float_as_int(t.y) - offQ);
    return point_t(t);
  }
};

// ------------------------------------------------------------------ TMA 1-D bulk copy (cp.async.bulk) + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// order this CTA's earlier generic-proxy shared-memory accesses (made visible to the issuing thread by a barrier)
// before a following async-proxy (TMA) write to the same bytes — needed when a TMA refills a reused buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

}  // namespace kk
