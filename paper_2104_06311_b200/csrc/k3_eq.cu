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
//   (3) R = Σ conj(φ̃)φ̃ᵀ, p = Σ conj(φ̃)d;  θ₁ = (R + λI)⁻¹(p + λθ₀)        (fp64 Cholesky)
//   (4) y¹ = φ̃ᵀθ₁;  γ = Σ y¹·conj(D(y¹)) / Σ|D(y¹)|²;  u = y¹/|γ|           (unbias)
//   (5) per window b: c_b = Σ u·conj(D(u)),  z = u·conj(c_b)/|c_b|           (CPR: e^{−i·arg c_b})
//   (6) label = D(z); counts vs reference labels.
//
// R is assembled from its structure instead of a dense 2L×2L accumulation: with u_k[j] = y[2k − j],
//   R11[i][j] = S(i, j−i) (j ≥ i), S(i,d) = Σ_k conj(y[2k−i])·y[2k−i−d];   R22 = conj(R11)
//   R21[i][j] = T(min(i,j), |j−i|),  T(i,d) = Σ_k y[2k−i]·y[2k−i−d];      R12 = conj(R21)
// The CTA accumulates S and T only for i ∈ {−K, −K+1} (all lags d), i.e. 4L complex MACs per symbol,
// and walks i upward by 2 with the exact sliding-window correction
//   S(i+2, d) = S(i, d) + term_i(k0 − 1) − term_i(k1 − 1).
// Exactly the same matrix as the dense sum (up to rounding order).
//
// Mapping: one CTA (256 threads) per frame; thread t owns symbols t + 256·s (s < 16) so that every warp
// access to the frame's 2-sps samples is a contiguous 256-B shared-memory load (the samples are stored
// de-interleaved by parity). Block reductions: in-warp transpose-reduce (31 shuffles for 32 values),
// then an fp64 sum over the 8 warps in fixed order (deterministic).
#include "kk_device.cuh"
#include "kk_params.h"

namespace kk {

constexpr int K3_THREADS = 256;
constexpr int K3_WARPS = 8;
constexpr int K3_SPT = kFrameSym / K3_THREADS;   // 16 symbols per thread
constexpr int K3_G = 8;                          // lags / taps per accumulation pass

struct K3Smem {
  // dynamic layout offsets (bytes)
  int ye, yo, red, dred, S, T, P1, P2, A, rhs, th, misc, total;
};

__host__ __device__ inline K3Smem k3_layout(int K) {
  K3Smem l;
  const int L = 2 * K + 1, n = 2 * L, nd = 2 * K + 1;
  int o = 0;
  auto take = [&](int bytes) { int r = o; o += (bytes + 15) & ~15; return r; };
  l.ye = take((kFrameSym + K + 1) * 8);
  l.yo = take((kFrameSym + K + 1) * 8);
  l.red = take(K3_WARPS * 32 * 4);
  l.dred = take(32 * 8);
  l.S = take(2 * nd * 16);
  l.T = take(2 * nd * 16);
  l.P1 = take(L * 16);
  l.P2 = take(L * 16);
  l.A = take(n * n * 16);
  l.rhs = take(n * 16);
  l.th = take(n * 8);
  l.misc = take(64 * 4);
  l.total = o;
  return l;
}

// Sum 32 per-thread floats over the CTA: result (fp64) in dres[0..31] for all threads after return.
__device__ __forceinline__ void block_reduce32(float (&v)[32], float* red, double* dres, int lane, int warp) {
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
  red[warp * 32 + lane] = v[0];   // lane l holds the warp sum of element l
  __syncthreads();
  if (warp == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < K3_WARPS; ++w) s += (double)red[w * 32 + lane];
    dres[lane] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ double2 dmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 dmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int M>
__device__ __forceinline__ Decision slice_m(float2 z) { return slice<M>(z); }

__device__ __forceinline__ Decision slice_rt(float2 z, int M) {
  switch (M) {
    case 4: return slice<4>(z);
    case 8: return slice<8>(z);
    case 16: return slice<16>(z);
    case 32: return slice<32>(z);
    default: return slice<64>(z);
  }
}

__global__ void __launch_bounds__(K3_THREADS, 2)
k3_eq_kernel(const float2* __restrict__ y, int64_t frame0, int K, const float2* __restrict__ w_cd,
             const int* __restrict__ clampcnt, int64_t clamp_frame_off, const uint8_t* __restrict__ ref,
             uint8_t* __restrict__ dec, float2* __restrict__ zout, unsigned long long* __restrict__ counters,
             K3Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const K3Smem lay = k3_layout(K);
  float2* ye = reinterpret_cast<float2*>(smem + lay.ye);
  float2* yo = reinterpret_cast<float2*>(smem + lay.yo);
  float* red = reinterpret_cast<float*>(smem + lay.red);
  double* dred = reinterpret_cast<double*>(smem + lay.dred);
  double2* Sd = reinterpret_cast<double2*>(smem + lay.S);
  double2* Td = reinterpret_cast<double2*>(smem + lay.T);
  double2* P1 = reinterpret_cast<double2*>(smem + lay.P1);
  double2* P2 = reinterpret_cast<double2*>(smem + lay.P2);
  double2* Am = reinterpret_cast<double2*>(smem + lay.A);
  double2* rhs = reinterpret_cast<double2*>(smem + lay.rhs);
  float2* th = reinterpret_cast<float2*>(smem + lay.th);
  int* misc = reinterpret_cast<int*>(smem + lay.misc);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fl = blockIdx.x;
  const int64_t f = frame0 + fl;
  const int L = 2 * K + 1, nd = 2 * K + 1;
  const bool wl = p.widely_linear != 0;
  const int n = wl ? 2 * L : L;
  const int M = (int)p.schedule[(int)(((f / p.segment_frames) % p.n_segments + p.n_segments) % p.n_segments)];
  const int bi = (M == 4) ? 0 : (M == 8) ? 1 : (M == 16) ? 2 : (M == 32) ? 3 : 4;
  const int nbits = bi + 2;

  // ---- frame-level clamp count (K1 per-block counts) → dead-frame rule
  int ccount = 0;
  if (warp == 0) {
    int c = clampcnt[clamp_frame_off + (int64_t)fl * 32 + lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) misc[0] = c;
  }
  // ---- load the frame's 2-sps samples y[2k0 − K .. 2k0 + 8190 + K], de-interleaved by parity
  const float4* yf = reinterpret_cast<const float4*>(y + (int64_t)fl * (2 * kFrameSym));
  const int npair = kFrameSym + K;   // pairs (ys[2c], ys[2c+1]); the last odd element is unused padding
  for (int c = tid; c < npair; c += K3_THREADS) {
    const float4 v = __ldg(yf + c);
    ye[c] = make_float2(v.x, v.y);
    yo[c] = make_float2(v.z, v.w);
  }
  __syncthreads();
  ccount = misc[0];
  const bool dead = (ccount >= kFrameSamp);
  // y_s[i] (i = tap-local index, y_s[i] = y[2k0 − K + i]) for local symbol kl: y_s[2kl + i]
  auto Y = [&](int idx) -> float2 { return (idx & 1) ? yo[idx >> 1] : ye[idx >> 1]; };

  float2 u[K3_SPT];
  int bad = 0;
  if (!dead) {
    // ---- (1) pass 1 with θ₀ = [w_cd; 0]: y⁰_k = Σ_j w_j y[2k − j] = Σ_{a} w_cd[a]·y_s[2kl + 2K − a]
#pragma unroll
    for (int s = 0; s < K3_SPT; ++s) u[s] = make_float2(0.f, 0.f);
    for (int a = 0; a < L; ++a) {
      const float2 w = __ldg(&w_cd[a]);
      const int off = 2 * K - a;
#pragma unroll
      for (int s = 0; s < K3_SPT; ++s) cmac(u[s], w, Y(2 * (tid + K3_THREADS * s) + off));
    }
    float pw[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) pw[i] = 0.f;
#pragma unroll
    for (int s = 0; s < K3_SPT; ++s) pw[0] = fmaf(u[s].x, u[s].x, fmaf(u[s].y, u[s].y, pw[0]));
    block_reduce32(pw, red, dred, lane, warp);
    const double P0 = dred[0] / (double)kFrameSym;
    float g = (P0 > 0.0 && isfinite(P0)) ? (float)(1.0 / sqrt(P0)) : 1.0f;
    if (!(P0 > 0.0 && isfinite(P0))) bad = 1;
    // ---- (2) decisions on the AGC'd pass-1 output
    float2 dk[K3_SPT];
#pragma unroll
    for (int s = 0; s < K3_SPT; ++s) dk[s] = slice_rt(cscale(u[s], g), M).pt;

    // ---- (3a) structured R: S(i,d), T(i,d) for base i = −K + rho (rho ∈ {0,1}), lags d in groups of 8
    //      y[2k − i] = y_s[2kl + K − i] = y_s[2kl + 2K − rho];   y[2k − i − d] = y_s[2kl + 2K − rho − d]
    for (int rho = 0; rho < 2; ++rho) {
      for (int d0 = 0; d0 < nd; d0 += K3_G) {
        float acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.f;
#pragma unroll 2
        for (int s = 0; s < K3_SPT; ++s) {
          const int ia = 2 * (tid + K3_THREADS * s) + 2 * K - rho;
          const float2 ya = Y(ia);
#pragma unroll
          for (int g8 = 0; g8 < K3_G; ++g8) {
            const int d = d0 + g8;
            if (d < nd) {
              const float2 yb = Y(ia - d);
              float2 sacc = make_float2(acc[4 * g8], acc[4 * g8 + 1]);
              float2 tacc = make_float2(acc[4 * g8 + 2], acc[4 * g8 + 3]);
              cmac_conj(sacc, ya, yb);
              cmac(tacc, ya, yb);
              acc[4 * g8] = sacc.x; acc[4 * g8 + 1] = sacc.y; acc[4 * g8 + 2] = tacc.x; acc[4 * g8 + 3] = tacc.y;
            }
          }
        }
        block_reduce32(acc, red, dred, lane, warp);
        if (tid < K3_G) {
          const int d = d0 + tid;
          if (d < nd) {
            Sd[rho * nd + d] = make_double2(dred[4 * tid], dred[4 * tid + 1]);
            Td[rho * nd + d] = make_double2(dred[4 * tid + 2], dred[4 * tid + 3]);
          }
        }
      }
    }
    // ---- (3b) p1[j] = Σ conj(y[2k−j])·d_k, p2[j] = Σ y[2k−j]·d_k; y[2k − j] = y_s[2kl + K − j], a = j + K
    for (int a0 = 0; a0 < L; a0 += K3_G) {
      float acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = 0.f;
#pragma unroll
      for (int s = 0; s < K3_SPT; ++s) {
        const int base = 2 * (tid + K3_THREADS * s) + 2 * K;
        const float2 dd = dk[s];
#pragma unroll
        for (int g8 = 0; g8 < K3_G; ++g8) {
          const int a = a0 + g8;
          if (a < L) {
            const float2 yv = Y(base - a);
            float2 p1 = make_float2(acc[4 * g8], acc[4 * g8 + 1]);
            float2 p2 = make_float2(acc[4 * g8 + 2], acc[4 * g8 + 3]);
            cmac_conj(p1, yv, dd);
            cmac(p2, yv, dd);
            acc[4 * g8] = p1.x; acc[4 * g8 + 1] = p1.y; acc[4 * g8 + 2] = p2.x; acc[4 * g8 + 3] = p2.y;
          }
        }
      }
      block_reduce32(acc, red, dred, lane, warp);
      if (tid < K3_G && a0 + tid < L) {
        P1[a0 + tid] = make_double2(dred[4 * tid], dred[4 * tid + 1]);
        P2[a0 + tid] = make_double2(dred[4 * tid + 2], dred[4 * tid + 3]);
      }
    }
    __syncthreads();

    // ---- (3c) assemble R + λI and rhs = p + λθ₀ (fp64), then Cholesky solve — warp 0
    if (warp == 0) {
      // S(i,d) for all i ∈ [−K, K − d] by the sliding recurrence; store R11 / R21 blocks directly.
      // y_s local index of y[2k − i] for the edge symbols: k0 − 1 → K − 2 − i ; k1 − 1 → 8192 + K − 2 − i
      for (int d = lane; d < nd; d += 32) {
        for (int rho = 0; rho < 2; ++rho) {
          double2 sv = Sd[rho * nd + d], tv = Td[rho * nd + d];
          for (int i = -K + rho; i + d <= K; i += 2) {
            const int r = i + K, c = i + d + K;     // R11[r][c] (c ≥ r), R21[r][c]
            Am[r * n + c] = sv;
            Am[c * n + r] = make_double2(sv.x, -sv.y);
            if (wl) {
              // R21 = T_sym, R12 = conj(T_sym), R22 = conj(R11)
              Am[(L + r) * n + c] = tv; Am[(L + c) * n + r] = tv;
              Am[r * n + (L + c)] = make_double2(tv.x, -tv.y); Am[c * n + (L + r)] = make_double2(tv.x, -tv.y);
              Am[(L + r) * n + (L + c)] = make_double2(sv.x, -sv.y);
              Am[(L + c) * n + (L + r)] = sv;
            }
            // advance i → i + 2
            if (i + 2 + d > K) break;
            const int lo1 = K - 2 - i, lo2 = lo1 - d;
            const int hi1 = 2 * kFrameSym + K - 2 - i, hi2 = hi1 - d;
            const float2 a1 = Y(lo1), a2 = Y(lo2), b1 = Y(hi1), b2 = Y(hi2);
            sv.x += (double)a1.x * a2.x + (double)a1.y * a2.y - ((double)b1.x * b2.x + (double)b1.y * b2.y);
            sv.y += (double)a1.x * a2.y - (double)a1.y * a2.x - ((double)b1.x * b2.y - (double)b1.y * b2.x);
            tv.x += (double)a1.x * a2.x - (double)a1.y * a2.y - ((double)b1.x * b2.x - (double)b1.y * b2.y);
            tv.y += (double)a1.x * a2.y + (double)a1.y * a2.x - ((double)b1.x * b2.y + (double)b1.y * b2.x);
          }
        }
      }
      __syncwarp();
      double tr = 0.0;
      for (int a = 0; a < n; ++a) tr += Am[a * n + a].x;
      const double lam = (double)p.ridge * tr / (double)n;
      for (int a = lane; a < n; a += 32) {
        Am[a * n + a].x += lam;
        const double2 pv = (a < L) ? P1[a] : P2[a - L];
        double2 t0 = make_double2(0.0, 0.0);
        if (a < L) { const float2 w = w_cd[a]; t0 = make_double2((double)g * w.x, (double)g * w.y); }
        rhs[a] = make_double2(pv.x + lam * t0.x, pv.y + lam * t0.y);
      }
      __syncwarp();
      // right-looking Cholesky A = L·Lᴴ (lower), in place
      int fail = 0;
      for (int k = 0; k < n; ++k) {
        const double dkk = Am[k * n + k].x;
        fail |= !(dkk > 0.0) || !isfinite(dkk);
        const double lkk = sqrt(fabs(dkk) + 1e-300);
        const double inv = 1.0 / lkk;
        __syncwarp();
        for (int i = k + 1 + lane; i < n; i += 32) {
          Am[i * n + k] = make_double2(Am[i * n + k].x * inv, Am[i * n + k].y * inv);
        }
        if (lane == 0) Am[k * n + k] = make_double2(lkk, 0.0);
        __syncwarp();
        for (int i = k + 1 + lane; i < n; i += 32) {
          const double2 lik = Am[i * n + k];
          for (int j = k + 1; j <= i; ++j) {
            const double2 t = dmulc(lik, Am[j * n + k]);
            Am[i * n + j].x -= t.x; Am[i * n + j].y -= t.y;
          }
        }
        __syncwarp();
      }
      // forward: L z = rhs ; backward: Lᴴ θ = z  (column-oriented, lanes over rows)
      for (int k = 0; k < n; ++k) {
        const double inv = 1.0 / Am[k * n + k].x;
        if (lane == 0) rhs[k] = make_double2(rhs[k].x * inv, rhs[k].y * inv);
        __syncwarp();
        const double2 zk = rhs[k];
        for (int i = k + 1 + lane; i < n; i += 32) {
          const double2 t = dmul(Am[i * n + k], zk);
          rhs[i].x -= t.x; rhs[i].y -= t.y;
        }
        __syncwarp();
      }
      for (int k = n - 1; k >= 0; --k) {
        const double inv = 1.0 / Am[k * n + k].x;
        if (lane == 0) rhs[k] = make_double2(rhs[k].x * inv, rhs[k].y * inv);
        __syncwarp();
        const double2 xk = rhs[k];
        for (int i = lane; i < k; i += 32) {   // rhs[i] -= conj(L[k][i]) · x_k
          const double2 lki = Am[k * n + i];
          const double2 t = make_double2(lki.x * xk.x + lki.y * xk.y, lki.x * xk.y - lki.y * xk.x);
          rhs[i].x -= t.x; rhs[i].y -= t.y;
        }
        __syncwarp();
      }
      for (int a = 0; a < n; ++a) fail |= !isfinite(rhs[a].x) || !isfinite(rhs[a].y);
      for (int a = lane; a < 2 * L; a += 32) {
        float2 v;
        if (fail) {
          v = (a < L) ? make_float2(g * w_cd[a].x, g * w_cd[a].y) : make_float2(0.f, 0.f);
        } else {
          v = (a < n) ? make_float2((float)rhs[a].x, (float)rhs[a].y) : make_float2(0.f, 0.f);
        }
        th[a] = v;
      }
      if (lane == 0) misc[1] = fail;
    }
    __syncthreads();
    bad |= misc[1];

    // ---- (4) pass 2: y¹_k = Σ_a w_a·y_s[2kl + 2K − a] + v_a·conj(y_s[...])
#pragma unroll
    for (int s = 0; s < K3_SPT; ++s) u[s] = make_float2(0.f, 0.f);
    for (int a = 0; a < L; ++a) {
      const float2 w = th[a], v = th[L + a];
      const int off = 2 * K - a;
#pragma unroll
      for (int s = 0; s < K3_SPT; ++s) {
        const float2 yv = Y(2 * (tid + K3_THREADS * s) + off);
        cmac(u[s], w, yv);
        cmac(u[s], v, cconj(yv));
      }
    }
    // gain unbias γ = Σ y¹·conj(D(y¹)) / Σ|D(y¹)|²
    {
      float acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = 0.f;
#pragma unroll
      for (int s = 0; s < K3_SPT; ++s) {
        const float2 dd = slice_rt(u[s], M).pt;
        const float2 c = cmulc(u[s], dd);
        acc[0] += c.x; acc[1] += c.y; acc[2] = fmaf(dd.x, dd.x, fmaf(dd.y, dd.y, acc[2]));
      }
      block_reduce32(acc, red, dred, lane, warp);
      const double gr = dred[0] / dred[2], gi = dred[1] / dred[2];
      const double ag = sqrt(gr * gr + gi * gi);
      float sc = 1.0f;
      if (ag > 0.0 && isfinite(ag)) sc = (float)(1.0 / ag); else bad = 1;
#pragma unroll
      for (int s = 0; s < K3_SPT; ++s) u[s] = cscale(u[s], sc);
    }
    // ---- (5) CPR: window index of symbol tid + 256 s is s / (W/256)
    {
      float acc[32];
#pragma unroll
      for (int s = 0; s < K3_SPT; ++s) {
        const float2 dd = slice_rt(u[s], M).pt;
        const float2 c = cmulc(u[s], dd);
        acc[2 * s] = c.x; acc[2 * s + 1] = c.y;
      }
      block_reduce32(acc, red, dred, lane, warp);
      const int per = p.cpr_window / K3_THREADS;   // s-values per window (1, 2, 4, 8, 16)
#pragma unroll
      for (int s = 0; s < K3_SPT; ++s) {
        const int w0 = (s / per) * per;
        double cr = 0.0, ci = 0.0;
        for (int q = 0; q < per; ++q) { cr += dred[2 * (w0 + q)]; ci += dred[2 * (w0 + q) + 1]; }
        const double mag = sqrt(cr * cr + ci * ci);
        float2 rot = make_float2(1.f, 0.f);
        if (mag > 0.0) rot = make_float2((float)(cr / mag), (float)(-ci / mag));
        u[s] = cmul(u[s], rot);
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < K3_SPT; ++s) u[s] = make_float2(0.f, 0.f);
  }

  // ---- (6) decisions, counts, outputs
  int serr = 0, berr = 0;
  const int64_t sym0 = (int64_t)fl * kFrameSym;
#pragma unroll
  for (int s = 0; s < K3_SPT; ++s) {
    const int kl = tid + K3_THREADS * s;
    const int lab = slice_rt(u[s], M).lab;
    if (ref) {
      const int r = ref[sym0 + kl];
      serr += (lab != r);
      berr += __popc(lab ^ r);
    }
    if (dec) dec[sym0 + kl] = (uint8_t)lab;
    if (zout) zout[sym0 + kl] = u[s];
  }
  if (ref) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      serr += __shfl_xor_sync(0xffffffffu, serr, o);
      berr += __shfl_xor_sync(0xffffffffu, berr, o);
    }
    if (lane == 0) { misc[8 + warp] = serr; misc[16 + warp] = berr; }
  }
  __syncthreads();
  if (tid == 0) {
    if (ref) {
      long long se = 0, be = 0;
      for (int w = 0; w < K3_WARPS; ++w) { se += misc[8 + w]; be += misc[16 + w]; }
      if (se) atomicAdd(&counters[5 + bi], (unsigned long long)se);
      if (be) atomicAdd(&counters[15 + bi], (unsigned long long)be);
    }
    atomicAdd(&counters[bi], (unsigned long long)kFrameSym);
    atomicAdd(&counters[10 + bi], (unsigned long long)kFrameSym * nbits);
    if (ccount) atomicAdd(&counters[20], (unsigned long long)ccount);
    atomicAdd(&counters[21], 1ull);
    if (dead) atomicAdd(&counters[22], 1ull);
    if (!dead && bad) atomicAdd(&counters[23], 1ull);
  }
}

size_t k3_smem_bytes(int K) { return (size_t)k3_layout(K).total; }

void launch_k3(const float2* y, int64_t frame0, int64_t n_frames, int K, const float2* w_cd, const int* clampcnt,
               int64_t clamp_frame_off, const uint8_t* ref, uint8_t* dec, float2* z, unsigned long long* counters,
               const K3Params& p, cudaStream_t s) {
  const size_t smem = k3_smem_bytes(K);
  cudaFuncSetAttribute(k3_eq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k3_eq_kernel<<<(unsigned)n_frames, K3_THREADS, smem, s>>>(y, frame0, K, w_cd, clampcnt, clamp_frame_off, ref, dec,
                                                            z, counters, p);
}

}  // namespace kk
