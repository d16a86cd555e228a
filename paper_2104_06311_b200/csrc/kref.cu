// kref.cu — the transmitter's known reference labels, generated on the device (kk_config.ref_prbs: 1 = the
// synthetic transmitter's counter hash, 2 = the ITU-T O.150 PRBS-31 stream).
//
// the BER is counted against the transmitted sequence, which the real-time receiver knows (a
// pattern synchronised to the received stream), so it need not cross PCIe with the samples. The sequence is the
// synthetic transmitter's (kkgen.symbol_labels): label(k) = H(seed, k) & (M(k) − 1) for global
// symbol k, with H the counter-based 32-bit hash (murmur3 fmix32 rounds keyed by the seed; stream 1) and M(k) the
// QAM order of k's frame from the R26 schedule. Integer arithmetic only — bit-exact with the generator.
#include <cstdint>
#include <cuda_runtime.h>

namespace kk {

__device__ __forceinline__ uint32_t fmix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return x;
}

// one thread per 16 consecutive symbols (one 16-B store); n_sym is a multiple of 4096 (whole frames)
__global__ void ref_prbs_kernel(uint8_t* __restrict__ out, int64_t sym0, int64_t n_sym, uint32_t key,
                                const uint8_t* __restrict__ schedule, int n_segments, int64_t segment_frames) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (16 * g >= n_sym) return;
  const int64_t k0 = sym0 + 16 * g;
  const int64_t f = k0 / 4096;                      // 16 | 4096: one frame per thread
  const uint32_t mask = (uint32_t)schedule[(int)(((f / segment_frames) % n_segments + n_segments) % n_segments)] - 1u;
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int64_t k = k0 + i;
    const uint32_t lo = (uint32_t)k, hi = (uint32_t)(k >> 32);
    uint32_t h = fmix32(lo ^ key);
    h = fmix32(h ^ hi ^ 0x68E31DA4u);
    h = fmix32(h ^ key);
    w[i >> 2] |= (h & mask) << (8 * (i & 3));
  }
  reinterpret_cast<uint4*>(out)[g] = make_uint4(w[0], w[1], w[2], w[3]);
}

// ---- ITU-T O.150 PRBS-31 (x^31 + x^28 + 1) label stream (kk_config.ref_prbs = 2): bit b[n] = b[n−28] ⊕ b[n−31],
// b[0..30] = the bits of W0(ref_seed); symbol k owns bits 6k … 6k+5 (slot, LSB first), label = slot & (M(k) − 1).
// The 31-bit window W_n = Σ_i b[n+i]·2^i evolves linearly over GF(2), W_{n+1} = (W_n >> 1) | ((b[n] ⊕ b[n+3]) << 30),
// so each thread jumps to its 96-bit block with the binary powers A^(2^j) (constant memory) — the same stream as
// kkgen.prbs31_slots, bit for bit, at any global position.
constexpr uint32_t kPrbsPeriod = 0x7FFFFFFFu;       // 2^31 − 1: the order of A
__constant__ uint32_t c_prbs_pow[31][31];           // [j][i] = A^(2^j)·e_i

__device__ __forceinline__ uint32_t gf2_apply(const uint32_t (&cols)[31], uint32_t w) {
  uint32_t r = 0u;
#pragma unroll
  for (int i = 0; i < 31; ++i) r ^= ((w >> i) & 1u) ? cols[i] : 0u;
  return r;
}

__global__ void ref_prbs31_kernel(uint8_t* __restrict__ out, int64_t sym0, int64_t n_sym, uint32_t w0,
                                  const uint8_t* __restrict__ schedule, int n_segments, int64_t segment_frames) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (16 * g >= n_sym) return;
  const int64_t k0 = sym0 + 16 * g;                 // a multiple of 16 (sym0: whole frames)
  const int64_t f = k0 / 4096;
  const uint32_t mask = (uint32_t)schedule[(int)(((f / segment_frames) % n_segments + n_segments) % n_segments)] - 1u;
  const uint32_t e = (uint32_t)(((uint64_t)(k0 / 16) * 96u) % kPrbsPeriod);
  uint32_t w = w0;
  for (int j = 0; j < 31; ++j)
    if ((e >> j) & 1u) w = gf2_apply(c_prbs_pow[j], w);
  constexpr uint32_t m28 = (1u << 28) - 1u;
  const uint32_t n1 = ((w >> 3) ^ w) & m28;                      // b[31 .. 58]
  const uint32_t w1 = (w >> 28) | (n1 << 3);
  const uint32_t n2 = ((w1 >> 3) ^ w1) & m28;                    // b[59 .. 86]
  const uint32_t w2 = (w1 >> 28) | (n2 << 3);
  const uint32_t n3 = ((w2 >> 3) ^ w2) & m28;                    // b[87 .. 114]
  const uint64_t lo = (uint64_t)w | ((uint64_t)n1 << 31) | ((uint64_t)(n2 & 31u) << 59);
  const uint64_t hi = (uint64_t)(n2 >> 5) | ((uint64_t)n3 << 23);
  uint32_t wd[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int off = 6 * i;
    const uint64_t v = off < 64 ? ((lo >> off) | (off ? (hi << (64 - off)) : 0ull)) : (hi >> (off - 64));
    wd[i >> 2] |= ((uint32_t)v & 63u & mask) << (8 * (i & 3));
  }
  reinterpret_cast<uint4*>(out)[g] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

uint32_t ref_prbs31_w0(uint32_t seed) {               // kkgen.prbs31_w0
  const uint32_t w = (uint32_t)(seed * 0x9E3779B1u) >> 1;
  return w ? w : 1u;
}

cudaError_t ref_prbs31_init() {                       // A^(2^j) columns → constant memory (once per process)
  static bool done = false;
  if (done) return cudaSuccess;
  uint32_t pw[31][31];
  for (int i = 0; i < 31; ++i) {
    const uint32_t v = 1u << i;
    pw[0][i] = (v >> 1) | ((((v) ^ (v >> 3)) & 1u) << 30);
  }
  for (int j = 1; j < 31; ++j)
    for (int i = 0; i < 31; ++i) {
      uint32_t r = 0u;
      for (int t = 0; t < 31; ++t) if ((pw[j - 1][i] >> t) & 1u) r ^= pw[j - 1][t];
      pw[j][i] = r;
    }
  const cudaError_t e = cudaMemcpyToSymbol(c_prbs_pow, pw, sizeof(pw));
  if (e == cudaSuccess) done = true;
  return e;
}

void launch_ref_prbs31(uint8_t* out, int64_t sym0, int64_t n_sym, uint32_t w0, const uint8_t* schedule,
                       int n_segments, int64_t segment_frames, cudaStream_t s) {
  const int64_t threads = n_sym / 16;
  const int bs = 256;
  ref_prbs31_kernel<<<(unsigned)((threads + bs - 1) / bs), bs, 0, s>>>(out, sym0, n_sym, w0, schedule, n_segments,
                                                                        segment_frames);
}

uint32_t ref_prbs_key(uint32_t seed) {              // H's key for stream 1 (host side, once per context)
  uint32_t x = (seed * 0x9E3779B1u) ^ (1u * 0x7F4A7C15u);
  x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16;
  return x;
}

void launch_ref_prbs(uint8_t* out, int64_t sym0, int64_t n_sym, uint32_t key, const uint8_t* schedule,
                     int n_segments, int64_t segment_frames, cudaStream_t s) {
  const int64_t threads = n_sym / 16;
  const int bs = 256;
  ref_prbs_kernel<<<(unsigned)((threads + bs - 1) / bs), bs, 0, s>>>(out, sym0, n_sym, key, schedule, n_segments,
                                                                      segment_frames);
}

}  // namespace kk
