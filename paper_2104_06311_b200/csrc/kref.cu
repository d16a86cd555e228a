// kref.cu — the transmitter's known reference labels, generated on the device (kk_config.ref_prbs).
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
