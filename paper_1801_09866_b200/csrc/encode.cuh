// encode.cuh -- step (a1): the compression key of a history vector, ONE device
// implementation shared by every producer of a code (the tcgen05 GRU
// epilogues, the FP32 path's k_encode_rows, the root state of k_reset_root
// and the inspection call rnnlm_encode_states), so the codes the tests probe
// are produced by the same instructions as the codes the cache compares.
//
// "we propose to quantize the history vectors by controlling the precision of
// history vector itself by rounding up to a specified decimal point.  We also
// consider an extreme case, in which we store only the signs of each element"
// (Table 1).  Readings 3-6:
//   sign     bit_i = (h_i >= 0.0f)                  (IEEE compare: -0 -> 1)
//   round:k  q_i = roundf(__fmul_rn(h_i, 10^k))     (fp32 product, half away)
//            int8 for k <= 2, little-endian int16 for k = 3, 4
//   off      the fp32 bit pattern (the state row itself is the code)
// Packing: sign bits LSB-first in 32-bit words; round codes in element order.
// Alongside the code, a 64-bit hash Σ mix64(word index << 32 | word) over the
// code's 32-bit words (off mode: over the elements' bit patterns).  The terms
// add, so chunks of a row combine in any order (one atomicAdd per epilogue
// tile); the hash only picks the hidden cache's probe start -- decisions always
// compare the full code.
#pragma once

#include "rnnlm_impl.cuh"

namespace rnnlm_dev {

struct KeySpec {
  uint32_t mode, digits, H;
  float scale;                      // 10^digits in fp32 (round mode)
};

__device__ __forceinline__ KeySpec key_spec(const Params &P) {
  return KeySpec{P.key_mode, P.round_digits, P.H, P.round_scale};
}

__device__ __forceinline__ uint32_t rnd8(float h, float s) {
  return (uint32_t)(uint8_t)(int8_t)(int)roundf(__fmul_rn(h, s));
}
__device__ __forceinline__ uint32_t rnd16(float h, float s) {
  return (uint32_t)(uint16_t)(int16_t)(int)roundf(__fmul_rn(h, s));
}

// Code words and hash terms of the 16 state elements h[0..15] = units
// u0 .. u0+15 (u0 % 16 == 0).  Units >= H are absent: their bits / codes are
// zero, and code words that hold only absent units are neither written nor
// hashed.  code == nullptr: hash only.  Sign words hold 32 units, so the
// first half of a word (u0 % 32 == 0) is parked in signacc and the word is
// written and hashed by the call for its second half (always made, see
// encode32).
__device__ __forceinline__ unsigned long long encode16(const KeySpec &k, const float *h, uint32_t u0,
                                                       uint8_t *code, uint32_t &signacc) {
  unsigned long long hs = 0;
  const bool full = u0 + 16 <= k.H;
  if (k.mode == RNNLM_KEY_SIGN) {
    uint32_t b = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) b |= ((full || u0 + j < k.H) && h[j] >= 0.0f ? 1u : 0u) << j;
    if ((u0 & 31) == 0) {
      signacc = b;
    } else if (u0 - 16 < k.H) {
      const uint32_t word = signacc | (b << 16), wi = u0 >> 5;
      if (code) reinterpret_cast<uint32_t *>(code)[wi] = word;
      hs += mix64(((unsigned long long)wi << 32) | word);
    }
  } else if (k.mode == RNNLM_KEY_ROUND && k.digits <= 2) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (full || u0 + 4 * i + j < k.H) word |= rnd8(h[4 * i + j], k.scale) << (8 * j);
      w[i] = word;
      if (full || u0 + 4 * i < k.H) hs += mix64(((unsigned long long)(u0 / 4 + i) << 32) | word);
    }
    if (code) {
      if (full) {
        *reinterpret_cast<uint4 *>(code + u0) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (u0 + 4 * i < k.H) reinterpret_cast<uint32_t *>(code)[u0 / 4 + i] = w[i];
      }
    }
  } else if (k.mode == RNNLM_KEY_ROUND) {
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (full || u0 + 2 * i + j < k.H) word |= rnd16(h[2 * i + j], k.scale) << (16 * j);
      w[i] = word;
      if (full || u0 + 2 * i < k.H) hs += mix64(((unsigned long long)(u0 / 2 + i) << 32) | word);
    }
    if (code) {
      if (full) {
        *reinterpret_cast<uint4 *>(code + 2 * u0) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4 *>(code + 2 * u0 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (u0 + 2 * i < k.H) reinterpret_cast<uint32_t *>(code)[u0 / 2 + i] = w[i];
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (full || u0 + j < k.H) hs += mix64(((unsigned long long)(u0 + j) << 32) | __float_as_uint(h[j]));
  }
  return hs;
}

// The 32 elements h[0..31] = units u0 .. u0+31 (u0 % 32 == 0): both halves.
__device__ __forceinline__ unsigned long long encode32(const KeySpec &k, const float *h, uint32_t u0,
                                                       uint8_t *code) {
  uint32_t signacc = 0;
  unsigned long long hs = encode16(k, h, u0, code, signacc);
  hs += encode16(k, h + 16, u0 + 16, code, signacc);
  return hs;
}

// One warp encodes one row h[0..H) into code (nullptr: hash only; the pad
// bytes up to cstride are zeroed).  Lane l takes the 32-unit chunks l, l+32,
// ...  Returns the row's code hash in every lane.
__device__ __forceinline__ unsigned long long encode_row_warp(const KeySpec &k, uint32_t cstride,
                                                              const float *__restrict__ h,
                                                              uint8_t *__restrict__ code) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long hs = 0;
  for (uint32_t u0 = lane * 32; u0 < k.H; u0 += 32 * 32) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = u0 + j < k.H ? h[u0 + j] : 0.0f;
    hs += encode32(k, v, u0, code);
  }
  if (code && k.mode != RNNLM_KEY_OFF) {
    const uint32_t nbytes = k.mode == RNNLM_KEY_SIGN ? (k.H + 31) / 32 * 4
                            : k.digits <= 2          ? (k.H + 3) / 4 * 4
                                                     : (k.H + 1) / 2 * 4;
    for (uint32_t wi = nbytes / 4 + lane; wi < cstride / 4; wi += 32) reinterpret_cast<uint32_t *>(code)[wi] = 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
  return hs;
}

}  // namespace rnnlm_dev
