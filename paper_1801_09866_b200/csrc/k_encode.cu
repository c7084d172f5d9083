// k_encode.cu -- step (a1): compression key of a history vector.
//
// The code (readings 3-6) is a pure function of the stored fp32 state, so it
// is computed ONCE when a state is created and stored with its slot, together
// with a 64-bit hash of the code words used as the probe position of the
// hidden-state cache; cache decisions always compare the full code.  The
// encoder itself is encode.cuh's encode32, shared with the tcgen05 epilogues.
#include "encode.cuh"

namespace rnnlm_dev {

// New states of this call: rows r < counts[1] (GRU rows), code + hash per row.
__global__ void k_encode_rows(Params P) {
  pdl_entry();
  const uint32_t rows = P.counts[1];
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    const uint32_t dst = P.row_dst[r];
    if (dst == NONE) continue;
    uint8_t *code = P.key_mode == RNNLM_KEY_OFF ? nullptr : P.codes + (size_t)dst * P.cstride;
    const unsigned long long hs = encode_row_warp(key_spec(P), P.cstride, P.state + (size_t)dst * P.H, code);
    if ((threadIdx.x & 31) == 0) P.codehash[dst] = hs;
  }
}

// Utterance root of sessions [lo, hi): handle 0 -> slot 0, zero state, ctx [<s>].
__global__ void k_reset_root(Params P, uint32_t lo) {
  const uint32_t s = lo + blockIdx.x;
  const size_t row = (size_t)s * P.cap;
  for (uint32_t i = threadIdx.x; i < P.H; i += blockDim.x) {
    P.state[row * P.H + i] = 0.0f;
  }
  if (threadIdx.x == 0) {
    Rec r;
    r.slot = 0;
    for (int j = 0; j < MAX_CTX; ++j) r.ctx[j] = NONE;
    if (P.N > 1) r.ctx[0] = 0u;                       // <s>
    P.rec[row] = r;
  }
  __syncthreads();
  if (threadIdx.x < 32 && P.cache) {
    uint8_t *code = P.key_mode == RNNLM_KEY_OFF ? nullptr : P.codes + row * P.cstride;
    const unsigned long long hs = encode_row_warp(key_spec(P), P.cstride, P.state + row * P.H, code);
    if (threadIdx.x == 0) P.codehash[row] = hs;
  }
}

// rnnlm_encode_states: arbitrary rows -> code_bytes per row (packed output).
__global__ void k_encode_states(Params P, uint32_t n, const float *__restrict__ states,
                                uint8_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t sm_code[];
  const int wib = threadIdx.x >> 5;
  const uint32_t r = blockIdx.x * (blockDim.x >> 5) + wib;
  if (r >= n) return;
  const float *h = states + (size_t)r * P.H;
  uint8_t *dst = out + (size_t)r * P.code_bytes;
  if (P.key_mode == RNNLM_KEY_OFF) {
    for (uint32_t b = threadIdx.x & 31; b < P.code_bytes; b += 32)
      dst[b] = reinterpret_cast<const uint8_t *>(h)[b];
    return;
  }
  uint8_t *code = sm_code + (size_t)wib * P.cstride;
  encode_row_warp(key_spec(P), P.cstride, h, code);
  __syncwarp();
  for (uint32_t b = threadIdx.x & 31; b < P.code_bytes; b += 32) dst[b] = code[b];
}

// rnnlm_read_codes: stored code of each handle's state.
__global__ void k_read_codes(Params P, uint32_t sess, uint32_t n, const uint32_t *__restrict__ h,
                             uint8_t *__restrict__ out) {
  const uint32_t i = blockIdx.x;
  if (i >= n) return;
  const uint32_t hd = h[i];
  uint8_t *dst = out + (size_t)i * P.code_bytes;
  const bool ok = sess < P.S && hd < P.ctr[sess].next_handle;
  const size_t slot = ok ? (size_t)sess * P.cap + P.rec[(size_t)sess * P.cap + hd].slot : 0;
  for (uint32_t b = threadIdx.x; b < P.code_bytes; b += blockDim.x) {
    uint8_t v = 0xFF;
    if (ok) v = P.key_mode == RNNLM_KEY_OFF
                    ? reinterpret_cast<const uint8_t *>(P.state + slot * P.H)[b]
                    : P.codes[slot * P.cstride + b];
    dst[b] = v;
  }
}

}  // namespace rnnlm_dev

namespace rnnlm_host {
using namespace rnnlm_dev;

int launch_encode_rows(const Params &P, uint32_t max_rows, int num_sms, cudaStream_t s) {
  if (!P.cache || max_rows == 0) return 0;
  uint32_t blocks = (max_rows + 7) / 8;
  const uint32_t cap = (uint32_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  launch_pdl(k_encode_rows, blocks, 256, 0, s, P);
  return 1;
}

int launch_reset_root(const Params &P, uint32_t lo, uint32_t hi, cudaStream_t s) {
  if (hi <= lo) return 0;
  k_reset_root<<<hi - lo, 256, 0, s>>>(P, lo);
  return 1;
}

int launch_encode_states(const Params &P, uint32_t n, const float *states, uint8_t *out,
                         cudaStream_t s) {
  if (!n) return 0;
  const int wpb = 4;
  k_encode_states<<<(n + wpb - 1) / wpb, 32 * wpb, wpb * P.cstride, s>>>(P, n, states, out);
  return 1;
}

int launch_read_codes(const Params &P, uint32_t sess, uint32_t n, const uint32_t *h, uint8_t *out,
                      cudaStream_t s) {
  if (!n) return 0;
  k_read_codes<<<n, 128, 0, s>>>(P, sess, n, h, out);
  return 1;
}
}  // namespace rnnlm_host
