// k_gru_tc.cu -- step (a5), tensor-core paths on sm_100a (tcgen05 + TMEM + TMA):
// BF16 operands (kind::f16), TF32 operands (kind::tf32), and 3xTF32 (kind::tf32
// over [hi | lo] operand parts in three K segments: the FP32 path's accuracy).
//
// The GRU gate contraction of the frame's MISS rows (the
// frame's (h || x) rows form one block) is a real dense contraction:
// [Q, E+H] x [E+H, 3H] for Q misses (Chung form, reading 1), executed as
//
//   gather   A1[r] = [x | bf16(h)] (x = E[word] bf16, h = the fp32 parent
//            state), one warp per row, 16-byte vector copies (k_gather_a1).
//   phase 1  z, r: A = A1 (TMA), B = W1 [(H/128) x 256 rows][E+H] bf16 (TMA;
//            per 128-unit block 128 rows [Wz|Uz] then 128 rows [Wr|Ur]),
//            tile 128 x 256, K = E+H.  Epilogue: z = s(.+bz) (fp32) and
//            r.h = s(.+br) * h (bf16, phase-2 A operand).
//   phase 2  candidate: A = [x | r.h] (x chunks from A1, recurrent chunks from
//            the r.h rows, both TMA), B = W2 [H rows][E+H] = [Wh | Uh] (TMA),
//            tile 128 x 256, K = E+H: the accumulator is Wh x + Uh (r.h)
//            directly (no fp32 round trip of Wh x).  Epilogue:
//            c = tanh(. + bh), h' = (1-z) h + z c, the new fp32 state and
//            (a1) its compression code + code-hash contribution
//            (hash terms add, so the N-tiles of a row combine with one 64-bit
//            atomicAdd each, order-independent).
//
// Both phases run in ONE persistent kernel (grid <= #SMs) over a merged tile
// list in which the phase-2 tiles of an M-tile trail its phase-1 tiles; a
// per-M-tile counter (release by the phase-1 epilogues, acquire by the TMA
// producer of the phase-2 tile) carries the r.h / z dependency, so phase 2 of
// early rows overlaps phase 1 of later rows and neither phase has a wave
// tail.  Warp-specialised: one TMA producer thread, one MMA-issuing thread
// (tcgen05.mma.cta_group::1.kind::f16, M = 128, N = 256), eight epilogue
// warps (tcgen05.ld.32x32b: TMEM lane quarter = warp % 4, two warps per
// quarter split the columns).  Pipelines
// are mbarrier rings (full / empty per smem stage, full / empty per TMEM
// accumulator; two 256-column accumulators, so the epilogue of tile i
// overlaps the MMAs of tile i+1).  Rows >= Q read stale A rows and are
// discarded.
//
// Variants of the same kernel template (k_gru_tc<T, CELL>): CELL 1 = the
// linear-before-reset GRU (one phase, tiles of 64 units x [Wh x | z | r | Uh h]
// over W3, see mma_loop), CELL 2 = the vanilla RNN (one phase, A1 x [Wh | Uh]);
// phase-2 / RNN tiles narrow to 128 units when H % 256 != 0 (a.bn2); the CTA
// pair k_gru_tc2 (cta_group::2, M = 256) runs the bf16 GRU cell when
// H % 256 == 0 (RNNLM_TC_PAIR=0 selects one CTA per tile), and RNNLM_TC_DIAG selects the timing diagnostics of
// DESIGN.md section 5.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "rnnlm_impl.cuh"
#include "tc_common.cuh"
#include "encode.cuh"

namespace rnnlm_tc {
using namespace rnnlm_dev;

constexpr int BM = 128;          // UMMA M (rows per tile)
constexpr int BK = 64;           // K elements per smem stage (= one 128-byte swizzle atom)
constexpr int UB = 128;          // units per phase-1 block
constexpr int BN = 256;          // UMMA N of both phases (phase 1: z|r of 128 units; phase 2: 256 units)
#ifndef RNNLM_TC_ST
#define RNNLM_TC_ST 4
#endif
constexpr int ST = RNNLM_TC_ST;  // smem pipeline stages (one-CTA kernel; GRU, LBR cells)
#ifndef RNNLM_TC_ST_RNN
#define RNNLM_TC_ST_RNN 3
#endif
// the RNN cell's kernel is short and its step is bound by the side-stream
// scoring that shares its SMs: 3 stages leave that scoring 48 KB more L1
// (1,274-1,326 vs 1,068-1,071 M q/s, profiles/ab_st1_r1.txt)
template <int CELL>
__host__ __device__ constexpr int st_of() { return CELL == RNNLM_CELL_RNN ? RNNLM_TC_ST_RNN : ST; }
constexpr int A_BYTES = BM * BK * 2;          // 16 KB
constexpr int B_BYTES = BN * BK * 2;          // 32 KB
constexpr int TMEM_COLS = 512;                // 2 accumulators x 256 columns
constexpr int STG_BYTES = 32 * 128;           // epilogue staging buffer per epilogue warp

// Operand element type of the fused kernel: bf16 (kind::f16) or fp32 read as
// TF32 (kind::tf32).  A smem stage is one 128-byte swizzle atom of K either
// way (64 bf16 / 32 fp32 elements), four 32-byte MMA K-steps per stage.
template <typename T> struct Op;
template <> struct Op<__nv_bfloat16> {
  static constexpr int BKE = 64;
  static constexpr uint32_t FMT = 1;
  static __device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    umma_bf16(d, a, b, id, acc);
  }
};
template <> struct Op<float> {
  static constexpr int BKE = 32;
  static constexpr uint32_t FMT = 2;
  static __device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    umma_tf32(d, a, b, id, acc);
  }
};

// fp32 -> TF32 (10 explicit mantissa bits), round to nearest, ties away; the
// result is an fp32 bit pattern with the low 13 bits zero, which the MMA
// reads exactly (no truncation of the operand inside the tensor core).
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float4 to_tf32(float4 v) {
  return make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
}

// fp32 -> bf16 parts v = hi + mid + lo (each round to nearest even of the
// remainder, which is exact in fp32): |v - hi - mid - lo| <= 2^-27 |v|, and
// every part times a bf16 weight part is exact in the fp32 accumulator.
__device__ __forceinline__ float bf16_part(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
__device__ __forceinline__ void split3(float v, float &hi, float &mid, float &lo) {
  hi = bf16_part(v);
  const float r = v - hi;
  mid = bf16_part(r);
  lo = bf16_part(r - mid);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {      // a, b already on the bf16 grid
  return (__float_as_uint(a) >> 16) | (__float_as_uint(b) & 0xFFFF0000u);
}
__device__ __forceinline__ void split3_bf16x4(float4 v, uint2 *p) {
  float h[4], m[4], l[4];
  split3(v.x, h[0], m[0], l[0]);
  split3(v.y, h[1], m[1], l[1]);
  split3(v.z, h[2], m[2], l[2]);
  split3(v.w, h[3], m[3], l[3]);
  p[0] = make_uint2(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3]));
  p[1] = make_uint2(pack_bf16x2(m[0], m[1]), pack_bf16x2(m[2], m[3]));
  p[2] = make_uint2(pack_bf16x2(l[0], l[1]), pack_bf16x2(l[2], l[3]));
}

__device__ __forceinline__ float sigm(float a) { return __fdividef(1.0f, 1.0f + __expf(-a)); }
// tanh via exp (relative error ~1e-6; the bf16 path's bar is 1e-3)
__device__ __forceinline__ float tanh_fast(float a) {
  const float e = __expf(2.0f * fminf(fmaxf(a, -15.0f), 15.0f));
  return __fdividef(e - 1.0f, e + 1.0f);
}
__device__ __forceinline__ void ld_bias16(const float *p, float *b) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(p) + j);
    b[4 * j] = v.x; b[4 * j + 1] = v.y; b[4 * j + 2] = v.z; b[4 * j + 3] = v.w;
  }
}

// Split (fp32-accurate) modes: a tile's accumulator sums the products
// A_pa . W_pw of operand parts over K segments, pa + pw <= P - 1 (the terms
// of order < 2^-(P * bits) relative), identically-zero parts skipped.  One
// segment = K-chunks [k0, k1) of weight part pw against the A parts
// pa0 .. pa0 + npa - 1: one smem stage holds one weight chunk and npa A
// chunks (the CTA-pair kernel loads each weight chunk once for all three
// BF16X3 parts); the one-CTA kernel runs npa = 1 segments.  The plain modes
// have the single segment (pa0 0, npa 1, pw 0, [0, KC)).
struct SplitSeg {
  uint8_t pa0, npa, pw, pad;
  uint16_t k0, k1;
};
constexpr int MAX_SEG = 12;

struct TcArgs {
  uint32_t E, H, nub;              // nub = H / 128 phase-1 unit blocks
  const __nv_bfloat16 *emb16;
  const float *state;
  const float *bzr;                // [nub][2][128] (bz, br)
  const float *bh;                 // [H]
  float *state_out;
  const uint32_t *row_src, *row_dst, *row_word, *counts;
  float *g_z;                      // [B_max][H]
  __nv_bfloat16 *g_rh16;           // [B_max][H]
  __nv_bfloat16 *a1;               // [B_max][E+H] gathered phase-1 A operand (bf16 path)
  const float *emb;                // [V][E] fp32 (TF32 path)
  float *a1f;                      // [B_max][E+H] gathered phase-1 A operand (TF32 path)
  float *g_rhf;                    // [B_max][H] r.h, phase-2 A operand (TF32 path)
  uint32_t *done1;                 // per M-tile phase-1 epilogue arrivals (zeroed by the gather)
  uint32_t *tile_ctr;              // dynamic tile scheduler (zeroed by the gather)
  uint32_t lag;                    // phase-2 tiles trail phase-1 tiles by this many M-tiles
  uint32_t gm;                     // CTA pair, separated phases: tile groups of gm M-tiles (see tile_of)
  uint32_t pack;                   // CTA pair, 3-part stages: single-part segments carry 2 K-chunks per stage
  uint32_t diag;                   // timing diagnostics: 1 no MMA, 2 no TMA, 3 no epilogue, 4 = 3 + no phase
                                   // dependency, 6 = 1 + 2 (results invalid); 5 cycle counters (results valid)
  unsigned long long *prof;        // diag 5: per-CTA cycle counters, else nullptr
  // cell variant GRU_LBR: one phase, tiles of 64 units x
  // (z | r | Wh x | Uh h), B = W3 [(H/64) x 192 rows][E+H]
  const float *bz, *br;            // [H] (LBR epilogue)
  uint32_t bn2;                    // units per phase-2 (and RNN) tile: 256, or 128 when H % 256 != 0
  uint32_t x3_xlo;                 // split modes: 1 = the embedding has non-zero lower parts (they are
                                   // gathered); 0 = every entry is exact in the operand type
  uint32_t x3;                     // split (fp32-accurate) modes: number of operand parts P of every
                                   // activation, v = sum_p part_p: 2 = RNNLM_MATH_TF32X3 ([hi | lo] TF32,
                                   // TF32 instance), 3 = RNNLM_MATH_BF16X3 ([hi | mid | lo] bf16); 0 = plain.
                                   // A1 rows are P (E+H) wide, r.h rows P H, weight rows PW (E+H)
  uint32_t nseg;                   // K segments of one tile (plain: 1); see SplitSeg
  SplitSeg seg[MAX_SEG];
  // (a1) compression of the new state, fused into the phase-2 epilogue
  uint32_t cache, key_mode, round_digits, cstride;
  float round_scale;
  uint8_t *codes;
  unsigned long long *codehash;
};

__host__ __device__ __forceinline__ uint32_t seg_chunks(const TcArgs &a) {
  uint32_t n = 0;
  for (uint32_t s = 0; s < a.nseg; ++s) n += a.seg[s].k1 - a.seg[s].k0;
  return n;
}

// Cycle counters of the RNNLM_TC_DIAG=5 profile: compiled in only with
// -DRNNLM_TC_PROF=1 (scripts/diag_r2.sh); otherwise every counter is the
// constant 0 and the producer / MMA / epilogue loops carry no clock reads
#ifndef RNNLM_TC_PROF
#define RNNLM_TC_PROF 0
#endif
__device__ __forceinline__ unsigned long long pclk() {
  if constexpr (RNNLM_TC_PROF != 0) return clock64();
  else return 0ull;
}
__device__ __forceinline__ unsigned long long gtimer() {       // ns (diag 5 timeline)
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// diag 5: the gather's last block end time, max over blocks (prof slot 1023 * 16)
struct GatherClock {
  unsigned long long *prof;
  __device__ ~GatherClock() {
    if (!prof) return;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(prof + 1023 * 16, gtimer());
  }
};

// ---------------------------------------------------------------- A gather
// Phase-1 A operand: row r = [E[word_r] | bf16(state[src_r])] (bf16, K-major,
// dense), one warp per row, 16-byte loads/stores (the paper's per-frame
// (h || x) block, built in HBM instead of host memory).  States are
// stored only in fp32; the bf16 operand copy is made here.
template <typename T>
__global__ void __launch_bounds__(256) k_gather_a1(TcArgs a) {
  pdl_entry();
  const GatherClock clock_end{a.prof};
  const uint32_t Q = a.counts[1];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t K1 = a.E + a.H;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (Q + BM - 1) / BM; i += gridDim.x * blockDim.x)
    a.done1[i] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.tile_ctr = 0u;
  if constexpr (sizeof(T) == 2) {
    if (a.x3) {
      // BF16X3: [x_hi | h_hi | x_mid | h_mid | x_lo | h_lo], v = hi + mid + lo
      // (split3); x parts from the fp32 embedding (x_mid, x_lo only when some
      // entry is not bf16-exact: otherwise their segments are skipped and
      // never read).  Four 16-byte loads per lane are in flight before the
      // first store.
      const uint32_t nk = K1 / 4, nx = a.E / 4;
      for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < Q; r += nw) {
        const float4 *x = reinterpret_cast<const float4 *>(a.emb + (size_t)a.row_word[r] * a.E);
        const float4 *h = reinterpret_cast<const float4 *>(a.state + (size_t)a.row_src[r] * a.H);
        uint2 *dst = reinterpret_cast<uint2 *>(a.a1 + (size_t)r * 3 * K1);
        uint32_t i1 = 0;                              // first float4 index taken from fp32 rows
        if (!a.x3_xlo && a.emb16) {                   // bf16-exact embedding: x = x_hi, copied from the bf16 rows
          const uint4 *x16 = reinterpret_cast<const uint4 *>(a.emb16 + (size_t)a.row_word[r] * a.E);
          uint4 *d16 = reinterpret_cast<uint4 *>(dst);
          for (uint32_t i = lane; i < a.E / 8; i += 32) d16[i] = __ldg(x16 + i);
          i1 = nx;
        }
        for (uint32_t i0 = i1 + lane; i0 < nk; i0 += 128) {
          float4 v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t i = i0 + 32 * j;
            if (i < nk) v[j] = i < nx ? __ldg(x + i) : __ldg(h + (i - nx));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t i = i0 + 32 * j;
            if (i >= nk) continue;
            uint2 p[3];
            split3_bf16x4(v[j], p);
            dst[i] = p[0];
            if (i >= nx || a.x3_xlo) { dst[nk + i] = p[1]; dst[2 * nk + i] = p[2]; }
          }
        }
      }
      return;
    }
    // bf16: every load of a row chunk (4 x 16 B of x, 8 x 16 B of h per lane)
    // is issued before its stores, and the next row's indices are fetched
    // while the current row is copied, so a warp keeps ~12 loads in flight
    const uint32_t nx = a.E / 8, nh = a.H / 8, nmax = nx > nh ? nx : nh;
    uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t wd = r < Q ? a.row_word[r] : 0u, src = r < Q ? a.row_src[r] : 0u;
    for (; r < Q; r += nw) {
      const uint4 *x = reinterpret_cast<const uint4 *>(a.emb16 + (size_t)wd * a.E);
      const float4 *h = reinterpret_cast<const float4 *>(a.state + (size_t)src * a.H);
      uint4 *dst = reinterpret_cast<uint4 *>(a.a1 + (size_t)r * K1);
      const uint32_t rn = r + nw;
      if (rn < Q) { wd = a.row_word[rn]; src = a.row_src[rn]; }
      for (uint32_t i0 = lane; i0 < nmax; i0 += 128) {
        uint4 xv[4];
        float4 hu[4], hv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t i = i0 + 32 * j;
          if (i < nx) xv[j] = __ldg(x + i);
          if (i < nh) { hu[j] = __ldg(h + 2 * i); hv[j] = __ldg(h + 2 * i + 1); }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t i = i0 + 32 * j;
          if (i < nx) dst[i] = xv[j];
          if (i < nh) {
            const float4 u = hu[j], v = hv[j];
            __nv_bfloat162 b0 = __floats2bfloat162_rn(u.x, u.y), b1 = __floats2bfloat162_rn(u.z, u.w);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v.x, v.y), b3 = __floats2bfloat162_rn(v.z, v.w);
            dst[nx + i] = make_uint4(*reinterpret_cast<uint32_t *>(&b0), *reinterpret_cast<uint32_t *>(&b1),
                                     *reinterpret_cast<uint32_t *>(&b2), *reinterpret_cast<uint32_t *>(&b3));
          }
        }
      }
    }
    return;
  }
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < Q; r += nw) {
    {
      // TF32 operands are the fp32 values themselves (the MMA reads their TF32 part)
      const float4 *x = reinterpret_cast<const float4 *>(a.emb + (size_t)a.row_word[r] * a.E);
      const float4 *h = reinterpret_cast<const float4 *>(a.state + (size_t)a.row_src[r] * a.H);
      const uint32_t nx = a.E / 4, nh = a.H / 4;
      if (!a.x3) {
        float4 *dst = reinterpret_cast<float4 *>(a.a1f + (size_t)r * K1);
        for (uint32_t i = lane; i < nx; i += 32) dst[i] = to_tf32(__ldg(x + i));
        for (uint32_t i = lane; i < nh; i += 32) dst[nx + i] = to_tf32(h[i]);
      } else {  // [hi(x) | hi(h) | lo(x) | lo(h)], lo = tf32(v - hi)
        float4 *dst = reinterpret_cast<float4 *>(a.a1f + (size_t)r * 2 * K1);
        const uint32_t nk = nx + nh;
        for (uint32_t i = lane; i < nk; i += 32) {
          const float4 v = i < nx ? __ldg(x + i) : h[i - nx];
          const float4 hi = to_tf32(v);
          dst[i] = hi;
          if (i >= nx || a.x3_xlo)                       // x_lo == 0 is never read (skipped segment)
            dst[nk + i] = to_tf32(make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w));
        }
      }
    }
  }
}

constexpr int EPI_WARPS = 8;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
// Register cap of the fused kernels: three of its warps share an SM sub-partition,
// and 3 x 160 x 32 registers leave 1,024 of the sub-partition's 16,384 for one
// warp of k_score capped at 32 registers (k_score.cu), so the side-stream
// scoring runs beside the GRU.  160 / 32 against 152 / 48: GRU 210.4 -> 207.9 us
// (BF16X3), 143.0 -> 139.1 us (bf16), no spills left in the GRU
// (profiles/ab_maxreg_r2.txt); 168 evicts the scoring warp altogether.
#ifndef GRU_MAXREG
#define GRU_MAXREG 160
#endif

constexpr int TQ = 4;            // depth of the tile-id ring (producer -> MMA / epilogue)
constexpr uint32_t NO_TILE = 0xFFFFFFFFu;

struct Smem {
  uint8_t *sA, *sB, *stg;
  uint64_t *full, *empty, *tfull, *tempty, *qfull, *qempty;
  uint32_t *tmem_base;
  uint32_t *tile_q;
};

__device__ __forceinline__ Smem carve(uint8_t *raw, int nst) {
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  Smem m;
  m.sA = smem;
  m.sB = smem + nst * A_BYTES;
  m.stg = m.sB + nst * B_BYTES;
  m.full = reinterpret_cast<uint64_t *>(m.stg + EPI_WARPS * STG_BYTES);
  m.empty = m.full + nst;
  m.tfull = m.empty + nst;
  m.tempty = m.tfull + 2;
  m.qfull = m.tempty + 2;
  m.qempty = m.qfull + TQ;
  m.tmem_base = reinterpret_cast<uint32_t *>(m.qempty + TQ);
  m.tile_q = m.tmem_base + 4;
  return m;
}

__device__ __forceinline__ void setup(const Smem &m, int warp, int nst) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { mbar_init(&m.full[s], 1); mbar_init(&m.empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&m.tfull[s], 1); mbar_init(&m.tempty[s], EPI_WARPS * 32); }
    // tile ids: the producer publishes, the MMA lane and one lane per epilogue warp release
    for (int s = 0; s < TQ; ++s) { mbar_init(&m.qfull[s], 1); mbar_init(&m.qempty[s], 1 + EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(m.tmem_base, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

__device__ __forceinline__ void teardown(const Smem &m, int warp, uint32_t tmem_base) {
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------- tile schedule
// One persistent kernel runs both phases.  Per M-tile m (128 rows) there are
// nub phase-1 tiles P1(m, j) (z|r of units [128j, 128j+128)) and nt phase-2
// tiles P2(m, j) (candidate of units [256j, 256j+256)).  Global order: step s
// holds P1(s, *) then P2(s - L, *), so a phase-2 tile comes ~L M-tiles after
// the phase-1 tiles it depends on (r.h of ALL units of its rows).  CTAs claim
// tiles from a global atomic counter, so tiles are started in increasing
// index order by CTAs that are running; a tile only waits on tiles with
// smaller indices, which were claimed earlier by running CTAs, so the kernel
// makes progress whatever the number of co-resident CTAs.
struct Tile {
  uint32_t kind, m, j;             // kind 0: phase 1, 1: phase 2
};

// Fully separated phases (L >= mt) in groups of gm M-tiles: inside a group the
// tiles run N-tile-major, so gm consecutive tiles read the same weight chunks
// at about the same time (the L2 serves concurrent identical requests once);
// gm = 1 is M-tile-major (the n1 / n2 tiles of an M-tile share its A rows).
__device__ __forceinline__ void grouped(uint32_t t, uint32_t mt, uint32_t n, uint32_t gm, uint32_t &m, uint32_t &j) {
  const uint32_t g = t / (gm * n), r = t - g * gm * n;
  const uint32_t gsz = mt - g * gm < gm ? mt - g * gm : gm;
  j = r / gsz;
  m = g * gm + r % gsz;
}

__device__ __forceinline__ Tile tile_of(uint32_t t, uint32_t mt, uint32_t n1, uint32_t n2, uint32_t L,
                                        uint32_t gm = 1) {
  Tile x;
  if (gm > 1 && L >= mt) {
    if (t < mt * n1) { x.kind = 0; grouped(t, mt, n1, gm, x.m, x.j); }
    else { x.kind = 1; grouped(t - mt * n1, mt, n2, gm, x.m, x.j); }
    return x;
  }
  const uint32_t a = L * n1, b = (mt - L) * (n1 + n2);
  if (t < a) {
    x.kind = 0; x.m = t / n1; x.j = t % n1;
  } else if (t < a + b) {
    const uint32_t u = t - a, s = L + u / (n1 + n2), j = u % (n1 + n2);
    if (j < n1) { x.kind = 0; x.m = s; x.j = j; }
    else { x.kind = 1; x.m = s - L; x.j = j - n1; }
  } else {
    const uint32_t u = t - a - b;
    x.kind = 1; x.m = mt - L + u / n2; x.j = u % n2;
  }
  return x;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_phase1(const uint32_t *cnt, uint32_t target) {
  while (ld_acquire(cnt) < target) __nanosleep(128);
}

// Next tile id from the producer's ring (MMA lane / epilogue warps).
__device__ __forceinline__ uint32_t next_tile(const Smem &m, uint32_t it, bool release_lane) {
  const uint32_t slot = it % TQ;
  mbar_wait(&m.qfull[slot], (it / TQ) & 1);
  const uint32_t t = *reinterpret_cast<volatile uint32_t *>(&m.tile_q[slot]);
  __syncwarp();
  if (release_lane) mbar_arrive(&m.qempty[slot]);
  return t;
}

// MMA issuer: KC chunks of 4 x (M=128, N=256, K=32 bytes) per tile, both phases.
// LBR tiles: accumulator columns [Wh x | z | r | Uh h] (64 each).  W3 rows
// carry [Wh; Wz; Wr] in their x half and [Uz; Ur; Uh] in their h half, so
// every K-chunk is ONE N = 192 MMA: x chunks into columns 0-191, h chunks
// into columns 64-255 (no product of a zero block).  The first h K-step
// splits into N = 128 (accumulate into z | r) + N = 64 (initialise Uh h).
// Phase-2 (and RNN) tiles are 128 units wide (N = 128) when H % 256 != 0.
template <typename T, bool LBR>
__device__ __forceinline__ void mma_loop(const Smem &m, uint32_t tmem_base, uint32_t KC, uint32_t kx, int lane,
                                         uint32_t diag, unsigned long long *prof, bool narrow, bool rnn,
                                         uint32_t mt, uint32_t n1, uint32_t n2, uint32_t L, int nst) {
  uint32_t stage = 0, phase = 0;
  const uint32_t id256 = idesc_of(Op<T>::FMT, BM, BN);
  const uint32_t id192 = idesc_of(Op<T>::FMT, BM, 192), id128 = idesc_of(Op<T>::FMT, BM, 128),
                 id64 = idesc_of(Op<T>::FMT, BM, 64);
  unsigned long long w_full = 0, w_tempty = 0, t0;
  for (uint32_t it = 0;; ++it) {
    const uint32_t tid = next_tile(m, it, lane == 0);
    if (tid == NO_TILE) break;
    const uint32_t id = (narrow && (rnn || tile_of(tid, mt, n1, n2, L).kind == 1)) ? id128 : id256;
    const uint32_t acc = it & 1;
    t0 = pclk();
    mbar_wait(&m.tempty[acc], ((it >> 1) & 1) ^ 1);
    w_tempty += pclk() - t0;
    tc_fence_after();
    const uint32_t tm = tmem_base + acc * BN;
    for (uint32_t kc = 0; kc < KC; ++kc) {
      t0 = pclk();
      mbar_wait(&m.full[stage], phase);
      w_full += pclk() - t0;
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(m.sA + stage * A_BYTES), b0 = smem_u32(m.sB + stage * B_BYTES);
        if (diag != 1 && diag != 6) {
          if constexpr (!LBR) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              Op<T>::mma(tm, sdesc(a0 + k * 32), sdesc(b0 + k * 32), id, (kc | k) != 0);
          } else if (kc < kx) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              Op<T>::mma(tm, sdesc(a0 + k * 32), sdesc(b0 + k * 32), id192, (kc | k) != 0);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (kc == kx && k == 0) {
                Op<T>::mma(tm + 64, sdesc(a0), sdesc(b0), id128, 1u);
                Op<T>::mma(tm + 192, sdesc(a0), sdesc(b0 + 16384), id64, 0u);
              } else {
                Op<T>::mma(tm + 64, sdesc(a0 + k * 32), sdesc(b0 + k * 32), id192, 1u);
              }
            }
          }
        }
        umma_commit(&m.empty[stage]);
        if (kc == KC - 1) umma_commit(&m.tfull[acc]);
      }
      __syncwarp();
      if (++stage == nst) { stage = 0; phase ^= 1; }
    }
  }
  if (prof && lane == 0) { prof[2] = w_full; prof[3] = w_tempty; }
}

// (a1) compression code of the new state: encode.cuh's encode32 (the same
// device code as k_encode_rows and rnnlm_encode_states).
__device__ __forceinline__ KeySpec key_spec(const TcArgs &a) {
  return KeySpec{a.key_mode, a.round_digits, a.H, a.round_scale};
}


// ---------------------------------------------------------------- epilogue I/O
// An epilogue thread owns one tile row (its TMEM lane) and walks its columns
// in chunks of 32.  Row-per-thread global accesses would touch 32 different
// lines per warp instruction (the L1 wavefront rate then bounds the epilogue,
// not the MMAs), so:
//  * z (internal scratch) lives in 128-row blocks, zq4() below, in which a
//    warp's 32 rows x 4 units are 512 contiguous bytes;
//  * rows the layout is not ours to choose (parent states, the new states,
//    the r.h / A1 rows) move through a per-warp 32-row staging buffer in
//    shared memory: the warp reads / writes RB contiguous bytes of each of
//    512 / RB rows per instruction, and each thread exchanges its own row
//    with the buffer.  16-byte chunks are XOR-swizzled so both access
//    patterns are bank-conflict-free.

// float4 index of z(row, u), u a multiple of 4: blocks of 128 rows x 4 units
__device__ __forceinline__ size_t zq4(uint32_t row, uint32_t u, uint32_t H) {
  return ((((size_t)(row >> 7) * (H >> 4) + (u >> 4)) * 4 + ((u & 15) >> 2)) << 7) + (row & 127);
}

template <int RB>
__device__ __forceinline__ uint32_t stg_off(uint32_t r, uint32_t c) {
  if constexpr (RB == 128) return r * 128 + ((c ^ (r & 7)) << 4);
  else return r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
}

// rows -> staging: lane l contributes its row's pointer (nullptr: not loaded)
template <int RB>
__device__ __forceinline__ void coop_load(uint8_t *stg, const void *row_ptr, uint32_t lane) {
  constexpr int CPR = RB / 16, RPI = 32 / CPR;         // 16-B chunks per row, rows per instruction
  uint4 v[CPR];
#pragma unroll
  for (int i = 0; i < CPR; ++i) {
    const uint32_t r = i * RPI + lane / CPR, c = lane % CPR;
    const uint8_t *p = reinterpret_cast<const uint8_t *>(
        __shfl_sync(0xFFFFFFFFu, reinterpret_cast<unsigned long long>(row_ptr), r));
    v[i] = p ? *reinterpret_cast<const uint4 *>(p + c * 16) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int i = 0; i < CPR; ++i) {
    const uint32_t r = i * RPI + lane / CPR, c = lane % CPR;
    *reinterpret_cast<uint4 *>(stg + stg_off<RB>(r, c)) = v[i];
  }
  __syncwarp();
}
// staging -> rows (after each lane wrote its own row); nullptr rows are skipped
template <int RB>
__device__ __forceinline__ void coop_store(uint8_t *stg, void *row_ptr, uint32_t lane) {
  constexpr int CPR = RB / 16, RPI = 32 / CPR;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < CPR; ++i) {
    const uint32_t r = i * RPI + lane / CPR, c = lane % CPR;
    uint8_t *p = reinterpret_cast<uint8_t *>(
        __shfl_sync(0xFFFFFFFFu, reinterpret_cast<unsigned long long>(row_ptr), r));
    const uint4 v = *reinterpret_cast<const uint4 *>(stg + stg_off<RB>(r, c));
    if (p) *reinterpret_cast<uint4 *>(p + c * 16) = v;
  }
  __syncwarp();
}
// this lane's row of the staging buffer, as 32 fp32 / 32 bf16 values
__device__ __forceinline__ void own_row_f32(const uint8_t *stg, uint32_t lane, float *x) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 t = *reinterpret_cast<const float4 *>(stg + stg_off<128>(lane, c));
    x[4 * c] = t.x; x[4 * c + 1] = t.y; x[4 * c + 2] = t.z; x[4 * c + 3] = t.w;
  }
}
__device__ __forceinline__ void put_row_f32(uint8_t *stg, uint32_t lane, const float *x) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4 *>(stg + stg_off<128>(lane, c)) =
        make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
}
__device__ __forceinline__ void own_row_bf16(const uint8_t *stg, uint32_t lane, float *x) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 t = *reinterpret_cast<const uint4 *>(stg + stg_off<64>(lane, c));
    const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x[8 * c + 2 * j] = __uint_as_float(w[j] << 16);
      x[8 * c + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
    }
  }
}
__device__ __forceinline__ void put_row_bf16(uint8_t *stg, uint32_t lane, const float *x) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 t2 = __floats2bfloat162_rn(x[8 * c + 2 * j], x[8 * c + 2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t *>(&t2);
    }
    *reinterpret_cast<uint4 *>(stg + stg_off<64>(lane, c)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
// BF16X3: the bf16 part of x (round to nearest even) into the staging row,
// x keeps the (exact) remainder; three calls store hi, mid, lo
__device__ __forceinline__ void put_row_bf16_part(uint8_t *stg, uint32_t lane, float *x) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float p0 = bf16_part(x[8 * c + 2 * j]), p1 = bf16_part(x[8 * c + 2 * j + 1]);
      x[8 * c + 2 * j] -= p0;
      x[8 * c + 2 * j + 1] -= p1;
      w[j] = pack_bf16x2(p0, p1);
    }
    *reinterpret_cast<uint4 *>(stg + stg_off<64>(lane, c)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
// 32 consecutive accumulator columns of this thread's TMEM lane (wait separately)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
  tmem_ld16(taddr, v);
  tmem_ld16(taddr + 16, v + 16);
}

// Epilogue knock-outs for timing experiments only (build flag -DEPI_KO=bits, results
// invalid): 1 no global loads of parent states / z, 2 no global stores, 4 no code
// encoding, 8 no transcendental math.  The default build has none.
#ifndef EPI_KO
#define EPI_KO 0
#endif
constexpr bool KO_LOAD = EPI_KO & 1, KO_STORE = EPI_KO & 2, KO_ENC = EPI_KO & 4, KO_MATH = EPI_KO & 8,
               KO_Z = EPI_KO & 16;    // 16: no z round trip (phase-1 z stores, phase-2 z loads)

// Phase-1 epilogue of one thread: row `row` of the tile, the 128 z columns
// (gate 0) or r columns (gate 1) of unit block ub.  The parent state h of
// r.h is, on the bf16 path, the bf16 copy in the row's A1 row (the value
// phase 1 multiplied); on the TF32 path the exact fp32 state.
template <typename T>
__device__ __forceinline__ void epi_phase1(const TcArgs &a, uint32_t tacc, uint32_t row, bool valid,
                                           int half, uint32_t ub, uint8_t *stg, uint32_t lane) {
  // the two epilogue warps of a TMEM lane quarter split the tile's 128 units:
  // each takes 64 units, their z columns (tacc + u) and r columns (tacc + 128
  // + u), so both do the same work (r.h, with its parent-state loads and
  // operand-part stores, costs ~2-3x z)
  const uint32_t u0 = ub * UB + half * 64;
#pragma unroll 1
  for (int cc = 0; cc < 4; ++cc) {
    const int gate = cc >> 1, c = cc & 1;               // z chunks 0, 1, then r chunks 0, 1
    const float *bias = a.bzr + (size_t)ub * 2 * UB + gate * UB + half * 64;
    float v[32], b[32];
    tmem_ld32(tacc + gate * UB + half * 64 + c * 32, v);
    ld_bias16(bias + c * 32, b);
    ld_bias16(bias + c * 32 + 16, b + 16);
    if (gate == 0) {
      tmem_ld_wait();
      if (valid && !KO_STORE && !KO_Z) {
        float4 *zq = reinterpret_cast<float4 *>(a.g_z) + zq4(row, u0 + c * 32, a.H);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          zq[j << 7] = make_float4(sigm(v[4 * j] + b[4 * j]), sigm(v[4 * j + 1] + b[4 * j + 1]),
                                   sigm(v[4 * j + 2] + b[4 * j + 2]), sigm(v[4 * j + 3] + b[4 * j + 3]));
      }
    } else {
      float hv[32];
      if (sizeof(T) == 2 && !a.x3) {
        coop_load<64>(stg, valid && !KO_LOAD ? a.a1 + (size_t)row * (a.E + a.H) + a.E + u0 + c * 32 : nullptr, lane);
        own_row_bf16(stg, lane, hv);
      } else {
        coop_load<128>(stg, valid && !KO_LOAD ? a.state + (size_t)a.row_src[row] * a.H + u0 + c * 32 : nullptr, lane);
        own_row_f32(stg, lane, hv);
      }
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) hv[j] *= KO_MATH ? v[j] + b[j] : sigm(v[j] + b[j]);
      __syncwarp();
      if constexpr (sizeof(T) == 2) {
        if (!a.x3) {
          put_row_bf16(stg, lane, hv);
          coop_store<64>(stg, valid && !KO_STORE ? a.g_rh16 + (size_t)row * a.H + u0 + c * 32 : nullptr, lane);
        } else {  // BF16X3: r.h as [hi | mid | lo] rows of 3H
#pragma unroll 1
          for (int p = 0; p < 3; ++p) {
            put_row_bf16_part(stg, lane, hv);
            coop_store<64>(stg, valid && !KO_STORE ? a.g_rh16 + (size_t)row * 3 * a.H + p * a.H + u0 + c * 32 : nullptr, lane);
          }
        }
      } else if (!a.x3) {
#pragma unroll
        for (int j = 0; j < 32; ++j) hv[j] = to_tf32(hv[j]);
        put_row_f32(stg, lane, hv);
        coop_store<128>(stg, valid ? a.g_rhf + (size_t)row * a.H + u0 + c * 32 : nullptr, lane);
      } else {  // 3xTF32: r.h as [hi | lo] rows of 2H
        float lo[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float hi = to_tf32(hv[j]);
          lo[j] = to_tf32(hv[j] - hi);
          hv[j] = hi;
        }
        put_row_f32(stg, lane, hv);
        coop_store<128>(stg, valid ? a.g_rhf + (size_t)row * 2 * a.H + u0 + c * 32 : nullptr, lane);
        put_row_f32(stg, lane, lo);
        coop_store<128>(stg, valid ? a.g_rhf + (size_t)row * 2 * a.H + a.H + u0 + c * 32 : nullptr, lane);
      }
    }
  }
}

// Phase-2 epilogue of one thread: row `row`, 128 units starting at n0.
__device__ __forceinline__ void epi_phase2(const TcArgs &a, uint32_t tbase, uint32_t row, bool valid,
                                           uint32_t n0, uint32_t units, uint8_t *stg, uint32_t lane) {
  const uint32_t dst = valid ? a.row_dst[row] : NONE;
  const bool live = dst != NONE;
  const float *hp = live ? a.state + (size_t)a.row_src[row] * a.H + n0 : nullptr;
  float *hout = live ? a.state_out + (size_t)dst * a.H + n0 : nullptr;
  uint8_t *code = (a.cache && a.key_mode != RNNLM_KEY_OFF && live) ? a.codes + (size_t)dst * a.cstride : nullptr;
  const float4 *zq = reinterpret_cast<const float4 *>(a.g_z) + zq4(live ? row : 0, n0, a.H);
  unsigned long long hs = 0;
#pragma unroll 1
  for (uint32_t c = 0; c < units / 32; ++c) {           // chunks of 32 units
    float v[32], b[32], z[32], h[32];
    tmem_ld32(tbase + c * 32, v);
    if (KO_Z) {
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = 0.5f;
    } else if (live && !KO_LOAD) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 t = zq[(c * 8 + j) << 7];
        z[4 * j] = t.x; z[4 * j + 1] = t.y; z[4 * j + 2] = t.z; z[4 * j + 3] = t.w;
      }
    }
    ld_bias16(a.bh + n0 + c * 32, b);
    ld_bias16(a.bh + n0 + c * 32 + 16, b + 16);
    coop_load<128>(stg, hp && !KO_LOAD ? hp + c * 32 : nullptr, lane);
    own_row_f32(stg, lane, h);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) h[j] = (1.0f - z[j]) * h[j] + z[j] * (KO_MATH ? v[j] + b[j] : tanh_fast(v[j] + b[j]));
    __syncwarp();
    put_row_f32(stg, lane, h);
    coop_store<128>(stg, hout && !KO_STORE ? hout + c * 32 : nullptr, lane);
    if (a.cache && live && !KO_ENC) hs += encode32(key_spec(a), h, n0 + c * 32, code);
  }
  if (a.cache && live) atomicAdd(&a.codehash[dst], hs);
}
// Vanilla-RNN epilogue of one thread (cell variant): row
// `row`, 128 units from n0; accumulator = Wh x + Uh h; h' = sigma(. + bh),
// the new fp32 state (staged row store) and its compression code.
__device__ __forceinline__ void epi_rnn(const TcArgs &a, uint32_t tbase, uint32_t row, bool valid, uint32_t n0,
                                        uint32_t units, uint8_t *stg, uint32_t lane) {
  const uint32_t dst = valid ? a.row_dst[row] : NONE;
  const bool live = dst != NONE;
  float *hout = live ? a.state_out + (size_t)dst * a.H + n0 : nullptr;
  uint8_t *code = (a.cache && a.key_mode != RNNLM_KEY_OFF && live) ? a.codes + (size_t)dst * a.cstride : nullptr;
  unsigned long long hs = 0;
#pragma unroll 1
  for (uint32_t c = 0; c < units / 32; ++c) {           // chunks of 32 units
    float v[32], b[32];
    tmem_ld32(tbase + c * 32, v);
    ld_bias16(a.bh + n0 + c * 32, b);
    ld_bias16(a.bh + n0 + c * 32 + 16, b + 16);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = sigm(v[j] + b[j]);
    __syncwarp();
    put_row_f32(stg, lane, v);
    coop_store<128>(stg, hout ? hout + c * 32 : nullptr, lane);
    if (a.cache && live) hs += encode32(key_spec(a), v, n0 + c * 32, code);
  }
  if (a.cache && live) atomicAdd(&a.codehash[dst], hs);
}

// LBR epilogue of one thread (cell variant): row `row`, the 32
// units [64 ub + 32 half, +32) of the tile's 64; accumulator columns: Wh x
// at 0-63, z at 64-127, r at 128-191, Uh h at 192-255 (tacc = the lane
// quarter's column 0).  c = tanh(Wh x + bh + r . (Uh h)), h' = (1 - z) h + z c,
// the new fp32 state (staged row store) and its compression code.
__device__ __forceinline__ void epi_lbr(const TcArgs &a, uint32_t tacc, uint32_t row, bool valid, int half,
                                        uint32_t ub, uint8_t *stg, uint32_t lane) {
  const uint32_t dst = valid ? a.row_dst[row] : NONE;
  const bool live = dst != NONE;
  const uint32_t u0 = ub * 64 + half * 32, c0 = half * 32;
  coop_load<128>(stg, live ? a.state + (size_t)a.row_src[row] * a.H + u0 : nullptr, lane);
  uint8_t *code = (a.cache && a.key_mode != RNNLM_KEY_OFF && live) ? a.codes + (size_t)dst * a.cstride : nullptr;
  unsigned long long hs = 0;
  uint32_t signacc = 0;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    float vz[16], vr[16], vx[16], vu[16], h[16];
    tmem_ld16(tacc + c0 + g * 16, vx);
    tmem_ld16(tacc + 64 + c0 + g * 16, vz);
    tmem_ld16(tacc + 128 + c0 + g * 16, vr);
    tmem_ld16(tacc + 192 + c0 + g * 16, vu);
#pragma unroll
    for (int c = 0; c < 4; ++c) {                   // this lane's 16 staged state values of group g
      const float4 t4 = *reinterpret_cast<const float4 *>(stg + stg_off<128>(lane, 4 * g + c));
      h[4 * c] = t4.x; h[4 * c + 1] = t4.y; h[4 * c + 2] = t4.z; h[4 * c + 3] = t4.w;
    }
    tmem_ld_wait();
    const float4 *bz4 = reinterpret_cast<const float4 *>(a.bz + u0 + g * 16);
    const float4 *br4 = reinterpret_cast<const float4 *>(a.br + u0 + g * 16);
    const float4 *bh4 = reinterpret_cast<const float4 *>(a.bh + u0 + g * 16);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float4 z4 = __ldg(bz4 + c), r4 = __ldg(br4 + c), h4 = __ldg(bh4 + c);
      const float bz[4] = {z4.x, z4.y, z4.z, z4.w}, br[4] = {r4.x, r4.y, r4.z, r4.w},
                  bh[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = 4 * c + t;
        const float z = sigm(vz[j] + bz[t]), r = sigm(vr[j] + br[t]);
        const float cand = tanh_fast(vx[j] + bh[t] + r * vu[j]);
        h[j] = (1.0f - z) * h[j] + z * cand;
      }
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<float4 *>(stg + stg_off<128>(lane, 4 * g + c)) =
          make_float4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
    if (a.cache && live) hs += encode16(key_spec(a), h, u0 + g * 16, code, signacc);
  }
  coop_store<128>(stg, live ? a.state_out + (size_t)dst * a.H + u0 : nullptr, lane);
  if (a.cache && live) atomicAdd(&a.codehash[dst], hs);
}

// =============================================================== fused GRU kernel
// warp 0: TMA producer (waits on the phase-1 counter before a phase-2 tile);
// warp 1: TMEM allocation + MMA issue; warps 2-9: epilogue, TMEM lane quarter
// = warp % 4, column half = (warp - 2) / 4.
template <typename T, int CELL>
__global__ void __maxnreg__(GRU_MAXREG)
    k_gru_tc(const __grid_constant__ CUtensorMap map_a1, const __grid_constant__ CUtensorMap map_w1,
             const __grid_constant__ CUtensorMap map_rh, const __grid_constant__ CUtensorMap map_w2,
             TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  constexpr int NST = st_of<CELL>();
  const Smem m = carve(smem_raw, NST);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // GRU: per M-tile nub phase-1 + H/256 phase-2 tiles; LBR: H/64 one-phase
  // tiles over W3; RNN: H/256 one-phase tiles of A1 x W2 = [Wh | Uh]
  constexpr bool LBR = CELL == RNNLM_CELL_GRU_LBR, RNN = CELL == RNNLM_CELL_RNN;
  const uint32_t n1 = LBR ? a.H / 64 : (RNN ? a.H / a.bn2 : a.nub), n2 = (LBR || RNN) ? 0u : a.H / a.bn2;
  constexpr int BKE = Op<T>::BKE;
  const uint32_t kx = a.E / BKE;
  const uint32_t KCt = seg_chunks(a);                    // K-chunks per tile over every split segment
  const uint32_t target = n1 * EPI_WARPS;               // phase-1 arrivals per M-tile
  if (threadIdx.x == 0) {
    prefetch_map(&map_a1); prefetch_map(&map_w1); prefetch_map(&map_rh); prefetch_map(&map_w2);
  }
  setup(m, warp, NST);
  pdl_entry();
  const uint32_t Q = a.counts[1];
  const uint32_t mt = (Q + BM - 1) / BM;
  const uint32_t L = mt < a.lag ? mt : a.lag;
  const uint32_t ntiles = mt * (n1 + n2);
  const uint32_t tmem_base = *m.tmem_base;
  unsigned long long *prof = a.prof ? a.prof + blockIdx.x * 16 : nullptr;
  const unsigned long long k_t0 = pclk();
  if (prof && threadIdx.x == 0) prof[14] = gtimer();

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      unsigned long long w_empty = 0, w_dep = 0, t0;
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % TQ;
        mbar_wait(&m.qempty[slot], ((it / TQ) & 1) ^ 1);
        uint32_t t = atomicAdd(a.tile_ctr, 1u);
        if (t >= ntiles) t = NO_TILE;
        m.tile_q[slot] = t;
        mbar_arrive(&m.qfull[slot]);
        if (t == NO_TILE) break;
        const Tile x = tile_of(t, mt, n1, n2, L);
        const uint32_t m0 = x.m * BM;
        if (x.kind == 1 && a.diag != 4) {
          t0 = pclk();
          wait_phase1(a.done1 + x.m, target);
          w_dep += pclk() - t0;
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        if (prof) prof[9 + x.kind] += 1;
        for (uint32_t sg = 0; sg < a.nseg; ++sg)
        for (uint32_t kc = a.seg[sg].k0; kc < a.seg[sg].k1; ++kc) {
          // split modes: A part pa, weight part pw of this segment (column offsets into the part blocks)
          const int a_off = (int)(a.seg[sg].pa0 * (a.E + a.H)), b_off = (int)(a.seg[sg].pw * (a.E + a.H));
          const int rh_off = (int)(a.seg[sg].pa0 * a.H);
          t0 = pclk();
          mbar_wait(&m.empty[stage], phase ^ 1);
          w_empty += pclk() - t0;
          if (a.diag == 2 || a.diag == 6) {
            mbar_arrive(&m.full[stage]);
            if (++stage == NST) { stage = 0; phase ^= 1; }
            continue;
          }
          // B rows this tile loads: 192 (LBR), bn2 (phase 2, RNN), 256 (phase 1)
          const uint32_t b_rows = LBR ? 192u : ((x.kind == 1 || RNN) ? a.bn2 : (uint32_t)BN);
          mbar_expect_tx(&m.full[stage], A_BYTES + b_rows * 128);
          const uint32_t dA = smem_u32(m.sA + stage * A_BYTES), dB = smem_u32(m.sB + stage * B_BYTES);
          if (x.kind == 0) {
            tma_load_2d(dA, &map_a1, &m.full[stage], a_off + (int)(kc * BKE), (int)m0);
            tma_load_2d(dB, &map_w1, &m.full[stage], b_off + (int)(kc * BKE), (int)(x.j * b_rows));
          } else {
            if (kc < kx) tma_load_2d(dA, &map_a1, &m.full[stage], a_off + (int)(kc * BKE), (int)m0);
            else tma_load_2d(dA, &map_rh, &m.full[stage], rh_off + (int)((kc - kx) * BKE), (int)m0);
            tma_load_2d(dB, &map_w2, &m.full[stage], b_off + (int)(kc * BKE), (int)(x.j * b_rows));
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
      if (prof) { prof[0] = w_empty; prof[1] = w_dep; }
    }
  } else if (warp == 1) {
    mma_loop<T, LBR>(m, tmem_base, KCt, kx, lane, a.diag, prof, a.bn2 != BN, RNN, mt, n1, n2, L, NST);
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r_in = q * 32 + lane;
    unsigned long long w_tfull = 0, b1 = 0, b2 = 0, t0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t t = next_tile(m, it, lane == 0);
      if (t == NO_TILE) break;
      const Tile x = tile_of(t, mt, n1, n2, L);
      const uint32_t acc = it & 1;
      t0 = pclk();
      mbar_wait(&m.tfull[acc], (it >> 1) & 1);
      w_tfull += pclk() - t0;
      t0 = pclk();
      tc_fence_after();
      const uint32_t row = x.m * BM + r_in;
      const bool valid = row < Q;
      // column half of the tile: 128 of 256 (phase 1 / LBR / wide tiles) or 64 of 128
      const uint32_t hw = (x.kind == 1 || RNN) ? a.bn2 / 2 : (uint32_t)(BN / 2);
      const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16) + half * hw;
      if (a.diag == 3 || a.diag == 4) {                   // timing only: no epilogue work
        float v[16];
        tmem_ld16(tbase, v);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&m.tempty[acc]);
        if (x.kind == 0) {
          __syncwarp();
          if (lane == 0) { __threadfence(); atomicAdd(a.done1 + x.m, 1u); }
        }
        continue;
      }
      if constexpr (RNN) {
        epi_rnn(a, tbase, row, valid, x.j * a.bn2 + half * hw, hw, m.stg + (warp - 2) * STG_BYTES, lane);
        tc_fence_before();
        mbar_arrive(&m.tempty[acc]);
        b1 += pclk() - t0;
      } else if constexpr (LBR) {
        epi_lbr(a, tbase - half * (BN / 2), row, valid, half, x.j, m.stg + (warp - 2) * STG_BYTES, lane);
        tc_fence_before();
        mbar_arrive(&m.tempty[acc]);
        b1 += pclk() - t0;
      } else if (x.kind == 0) {
        epi_phase1<T>(a, tbase - half * hw, row, valid, half, x.j, m.stg + (warp - 2) * STG_BYTES, lane);
        tc_fence_before();
        mbar_arrive(&m.tempty[acc]);
        // publish this warp's z / r.h columns to the phase-2 tiles of the M-tile
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(a.done1 + x.m, 1u);
        }
        b1 += pclk() - t0;
      } else {
        wait_phase1(a.done1 + x.m, target);               // acquire z of this M-tile
        epi_phase2(a, tbase, row, valid, x.j * a.bn2 + half * hw, hw, m.stg + (warp - 2) * STG_BYTES, lane);
        tc_fence_before();
        mbar_arrive(&m.tempty[acc]);
        b2 += pclk() - t0;
      }
    }
    if (prof && lane == 0 && (warp == 2 || warp == 6)) {
      const int o = warp == 2 ? 4 : 11;
      prof[o] = w_tfull; prof[o + 1] = b1; prof[o + 2] = b2;
    }
  }
  if (prof && threadIdx.x == 0) prof[8] = pclk() - k_t0;
  teardown(m, warp, tmem_base);
  if (prof && threadIdx.x == 0) prof[15] = gtimer();       // every warp of the CTA is done
}

// =============================================================== CTA-pair variant
// Same tile stream and epilogues, but each tile is 256 rows computed by a CTA
// pair (cluster of 2) with tcgen05.mma.cta_group::2 (M = 256, N = 256): each
// CTA TMA-loads its own 128 A rows and HALF of the B tile (128 of 256 rows);
// the pair's tensor cores read the peer's B half directly, so every SM pulls
// 32 KB per K-chunk from L2 instead of 48 KB (the one-CTA kernel is
// L2->SM-bandwidth bound).  The leader CTA claims tiles, issues the MMAs and
// owns the pipeline barriers that both CTAs' TMA and epilogues signal.
#ifndef RNNLM_TC_STP
#define RNNLM_TC_STP 5
#endif
// pair-kernel smem stages (32 KB each): 5 measured faster than 6 on the bench
// workload (547-549 vs 537-540 M q/s, kernel 194.8 vs 197.6 us, same box)
constexpr int BP_BYTES = (BN / 2) * BK * 2;    // 16 KB: this CTA's half of a B chunk
// stages per A parts per stage: NA = 1 (plain bf16: 32-KB stages), NA = 3
// (BF16X3: one weight chunk + three A part chunks, 64-KB stages, 3 of them)
template <int NA>
__host__ __device__ constexpr int stp_of() { return NA == 1 ? RNNLM_TC_STP : 3; }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// wait with cluster-scope acquire (the phase may have been completed by the peer CTA)
__device__ __forceinline__ void mbar_wait_cl(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// arrive on a (possibly remote) barrier with the default CTA-scope release: the
// TMEM-free signal only orders this warp's completed tcgen05.ld (waited and
// fenced with tcgen05.fence::before_thread_sync) before the peer's MMA, no
// global memory, so it needs no cluster-scope release (MEMBAR) per tile
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cl_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cl_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ void st_cl_u32(uint32_t cl_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cl_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *map, uint32_t mbar_cl,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar_cl), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this smem offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)), "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

struct SmemP {
  uint8_t *sA, *sB, *stg;
  uint64_t *full, *empty, *tfull, *tempty, *qfull, *qempty;
  uint32_t *tmem_base, *tile_q;
};

template <int NA>
__device__ __forceinline__ SmemP carve_pair(uint8_t *raw) {
  constexpr int STP = stp_of<NA>();
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  SmemP m;
  m.sA = smem;
  m.sB = smem + STP * NA * A_BYTES;
  m.stg = m.sB + STP * BP_BYTES;
  m.full = reinterpret_cast<uint64_t *>(m.stg + EPI_WARPS * STG_BYTES);
  m.empty = m.full + STP;
  m.tfull = m.empty + STP;
  m.tempty = m.tfull + 2;
  m.qfull = m.tempty + 2;
  m.qempty = m.qfull + TQ;
  m.tmem_base = reinterpret_cast<uint32_t *>(m.qempty + TQ);
  m.tile_q = m.tmem_base + 4;
  return m;
}

// warp 0: TMA producer (both CTAs; the leader also claims the tiles);
// warp 1: TMEM allocation (both) + MMA issue (leader only);
// warps 2-9: epilogue of this CTA's 128 rows.
// Both CTAs' TMA loads of a stage complete on the LEADER's full barrier
// (cp.async.bulk.tensor .cta_group::2), which the leader arms with the bytes
// of both halves; the MMA commit releases the stage in both CTAs at once
// (multicast), so no CTA-to-CTA handshake sits on the K loop.
template <int NA, int BN2>
__global__ void __maxnreg__(GRU_MAXREG)
    k_gru_tc2(const __grid_constant__ CUtensorMap map_a1, const __grid_constant__ CUtensorMap map_w1h,
              const __grid_constant__ CUtensorMap map_rh, const __grid_constant__ CUtensorMap map_w2h,
              TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  constexpr int STP = stp_of<NA>();
  const unsigned long long t_entry = a.prof ? gtimer() : 0ull;   // diag 5: kernel entry (before setup)
  const SmemP m = carve_pair<NA>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const uint32_t n1 = a.nub, n2 = a.H / BN2;             // phase-2 tiles of BN2 = 256 or 128 units
  const uint32_t kx = a.E / BK, KCt = seg_chunks(a);
  const uint32_t target = n1 * 2 * EPI_WARPS;           // phase-1 arrivals per 256-row tile
  // tile-ring consumers (arrivals on the leader's qempty per slot): the
  // leader's MMA lane, the peer's producer, both CTAs' epilogue warps
  constexpr uint32_t RING_CONSUMERS = 2 + 2 * EPI_WARPS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STP; ++s) { mbar_init(&m.full[s], 1); mbar_init(&m.empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&m.tfull[s], 1); mbar_init(&m.tempty[s], 2 * EPI_WARPS); }
    for (int s = 0; s < TQ; ++s) { mbar_init(&m.qfull[s], 1); mbar_init(&m.qempty[s], RING_CONSUMERS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&map_a1); prefetch_map(&map_w1h); prefetch_map(&map_rh); prefetch_map(&map_w2h);
  }
  if (warp == 1) tmem_alloc_pair(m.tmem_base, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();                                      // the peer's barriers exist
  pdl_entry();
  const uint32_t Q = a.counts[1];
  const uint32_t mt = (Q + 2 * BM - 1) / (2 * BM);
  const uint32_t L = mt < a.lag / 2 ? mt : a.lag / 2;
  const uint32_t ntiles = mt * (n1 + n2);
  const uint32_t tmem_base = *m.tmem_base;
  const uint32_t full0 = mapa(smem_u32(&m.full[0]), 0);       // the leader's barriers
  const uint32_t tempty0 = mapa(smem_u32(&m.tempty[0]), 0);
  const uint32_t qempty0 = mapa(smem_u32(&m.qempty[0]), 0);
  unsigned long long *prof = a.prof ? a.prof + blockIdx.x * 16 : nullptr;
  const unsigned long long k_t0 = pclk();
  if (prof && threadIdx.x == 0) { prof[14] = gtimer(); prof[7] = t_entry; }

  // tile id of ring slot `it`; one lane releases the slot on the leader's qempty
  auto take = [&](uint32_t it, bool release) -> uint32_t {
    const uint32_t slot = it % TQ;
    mbar_wait_cl(&m.qfull[slot], (it / TQ) & 1);
    const uint32_t t = *reinterpret_cast<volatile uint32_t *>(&m.tile_q[slot]);
    __syncwarp(__activemask());
    if (release) mbar_arrive_cl(qempty0 + slot * 8);
    return t;
  };

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      unsigned long long w_empty = 0, w_dep = 0, t0;
      for (uint32_t it = 0;; ++it) {
        uint32_t t;
        if (leader) {
          const uint32_t slot = it % TQ;
          mbar_wait_cl(&m.qempty[slot], ((it / TQ) & 1) ^ 1);
          t = atomicAdd(a.tile_ctr, 1u);
          if (t >= ntiles) t = NO_TILE;
          m.tile_q[slot] = t;
          st_cl_u32(mapa(smem_u32(&m.tile_q[slot]), 1), t);
          mbar_arrive(&m.qfull[slot]);
          mbar_arrive_cl(mapa(smem_u32(&m.qfull[slot]), 1));
        } else {
          t = take(it, true);
        }
        if (t == NO_TILE) break;
        const Tile x = tile_of(t, mt, n1, n2, L, a.gm);
        const uint32_t m0 = x.m * 2 * BM + rank * BM;
        const uint32_t bh = x.kind == 1 ? (uint32_t)(BN2 / 2) : (uint32_t)(BN / 2);   // B rows this CTA loads
        const uint32_t b0row = x.j * 2 * bh + rank * bh;
        if (x.kind == 1 && a.diag != 4) {
          t0 = pclk();
          wait_phase1(a.done1 + x.m, target);
          w_dep += pclk() - t0;
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        if (prof) prof[9 + x.kind] += 1;
        for (uint32_t sg = 0; sg < a.nseg; ++sg) {
          // this segment: weight part pw, A parts pa0 .. pa0 + npa - 1 (column offsets into the part blocks)
          const uint32_t pa0 = a.seg[sg].pa0, npa = NA == 1 ? 1u : a.seg[sg].npa;
          const int b_off = (int)(a.seg[sg].pw * (a.E + a.H));
          // packed single-part stage (3-part ring): A(kc), A(kc+1) in A slots 0, 1, B(kc) in the
          // B slot and B(kc+1) in A slot 2, so the stage carries as many bytes as a 3-part stage
          const uint32_t step = (NA == 3 && npa == 1 && a.pack) ? 2u : 1u;
          for (uint32_t kc = a.seg[sg].k0; kc < a.seg[sg].k1; kc += step) {
            const uint32_t nk = kc + step <= a.seg[sg].k1 ? step : 1u;   // K-chunks in this stage
            t0 = pclk();
            mbar_wait(&m.empty[stage], phase ^ 1);
            w_empty += pclk() - t0;
            if (a.diag == 2 || a.diag == 6) {
              if (leader) mbar_arrive(&m.full[stage]);
              if (++stage == STP) { stage = 0; phase ^= 1; }
              continue;
            }
            if (leader) mbar_expect_tx(&m.full[stage], 2 * (npa * nk * A_BYTES + nk * bh * BK * 2));
            const uint32_t fb = full0 + stage * 8;
            const uint32_t dA = smem_u32(m.sA + stage * NA * A_BYTES), dB = smem_u32(m.sB + stage * BP_BYTES);
            const CUtensorMap *mapb = x.kind == 0 ? &map_w1h : &map_w2h;
            if (nk == 2) {
#pragma unroll
              for (uint32_t c = 0; c < 2; ++c) {
                const uint32_t k = kc + c;
                if (x.kind == 0 || k < kx)
                  tma_load_2d_pair(dA + c * A_BYTES, &map_a1, fb, (int)(pa0 * (a.E + a.H) + k * BK), (int)m0);
                else
                  tma_load_2d_pair(dA + c * A_BYTES, &map_rh, fb, (int)(pa0 * a.H + (k - kx) * BK), (int)m0);
              }
              tma_load_2d_pair(dB, mapb, fb, b_off + (int)(kc * BK), (int)b0row);
              tma_load_2d_pair(dA + 2 * A_BYTES, mapb, fb, b_off + (int)((kc + 1) * BK), (int)b0row);
            } else {
#pragma unroll
              for (uint32_t p = 0; p < (uint32_t)NA; ++p) {
                if (p >= npa) break;
                const uint32_t pa = pa0 + p;
                if (x.kind == 0 || kc < kx)
                  tma_load_2d_pair(dA + p * A_BYTES, &map_a1, fb, (int)(pa * (a.E + a.H) + kc * BK), (int)m0);
                else
                  tma_load_2d_pair(dA + p * A_BYTES, &map_rh, fb, (int)(pa * a.H + (kc - kx) * BK), (int)m0);
              }
              tma_load_2d_pair(dB, mapb, fb, b_off + (int)(kc * BK), (int)b0row);
            }
            if (++stage == STP) { stage = 0; phase ^= 1; }
          }
        }
      }
      if (prof) { prof[0] = w_empty; prof[1] = w_dep; }
    }
  } else if (warp == 1) {
    if (leader) {
      uint32_t stage = 0, phase = 0;
      const uint32_t id1 = idesc_bf16(2 * BM, BN), id2 = idesc_bf16(2 * BM, BN2);
      uint32_t KSt = 0;                                 // smem stages per tile (packed single-part stages)
      for (uint32_t sg = 0; sg < (NA == 1 ? 1u : a.nseg); ++sg) {
        const uint32_t len = NA == 1 ? KCt : (uint32_t)(a.seg[sg].k1 - a.seg[sg].k0);
        KSt += (NA == 3 && a.seg[sg].npa == 1 && a.pack) ? (len + 1) / 2 : len;
      }
      const uint32_t p2_first = L >= mt ? mt * n1 : 0xFFFFFFFFu;     // separated phases: phase 2 = the tail
      unsigned long long w_full = 0, w_tempty = 0, t0;
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % TQ;                  // the leader MMA lane reads its own ring
        mbar_wait(&m.qfull[slot], (it / TQ) & 1);
        const uint32_t t = *reinterpret_cast<volatile uint32_t *>(&m.tile_q[slot]);
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(qempty0 + slot * 8);
        if (t == NO_TILE) break;
        const uint32_t id = BN2 == BN ? id1
                            : ((t >= p2_first || (p2_first == 0xFFFFFFFFu && tile_of(t, mt, n1, n2, L, a.gm).kind == 1))
                                   ? id2 : id1);
        const uint32_t acc = it & 1;
        t0 = pclk();
        mbar_wait_cl(&m.tempty[acc], ((it >> 1) & 1) ^ 1);   // arrivals from both CTAs
        w_tempty += pclk() - t0;
        tc_fence_after();
        const uint32_t tm = tmem_base + acc * BN;
        uint32_t kc = 0;                                  // stage count of this tile
        // NA == 1: every stage holds one A chunk, the segment walk is not needed
        for (uint32_t sg = 0; sg < (NA == 1 ? 1u : a.nseg); ++sg) {
          const uint32_t npa = NA == 1 ? 1u : a.seg[sg].npa;
          const uint32_t c0 = NA == 1 ? 0u : a.seg[sg].k0, c1 = NA == 1 ? KCt : a.seg[sg].k1;
          const uint32_t step = (NA == 3 && npa == 1 && a.pack) ? 2u : 1u;   // packed stages (producer)
          for (uint32_t c = c0; c < c1; c += step, ++kc) {
            const uint32_t nk = c + step <= c1 ? step : 1u;
            t0 = pclk();
            // both CTAs' bytes landed (complete_tx on this barrier); the MMA reads them
            // through the async proxy, so a CTA-scope wait suffices -- a cluster-scope
            // acquire would invalidate this SM's L1 (CCTL.IVALL) on every stage
            mbar_wait(&m.full[stage], phase);
            w_full += pclk() - t0;
            tc_fence_after();
            if (lane == 0) {
              const uint32_t a0 = smem_u32(m.sA + stage * NA * A_BYTES), b0 = smem_u32(m.sB + stage * BP_BYTES);
              if (a.diag != 1 && a.diag != 6) {
                if (nk == 2) {                            // A(c) . B(c), then A(c+1) . B(c+1) (in A slot 2)
#pragma unroll
                  for (uint32_t q = 0; q < 2; ++q)
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                      umma_bf16_pair(tm, sdesc(a0 + q * A_BYTES + k * 32),
                                     sdesc((q ? a0 + 2 * A_BYTES : b0) + k * 32), id, (kc | q | k) != 0);
                } else {
#pragma unroll
                  for (uint32_t p = 0; p < (uint32_t)NA; ++p)
                    if (p < npa)
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                      umma_bf16_pair(tm, sdesc(a0 + p * A_BYTES + k * 32), sdesc(b0 + k * 32), id, (kc | p | k) != 0);
                }
              }
              umma_commit_pair(&m.empty[stage]);
              if (kc == KSt - 1) umma_commit_pair(&m.tfull[acc]);
            }
            __syncwarp();
            if (++stage == STP) { stage = 0; phase ^= 1; }
          }
        }
      }
      if (prof && lane == 0) { prof[2] = w_full; prof[3] = w_tempty; }
    }
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r_in = q * 32 + lane;
    uint8_t *stg = m.stg + (warp - 2) * STG_BYTES;
    unsigned long long w_tfull = 0, b1 = 0, b2 = 0, t0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t t = take(it, lane == 0);
      if (t == NO_TILE) break;
      const Tile x = tile_of(t, mt, n1, n2, L, a.gm);
      const uint32_t acc = it & 1;
      t0 = pclk();
      mbar_wait(&m.tfull[acc], (it >> 1) & 1);
      w_tfull += pclk() - t0;
      t0 = pclk();
      tc_fence_after();
      const uint32_t row = x.m * 2 * BM + rank * BM + r_in;
      const bool valid = row < Q;
      const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16) + half * (BN / 2);
      if (a.diag == 3 || a.diag == 4) {                   // timing only: no epilogue work
        float v[16];
        tmem_ld16(tbase, v);
        tmem_ld_wait();
      } else if (x.kind == 0) {
        epi_phase1<__nv_bfloat16>(a, tbase - half * (BN / 2), row, valid, half, x.j, stg, lane);
      } else {
        wait_phase1(a.done1 + x.m, target);
        epi_phase2(a, tbase - half * (BN / 2) + half * (BN2 / 2), row, valid, x.j * BN2 + half * (BN2 / 2),
                   BN2 / 2, stg, lane);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty0 + acc * 8);
      if (x.kind == 0) {
        // publish this CTA's z / r.h columns to the phase-2 tiles of the pair tile:
        // every writer orders its generic stores for the async proxy (the phase-2
        // TMA reads r.h), the 8 epilogue warps meet on a named barrier, and one
        // thread releases them at GPU scope with ONE fence + counter add
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(EPI_WARPS * 32) : "memory");
        if (warp == 2 && lane == 0) {
          __threadfence();
          atomicAdd(a.done1 + x.m, (uint32_t)EPI_WARPS);
        }
        b1 += pclk() - t0;
      } else {
        b2 += pclk() - t0;
      }
    }
    if (prof && lane == 0 && (warp == 2 || warp == 6)) {
      const int o = warp == 2 ? 4 : 11;
      prof[o] = w_tfull; prof[o + 1] = b1; prof[o + 2] = b2;
    }
  }
  if (prof && threadIdx.x == 0) prof[8] = pclk() - k_t0;
  tc_fence_before();
  __syncthreads();
  if (prof && threadIdx.x == 0) prof[15] = gtimer();       // every warp of the CTA is done
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}
template <int NA>
constexpr size_t smem_pair() { return 1024 + stp_of<NA>() * (NA * A_BYTES + BP_BYTES) + EPI_WARPS * STG_BYTES + 256; }
static_assert(smem_pair<3>() <= 232448, "BF16X3 pair stages exceed the 227-KB smem limit");

constexpr size_t smem_of(int nst) { return 1024 + nst * (A_BYTES + B_BYTES) + EPI_WARPS * STG_BYTES + 256; }
constexpr size_t SMEM = smem_of(ST), SMEM_RNN = smem_of(st_of<RNNLM_CELL_RNN>());

// ---------------------------------------------------------------- host side
struct TcState {
  uint32_t E = 0, H = 0, nub = 0, bmax = 0;
  bool tf32 = false;               // operands fp32 read as TF32 (else bf16)
  void *w1 = nullptr, *w2 = nullptr, *rh = nullptr, *a1 = nullptr;
  uint32_t *done1 = nullptr;
  int pair = 0;                    // 0: one-CTA kernel; 1: cta_group::2 pair (bf16 GRU default; RNNLM_TC_PAIR)
  uint32_t diag = 0;               // RNNLM_TC_DIAG: timing diagnostics (see TcArgs::diag)
  unsigned long long *prof = nullptr;
  float *bzr = nullptr, *bh = nullptr;
  uint32_t x3 = 0;                 // split modes: operand parts P (2: TF32X3, 3: BF16X3); 0: plain
  uint32_t wparts = 1;             // weight parts with a non-zero entry (1: every weight is exact in T)
  bool x3_xlo = true;              // some embedding entry is not exact in the operand type
  bool lbr = false;                // cell GRU_LBR: one-phase tiles over W3
  bool rnn = false;                // cell RNN: one-phase tiles over W2 = [Wh | Uh]
  void *w3 = nullptr;
  float *bz = nullptr, *br = nullptr;
  CUtensorMap map_w1, map_w2, map_a1, map_rh, map_w1h, map_w2h, map_w2q, map_w3;
  bool bound = false;
};

}  // namespace rnnlm_tc

namespace rnnlm_host {
using namespace rnnlm_tc;

int gru_tc_supported(uint32_t E, uint32_t H) {
  return E % BK == 0 && H % UB == 0 && E >= BK && H >= UB;      // phase-2 tiles narrow to 128 units
}

template <typename T>
static T cv_op(float v) {
  if constexpr (sizeof(T) == 2) {
    return __float2bfloat16_rn(v);
  } else {  // round to TF32 (nearest, ties away; same as cvt.rna.tf32.f32 on the activations)
    uint32_t b;
    std::memcpy(&b, &v, 4);
    b = (b + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &b, 4);
    return r;
  }
}

// LBR cell: W3 = per 64-unit block 192 rows (K-major, E + H columns); row
// g * 64 + i carries [Wh, Wz, Wr][g] row i in its x half and [Uz, Ur, Uh][g]
// row i in its h half (see mma_loop).
template <typename T>
static bool upload_w3(TcState *t, const rnnlm_weights *w, uint32_t E, uint32_t H) {
  const size_t K1 = E + H;
  std::vector<T> w3((size_t)3 * H * K1);
  const float *Wg[3] = {w->Wh, w->Wz, w->Wr};
  const float *Ug[3] = {w->Uz, w->Ur, w->Uh};
  for (size_t u = 0; u < H; ++u)
    for (int g = 0; g < 3; ++g) {
      T *row = w3.data() + ((u / 64) * 192 + g * 64 + u % 64) * K1;
      for (size_t k = 0; k < E; ++k) row[k] = cv_op<T>(Wg[g][u * E + k]);
      for (size_t k = 0; k < H; ++k) row[E + k] = cv_op<T>(Ug[g][u * H + k]);
    }
  return cudaMalloc(&t->w3, w3.size() * sizeof(T)) == cudaSuccess &&
         cudaMemcpy(t->w3, w3.data(), w3.size() * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess;
}

template <typename T>
static bool upload_w(TcState *t, const rnnlm_weights *w, uint32_t E, uint32_t H) {
  // rows of K1 = E + H operands; in the split modes each row is [part 0 | .. | part P-1] (P K1)
  const size_t K1 = E + H, NP = t->x3 ? t->x3 : 1, RW = NP * K1;
  std::vector<T> w1((size_t)2 * H * RW), w2((size_t)H * RW);
  auto cv = [](float v) -> T {
    if constexpr (sizeof(T) == 2) {
      return __float2bfloat16_rn(v);
    } else {  // round to TF32 (nearest, ties away; same as cvt.rna.tf32.f32 on the activations)
      uint32_t b;
      std::memcpy(&b, &v, 4);
      b = (b + 0x1000u) & 0xFFFFE000u;
      float r;
      std::memcpy(&r, &b, 4);
      return r;
    }
  };
  const float *Wg[2] = {w->Wz, w->Wr};
  const float *Ug[2] = {w->Uz, w->Ur};
  bool any_lo = false;
  // one weight into (row, k): its (TF32 / bf16) value, and in the split modes
  // the parts of the successive remainders at k + p K1 (exact fp32 differences)
  auto put = [&](T *row, size_t k, float v) {
    float r = v;
    for (size_t p = 0; p < NP; ++p) {
      row[p * K1 + k] = cv(r);
      r -= (float)row[p * K1 + k];
      if (p > 0 && (float)row[p * K1 + k] != 0.0f) any_lo = true;
    }
  };
  for (size_t u = 0; u < H; ++u) {
    const size_t ub = u / UB, uu = u % UB;
    for (int g = 0; g < 2; ++g) {
      T *row = w1.data() + (ub * BN + g * UB + uu) * RW;
      for (size_t k = 0; k < E; ++k) put(row, k, Wg[g][u * E + k]);
      for (size_t k = 0; k < H; ++k) put(row, E + k, Ug[g][u * H + k]);
    }
    T *row2 = w2.data() + u * RW;
    for (size_t k = 0; k < E; ++k) put(row2, k, w->Wh[u * E + k]);
    for (size_t k = 0; k < H; ++k) put(row2, E + k, w->Uh[u * H + k]);
  }
  t->wparts = any_lo ? (uint32_t)NP : 1u;
  return cudaMalloc(&t->w1, w1.size() * sizeof(T)) == cudaSuccess &&
         cudaMalloc(&t->w2, w2.size() * sizeof(T)) == cudaSuccess &&
         cudaMemcpy(t->w1, w1.data(), w1.size() * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(t->w2, w2.data(), w2.size() * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess;
}

int gru_tc_prepare(const rnnlm_weights *w, uint32_t V, uint32_t E, uint32_t H, int tf32, int x3, int cell,
                   void **state_out) {
  *state_out = nullptr;
  TcState *t = new TcState;
  t->E = E; t->H = H; t->nub = H / UB; t->tf32 = tf32 != 0;
  t->x3 = (x3 == 2 && t->tf32) || (x3 == 3 && !t->tf32) ? (uint32_t)x3 : 0u;
  if (t->x3) {                    // is every embedding entry exact in T (TF32: low 13, bf16: low 16 bits zero)?
    const uint32_t low = t->tf32 ? 0x1FFFu : 0xFFFFu;
    t->x3_xlo = false;
    for (size_t i = 0; i < (size_t)E * V; ++i) {
      uint32_t b;
      std::memcpy(&b, &w->emb[i], 4);
      if (b & low) { t->x3_xlo = true; break; }
    }
  }
  t->lbr = cell == RNNLM_CELL_GRU_LBR;
  t->rnn = cell == RNNLM_CELL_RNN;
  // the CTA pair (cta_group::2) is the default for the bf16 GRU: ~1.3 % faster kernel
  // than one CTA per tile at the bench size (198.5 vs 201.1 us, three runs each);
  // RNNLM_TC_PAIR=0 selects the one-CTA kernel, which runs every other mode
  t->pair = 1;
  if (const char *e = getenv("RNNLM_TC_PAIR")) t->pair = atoi(e);
  if (t->tf32 || cell) t->pair = 0;
  if (const char *e = getenv("RNNLM_TC_DIAG")) t->diag = (uint32_t)atoi(e);
  const size_t K1 = E + H;
  std::vector<float> bzr((size_t)2 * H), bh(H);
  const float *bg[2] = {w->bz, w->br};
  for (size_t u = 0; u < H; ++u) {
    const size_t ub = u / UB, uu = u % UB;
    for (int g = 0; g < 2; ++g) bzr[ub * BN + g * UB + uu] = bg[g][u];
    bh[u] = w->bh[u];
  }
  bool ok = t->tf32 ? upload_w<float>(t, w, E, H) : upload_w<__nv_bfloat16>(t, w, E, H);
  if (t->lbr) {
    ok = ok && (t->tf32 ? upload_w3<float>(t, w, E, H) : upload_w3<__nv_bfloat16>(t, w, E, H));
    ok = ok && cudaMalloc(&t->bz, (size_t)H * 4) == cudaSuccess && cudaMalloc(&t->br, (size_t)H * 4) == cudaSuccess &&
         cudaMemcpy(t->bz, w->bz, (size_t)H * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(t->br, w->br, (size_t)H * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         make_map(&t->map_w3, t->w3, K1, (uint64_t)H / 64 * 192, 192, t->tf32);
  }
  ok = ok && cudaMalloc(&t->bzr, bzr.size() * 4) == cudaSuccess &&
       cudaMalloc(&t->bh, bh.size() * 4) == cudaSuccess;
  ok = ok && cudaMemcpy(t->bzr, bzr.data(), bzr.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(t->bh, bh.data(), bh.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  const size_t RW = (t->x3 ? t->x3 : 1) * K1;
  ok = ok && make_map(&t->map_w1, t->w1, RW, 2 * (uint64_t)H, BN, t->tf32) &&
       make_map(&t->map_w2, t->w2, RW, H, H % BN ? UB : BN, t->tf32);
  if (H % BN) t->pair = 0;        // the CTA pair keeps 256-unit phase-2 tiles
  if (!t->tf32)
    ok = ok && make_map(&t->map_w1h, t->w1, RW, 2 * (uint64_t)H, BN / 2) &&
         make_map(&t->map_w2h, t->w2, RW, H, BN / 2) && make_map(&t->map_w2q, t->w2, RW, H, BN / 4);
  ok = ok && cudaFuncSetAttribute(k_gru_tc<__nv_bfloat16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc<float, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc<__nv_bfloat16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc<float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc<__nv_bfloat16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_RNN) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc<float, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_RNN) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc2<1, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pair<1>()) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc2<3, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pair<3>()) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc2<1, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pair<1>()) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_gru_tc2<3, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pair<3>()) == cudaSuccess;
  *state_out = t;
  if (!ok) {
    (void)cudaGetLastError();
    return -1;
  }
  return 0;
}

// The activation maps need the engine's scratch; bound once per engine.
int gru_tc_bind(void *state, void *rh, uint32_t bmax) {
  TcState *t = static_cast<TcState *>(state);
  t->rh = rh;
  t->bmax = bmax;
  const size_t es = t->tf32 ? 4 : 2;
  const size_t xw = t->x3 ? t->x3 : 1;                 // split modes: P operand parts per row
  if (cudaMalloc(&t->a1, (size_t)bmax * (t->E + t->H) * es * xw) != cudaSuccess ||
      cudaMalloc(&t->done1, ((size_t)bmax / BM + 4) * sizeof(uint32_t)) != cudaSuccess) {
    (void)cudaGetLastError();
    return -1;
  }
  t->bound = make_map(&t->map_rh, rh, t->H * xw, bmax, BM, t->tf32) &&
             make_map(&t->map_a1, t->a1, (t->E + t->H) * xw, bmax, BM, t->tf32);
  return t->bound ? 0 : -1;
}

// The gate weights in their K-major row layouts (bf16, or TF32-rounded fp32):
// W1 rows [Wz|Uz], [Wr|Ur] per 128-unit block, W2 rows [Wh|Uh]; row width in
// elements.  The GEMV path (k_gemv.cu) reads them directly.  Returns -1 for
// 3xTF32 (its rows hold [hi | lo] parts).
int gru_tc_weights(void *state, const void **w1, const void **w2, uint32_t *rw) {
  TcState *t = static_cast<TcState *>(state);
  if (!t || t->x3) return -1;
  *w1 = t->w1; *w2 = t->w2; *rw = t->E + t->H;
  return 0;
}

// K segments of the split modes (see SplitSeg): the terms A_pa . W_pw with
// pa + pw < P, lowest order first; weight parts that are all zero and, over
// the x columns, embedding parts that are all zero are skipped.
// RNNLM_SPLIT_ALL_SEGMENTS (A/B) runs the identically-zero products anyway.
static void make_segs(TcArgs &a, const TcState *t, bool grouped) {
  const uint32_t bke = t->tf32 ? 32u : 64u;
  const uint32_t kx = t->E / bke, KC = (t->E + t->H) / bke;
  a.nseg = 0;
  auto add = [&](uint32_t npa, uint32_t pw, uint32_t k0, uint32_t k1) {   // A parts 0 .. npa - 1
    if (grouped) {
      a.seg[a.nseg++] = SplitSeg{0, (uint8_t)npa, (uint8_t)pw, 0, (uint16_t)k0, (uint16_t)k1};
    } else {
      for (uint32_t p = 0; p < npa; ++p)
        a.seg[a.nseg++] = SplitSeg{(uint8_t)p, 1, (uint8_t)pw, 0, (uint16_t)k0, (uint16_t)k1};
    }
  };
  if (!t->x3) {
    add(1, 0, 0, KC);
    return;
  }
  const bool all = getenv("RNNLM_SPLIT_ALL_SEGMENTS") != nullptr;
  const uint32_t P = t->x3, PW = all ? P : t->wparts;
  const bool xlo = all || t->x3_xlo;
  for (uint32_t pw = 0; pw < PW; ++pw) {
    const uint32_t nh = P - pw;                  // A parts pa with pa + pw <= P - 1
    const uint32_t nx = xlo ? nh : 1;            // over the x columns only part 0 may be non-zero
    if (nx == nh) {
      add(nh, pw, 0, KC);
    } else {
      add(nx, pw, 0, kx);
      add(nh, pw, kx, KC);
    }
  }
}

// Tensor-core products per useful multiply-add of a split mode (the chunks
// of every segment over the chunks of K); 0 for the plain modes.
double gru_tc_x3_products(void *state) {
  TcState *t = static_cast<TcState *>(state);
  if (!t || !t->x3) return 0.0;
  TcArgs a;
  make_segs(a, t, true);
  double chunks = 0;
  for (uint32_t i = 0; i < a.nseg; ++i) chunks += (double)a.seg[i].npa * (a.seg[i].k1 - a.seg[i].k0);
  return chunks * (t->tf32 ? 32.0 : 64.0) / (double)(t->E + t->H);
}

void gru_tc_release(void *state) {
  TcState *t = static_cast<TcState *>(state);
  if (!t) return;
  cudaFree(t->w1);
  cudaFree(t->w2);
  cudaFree(t->w3);
  cudaFree(t->bz);
  cudaFree(t->br);
  cudaFree(t->a1);
  cudaFree(t->done1);
  cudaFree(t->prof);
  cudaFree(t->bzr);
  cudaFree(t->bh);
  delete t;
}

int launch_gru_tc(const Params &P, void *state, uint32_t max_rows, int num_sms, cudaStream_t s,
                  cudaEvent_t ev_gathered, cudaEvent_t ev_phase1, cudaEvent_t ev_fork) {
  TcState *t = static_cast<TcState *>(state);
  if (!max_rows || !t || !t->bound) return 0;
  TcArgs a;
  a.E = P.E; a.H = P.H; a.nub = t->nub;
  a.emb16 = P.emb16; a.state = P.state; a.bzr = t->bzr; a.bh = t->bh;
  a.state_out = P.state;
  a.row_src = P.row_src; a.row_dst = P.row_dst; a.row_word = P.row_word; a.counts = P.counts;
  a.g_z = P.g_z; a.g_rh16 = P.g_rh16; a.g_rhf = P.g_rh;
  a.a1 = static_cast<__nv_bfloat16 *>(t->a1); a.a1f = static_cast<float *>(t->a1); a.emb = P.emb;
  a.cache = P.cache; a.key_mode = P.key_mode; a.round_digits = P.round_digits;
  a.cstride = P.cstride; a.round_scale = P.round_scale; a.codes = P.codes; a.codehash = P.codehash;
  a.done1 = t->done1;
  a.tile_ctr = t->done1 + (t->bmax / BM + 2);
  // phase-2 tiles trail their phase-1 tiles by this many 128-row M-tiles (RNNLM_TC_LAG);
  // one CTA per tile, measured: 24: 504, 48: 521, 96-1000: 530-535 M q/s on the bench
  // workload -- keeping the two
  // phases apart (each phase's weights hot in L2) beats interleaving them tightly
  // CTA pair (5-stage ring): lag 32: 537-540, 48: 543-545, 64: 548-551, 96: 543-553,
  // 128: 546-549 M q/s, kernel 199.5 / 196.5 / 193.3 / 193.7 / 195.4 us (profiles/ab_lag_r1.txt)
  // BF16X3 on the pair: every phase-1 tile before any phase-2 tile -- lag 16 / 32 / 64 / 128 / 1000:
  // 264 / 248 / 235 / 228 / 228 us per bench step (profiles/ab_lag_r2.txt)
  a.lag = getenv("RNNLM_TC_LAG") ? (uint32_t)atoi(getenv("RNNLM_TC_LAG"))
                                 : (t->pair ? (t->x3 ? 1000u : 64u) : 128u);
  a.gm = getenv("RNNLM_TC_GM") ? (uint32_t)atoi(getenv("RNNLM_TC_GM")) : 1u;
  a.pack = getenv("RNNLM_TC_PACK") ? (uint32_t)atoi(getenv("RNNLM_TC_PACK")) : 1u;
  if (!a.gm) a.gm = 1;
  a.diag = t->diag;
  a.bz = t->bz; a.br = t->br;
  a.bn2 = P.H % BN ? UB : BN;
  a.x3 = t->x3;
  a.x3_xlo = (t->x3_xlo || getenv("RNNLM_SPLIT_ALL_SEGMENTS")) ? 1u : 0u;
  // the CTA pair loads each weight chunk once for all A parts (RNNLM_TC_GROUP=0: one part per stage)
  const bool grouped = t->pair && !(getenv("RNNLM_TC_GROUP") && atoi(getenv("RNNLM_TC_GROUP")) == 0);
  make_segs(a, t, grouped);
  a.prof = nullptr;
  if (t->diag == 5) {
    if (!t->prof) cudaMalloc(&t->prof, 1024 * 16 * sizeof(unsigned long long));
    cudaMemsetAsync(t->prof, 0, 1024 * 16 * sizeof(unsigned long long), s);
    a.prof = t->prof;
  }
  const uint32_t mt = (max_rows + BM - 1) / BM;
  uint32_t g1 = t->lbr ? mt * (P.H / 64) : (t->rnn ? mt * (P.H / a.bn2) : mt * (t->nub + P.H / a.bn2));
  if (g1 > (uint32_t)num_sms) g1 = num_sms;
  uint32_t gg = (max_rows + 7) / 8;
  // resident blocks per SM: 4 for the fp32-operand gather (40 registers), 3 for
  // the bf16 gather (70 registers: a row chunk's 12 loads are held at once)
  uint32_t bps = t->tf32 ? 4u : 3u;
  if (const char *e = getenv("RNNLM_TC_GATHER_BPS")) bps = (uint32_t)atoi(e);
  if (gg > (uint32_t)num_sms * bps) gg = num_sms * bps;
  // side-stream fork before the gather (RNNLM_FORK_EARLY=1; A/B) or after it
  static const bool fork_early = getenv("RNNLM_FORK_EARLY") && atoi(getenv("RNNLM_FORK_EARLY")) != 0;
  if (ev_fork && fork_early) cudaEventRecord(ev_fork, s);
  if (t->tf32) launch_pdl(k_gather_a1<float>, gg, 256, 0, s, a);
  else launch_pdl(k_gather_a1<__nv_bfloat16>, gg, 256, 0, s, a);
  if (ev_gathered) cudaEventRecord(ev_gathered, s);
  if (ev_fork && !fork_early) cudaEventRecord(ev_fork, s);
  if (t->pair) {
    // Phase-2 tiles of 128 units for calls of up to RNNLM_TC_P2N_MAX queries (default 32,768:
    // 16 streams x 2,048), else 256: a small frame's GRU is two dependent tile waves, and
    // half-width phase-2 tiles halve the second one (8 / 16 streams: 138 -> 150 / 228 -> 245
    // M q/s) while costing ~10 % at 64 streams.  Splitting N does not change any output
    // element's accumulation, so results are bitwise the same either way.
    const uint32_t p2max = getenv("RNNLM_TC_P2N_MAX") ? (uint32_t)atoi(getenv("RNNLM_TC_P2N_MAX")) : 32768u;
    a.bn2 = max_rows <= p2max ? 128u : (uint32_t)BN;
    uint32_t gp = ((max_rows + 2 * BM - 1) / (2 * BM)) * (t->nub + P.H / a.bn2) * 2;
    const uint32_t cap = (uint32_t)num_sms & ~1u;
    if (gp > cap) gp = cap;
    const CUtensorMap &m2 = a.bn2 == UB ? t->map_w2q : t->map_w2h;
    // plain bf16 runs on the 3-part ring too: packed 64-KB stages of 2 K-chunks, 6 chunks in flight
    // instead of 5 (RNNLM_TC_BF16_NA3=0: the 5-deep 32-KB ring; 143.6 -> 141.7 us, profiles/ab_pack_r2.txt)
    const bool na3 = grouped && (t->x3 || !(getenv("RNNLM_TC_BF16_NA3") && atoi(getenv("RNNLM_TC_BF16_NA3")) == 0));
    if (na3) {
      if (a.bn2 == UB) launch_pdl_cluster(k_gru_tc2<3, UB>, gp, THREADS, smem_pair<3>(), s, 2, t->map_a1, t->map_w1h, t->map_rh, m2, a);
      else launch_pdl_cluster(k_gru_tc2<3, BN>, gp, THREADS, smem_pair<3>(), s, 2, t->map_a1, t->map_w1h, t->map_rh, m2, a);
    } else {
      if (a.bn2 == UB) launch_pdl_cluster(k_gru_tc2<1, UB>, gp, THREADS, smem_pair<1>(), s, 2, t->map_a1, t->map_w1h, t->map_rh, m2, a);
      else launch_pdl_cluster(k_gru_tc2<1, BN>, gp, THREADS, smem_pair<1>(), s, 2, t->map_a1, t->map_w1h, t->map_rh, m2, a);
    }
  } else {
    if (t->lbr) {
      if (t->tf32) launch_pdl(k_gru_tc<float, 1>, g1, THREADS, SMEM, s, t->map_a1, t->map_w3, t->map_rh, t->map_w2, a);
      else launch_pdl(k_gru_tc<__nv_bfloat16, 1>, g1, THREADS, SMEM, s, t->map_a1, t->map_w3, t->map_rh, t->map_w2, a);
    } else if (t->rnn) {
      if (t->tf32) launch_pdl(k_gru_tc<float, 2>, g1, THREADS, SMEM_RNN, s, t->map_a1, t->map_w2, t->map_rh, t->map_w2, a);
      else launch_pdl(k_gru_tc<__nv_bfloat16, 2>, g1, THREADS, SMEM_RNN, s, t->map_a1, t->map_w2, t->map_rh, t->map_w2, a);
    } else {
      if (t->tf32) launch_pdl(k_gru_tc<float, 0>, g1, THREADS, SMEM, s, t->map_a1, t->map_w1, t->map_rh, t->map_w2, a);
      else launch_pdl(k_gru_tc<__nv_bfloat16, 0>, g1, THREADS, SMEM, s, t->map_a1, t->map_w1, t->map_rh, t->map_w2, a);
    }
  }
  if (ev_phase1) cudaEventRecord(ev_phase1, s);
  if (a.prof) {
    // diag 5: per-CTA cycle counters, averaged over the CTAs, to stderr
    std::vector<unsigned long long> h(1024 * 16);
    cudaMemcpyAsync(h.data(), t->prof, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    int nb = 0;
    double sum[16] = {0};
    for (int b = 0; b < 1023; ++b) {
      if (!h[b * 16 + 8]) continue;
      ++nb;
      for (int k = 0; k < 16; ++k) sum[k] += (double)h[b * 16 + k];
    }
    if (nb) {
      // CTA timeline (globaltimer ns): kernel span, mean CTA busy span, spread of the CTA end times
      unsigned long long s0 = ~0ull, e0 = ~0ull, s1 = 0, e1 = 0;
      double busy = 0;
      for (int b = 0; b < 1023; ++b) {
        if (!h[b * 16 + 8]) continue;
        const unsigned long long st = h[b * 16 + 14], en = h[b * 16 + 15];
        s0 = st < s0 ? st : s0; s1 = st > s1 ? st : s1; e0 = en < e0 ? en : e0; e1 = en > e1 ? en : e1;
        busy += (double)(en - st);
      }
      unsigned long long en0 = ~0ull;
      for (int b = 0; b < 1023; ++b)
        if (h[b * 16 + 8] && h[b * 16 + 7] && h[b * 16 + 7] < en0) en0 = h[b * 16 + 7];
      const unsigned long long gend = h[1023 * 16];
      fprintf(stderr, "[gru_tc timeline] span_us=%.1f mean_cta_busy_us=%.1f start_spread_us=%.1f end_spread_us=%.1f"
              " gather_end_to_first_entry_us=%.1f first_entry_to_first_start_us=%.1f\n",
              (e1 - s0) * 1e-3, busy / nb * 1e-3, (s1 - s0) * 1e-3, (e1 - e0) * 1e-3,
              (gend && en0 != ~0ull) ? ((double)en0 - (double)gend) * 1e-3 : -1.0,
              en0 != ~0ull ? ((double)s0 - (double)en0) * 1e-3 : -1.0);
      static const char *nm[16] = {"prod_wait_empty", "prod_wait_dep", "mma_wait_full", "mma_wait_tempty",
                                   "epi_z_wait_tfull", "epi_z_body_p1", "epi_z_body_p2", "-", "total",
                                   "tiles_p1", "tiles_p2", "epi_r_wait_tfull", "epi_r_body_p1", "epi_r_body_p2",
                                   "-", "-"};
      fprintf(stderr, "[gru_tc prof] pair=%d ctas=%d", t->pair, nb);
      for (int k = 0; k < 14; ++k)
        if (nm[k][0] != '-') fprintf(stderr, " %s=%.0f", nm[k], sum[k] / nb);
      fprintf(stderr, "\n");
    }
  }
  return 2;
}
}  // namespace rnnlm_host
