// Persistent, warp-specialised tcgen05 GEMM for the AtariNet torso (sm_100a).
//
//   D[128 x BN tile] = sum_kb A_kb[128 x 64] * B_kb[BN x 64]^T   (bf16 in, f32 in TMEM)
//
// Warp roles (256 threads, 1 CTA / SM, grid = min(tiles, #SMs)):
//   warp 0      TMA producer: per K-block one (or two) A boxes + B boxes -> smem ring
//   warp 1      MMA issuer:   4 x tcgen05.mma (K=16) per 64-wide K-block, commit -> empty[s]
//   warp 2      TMEM allocator (2 accumulator buffers of BN f32 columns)
//   warps 4..7  epilogue:     tcgen05.ld 32 columns at a time, fused bias / relu /
//                             relu-mask / layout remap, vector stores
// The accumulator is double buffered so the epilogue of tile i overlaps the
// MMAs of tile i+1.
//
// Operand addressing generalises "shifted GEMM" convolution: K-block kb of A
// is a TMA box of the activation matrix [rows, C] at row offset off[kb / cb]
// (one offset per filter tap), so stride-1 convolutions (and strided ones
// after space-to-depth) need no im2col buffer.  For weight gradients the
// reduction runs over rows and both operands are MN-major boxes.
#pragma once
#include "sm100.cuh"

namespace bp {

constexpr int kGemmThreads = 256;
constexpr int kMaxShifts = 16;

enum AMode { A_KMAJOR = 0, A_MNMAJOR = 1 };
enum BMode { B_KMAJOR = 0, B_MNMAJOR = 1 };

// n / d for n < 2^31 by a precomputed multiplier (round-up method): q = (umulhi(n, mul) + n) >> shift
struct FDiv {
  uint32_t mul, shift;
};
inline FDiv fdiv_make(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  const unsigned long long m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
  return FDiv{(uint32_t)m, l};
}
BP_DEVICE uint32_t fdivu(uint32_t n, FDiv f) { return (__umulhi(n, f.mul) + n) >> f.shift; }

// the forward's two small jobs (network.cu prep_kernel): pack the heads operand
// Whf [32][576] bf16 = [Wp | bp ; Wv | bv] and write the augmented core columns [512, 576)
// [clip(r) | onehot(a) | 1 | 0] of every row.  Item space: [0, 32 * 576) heads elements, then
// n * 8 core chunks of 8 columns (one 16-byte store each).
struct PrepArgs {
  const float *wp, *bp, *wv, *bv;
  __nv_bfloat16* whf;
  const float* reward;
  const int64_t* last_action;
  __nv_bfloat16* core;
  int n, A;  // n == 0: no prep work
  unsigned long long* seed_state;  // non-null: advance the sampler's device-resident seed once
};

// graph-replayable sampling: every forward advances the device-resident seed (splitmix64 step)
// before its heads read it
BP_DEVICE void advance_seed_dev(unsigned long long* seed_state) {
  unsigned long long x = *seed_state + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  *seed_state = x ^ (x >> 31);
}

BP_DEVICE void prep_items(const PrepArgs& p, long long i0, long long stride) {
  constexpr int W = 576;
  const int core_w = 513 + p.A;
  const long long nh = 32 * W, total = nh + (long long)p.n * 8;
  for (long long i = i0; i < total; i += stride) {
    if (i < nh) {
      const int a = (int)(i / W), j = (int)(i % W);
      float v = 0.f;
      if (a < p.A) v = j < core_w ? p.wp[(size_t)a * core_w + j] : (j == core_w ? p.bp[a] : 0.f);
      else if (a == p.A) v = j < core_w ? p.wv[j] : (j == core_w ? p.bv[0] : 0.f);
      p.whf[i] = __float2bfloat16_rn(v);
      continue;
    }
    const long long c = i - nh, img = c >> 3;
    const int j0 = (int)(c & 7) * 8;
    const float r = fminf(fmaxf(p.reward[img], -1.f), 1.f);
    const long long la = p.last_action[img];
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = j0 + 2 * q + h;
        v2[h] = j == 0 ? r : j <= p.A ? (la == j - 1 ? 1.f : 0.f) : (j == p.A + 1 ? 1.f : 0.f);
      }
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(v2[0], v2[1]);
      w[q] = *reinterpret_cast<const uint32_t*>(&b2);
    }
    *reinterpret_cast<uint4*>(p.core + img * W + 512 + j0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

struct GemmArgs {
  // launch: grid cap (0 = one CTA per SM); pdl_late: the inputs are final before this kernel's
  // PDL predecessor started (e.g. the LSTM layer-1 weight gradients beside layer 0's
  // recurrence), so the kernel runs at once and waits for its predecessor only at the end
  int max_ctas, pdl_late;
  // tiling
  int m_tiles, n_tiles, splits;
  int num_kb;        // K blocks in total (K / 64 for K-major, rows / 64 for MN-major)
  int kb_per_split;  // K blocks per split
  // A operand
  int a_cb;                    // K-major: 64-wide channel blocks per shift
  int a_atoms_per_shift;       // MN-major: 64-wide M atoms per shift
  int a_nshifts;               // MN-major: number of shifts (atoms beyond are zero)
  int a_row_off[kMaxShifts];   // per-shift row offset (signed)
  // window mode (AW > 0, K-major A): one TMA box of a_win_rows rows starting at
  // m0 + a_min_off per channel block; tap s reads it at row (a_row_off[s] - a_min_off)
  int a_ntaps, a_min_off, a_win_rows;
  // B operand: K-major -> box (kb*64, n0); MN-major -> box (n0 + 64 j, kb*64)
  // epilogue
  int N;                 // full N (row-major ld of mask source / plain output)
  int M;                 // valid M rows (rows >= M are not stored)
  float alpha;           // v = alpha * acc (+ bias)
  const float* bias;     // [N] or null
  int relu;              // apply max(0, .)
  const uint32_t* mask_bits;  // relu-backward mask: bit (m * mask_ld + n) of this bit array; null = none
  int mask_ld;                // element row pitch of the masked activation (0 -> N)
  uint32_t* bits_out;         // forward: relu mask bits of the stored output, word = element offset / 32
  int out_f32;           // 1: f32 output, 0: bf16
  void* out;
  long long split_stride;  // elements between split partial outputs
  // row map: m -> (img, y, x) on a gh x gw grid; valid iff y < vh && x < vw
  int gh, gw, vh, vw, sy, sx;
  long long r_img, r_y, r_x, r_sub;
  // column map: C(n) = ((n/cdiv)/cq)*cs1 + ((n/cdiv)%cq)*cs2 + n%cdiv
  int cdiv, cq;
  long long cs1, cs2;
  // B MN-major addressing: box x = (kb / b_kb_per_tap) * b_tap_stride + n0 + 64 j,
  //                          box y = (kb % b_kb_per_tap) * 64
  int b_kb_per_tap;
  int b_tap_stride;
  // bias-gradient column sums of the stored (post-mask) values, deterministic:
  // colsum[(mt * 4 + epilogue_warp) * N + n] = sum over that warp's 32 rows (splits == 1)
  float* colsum;
  // optional per-tile timeline (test builds): trace[(blockIdx.x * trace_tiles + i) * 16 + event]
  unsigned long long* trace;
  int trace_tiles;
  // AtariNet heads epilogue (heads != 0): column j < A -> logits[m][j], j == A -> baseline[m]
  int heads, A;
  float* logits;   // [M][A] f32
  float* baseline; // [M] f32
  int64_t* actions;          // heads: optional fused Gumbel-max action per row (null = none)
  unsigned long long sample_seed;
  const unsigned long long* seed_state;  // non-null: the seed is read from device memory
  int greedy;                // heads sampling: argmax instead of Gumbel-max
  // AU8 (conv1): the A operand is built on chip from u8 frames instead of a bf16 grid.
  // Grid row r = img*441 + gy*21 + gx, channel ci*16 + ry*4 + rx of row r is
  // frame(img, ci)[4gy + ry][4gx + rx]; frame(img, ci) = u8 + plane * 7056 with
  // plane = u8_index ? clamp(u8_index[img*4 + ci], 0, u8_planes - 1) : img*4 + ci.
  const uint8_t* u8;
  const int32_t* u8_index;
  int u8_planes;
  long long u8_rows;  // valid grid rows (n * 441); rows beyond convert to zero
  __nv_bfloat16* u8_x0_out;  // optional: the converted grid rows of every tile also go to HBM
                             // as X0 [rows][64] bf16 (the conv1 weight-gradient operand)
  // epilogue divisors (filled by the launcher from gh*gw, gw, sy, sx, cdiv, cq)
  FDiv fd_per, fd_gw, fd_sy, fd_sx, fd_cdiv, fd_cq, fd_splits, fd_ntiles;
  long long col_stride;  // f32 output only: element stride between consecutive columns (0 = 1, vector stores)
  PrepArgs prep;         // prep.n > 0: the idle warp 3 of every CTA also does the forward's prep
                         // work (conv1: its outputs are read only by later kernels)
};

inline void gemm_prepare(GemmArgs& g) {
  g.fd_per = fdiv_make((uint32_t)(g.gh * g.gw));
  g.fd_gw = fdiv_make((uint32_t)g.gw);
  g.fd_sy = fdiv_make((uint32_t)g.sy);
  g.fd_sx = fdiv_make((uint32_t)g.sx);
  g.fd_cdiv = fdiv_make((uint32_t)g.cdiv);
  g.fd_cq = fdiv_make((uint32_t)g.cq);
  g.fd_splits = fdiv_make((uint32_t)g.splits);
  g.fd_ntiles = fdiv_make((uint32_t)g.n_tiles);
}

// BRES ("B resident", weight-stationary): every tile of the launch shares one B
// (n_tiles == 1, splits == 1) whose K-blocks fit in kBResBytes of shared memory; it
// is loaded once per CTA and only A streams through the pipeline, halving L2 traffic
// for the conv GEMMs (B = the conv weights, A = the activation grid).
constexpr uint32_t kBResBytes = 96 * 1024;

constexpr uint32_t kWinBytes = 20 * 1024;  // window stage: up to 160 rows x 128 B

// AU8 raw staging: per tile, 4 channel planes x up to 9 (img, gy) grid rows x 4 frame lines
// of 84 bytes (one 336-byte span per grid row), copied by bulk TMA from the u8 frames
constexpr int kRawRowBytes = 336;
constexpr int kRawRows = 9;
constexpr uint32_t kRawCiBytes = kRawRows * kRawRowBytes;  // 3024
constexpr uint32_t kRawBytes = 12288;                       // >= 4 * 3024, 1 KB multiple
constexpr int kRawStages = 4;
constexpr int kConvWarps = 8;  // AU8 converter warps (after the epilogue warps)

#ifndef BP_EPI_GROUPS
#define BP_EPI_GROUPS 3
#endif
constexpr int kEpiGroups = BP_EPI_GROUPS;

template <int BN, int AM, int BM, int BSWZ, bool BRES = false, int AW = 0, int AU8 = 0>
struct GemmCfg {
  // EPI epilogue warpgroups take the CTA's tiles in turn (the epilogue is the per-tile
  // bottleneck of these small-N GEMMs); one or two TMEM accumulators per group
  static constexpr int EPI = BN > 128 ? 1 : AU8 ? 2 : kEpiGroups;
  static constexpr int ACC = 2 * EPI * BN <= 512 ? 2 * EPI : EPI;
  static constexpr int CONV_WARP0 = 4 + 4 * EPI;  // AU8 converter warps follow the epilogue
  static constexpr int THREADS = 128 + 128 * EPI + (AU8 ? 32 * kConvWarps : 0);
  static constexpr uint32_t A_BYTES = AU8 == 2 ? 0 : AW ? kWinBytes : 128 * 64 * 2;
  static constexpr uint32_t B_BYTES = BN * 64 * 2;
  // AU8 == 2: the A operand (im2col rows, 4 taps x 64 channels) lives in TMEM, two buffers of
  // 128 columns after the accumulators; the "stages" are those two buffers (no smem ring)
  static constexpr uint32_t STAGE = AU8 == 2 ? 1024 : BRES ? A_BYTES : A_BYTES + B_BYTES;
  static constexpr uint32_t B_RES = AU8 ? 16 * 1024 : BRES ? kBResBytes : 0;
  static constexpr uint32_t RAW = AU8 ? kRawStages * kRawBytes : 0;
  static constexpr int STAGES = AU8 == 2 ? 2
      : (184 * 1024 - B_RES - RAW) / STAGE > 8 ? 8 : (184 * 1024 - B_RES - RAW) / STAGE;
  static constexpr uint32_t A_TMEM = ACC * BN;  // first TMEM column of the A buffers (AU8 == 2)
  static constexpr uint32_t TMEM_COLS = AU8 == 2 ? 512 : (ACC * BN <= 32) ? 32 : (ACC * BN <= 64) ? 64 : (ACC * BN <= 128) ? 128 : (ACC * BN <= 256) ? 256 : 512;
  static constexpr uint32_t OSTAGE = 4 * EPI * 2048;  // per epilogue warp: 32 rows x 64 B bf16 staging
  static constexpr size_t SMEM = (size_t)B_RES + RAW + (size_t)STAGES * STAGE + 1024 /*align*/ + 512 /*barriers*/ +
                                 4 * EPI * BN * sizeof(float) /*column sums*/ + 256 /*raw barriers + align*/ + OSTAGE;
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  static_assert(BM == B_KMAJOR || BSWZ == 128 || (BSWZ == 64 && BN == 32), "B swizzle");
};

BP_DEVICE unsigned long long gtimer() {  // SM cycle counter (per-CTA traces; %globaltimer ticks are ~1 us)
  return (unsigned long long)clock64();
}
BP_DEVICE void trace_ev(const GemmArgs& g, int i, int ev) {
  if (g.trace && i < g.trace_tiles) g.trace[((size_t)blockIdx.x * g.trace_tiles + i) * 16 + ev] = gtimer();
}

BP_DEVICE void tile_coords(const GemmArgs& g, int tile, int& mt, int& nt, int& sp) {
  const uint32_t r = fdivu((uint32_t)tile, g.fd_splits);
  sp = tile - (int)r * g.splits;
  mt = (int)fdivu(r, g.fd_ntiles);
  nt = (int)r - mt * g.n_tiles;
}

template <int AM>
BP_DEVICE void load_a(const GemmArgs& g, const CUtensorMap* tmA, int mt, int kb, uint8_t* sa, uint64_t* bar) {
  if constexpr (AM == A_KMAJOR) {
    const int s = kb / g.a_cb;
    const int cb = kb - s * g.a_cb;
    sm100::tma_load_2d(sa, tmA, bar, cb * 64, mt * 128 + g.a_row_off[s]);
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int atom = mt * 2 + j;
      const int s = atom / g.a_atoms_per_shift;
      const int cb = atom - s * g.a_atoms_per_shift;
      // shifts beyond the last are all-zero atoms: point the box fully out of bounds
      const int y = (s < g.a_nshifts) ? kb * 64 + g.a_row_off[s] : 0x3fffffff;
      sm100::tma_load_2d(sa + j * 8192, tmA, bar, cb * 64, y);
    }
  }
}

template <int BN, int BM, int BSWZ>
BP_DEVICE void load_b(const GemmArgs& g, const CUtensorMap* tmB, int nt, int kb, uint8_t* sb, uint64_t* bar) {
  if constexpr (BM == B_KMAJOR) {
    sm100::tma_load_2d(sb, tmB, bar, kb * 64, nt * BN);
  } else {
    const int tap = kb / g.b_kb_per_tap;
    const int x0 = tap * g.b_tap_stride + nt * BN;
    const int y = (kb - tap * g.b_kb_per_tap) * 64;
    if constexpr (BSWZ == 64) {
      sm100::tma_load_2d(sb, tmB, bar, x0, y);
    } else {
#pragma unroll
      for (int j = 0; j < BN / 64; ++j) sm100::tma_load_2d(sb + j * 8192, tmB, bar, x0 + j * 64, y);
    }
  }
}

template <int AM>
BP_DEVICE uint64_t a_desc(uint32_t base, int k) {
  if constexpr (AM == A_KMAJOR) return sm100::smem_desc(base + k * 32, 16, 1024, sm100::SWZ_128B);
  else return sm100::smem_desc(base + k * 2048, 8192, 1024, sm100::SWZ_128B);
}
template <int BM, int BSWZ>
BP_DEVICE uint64_t b_desc(uint32_t base, int k) {
  if constexpr (BM == B_KMAJOR) return sm100::smem_desc(base + k * 32, 16, 1024, sm100::SWZ_128B);
  else if constexpr (BSWZ == 64) return sm100::smem_desc(base + k * 1024, 16, 512, sm100::SWZ_64B);
  else return sm100::smem_desc(base + k * 2048, 8192, 1024, sm100::SWZ_128B);
}

BP_DEVICE uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

BP_DEVICE uint32_t ldg_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];\n" : "=r"(v) : "l"(p));
  return v;
}

// lane j ends with sum over the warp's 32 lanes of v[j] (31 shuffles, fixed order)
BP_DEVICE float warp_transpose_sum(float (&v)[32], int lane) {
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const bool upper = (lane & k) != 0;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const float send = upper ? v[i] : v[i + k];
      const float keep = upper ? v[i + k] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return v[0];
}

// Epilogue kinds (compile time; the hot GEMMs drop the runtime feature checks):
//   EPK_GEN   every feature from GemmArgs at run time (f32 partials, heads, tests);
//   EPK_FWD   conv / fc forward: alpha * acc + bias, ReLU, relu bits (when bits_out), bf16 out;
//   EPK_DGRAD data gradient: relu-backward mask, bf16 out, optional column sums.
//   EPK_HEADS the heads forward with the fused action sampler (inference only: the Philox code
//             stays out of the EPK_GEN instantiations, where it cost the heads / fc gradient
//             GEMMs 13 us per learner step in code size and registers).
//   EPK_F32   plain f32 output (split-K partials, weight gradients, LSTM projections), optional
//             transposed store (col_stride); no bias / activation / mask / column sums.
enum { EPK_GEN = 0, EPK_FWD = 1, EPK_DGRAD = 2, EPK_HEADS = 3, EPK_F32 = 4 };

// element offset of column n (the column map; n is warp-uniform)
BP_DEVICE long long col_offset(const GemmArgs& g, int n) {
  const uint32_t qd = fdivu((uint32_t)n, g.fd_cdiv), q1 = fdivu(qd, g.fd_cq);
  return (long long)q1 * g.cs1 + (long long)(qd - q1 * (uint32_t)g.cq) * g.cs2 + (long long)((uint32_t)n - qd * (uint32_t)g.cdiv);
}

// one row x 32 consecutive columns of the tile (called by all 32 lanes of an epilogue warp)
// roff: this lane's row offset (row map + split; -1: row not stored); sro[k]: roff of row
// 8k + lane/4 (the rows this lane writes in the staged store); mkw: the prefetched relu-mask
// word of this row chunk (when g.mask_bits); csum_acc: per-CTA running column sum for this
// lane's column (null: per-tile partial rows)
template <int EK>
BP_DEVICE void epilogue_chunk(const GemmArgs& g, long long roff, const long long (&sro)[4], int m, int n0,
                              int mt, int ew, int lane, float (&v)[32], uint32_t mkw, float* csum_acc,
                              uint32_t ostage) {
  if (n0 >= g.N) return;  // a partial last column tile (warp-uniform)
  const bool row_ok = roff >= 0;
  constexpr bool GEN = EK == EPK_GEN;
  constexpr bool F32 = EK == EPK_F32;
  if ((GEN || EK == EPK_HEADS) && g.heads) {
    if (row_ok) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {  // compile-time indices keep v[] in registers
        if (n0 + j < g.A) g.logits[(size_t)m * g.A + n0 + j] = v[j];
        else if (n0 + j == g.A) g.baseline[m] = v[j];
      }
      // fused sampling: the whole row (A + 1 <= 32 columns) is in this thread's registers
      if constexpr (EK == EPK_HEADS) {
        if (g.actions && n0 == 0)
          g.actions[m] = gumbel_argmax<32>(v, g.A, g.seed_state ? *g.seed_state : g.sample_seed,
                                           (unsigned long long)m, g.greedy != 0);
      }
    }
    return;
  }
  if (EK == EPK_FWD || (GEN && g.bias)) {  // alpha * acc + bias; the 32 bias values as 8 broadcast 16-byte loads
    const float4* b4 = reinterpret_cast<const float4*>(g.bias + n0);
    const float al = g.alpha;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = __ldg(b4 + q);
      v[4 * q] = fmaf(v[4 * q], al, b.x);
      v[4 * q + 1] = fmaf(v[4 * q + 1], al, b.y);
      v[4 * q + 2] = fmaf(v[4 * q + 2], al, b.z);
      v[4 * q + 3] = fmaf(v[4 * q + 3], al, b.w);
    }
  } else if (GEN && g.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= g.alpha;
  }
  if (EK == EPK_FWD || (GEN && g.relu)) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
  }
  if (EK == EPK_DGRAD || (GEN && g.mask_bits)) {  // (mkw is 0 for rows outside the grid)
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!((mkw >> i) & 1u)) v[i] = 0.f;
  }
  const long long coff = col_offset(g, n0);
  if (row_ok) {
    const long long off = roff + coff;
    if (EK != EPK_DGRAD && !F32 && g.bits_out) {
      uint32_t bits = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i) bits |= (v[i] > 0.f ? 1u : 0u) << i;
      g.bits_out[off >> 5] = bits;
    }
    if ((F32 || (GEN && g.out_f32)) && g.col_stride) {  // transposed store: per column, the warp's 32 rows are contiguous
      float* o = reinterpret_cast<float*>(g.out) + off;
#pragma unroll
      for (int i = 0; i < 32; ++i) o[(long long)i * g.col_stride] = v[i];
    } else if (F32 || (GEN && g.out_f32)) {
      float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(g.out) + off);
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  if (!F32 && (!GEN || !g.out_f32)) {
    // bf16 rows through a per-warp 2 KB staging buffer: every lane writes its 64-byte row chunk
    // (16-byte pieces XOR-swizzled by row pair: conflict-free), then each store instruction
    // writes 8 rows x 64 contiguous bytes (4 lanes per row) instead of 32 scattered 16-byte
    // pieces -- full sectors and 4x fewer L1 -> L2 write transactions
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(ostage + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)),
                   "r"(pack_bf16x2(v[8 * q], v[8 * q + 1])), "r"(pack_bf16x2(v[8 * q + 2], v[8 * q + 3])),
                   "r"(pack_bf16x2(v[8 * q + 4], v[8 * q + 5])), "r"(pack_bf16x2(v[8 * q + 6], v[8 * q + 7]))
                   : "memory");
    __syncwarp();
    char* outb = reinterpret_cast<char*>(g.out) + coff * 2;
    const int sub = lane & 3;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int row = k * 8 + (lane >> 2);
      uint32_t a, b, c, d;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                   : "r"(ostage + row * 64 + ((sub ^ ((row >> 1) & 3)) << 4)));
      if (sro[k] >= 0) *reinterpret_cast<uint4*>(outb + sro[k] * 2 + sub * 16) = make_uint4(a, b, c, d);
    }
    __syncwarp();  // the buffer is reused by the next chunk
  }
  if (EK != EPK_FWD && !F32 && g.colsum) {  // warp-uniform branch
    if (!row_ok) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    const float sum = warp_transpose_sum(v, lane);
    if (csum_acc) *csum_acc += sum;
    else g.colsum[(size_t)(mt * 4 + ew) * g.N + n0 + lane] = sum;
  }
}

// two u8 (bytes k, k+1 of w) -> packed bf16x2, exact: 0x4B0000bb as f32 is 2^23 + b; the two
// subtractions are one packed f32x2 add (FADD2)
BP_DEVICE uint32_t u8pair_bf16x2(uint32_t w, int k) {
  const uint32_t m0 = __byte_perm(w, 0x4B000000u, 0x7540u + k);
  const uint32_t m1 = __byte_perm(w, 0x4B000000u, 0x7540u + k + 1);
  uint32_t f0, f1;
  asm("{\n.reg .b64 a, c, d;\n"
      "mov.b64 a, {%2, %3};\n"
      "mov.b64 c, {%4, %4};\n"
      "add.rn.f32x2 d, a, c;\n"
      "mov.b64 {%0, %1}, d;\n}\n"
      : "=r"(f0), "=r"(f1)
      : "r"(m0), "r"(m1), "r"(0xCB000000u));  // -2^23
  return __byte_perm(f0, f1, 0x7632u);
}

// u8 plane of (img, ci) (AU8 frame source)
template <class Args>
BP_DEVICE const uint8_t* u8_plane(const Args& g, long long img, int ci) {
  long long p = img * 4 + ci;
  if (g.u8_index) {
    const int q = __ldg(g.u8_index + p);
    p = q < 0 ? 0 : q >= g.u8_planes ? g.u8_planes - 1 : q;
  }
  return g.u8 + p * 7056;
}

// AU8 producer (one warp): bulk-copy the frame lines behind grid rows [r0, r0 + nrows) into
// a raw stage laid out [ci][grid row - G0][336 B]; lanes 0..7 each copy one (image, ci) span.
template <class Args>
BP_DEVICE void u8_stage_issue(const Args& g, long long r0, int nrows, uint8_t* raw, uint64_t* bar, int lane) {
  const long long gmax = g.u8_rows / 21 - 1;  // last global grid row (img*21 + gy)
  const long long G0 = r0 / 21;
  long long G1 = (r0 + nrows - 1) / 21;
  G1 = G1 > gmax ? gmax : G1;
  // image segments: [G0, Gm] in image G0/21, [Gm+1, G1] in the next one
  const long long img0 = G0 / 21;
  const long long Gm = G1 < img0 * 21 + 20 ? G1 : img0 * 21 + 20;
  const uint32_t bytes0 = (uint32_t)(Gm - G0 + 1) * kRawRowBytes;
  const uint32_t bytes1 = G1 > Gm ? (uint32_t)(G1 - Gm) * kRawRowBytes : 0u;
  if (lane == 0) sm100::mbar_arrive_expect_tx(bar, 4 * (bytes0 + bytes1));
  __syncwarp();
  if (lane < 8) {
    const int ci = lane & 3, seg = lane >> 2;
    const uint32_t bytes = seg ? bytes1 : bytes0;
    if (bytes) {
      const long long img = img0 + seg;
      const int gy = seg ? 0 : (int)(G0 - img0 * 21);
      const uint8_t* src = u8_plane(g, img, ci) + gy * kRawRowBytes;
      uint8_t* dst = raw + ci * kRawCiBytes + (seg ? (uint32_t)(Gm - G0 + 1) * kRawRowBytes : 0u);
      bulk_g2s(dst, src, bytes, bar);
    }
  }
  __syncwarp();
}

// AU8 converters (kConvWarps warps, thread c): raw stage -> bf16 grid rows [r0, r0 + nrows)
// in the 128B-swizzled K-major layout (row rr at rr * 128, 16-byte chunk j at j ^ (rr & 7)).
// Explicit shared-space loads / stores (the stage pointers are generic).
BP_DEVICE uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}
// an opaque copy of a value, produced after the preceding (volatile) mbarrier wait, so that
// non-volatile loads addressed through it cannot be hoisted above the wait
BP_DEVICE uint32_t after_wait(uint32_t v) {
  uint32_t o;
  asm volatile("mov.b32 %0, %1;\n" : "=r"(o) : "r"(v) : "memory");
  return o;
}
BP_DEVICE void sts_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

template <class Args, int CW = kConvWarps>
BP_DEVICE void u8_stage_convert(const Args& g, long long r0, int nrows, const uint8_t* raw, uint8_t* a, int c,
                                 int own_rows) {
  constexpr int RSTEP = CW * 4;                        // rows per pass (8 chunks per row)
  constexpr int NIT = (160 + RSTEP - 1) / RSTEP;       // window rows <= 160
  // 32-bit grid-row arithmetic (grid rows < 2^31)
  const uint32_t r0u = (uint32_t)r0;
  const int x0 = (int)(r0u - fdivu(r0u, FDiv{0x86186187u, 5u}) * 21u);  // r0 % 21 (r0 < 2^31)
  const long long left = g.u8_rows - r0;
  const int valid = left < nrows ? (int)left : nrows;    // rows past the tensor -> 0
  const uint32_t sraw = after_wait(sm100::smem_addr(raw)), sa = sm100::smem_addr(a);
  const int j = c & 7;  // fixed chunk per thread
  const uint32_t cbase = sraw + (j >> 1) * kRawCiBytes + (j & 1) * 2 * 84;
  const int rr0 = c >> 3;
  // all loads of this thread's rows first (independent), then convert + store
  uint32_t w0[NIT], w1[NIT];
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int rr = rr0 + it * RSTEP;
    w0[it] = w1[it] = 0u;
    if (rr < valid) {
      const int q = x0 + rr;          // 32-bit: grid row offset G - G0 = q / 21, gx = q % 21
      const int gs = q / 21;
      const uint32_t src = cbase + gs * kRawRowBytes + 4 * (q - gs * 21);
      w0[it] = lds_u32(src);
      w1[it] = lds_u32(src + 84);
    }
  }
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int rr = rr0 + it * RSTEP;
    if (rr < nrows) {
      const uint4 v = make_uint4(u8pair_bf16x2(w0[it], 0), u8pair_bf16x2(w0[it], 2), u8pair_bf16x2(w1[it], 0),
                                 u8pair_bf16x2(w1[it], 2));
      sts_v4(sa + rr * 128 + ((j ^ (rr & 7)) << 4), v.x, v.y, v.z, v.w);
      // the tile's own rows (not the window halo) also to HBM: 128 B per row, coalesced
      if (g.u8_x0_out && rr < own_rows && rr < valid)
        __stcs(reinterpret_cast<uint4*>(g.u8_x0_out + (r0 + rr) * 64) + j, v);
    }
  }
}

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16: A (M = 128 rows = TMEM lanes, K along columns,
// two bf16 per 32-bit column) read from tensor memory
BP_DEVICE void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread i of the warp writes lane (base + i)
BP_DEVICE void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
BP_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// AU8 == 2 converter warp (quadrant q = TMEM lanes [32q, 32q + 32), half h = taps 2h, 2h + 1):
// the im2col row of tile row rr = 32q + lane for those taps -- 64 channels of window row
// rr + off_tap each -- converted from the raw stage and stored to the TMEM A buffer at
// column a_col + 32 tap.  Tap 0 is the tile's own row: it also goes to HBM as X0 (optional).
template <class Args>
BP_DEVICE void u8_im2col_tmem(const Args& g, long long r0, const uint8_t* raw, uint32_t tmem_a, int q, int h,
                              int lane) {
  const uint32_t r0u = (uint32_t)r0;
  const int x0 = (int)(r0u - fdivu(r0u, FDiv{0x86186187u, 5u}) * 21u);  // r0 % 21 (r0 < 2^31)
  const long long left = g.u8_rows - r0;
  const int rr = q * 32 + lane;
  const uint32_t sraw = after_wait(sm100::smem_addr(raw));
#pragma unroll
  for (int tt = 0; tt < 2; ++tt) {
    const int t = 2 * h + tt;
    const int wr = rr + g.a_row_off[t];
    uint32_t v[32];
    if (wr < left) {
      const int qq = x0 + wr;
      const int gs = qq / 21;
      const uint32_t base = sraw + gs * kRawRowBytes + 4 * (qq - gs * 21);
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) w[k] = lds_u32(base + (k >> 2) * kRawCiBytes + (k & 3) * 84);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        v[2 * k] = u8pair_bf16x2(w[k], 0);
        v[2 * k + 1] = u8pair_bf16x2(w[k], 2);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = 0u;
    }
    tmem_st_32x32b_x32(tmem_a + ((uint32_t)(q * 32) << 16) + (uint32_t)(t * 32), v);
    if (t == 0 && g.u8_x0_out && rr < left) {
      uint4* o = reinterpret_cast<uint4*>(g.u8_x0_out + (r0 + rr) * 64);
#pragma unroll
      for (int k = 0; k < 8; ++k) __stcs(o + k, make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
    }
  }
  tmem_st_wait();
}

template <int BN, int AM, int BM, int BSWZ, bool BRES = false, int AW = 0, int AU8 = 0, int EK = EPK_GEN>
__global__ void __launch_bounds__(GemmCfg<BN, AM, BM, BSWZ, BRES, AW, AU8>::THREADS, 1)
    umma_gemm_kernel(const __grid_constant__ GemmArgs g, const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB) {
  using C = GemmCfg<BN, AM, BM, BSWZ, BRES, AW, AU8>;
  static_assert(AW == 0 || (BRES && AM == A_KMAJOR), "window mode: K-major A with resident B");
  static_assert(AU8 == 0 || AW > 0, "u8 A operand: window mode (conv1 forward)");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bres = smem;                // resident B (BRES): K-block kb at kb * B_BYTES
  uint8_t* rawr = smem + C::B_RES;     // AU8 raw u8 stages
  uint8_t* ring = rawr + C::RAW;       // pipeline stages
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + C::ACC;
  uint64_t* bfull = tempty + C::ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  float* csum_smem = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bfull) + 64);  // [4 * EPI][BN]
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(csum_smem + 4 * C::EPI * BN);        // AU8
  uint64_t* raw_empty = raw_full + kRawStages;
  uint8_t* ostage_base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw_empty + kRawStages) + 127) &
                                                    ~uintptr_t(127));  // [4 * EPI][2048] bf16 staging

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      sm100::mbar_init(&full[s], AU8 ? kConvWarps : 1);  // AU8: one arrival per converter warp
      sm100::mbar_init(&empty[s], 1);
    }
    if constexpr (AU8 > 0) {
      for (int s = 0; s < kRawStages; ++s) {
        sm100::mbar_init(&raw_full[s], 1);
        sm100::mbar_init(&raw_empty[s], kConvWarps);
      }
    }
    for (int i = 0; i < C::ACC; ++i) {
      sm100::mbar_init(&tfull[i], 1);
      sm100::mbar_init(&tempty[i], 4);
    }
    sm100::mbar_init(bfull, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc(tmem_slot, C::TMEM_COLS);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!g.pdl_late) pdl_wait();  // the previous kernel's outputs (every global read below)

  const int ntiles = g.m_tiles * g.n_tiles * g.splits;
  // Warps 0 (TMA producer) and 1 (MMA issuer) run their loops converged with
  // warp-uniform state (uniform datapath, no per-lane divergence); one elected lane
  // issues each TMA / tcgen05.mma.
  if (warp == 0) {
    if constexpr (BRES) {  // the whole B, once
      if ((int)blockIdx.x < ntiles && sm100::elect_one()) {
        sm100::mbar_arrive_expect_tx(bfull, C::B_BYTES * g.num_kb);
        for (int kb = 0; kb < g.num_kb; ++kb)
          load_b<BN, BM, BSWZ>(g, &tmB, 0, kb, bres + kb * C::B_BYTES, bfull);
      }
      __syncwarp();
    }
    int stage = 0;
    uint32_t phase = 0;
    int ti = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      int mt, nt, sp;
      tile_coords(g, tile, mt, nt, sp);
      const int kb0 = sp * g.kb_per_split;
      const int kb1 = min(g.num_kb, kb0 + g.kb_per_split);
      if (lane == 0) trace_ev(g, ti, 0);
      if constexpr (AU8 > 0) {  // raw frame lines of the window -> raw stage (converters build A)
        sm100::mbar_wait(&raw_empty[stage], phase ^ 1);
        u8_stage_issue(g, (long long)mt * 128 + g.a_min_off, g.a_win_rows, rawr + stage * kRawBytes,
                       &raw_full[stage], lane);
        if (++stage == kRawStages) { stage = 0; phase ^= 1; }
      } else if constexpr (AW > 0) {  // one window per channel block feeds all taps
        for (int cb = 0; cb < g.a_cb; ++cb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (sm100::elect_one()) {
            sm100::mbar_arrive_expect_tx(&full[stage], g.a_win_rows * 128);
            sm100::tma_load_2d(ring + stage * C::STAGE, &tmA, &full[stage], cb * 64, mt * 128 + g.a_min_off);
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      } else {
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (sm100::elect_one()) {
            sm100::mbar_arrive_expect_tx(&full[stage], C::STAGE);
            uint8_t* sa = ring + stage * C::STAGE;
            load_a<AM>(g, &tmA, mt, kb, sa, &full[stage]);
            if constexpr (!BRES) load_b<BN, BM, BSWZ>(g, &tmB, nt, kb, sa + C::A_BYTES, &full[stage]);
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (lane == 0) trace_ev(g, ti, 1);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = sm100::idesc_bf16(128, BN, AM == A_MNMAJOR, BM == B_MNMAJOR);
    if constexpr (BRES) {
      if ((int)blockIdx.x < ntiles) sm100::mbar_wait(bfull, 0);
    }
    // constant high words of the shared-memory descriptors; only the start address varies
    const uint64_t a_hi = sm100::smem_desc(0, AM == A_KMAJOR ? 16 : 8192, 1024, sm100::SWZ_128B);
    const uint64_t b_hi = BM == B_KMAJOR ? sm100::smem_desc(0, 16, 1024, sm100::SWZ_128B)
                          : BSWZ == 64   ? sm100::smem_desc(0, 16, 512, sm100::SWZ_64B)
                                         : sm100::smem_desc(0, 8192, 1024, sm100::SWZ_128B);
    constexpr uint32_t a_kstep = AM == A_KMAJOR ? 32 : 2048;
    constexpr uint32_t b_kstep = BM == B_KMAJOR ? 32 : (BSWZ == 64 ? 1024 : 2048);
    int stage = 0, acc = 0;
    uint32_t phase = 0, aphase = 0;
    int ti = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      int mt, nt, sp;
      tile_coords(g, tile, mt, nt, sp);
      const int kb0 = sp * g.kb_per_split;
      const int kb1 = min(g.num_kb, kb0 + g.kb_per_split);
      sm100::mbar_wait(&tempty[acc], aphase ^ 1);
      sm100::tc_fence_after();
      if (lane == 0) trace_ev(g, ti, 2);
      const uint32_t d = tmem_base + acc * BN;
      if constexpr (AU8 == 2) {  // A = the im2col buffer in TMEM, B = the resident weights
        sm100::mbar_wait(&full[stage], phase);
        sm100::tc_fence_after();
        const uint32_t ta = tmem_base + C::A_TMEM + (uint32_t)stage * 128u;
        if (sm100::elect_one()) {
          for (int t = 0; t < g.a_ntaps; ++t) {
            const uint32_t sb = sm100::smem_addr(bres + t * C::B_BYTES);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16_ts(d, ta + (uint32_t)(t * 32 + k * 8), b_hi | ((sb + k * b_kstep) >> 4), idesc,
                          (t > 0 || k > 0) ? 1u : 0u);
          }
          sm100::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      } else if constexpr (AW > 0) {
        for (int cb = 0; cb < g.a_cb; ++cb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sw = sm100::smem_addr(ring + stage * C::STAGE);
          if (sm100::elect_one()) {
            for (int t = 0; t < g.a_ntaps; ++t) {
              const uint32_t sa = sw + (uint32_t)(g.a_row_off[t] - g.a_min_off) * 128u;
              const uint32_t sb = sm100::smem_addr(bres + (t * g.a_cb + cb) * C::B_BYTES);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                sm100::umma_f16(d, a_hi | ((sa + k * a_kstep) >> 4), b_hi | ((sb + k * b_kstep) >> 4), idesc,
                                (cb > 0 || t > 0 || k > 0) ? 1u : 0u);
            }
            sm100::umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      } else {
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_addr(ring + stage * C::STAGE);
          const uint32_t sb = BRES ? sm100::smem_addr(bres + kb * C::B_BYTES) : sa + C::A_BYTES;
          if (sm100::elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              sm100::umma_f16(d, a_hi | ((sa + k * a_kstep) >> 4), b_hi | ((sb + k * b_kstep) >> 4), idesc,
                              (kb > kb0 || k > 0) ? 1u : 0u);
            sm100::umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (sm100::elect_one()) sm100::umma_commit(&tfull[acc]);
      __syncwarp();
      if (lane == 0) trace_ev(g, ti, 3);
      if (++acc == C::ACC) { acc = 0; aphase ^= 1; }
    }
    pdl_trigger();  // every MMA of this CTA issued: the next kernel may start launching
  } else if (AU8 > 0 && warp >= C::CONV_WARP0) {
    // converters: raw stage -> swizzled bf16 window in the A ring (one tile per stage)
    const int c = threadIdx.x - 32 * C::CONV_WARP0;
    int rs = 0, stage = 0;
    uint32_t rph = 0, phase = 0;
    int ti = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      int mt, nt, sp;
      tile_coords(g, tile, mt, nt, sp);
      sm100::mbar_wait(&raw_full[rs], rph);
      sm100::mbar_wait(&empty[stage], phase ^ 1);
      if (c == 0) trace_ev(g, ti, 6);
      if constexpr (AU8 == 2) {
        sm100::tc_fence_after();
        const int cw = warp - C::CONV_WARP0;
        u8_im2col_tmem(g, (long long)mt * 128, rawr + rs * kRawBytes,
                       tmem_base + C::A_TMEM + (uint32_t)stage * 128u, warp & 3, cw >> 2, threadIdx.x & 31);
        sm100::tc_fence_before();  // tcgen05.st -> the MMA warp's reads, ordered by the barrier
      } else {
        u8_stage_convert(g, (long long)mt * 128 + g.a_min_off, g.a_win_rows, rawr + rs * kRawBytes,
                         ring + stage * C::STAGE, c, 128 - g.a_min_off);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> UMMA reads
      }
      if (c == 0) trace_ev(g, ti, 8);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        sm100::mbar_arrive(&full[stage]);
        sm100::mbar_arrive(&raw_empty[rs]);
      }
      if (c == 0) trace_ev(g, ti, 7);
      if (++rs == kRawStages) { rs = 0; rph ^= 1; }
      if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 3 && g.prep.n > 0) {
    if (blockIdx.x == 0 && lane == 0 && g.prep.seed_state) advance_seed_dev(g.prep.seed_state);
    prep_items(g.prep, (long long)blockIdx.x * 32 + lane, (long long)gridDim.x * 32);
  } else if (warp >= 4 && warp < 4 + 4 * C::EPI) {
    // epilogue warpgroup grp takes the CTA's tiles k = grp, grp + EPI, ... (accumulator k % ACC);
    // warp ew of a group reads TMEM lanes [32 ew, 32 ew + 32)
    const int grp = (warp - 4) >> 2, ew = (warp - 4) & 3;
    constexpr int NCH = BN / 32;
    const uint32_t ostage = sm100::smem_addr(ostage_base + (warp - 4) * 2048);
    // bias-gradient column sums: accumulated per CTA (per epilogue warp, in shared memory)
    // when every tile covers the same columns; otherwise written per tile
    const bool cta_colsum = EK != EPK_FWD && g.colsum && g.n_tiles == 1 && g.splits == 1;
    float* csum = csum_smem + (grp * 4 + ew) * BN;
    if (cta_colsum) {
      for (int c = 0; c < NCH; ++c) csum[c * 32 + lane] = 0.f;
    }
    // row map + relu-mask words of a tile (the masks are prefetched one tile ahead: when the
    // epilogue is the bottleneck the accumulator is already waiting, so loads issued just
    // before the tfull wait would not be hidden)
    struct RowInfo {
      int m, mt, nt, sp;
      bool ok;
      long long rbase;
      uint32_t mk[4];
    };
    auto row_info = [&](int tile) {
      RowInfo ri;
      tile_coords(g, tile, ri.mt, ri.nt, ri.sp);
      ri.m = ri.mt * 128 + ew * 32 + lane;
      ri.ok = ri.m < g.M;
      {  // precomputed-multiplier divisions (m < 2^31)
        const uint32_t mu = (uint32_t)ri.m;
        const uint32_t img = fdivu(mu, g.fd_per);
        const uint32_t rem = mu - img * (uint32_t)(g.gh * g.gw);
        const uint32_t y = fdivu(rem, g.fd_gw);
        const uint32_t x = rem - y * (uint32_t)g.gw;
        const uint32_t ys = fdivu(y, g.fd_sy), xs = fdivu(x, g.fd_sx);
        ri.ok = ri.ok && ((int)y < g.vh) && ((int)x < g.vw);
        ri.rbase = (long long)img * g.r_img + (long long)ys * g.r_y + (long long)xs * g.r_x +
                   (long long)((y - ys * (uint32_t)g.sy) * (uint32_t)g.sx + (x - xs * (uint32_t)g.sx)) * g.r_sub;
      }
      ri.mk[0] = ri.mk[1] = ri.mk[2] = ri.mk[3] = 0u;
      if ((EK == EPK_DGRAD || (EK == EPK_GEN && g.mask_bits)) && ri.ok) {
        const uint32_t* mp = g.mask_bits + (((size_t)ri.m * (g.mask_ld ? g.mask_ld : g.N) + ri.nt * BN) >> 5);
        const int nc = ri.nt * BN;  // only the chunks inside N (a partial last column tile)
        // volatile: issued here, a tile ahead of use (a plain __ldg may be sunk to its use)
        ri.mk[0] = ldg_volatile(mp);
        if (NCH > 1 && nc + 32 < g.N) ri.mk[1] = ldg_volatile(mp + 1);
        if (NCH > 2 && nc + 64 < g.N) ri.mk[2] = ldg_volatile(mp + 2);
        if (NCH > 3 && nc + 96 < g.N) ri.mk[3] = ldg_volatile(mp + 3);
      }
      return ri;
    };
    const int tile_step = C::EPI * gridDim.x;
    RowInfo nxt{};
    if ((int)blockIdx.x + grp * (int)gridDim.x < ntiles) nxt = row_info(blockIdx.x + grp * gridDim.x);
    for (int ti = grp, tile = blockIdx.x + grp * gridDim.x; tile < ntiles; ti += C::EPI, tile += tile_step) {
      const int acc = ti % C::ACC;
      const uint32_t aphase = (uint32_t)(ti / C::ACC) & 1u;
      const RowInfo cur = nxt;
      if (tile + tile_step < ntiles) nxt = row_info(tile + tile_step);
      const int m = cur.m, mt = cur.mt, nt = cur.nt, sp = cur.sp;
      const uint32_t mk0 = cur.mk[0], mk1 = cur.mk[1], mk2 = cur.mk[2], mk3 = cur.mk[3];
      // this lane's row offset (-1: not stored) and those of the rows it writes in the staged
      // bf16 store (row 8k + lane/4), once per tile
      const long long roff = cur.ok ? cur.rbase + (long long)sp * g.split_stride : -1ll;
      long long sro[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) sro[k] = __shfl_sync(0xffffffffu, roff, k * 8 + (lane >> 2));
      sm100::mbar_wait(&tfull[acc], aphase);
      sm100::tc_fence_after();
      if (ew == 0 && lane == 0) trace_ev(g, ti, 4);
      const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(ew * 32) << 16);
      if ((sp * g.kb_per_split) >= g.num_kb) {  // an empty split-K range: no MMA wrote the accumulator
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = 0u;
        for (int c = 0; c < NCH; ++c) tmem_st_32x32b_x32(tbase + c * 32, z);
        tmem_st_wait();
      }
      if constexpr (NCH <= 2 && C::EPI <= 2) {
        // TMEM loads one chunk ahead: the load of chunk c + 1 is in flight while chunk c is
        // processed (tcgen05.wait::ld waits for all earlier loads, so it is issued right after).
        // (BN <= 64; for 4 chunks the extra 32 live registers cost more than the overlap gains)
        uint32_t rbuf[2][32];
        sm100::tmem_ld_32x32b_x32(tbase, rbuf[0]);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          sm100::tmem_ld_wait();
          if (c + 1 < NCH) sm100::tmem_ld_32x32b_x32(tbase + (c + 1) * 32, rbuf[(c + 1) & 1]);
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rbuf[c & 1][i]);
          epilogue_chunk<EK>(g, roff, sro, m, nt * BN + c * 32, mt, ew, lane, v, c == 0 ? mk0 : mk1,
                         cta_colsum ? &csum[c * 32 + lane] : nullptr, ostage);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          uint32_t r[32];
          sm100::tmem_ld_32x32b_x32(tbase + c * 32, r);
          sm100::tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          const uint32_t mkw = c == 0 ? mk0 : c == 1 ? mk1 : c == 2 ? mk2 : mk3;
          epilogue_chunk<EK>(g, roff, sro, m, nt * BN + c * 32, mt, ew, lane, v, mkw,
                         cta_colsum ? &csum[c * 32 + lane] : nullptr, ostage);
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (ew == 0 && lane == 0) trace_ev(g, ti, 5);
    }
    if (cta_colsum) {  // fixed-order combine of the groups' sums, one row per lane quadrant
      if constexpr (C::EPI > 1) asm volatile("bar.sync 2, %0;\n" ::"n"(128 * C::EPI) : "memory");
      if (grp == 0) {
        for (int c = 0; c < NCH; ++c) {
          float v = csum[c * 32 + lane];
          for (int q = 1; q < C::EPI; ++q) v += csum_smem[(q * 4 + ew) * BN + c * 32 + lane];
          g.colsum[(size_t)(blockIdx.x * 4 + ew) * g.N + c * 32 + lane] = v;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  if (g.pdl_late) pdl_wait();  // completion stays transitive for the kernels after this one
}

// ============================================================================
// Weight-gradient "window" GEMM (conv weight gradients):
//   D[m][n] = sum_rows X[row + off(m)][c(m)] * dY[row][n],  m = (tap, channel)
// reduced over grid rows in K-blocks of 64.  Per K-block the producer loads ONE window of
// X rows [kb*64 + min_off, kb*64 + 64 + max_off) per 64-channel block (plus the dY box), and
// every M atom (tap, channel block) of every m-tile is a view into it: an M=128 MMA covers
// atoms (2mt, 2mt+1) with the A descriptor at atom 2mt and LBO = address(2mt+1) - address(2mt)
// (MN-major, 128B swizzle on absolute smem addresses, like the forward window mode).  One
// CTA owns all NMT m-tiles of its K range (NMT accumulators in TMEM), so X and dY cross
// L2 -> SM once per K-block instead of once per (m-tile, tap).
// Output: f32 partials out[split][Mpad][N] (split = the CTA's K range), reduced by finalize.
// ============================================================================
struct WgArgs {
  int num_kb, kb_per_split, splits;
  int a_cb;                       // 64-channel blocks of X (window count per stage)
  int nshifts, atoms_per_shift;   // atom a -> tap a / atoms_per_shift, block a % atoms_per_shift
  int row_off[kMaxShifts];        // per-tap row offset (>= 0)
  int min_off, win_rows;          // window rows (multiple of 8)
  int Mpad, N;
  int ones_atom;  // atom index holding all ones (its D rows = column sums of dY: the bias
                  // gradient), -1 = none; atoms past the taps and the ones atom are zero
  float* out;
  // optional (BN == 32 / BSWZ == 64 or BN == 64 / BSWZ == 128): column sums of the CTA's dY
  // rows (the bias gradient),
  // colsum[blockIdx.x][BN], summed by the otherwise idle warp 3 from the staged dY boxes
  float* colsum;
  unsigned long long* trace;
  int trace_tiles;
  // AU8 (conv1): the X windows are converted on chip from u8 frames (see GemmArgs)
  const uint8_t* u8;
  const int32_t* u8_index;
  int u8_planes;
  long long u8_rows;
  __nv_bfloat16* u8_x0_out;  // (unused here)
};

// CB: 64-channel blocks of X (windows per stage); WR: window rows (multiple of 8), sized per
// conv so that the stage ring holds as many K-blocks in flight as shared memory allows
template <int BN, int BSWZ, int NMT, int AU8 = 0, int CB = 1, int WR = 88>
struct WgCfg {
  static_assert(WR % 8 == 0 && WR <= 160, "window rows");
  static constexpr uint32_t WIN_BYTES = WR * 128;   // one window per channel block
  static constexpr uint32_t B_BYTES = BN * 64 * 2;
  static constexpr int MAX_CB = CB;
  static constexpr uint32_t STAGE = MAX_CB * WIN_BYTES + B_BYTES;  // 1 KB multiple
  static constexpr uint32_t ZERO = 8192;                           // the all-zero atom
  static constexpr uint32_t ONES = 8192;                           // the all-ones atom
  static constexpr uint32_t RAW = AU8 ? kRawStages * kRawBytes : 0;
  static constexpr int THREADS = 256 + (AU8 ? 32 * kConvWarps : 0);
  static constexpr int STAGES = (200 * 1024 - ZERO - ONES - RAW) / STAGE > 12 ? 12 : (200 * 1024 - ZERO - ONES - RAW) / STAGE;
  static constexpr uint32_t TMEM_COLS = (NMT * BN <= 32) ? 32 : (NMT * BN <= 64) ? 64 : (NMT * BN <= 128) ? 128
                                        : (NMT * BN <= 256) ? 256 : 512;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + ZERO + ONES + RAW + 1024 + 512;
  static_assert(NMT * BN <= 512, "TMEM");
};

template <int BN, int BSWZ, int NMT, int AU8 = 0, int CB = 1, int WR = 88>
__global__ void __launch_bounds__(WgCfg<BN, BSWZ, NMT, AU8, CB, WR>::THREADS, 1)
    umma_wgrad_win_kernel(const __grid_constant__ WgArgs g, const __grid_constant__ CUtensorMap tmX,
                          const __grid_constant__ CUtensorMap tmY) {
  using C = WgCfg<BN, BSWZ, NMT, AU8, CB, WR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                           // stages: [windows | dY box]
  // fixed atoms above the ring, ones below zero, so every atom pair has LBO > 0
  uint8_t* ones = ring + C::STAGES * C::STAGE;    // all-ones atom (bf16 1.0)
  uint8_t* zero = ones + C::ONES;                 // all-zero atom
  uint8_t* rawr = zero + C::ZERO;                 // AU8 raw u8 stages
  uint64_t* full = reinterpret_cast<uint64_t*>(rawr + C::RAW);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  uint64_t* raw_full = tfull + 2;
  uint64_t* raw_empty = raw_full + kRawStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (int)(C::ZERO / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(zero)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int i = threadIdx.x; i < (int)(C::ONES / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(ones)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmX);
    sm100::tma_prefetch_desc(&tmY);
    for (int s = 0; s < C::STAGES; ++s) {
      sm100::mbar_init(&full[s], AU8 ? 1 + kConvWarps : 1);  // AU8: + one arrival per converter warp
      sm100::mbar_init(&empty[s], g.colsum ? 2 : 1);         // + the column-sum warp
    }
    sm100::mbar_init(tfull, 1);
    if constexpr (AU8 > 0) {
      for (int s = 0; s < kRawStages; ++s) {
        sm100::mbar_init(&raw_full[s], 1);
        sm100::mbar_init(&raw_empty[s], kConvWarps);
      }
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc(tmem_slot, C::TMEM_COLS);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the previous kernel's outputs (every global read below)
  const uint32_t stage_tx = (AU8 ? 0 : g.a_cb * g.win_rows * 128) + C::B_BYTES;

  if (warp == 0) {
    int stage = 0, rs = 0;
    uint32_t phase = 0, rph = 0;
    for (int sp = blockIdx.x; sp < g.splits; sp += gridDim.x) {
      const int kb0 = sp * g.kb_per_split, kb1 = min(g.num_kb, kb0 + g.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        if constexpr (AU8 > 0) {  // raw frame lines of the window (converters build it)
          sm100::mbar_wait(&raw_empty[rs], rph ^ 1);
          u8_stage_issue(g, (long long)kb * 64 + g.min_off, g.win_rows, rawr + rs * kRawBytes, &raw_full[rs], lane);
          if (++rs == kRawStages) { rs = 0; rph ^= 1; }
        }
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        if (sm100::elect_one()) {
          uint8_t* st = ring + stage * C::STAGE;
          sm100::mbar_arrive_expect_tx(&full[stage], stage_tx);
          if constexpr (AU8 == 0)
            for (int cb = 0; cb < g.a_cb; ++cb)
              sm100::tma_load_2d(st + cb * C::WIN_BYTES, &tmX, &full[stage], cb * 64, kb * 64 + g.min_off);
          uint8_t* sb = st + C::MAX_CB * C::WIN_BYTES;
          if constexpr (BSWZ == 64) {
            sm100::tma_load_2d(sb, &tmY, &full[stage], 0, kb * 64);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) sm100::tma_load_2d(sb + j * 8192, &tmY, &full[stage], j * 64, kb * 64);
          }
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = sm100::idesc_bf16(128, BN, true, true);
    const uint64_t b_hi = BSWZ == 64 ? sm100::smem_desc(0, 16, 512, sm100::SWZ_64B)
                                     : sm100::smem_desc(0, 8192, 1024, sm100::SWZ_128B);
    constexpr uint32_t b_kstep = BSWZ == 64 ? 1024 : 2048;
    // per m-tile: the two atoms' addresses.  Window atoms are stage-relative offsets; the
    // zero / ones atoms are fixed shared addresses above the ring (flag bit 31)
    constexpr uint32_t kFixed = 0x80000000u;
    uint32_t a0[NMT], a1[NMT];
    const uint32_t zero_addr = sm100::smem_addr(zero), ones_addr = sm100::smem_addr(ones);
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt) {
      uint32_t ad[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int atom = 2 * mt + j;
        const int sft = atom / g.atoms_per_shift, cb = atom - sft * g.atoms_per_shift;
        if (atom == g.ones_atom) ad[j] = kFixed | ones_addr;
        else if (sft >= g.nshifts) ad[j] = kFixed | zero_addr;
        else ad[j] = cb * C::WIN_BYTES + (uint32_t)(g.row_off[sft] - g.min_off) * 128u;
      }
      a0[mt] = ad[0];
      a1[mt] = ad[1];
    }
    // one K range (split) per CTA: grid == splits (single accumulator set)
    int stage = 0;
    uint32_t phase = 0;
    for (int sp = blockIdx.x; sp < g.splits; sp += gridDim.x) {
      const int kb0 = sp * g.kb_per_split, kb1 = min(g.num_kb, kb0 + g.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        sm100::tc_fence_after();
        const uint32_t st = sm100::smem_addr(ring + stage * C::STAGE);
        const uint32_t sb = st + C::MAX_CB * C::WIN_BYTES;
        if (sm100::elect_one()) {
#pragma unroll
          for (int mt = 0; mt < NMT; ++mt) {
            const uint32_t sa = (a0[mt] & kFixed) ? (a0[mt] & ~kFixed) : st + a0[mt];
            const uint32_t sb1 = (a1[mt] & kFixed) ? (a1[mt] & ~kFixed) : st + a1[mt];
            const uint32_t lbo = sb1 - sa;  // the second atom is above the first (checked on the host)
            const uint64_t a_hi = sm100::smem_desc(0, lbo, 1024, sm100::SWZ_128B);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              sm100::umma_f16(tmem_base + mt * BN, a_hi | ((sa + k * 2048) >> 4),
                              b_hi | ((sb + k * b_kstep) >> 4), idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          sm100::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (sm100::elect_one()) sm100::umma_commit(tfull);
      __syncwarp();
    }
    pdl_trigger();  // every MMA of this CTA issued: the next kernel may start launching
  } else if (AU8 > 0 && warp >= 8) {
    // converters: raw stage -> swizzled bf16 window of the stage (then one arrival per warp)
    const int c = threadIdx.x - 256;
    int stage = 0, rs = 0;
    uint32_t phase = 0, rph = 0;
    for (int sp = blockIdx.x; sp < g.splits; sp += gridDim.x) {
      const int kb0 = sp * g.kb_per_split, kb1 = min(g.num_kb, kb0 + g.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        sm100::mbar_wait(&raw_full[rs], rph);
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        u8_stage_convert(g, (long long)kb * 64 + g.min_off, g.win_rows, rawr + rs * kRawBytes,
                         ring + stage * C::STAGE, c, 0);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> UMMA reads
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          sm100::mbar_arrive(&full[stage]);
          sm100::mbar_arrive(&raw_empty[rs]);
        }
        if (++rs == kRawStages) { rs = 0; rph ^= 1; }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 3 && g.colsum) {
    // bias gradient: column sums of the dY boxes (64 rows x BN bf16; BN = 32: 64B-swizzled rows,
    // the 16-byte chunk j of row r at r * 64 + ((j ^ ((r >> 1) & 3)) << 4); BN = 64: 128B rows,
    // at r * 128 + ((j ^ (r & 7)) << 4)).  Lane l sums chunk j = l % CPR (channels 8j .. 8j + 7)
    // of rows l / CPR + RPI i, in f32
    constexpr int CPR = BN * 2 / 16, RPI = 32 / CPR, NI = 64 / RPI;
    static_assert((BN == 32 && BSWZ == 64) || (BN == 64 && BSWZ == 128), "column-sum warp layout");
    float cs[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) cs[i] = 0.f;
    const int j = lane % CPR, r0 = lane / CPR;
    int stage = 0;
    uint32_t phase = 0;
    for (int sp = blockIdx.x; sp < g.splits; sp += gridDim.x) {
      const int kb0 = sp * g.kb_per_split, kb1 = min(g.num_kb, kb0 + g.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        const uint32_t sb = after_wait(sm100::smem_addr(ring + stage * C::STAGE + C::MAX_CB * C::WIN_BYTES));
        uint32_t w[NI][4];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int r = r0 + RPI * i;
          const uint32_t a = BN == 32 ? sb + r * 64 + ((j ^ ((r >> 1) & 3)) << 4) : sb + r * 128 + ((j ^ (r & 7)) << 4);
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                       : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3])
                       : "r"(a));
        }
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&empty[stage]);
#pragma unroll
        for (int i = 0; i < NI; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            cs[2 * q] += __uint_as_float(w[i][q] << 16);
            cs[2 * q + 1] += __uint_as_float(w[i][q] & 0xFFFF0000u);
          }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
    // lanes with the same chunk j (l = j + CPR k): fixed-order butterfly over k
#pragma unroll
    for (int o = CPR; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < 8; ++i) cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], o);
    if (lane < CPR) {
#pragma unroll
      for (int i = 0; i < 8; ++i) g.colsum[(size_t)blockIdx.x * BN + 8 * j + i] = cs[i];
    }
  } else if (warp >= 4 && warp < 8) {
    const int ew = warp - 4;
    int ti = 0;
    for (int sp = blockIdx.x; sp < g.splits; sp += gridDim.x, ++ti) {
      const int kb0 = sp * g.kb_per_split;
      const bool has_k = kb0 < g.num_kb;
      if (has_k) {
        sm100::mbar_wait(tfull, ti & 1);
        sm100::tc_fence_after();
      }
#pragma unroll 1
      for (int mt = 0; mt < NMT; ++mt) {
        const int m = mt * 128 + ew * 32 + lane;
        float* orow = g.out + ((size_t)sp * g.Mpad + m) * g.N;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          if (has_k) {
            sm100::tmem_ld_32x32b_x32(tmem_base + mt * BN + c * 32 + ((uint32_t)(ew * 32) << 16), r);
            sm100::tmem_ld_wait();
          }
          float4* o = reinterpret_cast<float4*>(orow + c * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            o[q] = has_k ? make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                       __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      sm100::tc_fence_before();
    }
  }
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace bp
