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

struct GemmArgs {
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
  // optional per-tile timeline (test builds): trace[(blockIdx.x * trace_tiles + i) * 8 + event]
  unsigned long long* trace;
  int trace_tiles;
  // AtariNet heads epilogue (heads != 0): column j < A -> logits[m][j], j == A -> baseline[m]
  int heads, A;
  float* logits;   // [M][A] f32
  float* baseline; // [M] f32
};

// BRES ("B resident", weight-stationary): every tile of the launch shares one B
// (n_tiles == 1, splits == 1) whose K-blocks fit in kBResBytes of shared memory; it
// is loaded once per CTA and only A streams through the pipeline, halving L2 traffic
// for the conv GEMMs (B = the conv weights, A = the activation grid).
constexpr uint32_t kBResBytes = 96 * 1024;

constexpr uint32_t kWinBytes = 20 * 1024;  // window stage: up to 160 rows x 128 B

template <int BN, int AM, int BM, int BSWZ, bool BRES = false, int AW = 0>
struct GemmCfg {
  static constexpr uint32_t A_BYTES = AW ? kWinBytes : 128 * 64 * 2;
  static constexpr uint32_t B_BYTES = BN * 64 * 2;
  static constexpr uint32_t STAGE = BRES ? A_BYTES : A_BYTES + B_BYTES;
  static constexpr uint32_t B_RES = BRES ? kBResBytes : 0;
  static constexpr int STAGES = (200 * 1024 - B_RES) / STAGE > 8 ? 8 : (200 * 1024 - B_RES) / STAGE;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr size_t SMEM = (size_t)B_RES + (size_t)STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/ +
                                 4 * BN * sizeof(float) /*column sums*/;
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  static_assert(BM == B_KMAJOR || BSWZ == 128 || (BSWZ == 64 && BN == 32), "B swizzle");
};

BP_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
BP_DEVICE void trace_ev(const GemmArgs& g, int i, int ev) {
  if (g.trace && i < g.trace_tiles) g.trace[((size_t)blockIdx.x * g.trace_tiles + i) * 8 + ev] = gtimer();
}

BP_DEVICE void tile_coords(const GemmArgs& g, int tile, int& mt, int& nt, int& sp) {
  sp = tile % g.splits;
  const int r = tile / g.splits;
  nt = r % g.n_tiles;
  mt = r / g.n_tiles;
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

// one row x 32 consecutive columns of the tile (called by all 32 lanes of an epilogue warp)
// mkw: the prefetched relu-mask word of this row chunk (when g.mask_bits);
// csum_acc: per-CTA running column sum for this lane's column (null: per-tile partial rows)
BP_DEVICE void epilogue_chunk(const GemmArgs& g, long long rbase, bool row_ok, int m, int n0,
                              int sp, int mt, int ew, int lane, float (&v)[32], uint32_t mkw,
                              float* csum_acc) {
  if (g.heads) {
    if (row_ok) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {  // compile-time indices keep v[] in registers
        if (n0 + j < g.A) g.logits[(size_t)m * g.A + n0 + j] = v[j];
        else if (n0 + j == g.A) g.baseline[m] = v[j];
      }
    }
    return;
  }
  if (g.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= g.alpha;
  }
  if (g.bias) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += __ldg(g.bias + n0 + i);
  }
  if (g.relu) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
  }
  if (g.mask_bits && row_ok) {
    const uint32_t w = mkw;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!((w >> i) & 1u)) v[i] = 0.f;
  }
  if (row_ok) {
    const int qd = n0 / g.cdiv;
    const long long cbase = (long long)(qd / g.cq) * g.cs1 + (long long)(qd % g.cq) * g.cs2 + (n0 % g.cdiv);
    const long long off = rbase + cbase + (long long)sp * g.split_stride;
    if (g.bits_out) {
      uint32_t bits = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i) bits |= (v[i] > 0.f ? 1u : 0u) << i;
      g.bits_out[off >> 5] = bits;
    }
    if (g.out_f32) {
      float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(g.out) + off);
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
      uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(g.out) + off);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        o[q] = make_uint4(pack_bf16x2(v[8 * q], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                          pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
    }
  }
  if (g.colsum) {  // warp-uniform branch
    if (!row_ok) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    const float sum = warp_transpose_sum(v, lane);
    if (csum_acc) *csum_acc += sum;
    else g.colsum[(size_t)(mt * 4 + ew) * g.N + n0 + lane] = sum;
  }
}

template <int BN, int AM, int BM, int BSWZ, bool BRES = false, int AW = 0>
__global__ void __launch_bounds__(kGemmThreads, 1)
    umma_gemm_kernel(const __grid_constant__ GemmArgs g, const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB) {
  using C = GemmCfg<BN, AM, BM, BSWZ, BRES, AW>;
  static_assert(AW == 0 || (BRES && AM == A_KMAJOR), "window mode: K-major A with resident B");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bres = smem;                // resident B (BRES): K-block kb at kb * B_BYTES
  uint8_t* ring = smem + C::B_RES;     // pipeline stages
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  float* csum_smem = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bfull) + 64);  // [4][BN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
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
      if constexpr (AW > 0) {  // one window per channel block feeds all taps
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
      if constexpr (AW > 0) {
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
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    constexpr int NCH = BN / 32;
    int acc = 0;
    uint32_t aphase = 0;
    // bias-gradient column sums: accumulated per CTA (per epilogue warp, in shared memory)
    // when every tile covers the same columns; otherwise written per tile
    const bool cta_colsum = g.colsum && g.n_tiles == 1 && g.splits == 1;
    float* csum = csum_smem + ew * BN;
    if (cta_colsum) {
      for (int c = 0; c < NCH; ++c) csum[c * 32 + lane] = 0.f;
    }
    int ti = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      int mt, nt, sp;
      tile_coords(g, tile, mt, nt, sp);
      const int m = mt * 128 + ew * 32 + lane;
      // row map
      bool row_ok = m < g.M;
      long long rbase = 0;
      {
        const int per = g.gh * g.gw;
        const int img = m / per;
        const int rem = m - img * per;
        const int y = rem / g.gw;
        const int x = rem - y * g.gw;
        row_ok = row_ok && (y < g.vh) && (x < g.vw);
        rbase = (long long)img * g.r_img + (long long)(y / g.sy) * g.r_y + (long long)(x / g.sx) * g.r_x +
                (long long)((y % g.sy) * g.sx + (x % g.sx)) * g.r_sub;
      }
      // prefetch the tile's relu-mask words (one u32 per 32 columns) before waiting for the
      // accumulator, so their latency overlaps the MMAs (masked GEMMs have BN <= 128)
      uint32_t mk0 = 0, mk1 = 0, mk2 = 0, mk3 = 0;
      if (g.mask_bits && row_ok) {
        const uint32_t* mp = g.mask_bits + (((size_t)m * (g.mask_ld ? g.mask_ld : g.N) + nt * BN) >> 5);
        mk0 = __ldg(mp);
        if (NCH > 1) mk1 = __ldg(mp + 1);
        if (NCH > 2) mk2 = __ldg(mp + 2);
        if (NCH > 3) mk3 = __ldg(mp + 3);
      }
      sm100::mbar_wait(&tfull[acc], aphase);
      sm100::tc_fence_after();
      if (ew == 0 && lane == 0) trace_ev(g, ti, 4);
      const bool has_k = (sp * g.kb_per_split) < g.num_kb;
#pragma unroll 1
      for (int c = 0; c < NCH; ++c) {
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(tmem_base + acc * BN + c * 32 + ((uint32_t)(ew * 32) << 16), r);
        sm100::tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = has_k ? __uint_as_float(r[i]) : 0.f;
        const uint32_t mkw = c == 0 ? mk0 : c == 1 ? mk1 : c == 2 ? mk2 : mk3;
        epilogue_chunk(g, rbase, row_ok, m, nt * BN + c * 32, sp, mt, ew, lane, v, mkw,
                       cta_colsum ? &csum[c * 32 + lane] : nullptr);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (ew == 0 && lane == 0) trace_ev(g, ti, 5);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (cta_colsum) {
      __syncwarp();
      for (int c = 0; c < NCH; ++c)
        g.colsum[(size_t)(blockIdx.x * 4 + ew) * g.N + c * 32 + lane] = csum[c * 32 + lane];
    }
  }
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace bp
