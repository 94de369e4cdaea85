// AtariNet (TorchBeast monobeast.AtariNet, no-LSTM path) forward + backward on sm_100a.
//
// Replaces the reference network seam mlp_forward_backward (model.py:176-203)
// with the north-star AtariNet: conv 8x8/4 -> 32, 4x4/2 -> 64, 3x3/1 -> 64,
// FC 3136 -> 512, core = [relu(fc), clip(r), onehot(last_action)], policy /
// baseline heads.  All dense contractions run on the tcgen05 GEMM engine
// (umma_gemm.cuh) with bf16 operands and f32 TMEM accumulation.
//
// Convolutions are "shifted GEMMs" on row-major NHWC grids, no im2col:
//   conv1: frames (u8, 4x84x84) -> space-to-depth by 4 -> X0 [N*21*21, 64] bf16
//          = a 2x2 stride-1 conv on a 21x21 grid (K = 4 taps x 64 = 256)
//   conv2: conv1 output written by conv1's epilogue directly in space-to-depth-2
//          layout X1 [N*10*10, 128] = a 2x2 stride-1 conv (K = 4 x 128 = 512)
//   conv3: X2 [N*9*9, 64], 3x3 stride-1 (K = 9 x 64 = 576)
//   fc   : X3 [N, 7*7*64] (feature order (y, x, c))
// Each output row of a shifted GEMM lives on the input grid; rows outside the
// valid output window are computed and discarded by the epilogue.  Backward
// data-gradients are shifted GEMMs with negated offsets against zero-padded
// gradient grids; weight gradients reduce over grid rows with MN-major operands
// and split-K partials reduced deterministically.
//
// Master parameters (f32, flat, see bp_atari_param_offsets) keep the conv / fc
// weights in GEMM layout [Cout][K] (K = (tap, input channel)); the Python module
// converts state_dicts to / from the upstream torch layouts.  A bf16 mirror of
// the flat buffer (written by the optimiser kernel, or bp_atari_pack_weights)
// is the GEMM operand for the forward (K-major B) and the data-gradients
// (MN-major B, same buffer); the policy / baseline heads are one GEMM over the
// augmented core [relu(fc) | clip(r) | onehot(a) | 1].
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "lstm.h"
#include "tma_host.h"
#include "umma_gemm.cuh"

namespace bp {

// ============================================================ param layout
enum {
  P_W1, P_B1, P_W2, P_B2, P_W3, P_B3, P_WFC, P_BFC,
  P_WIH0, P_WHH0, P_BIH0, P_BHH0, P_WIH1, P_WHH1, P_BIH1, P_BHH1,  // use_lstm only
  P_WP, P_BP, P_WV, P_BV, P_COUNT
};

static void param_offsets(int A, int lstm, int64_t* off) {
  const int64_t core = 512 + 1 + A;
  const int64_t g = lstm ? 4 * core * core : 0, b = lstm ? 4 * core : 0;
  const int64_t sizes[P_COUNT] = {256 * 32, 32, 512 * 64, 64, 576 * 64, 64, 3136 * 512, 512,
                                  g, g, b, b, g, g, b, b,
                                  A * core, A, core, 1};
  int64_t o = 0;
  for (int i = 0; i < P_COUNT; ++i) {
    off[i] = o;
    o += sizes[i];
  }
  off[P_COUNT] = o;
}

// ============================================================ tensor maps (tma_host.cu)
static int init_driver() { return tma_init(); }
#define g_num_sms tma_num_sms()

// bf16 row-major [rows][cols]; box {box_cols (inner), box_rows}
static int make_tmap(CUtensorMap* m, const void* ptr, long long rows, long long cols, int box_cols,
                     int box_rows, int swz) {
  return tma_make_2d(m, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, cols, box_cols, box_rows, swz);
}

// window mode for a shifted K-major A operand: taps share one TMA box per channel block
// conv1 A operand straight from the u8 frames (BP_CONV1_U8=0 or bp_atari_set_conv1_u8(0) restore
// the bf16 X0 grid path: space-to-depth kernel + TMA-loaded windows)
// mode 1 (default): converted windows in shared memory; mode 2: im2col rows in TMEM (A operand
// read by the MMA from tensor memory, no shared-memory A traffic, but 4x the conversion work:
// measured 102 vs 74 us)
static int g_conv1_u8 = -1;
static int conv1_u8_mode() {
  if (g_conv1_u8 < 0) {
    const char* e = std::getenv("BP_CONV1_U8");
    g_conv1_u8 = e ? (e[0] == '0' ? 0 : e[0] == '2' ? 2 : 1) : 1;
  }
  return g_conv1_u8;
}
static bool conv1_u8() { return conv1_u8_mode() != 0; }
// conv1 bias gradient: from the conv2 data-gradient epilogue's column sums (default), or from
// an all-ones atom in the conv1 window weight gradient (env BP_CONV1_ONES=1; one more M tile of
// MMAs -- the conv1 weight gradient is bound by the tensor pipe's shared-memory reads)
static bool conv1_ones() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("BP_CONV1_ONES");
    v = e && e[0] == '1' ? 1 : 0;
  }
  return v == 1;
}

static void set_window(GemmArgs& g, int taps) {
  int mn = 0, mx = 0;
  for (int t = 0; t < taps; ++t) {
    mn = g.a_row_off[t] < mn ? g.a_row_off[t] : mn;
    mx = g.a_row_off[t] > mx ? g.a_row_off[t] : mx;
  }
  g.a_ntaps = taps;
  g.a_min_off = mn;
  g.a_win_rows = (128 + mx - mn + 7) & ~7;
}

static GemmArgs base_args() {
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.splits = 1;
  g.a_cb = 1;
  g.a_atoms_per_shift = 1;
  g.a_nshifts = 1;
  g.alpha = 1.f;
  g.gh = g.gw = g.vh = g.vw = g.sy = g.sx = 1;
  g.cdiv = 1 << 30;
  g.cq = 1;
  g.b_kb_per_tap = 1 << 30;
  return g;
}

// conv weight gradients through the window kernel (umma_wgrad_win_kernel); 0 = per-tap
// atom boxes through umma_gemm_kernel (BP_WGRAD_WINDOW=0 / bp_atari_set_wgrad_window)
// small-batch inference tail (BP_SMALL_INFER=0: the GEMM fc epilogue + heads GEMM, A/B)
static bool small_infer() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BP_SMALL_INFER");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

static int g_wgrad_win = -1;
static bool wgrad_window() {
  if (g_wgrad_win < 0) {
    const char* e = std::getenv("BP_WGRAD_WINDOW");
    g_wgrad_win = (e && e[0] == '0') ? 0 : 1;
  }
  return g_wgrad_win != 0;
}

static void* g_trace_next = nullptr;
static int g_trace_tiles = 0, g_trace_skip = 0;

template <int BN, int BSWZ, int NMT, int AU8 = 0, int CB = 1, int WR = 88>
static int launch_wgrad_win(const WgArgs& g0, const CUtensorMap& tx, const CUtensorMap& ty, cudaStream_t s) {
  using Cfg = WgCfg<BN, BSWZ, NMT, AU8, CB, WR>;
  auto kern = umma_wgrad_win_kernel<BN, BSWZ, NMT, AU8, CB, WR>;
  WgArgs g = g0;
  if (g.win_rows > WR || g.a_cb > Cfg::MAX_CB || g.splits < 1 || (g.colsum && !((BN == 32 && BSWZ == 64) || (BN == 64 && BSWZ == 128)))) {
    set_error("wgrad window: %d rows / %d channel blocks unsupported", g.win_rows, g.a_cb);
    return BP_ERR_ARG;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) {
      set_error("wgrad smem attr: %s", cudaGetErrorString(e));
      return BP_ERR_LAUNCH;
    }
    attr = true;
  }
  launch_pdl(kern, dim3(g.splits), dim3(Cfg::THREADS), Cfg::SMEM, s, g, tx, ty);
  return check_launch("umma_wgrad_win_kernel");
}
template <int BN, int AM, int BM, int BSWZ, bool BRES = false, int AW = 0, int AU8 = 0, int EK = EPK_GEN>
static int launch_gemm(const GemmArgs& g0, const CUtensorMap& ta, const CUtensorMap& tb, cudaStream_t s) {
  GemmArgs g = g0;
  gemm_prepare(g);


  if (g_trace_next) {  // debug: per-tile role timeline of this launch (bp_gemm_trace_next)
    if (g_trace_skip > 0) {
      --g_trace_skip;
    } else {
      g.trace = reinterpret_cast<unsigned long long*>(g_trace_next);
      g.trace_tiles = g_trace_tiles;
      g_trace_next = nullptr;
    }
  }
  using Cfg = GemmCfg<BN, AM, BM, BSWZ, BRES, AW, AU8>;
  auto kern = umma_gemm_kernel<BN, AM, BM, BSWZ, BRES, AW, AU8, EK>;
  if (EK == EPK_FWD && (!g.bias || !g.relu || g.out_f32 || g.heads || g.mask_bits || g.colsum)) {
    set_error("gemm: forward epilogue needs bias + relu, bf16 out");
    return 1;
  }
  if (EK == EPK_DGRAD && (!g.mask_bits || g.out_f32 || g.heads || g.bias || g.relu || g.bits_out)) {
    set_error("gemm: data-gradient epilogue needs a mask, bf16 out");
    return 1;
  }
  if (EK == EPK_F32 && (!g.out_f32 || g.heads || g.bias || g.relu || g.mask_bits || g.bits_out || g.colsum ||
                        g.alpha != 1.f)) {
    set_error("gemm: EPK_F32 epilogue with unsupported features");
    return BP_ERR_ARG;
  }
  if (AW && (g.a_win_rows > 160 || g.a_win_rows < 128 || g.a_ntaps < 1 || g.a_ntaps > kMaxShifts)) {
    set_error("gemm: window rows %d / taps %d unsupported", g.a_win_rows, g.a_ntaps);
    return BP_ERR_ARG;
  }
  if (BRES && (g.n_tiles != 1 || g.splits != 1 || (size_t)g.num_kb * Cfg::B_BYTES > Cfg::B_RES)) {
    set_error("gemm: B-resident mode needs n_tiles == splits == 1 and B <= %u bytes", Cfg::B_RES);
    return BP_ERR_ARG;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) {
      set_error("gemm smem attr: %s", cudaGetErrorString(e));
      return BP_ERR_LAUNCH;
    }
    attr = true;
  }
  const int tiles = g.m_tiles * g.n_tiles * g.splits;
  const int cap = g.max_ctas > 0 && g.max_ctas < g_num_sms ? g.max_ctas : g_num_sms;
  const int grid = tiles < cap ? tiles : cap;
  launch_pdl(kern, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, s, g, ta, tb);
  return check_launch("umma_gemm_kernel");
}

// ============================================================ support kernels

constexpr int kCoreW = 576;  // augmented core row: 512 fc + clip(r) + onehot(A) + 1 + zero pad

// u8 frames [N,4,84,84] -> X0 [N*21*21, 64] bf16, channel = ci*16 + ry*4 + rx.
// Frame-stack dedup (plane_index != null): `frames` is a plane store [P][84][84] and channel
// ci of frame img is plane plane_index[img*4 + ci] (clamped to [0, num_planes)).
// The Y == 0 CTA of each image also writes the augmented core columns 512..575:
// [clip(reward), onehot(last_action) (A), 1 (bias), 0 ...]  (core order of upstream AtariNet).
__global__ void __launch_bounds__(128) frames_s2d_kernel(const uint8_t* __restrict__ frames,
                                                         const int32_t* __restrict__ plane_index,
                                                         int num_planes,
                                                         __nv_bfloat16* __restrict__ x0,
                                                         const float* __restrict__ reward,
                                                         const int64_t* __restrict__ last_action,
                                                         __nv_bfloat16* __restrict__ core, int A) {
  __shared__ __align__(16) uint8_t slab[4][4][84];
  const int img = blockIdx.x / 21, Y = blockIdx.x % 21;
  if (Y == 0 && threadIdx.x < 64) {
    const int j = threadIdx.x;
    float v = 0.f;
    if (j == 0) v = fminf(fmaxf(reward[img], -1.f), 1.f);
    else if (j <= A) v = (last_action[img] == j - 1) ? 1.f : 0.f;
    else if (j == A + 1) v = 1.f;
    core[(size_t)img * kCoreW + 512 + j] = __float2bfloat16_rn(v);
  }
  for (int w = threadIdx.x; w < 16 * 21; w += 128) {
    const int row = w / 21, col = w % 21;  // row = ci*4 + ry
    const int ci = row >> 2, ry = row & 3;
    size_t plane = (size_t)img * 4 + ci;
    if (plane_index) {
      const int pi = __ldg(plane_index + plane);
      plane = (size_t)(pi < 0 ? 0 : pi >= num_planes ? num_planes - 1 : pi);
    }
    const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(
        frames + (plane * 84 + (4 * Y + ry)) * 84) + col);
    *reinterpret_cast<uint32_t*>(&slab[ci][ry][4 * col]) = v;
  }
  __syncthreads();
  __nv_bfloat16* dst = x0 + ((size_t)img * 441 + (size_t)Y * 21) * 64;
  for (int c = threadIdx.x; c < 21 * 8; c += 128) {
    const int X = c >> 3, ch0 = (c & 7) * 8;
    const int ci = ch0 >> 4, ry0 = (ch0 & 15) >> 2;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ry = ry0 + (k >> 1), rx = (k & 1) * 2;
      const float a = (float)slab[ci][ry][4 * X + rx];
      const float b = (float)slab[ci][ry][4 * X + rx + 1];
      w[k] = pack_bf16x2(a, b);
    }
    *reinterpret_cast<uint4*>(dst + (size_t)X * 64 + ch0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// one launch for the forward's two small jobs: blocks [0, 36) pack the heads operand, the
// rest write the augmented core columns (u8 conv1 path)
__global__ void __launch_bounds__(512) prep_kernel(const float* __restrict__ wp, const float* __restrict__ bp,
                                                   const float* __restrict__ wv, const float* __restrict__ bv,
                                                   __nv_bfloat16* __restrict__ whf, const float* __restrict__ reward,
                                                   const int64_t* __restrict__ last_action,
                                                   __nv_bfloat16* __restrict__ core, int n, int A,
                                                   unsigned long long* seed_state) {
  pdl_trigger();  // conv1 may launch now: it sets up its pipeline, then waits for this kernel
  pdl_wait();
  if (seed_state && blockIdx.x == 0 && threadIdx.x == 0) advance_seed_dev(seed_state);  // (sampling)
  if (blockIdx.x < 36) {
    const int core_w = 513 + A;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 32 * kCoreW; i += 36 * blockDim.x) {
      const int a = i / kCoreW, j = i % kCoreW;
      float v = 0.f;
      if (a < A) v = j < core_w ? wp[(size_t)a * core_w + j] : (j == core_w ? bp[a] : 0.f);
      else if (a == A) v = j < core_w ? wv[j] : (j == core_w ? bv[0] : 0.f);
      whf[i] = __float2bfloat16_rn(v);
    }
    return;
  }
  // core columns [512, 576) of row img: 8 threads per row, one 16-byte store of 8 bf16 each
  const long long i = (long long)(blockIdx.x - 36) * blockDim.x + threadIdx.x;
  if (i >= (long long)n * 8) return;
  const long long img = i >> 3;
  const int j0 = (int)(i & 7) * 8;
  const float r = fminf(fmaxf(reward[img], -1.f), 1.f);
  const long long la = last_action[img];
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float v2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + 2 * q + h;
      v2[h] = j == 0 ? r : j <= A ? (la == j - 1 ? 1.f : 0.f) : (j == A + 1 ? 1.f : 0.f);
    }
    w[q] = pack_bf16x2(v2[0], v2[1]);
  }
  *reinterpret_cast<uint4*>(core + img * kCoreW + 512 + j0) = make_uint4(w[0], w[1], w[2], w[3]);
}

// G [N][64] bf16 = [d_logits (A) | d_baseline | 0 ...]
__global__ void pack_g_kernel(const float* __restrict__ dlog, const float* __restrict__ dbase,
                              __nv_bfloat16* __restrict__ G, int n, int A) {
  pdl_trigger();  // the heads data-gradient GEMM may set up (it waits for this kernel)
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // (row, 8-col chunk)
  if (i >= (long long)n * 8) return;
  const int row = (int)(i >> 3), c0 = (int)(i & 7) * 8;
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = c0 + k;
    v[k] = c < A ? dlog[(size_t)row * A + c] : (c == A ? dbase[row] : 0.f);
  }
  *reinterpret_cast<uint4*>(G + (size_t)row * 64 + c0) =
      make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                 pack_bf16x2(v[6], v[7]));
}

// flat f32 -> bf16 mirror (all parameters), vectorised
__global__ void cast_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, long long n) {
  const long long n4 = n >> 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    reinterpret_cast<uint2*>(dst)[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
  for (long long i = (n4 << 2) + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

// heads operand Whf [32][576]: row a < A = [Wp[a][0..core) | bp[a] | 0], row A = [Wv | bv | 0]
__global__ void pack_heads_kernel(const float* __restrict__ wp, const float* __restrict__ bp,
                                  const float* __restrict__ wv, const float* __restrict__ bv,
                                  __nv_bfloat16* __restrict__ whf, int A) {
  const int core = 513 + A;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 32 * kCoreW; i += 36 * blockDim.x) {
    const int a = i / kCoreW, j = i % kCoreW;
    float v = 0.f;
    if (a < A) v = j < core ? wp[(size_t)a * core + j] : (j == core ? bp[a] : 0.f);
    else if (a == A) v = j < core ? wv[j] : (j == core ? bv[0] : 0.f);
    whf[i] = __float2bfloat16_rn(v);
  }
}

// ---- finalize: deterministic reductions of every partial buffer into the f32 grads
struct FinJob {
  const float* partial;
  float* dst;
  int kind;     // 0 split-K [splits][Mpad][Npad] -> dst[n*M + m] * alpha (transpose to [Cout][K]);
                // 1 colsum [R][G*C] -> dst[c] = sum_r sum_g; 2 heads split-K routing
  int splits;   // kind 0/2: splits; kind 1: R (partial rows)
  int M, N;     // kind 0/2: valid rows (K) / cols (Cout); kind 1: M = G groups, N = C
  int Npad;
  long long Mpad;
  float alpha;
};
struct FinArgs {
  FinJob job[8];
  int njobs;
  int A;
  float* wp_grad;
  float* bp_grad;
  float* wv_grad;
  float* bv_grad;
};

BP_DEVICE float fin_partial(const FinJob& j, long long i, int r) {
  if (j.kind == 1) {  // r over rows * groups
    const int row = r / j.M, grp = r - row * j.M;
    return j.partial[(long long)row * j.M * j.N + (long long)grp * j.N + i];
  }
  const long long m = i / j.N, n = i % j.N;
  return j.partial[((long long)r * j.Mpad + m) * j.Npad + n];
}

BP_DEVICE void fin_store_mn(const FinArgs& a, const FinJob& j, int m, int n, float s);
BP_DEVICE void fin_store(const FinArgs& a, const FinJob& j, long long i, float s) {
  if (j.kind == 1) {
    j.dst[i] = s;
    return;
  }
  fin_store_mn(a, j, (int)(i / j.N), (int)(i % j.N), s);
}
// split-K outputs (kind 0: conv weights transposed to [Cout][K]; kind 2: heads), element (m, n)
BP_DEVICE void fin_store_mn(const FinArgs& a, const FinJob& j, int m, int n, float s) {
  s *= j.alpha;
  if (j.kind == 0) {
    j.dst[n * j.M + m] = s;
  } else {  // heads: D[jj][aa], core = 513 + A; row core is the bias (ones) column
    const int core = 513 + a.A;
    if (n < a.A) {
      if (m < core) a.wp_grad[n * core + m] = s;
      else if (m == core) a.bp_grad[n] = s;
    } else if (n == a.A) {
      if (m < core) a.wv_grad[m] = s;
      else if (m == core) a.bv_grad[0] = s;
    }
  }
}

// Split-K jobs: 32 outputs per block, the partials split over its 8 warps, fixed-order
// combine.  Column-sum jobs (thousands of partials, few outputs): one block per output,
// fixed strided split + fixed shared-memory tree.  All deterministic.
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ FinArgs a) {
  pdl_wait();
  const FinJob& j = a.job[blockIdx.y];
  if (j.kind == 1) {
    __shared__ float red[256];
    const int nparts = j.splits * j.M;
    for (int c = blockIdx.x; c < j.N; c += gridDim.x) {
      float s = 0.f;
      for (int r = threadIdx.x; r < nparts; r += 256) s += fin_partial(j, c, r);
      red[threadIdx.x] = s;
      __syncthreads();
      for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
      }
      if (threadIdx.x == 0) fin_store(a, j, c, red[0]);
      __syncthreads();
    }
    return;
  }
  // split-K: a block takes 32 consecutive outputs (lane = output: coalesced partial rows);
  // its 8 warps split the partials (warp w sums splits w, w + 8, ...; 8 loads in flight per
  // lane), then warp 0 adds the 8 warp sums in a fixed order.  The one-thread-per-output form
  // had 16 loads in flight on ~2 blocks per SM and was latency-bound.
  __shared__ float red8[8][32];
  const long long total = (long long)j.M * j.N;
  const long long pstride = j.Mpad * j.Npad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * 32; base < total; base += (long long)gridDim.x * 32) {
    const long long i = base + lane;
    float s = 0.f;
    // 32-bit index math (outputs < 2^31; a 64-bit division is a long software sequence)
    const uint32_t iu = (uint32_t)i, mu = iu / (uint32_t)j.N, nu = iu - mu * (uint32_t)j.N;
    if (i < total) {
      const float* p = j.partial + (long long)mu * j.Npad + nu;
      for (int r = warp; r < j.splits; r += 64) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int rr = r + 8 * q;
          v[q] = rr < j.splits ? __ldcs(p + (long long)rr * pstride) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) s += v[q];
      }
    }
    red8[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && i < total) {
      float t = red8[0][lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) t += red8[w][lane];
      fin_store_mn(a, j, (int)mu, (int)nu, t);
    }
    __syncthreads();
  }
}

// ============================================================ workspace plan
struct WgPlan {
  int m_tiles, n_tiles, num_kb, splits, kb_per;
  long long Mpad;
  int Npad;
  size_t off, floats;
};
struct NetPlan {
  WgPlan wg[4];       // conv1, conv2, conv3, heads (fc wgrad writes the grads directly)
  size_t cs_off[4];   // colsum partials: db1 (conv2 dgrad), db2, db3, dbfc
  int cs_rows[4], cs_n[4];
  size_t total_floats;
};

static void make_plan(int n, int sms, NetPlan* P, bool win) {
  const long long rows[4] = {(long long)n * 441, (long long)n * 100, (long long)n * 81, n};
  // conv3's 9 taps x 64 channels pad to 5 m-tiles (the 10th atom is the zero atom)
  // window mode: conv1 gets one more m-tile (the all-ones atom -> db1 rows, which spares the
  // conv2 dgrad epilogue its column sums); conv3's 9 taps leave atom 9 free for db3
  const int M[4] = {win && conv1_ones() ? 384 : 256, 512, 576, kCoreW};
  const int Ns[4] = {32, 64, 64, 64};
  size_t off = 0;
  for (int i = 0; i < 4; ++i) {
    WgPlan& w = P->wg[i];
    w.m_tiles = (M[i] + 127) / 128;
    w.n_tiles = 1;
    w.num_kb = (int)((rows[i] + 63) / 64);
    int sp = (i < 3 && win) ? sms : (sms + w.m_tiles - 1) / w.m_tiles;
    if (sp > w.num_kb) sp = w.num_kb;
    if (sp < 1) sp = 1;
    w.kb_per = (w.num_kb + sp - 1) / sp;
    w.splits = (w.num_kb + w.kb_per - 1) / w.kb_per;
    w.Mpad = (long long)w.m_tiles * 128;
    w.Npad = Ns[i];
    w.off = off;
    w.floats = (size_t)w.splits * w.Mpad * w.Npad;
    off += (w.floats + 63) & ~size_t(63);
  }
  // dgrad epilogue column sums: rows = 4 * m_tiles of the producing GEMM, width = its N
  const long long drows[4] = {(long long)n * 100, (long long)n * 81, n, n};
  const int dn[4] = {128, 64, 3136, 512};
  const bool cta_mode[4] = {true, true, false, false};  // producing GEMM has a single N tile
  for (int i = 0; i < 4; ++i) {
    const long long mt = (drows[i] + 127) / 128;
    P->cs_rows[i] = (int)(4 * (cta_mode[i] ? (mt < sms ? mt : sms) : mt));
    P->cs_n[i] = dn[i];
    P->cs_off[i] = off;
    off += ((size_t)P->cs_rows[i] * dn[i] + 63) & ~size_t(63);
  }
  P->total_floats = off;
}

}  // namespace bp

// ============================================================ C ABI
using namespace bp;

// Raw engine entry for unit tests: C[M][N] f32 = A . B^T with
//   a_mn = 0: A stored [M][K] (K-major), 1: A stored [K][M] (MN-major)
//   b_mn = 0: B stored [N][K],           1: B stored [K][N]
extern "C" int bp_gemm_bf16_test(const void* A, const void* B, void* C, int M, int N, int K,
                                 int a_mn, int b_mn, int splits, int out_bf16, void* stream) {
  if (int e = init_driver()) return e;
  cudaStream_t s = (cudaStream_t)stream;
  if (K % 64 || M % 64 || (!a_mn && M % 128) || splits < 1) {
    set_error("gemm_test: bad dims M=%d N=%d K=%d", M, N, K);
    return BP_ERR_ARG;
  }
  int BN = N >= 256 ? 256 : N;
  if (!(BN == 32 || BN == 64 || BN == 128 || BN == 256) || N % BN) {
    set_error("gemm_test: unsupported N=%d", N);
    return BP_ERR_ARG;
  }
  CUtensorMap ta, tb;
  int rc;
  GemmArgs g = base_args();
  g.m_tiles = (M + 127) / 128;
  g.n_tiles = N / BN;
  g.num_kb = K / 64;
  g.splits = splits;
  g.kb_per_split = (g.num_kb + splits - 1) / splits;
  g.N = N;
  g.M = g.m_tiles * 128;
  g.out_f32 = out_bf16 ? 0 : 1;
  g.out = C;
  g.r_img = N;
  g.split_stride = (long long)g.m_tiles * 128 * N;
  if (!a_mn) {
    g.a_cb = K / 64;
    if ((rc = make_tmap(&ta, A, M, K, 64, 128, 128))) return rc;
  } else {
    g.a_atoms_per_shift = M / 64;
    g.a_nshifts = 1;
    if ((rc = make_tmap(&ta, A, K, M, 64, 64, 128))) return rc;
  }
  if (!b_mn) {
    if ((rc = make_tmap(&tb, B, N, K, 64, BN, 128))) return rc;
  } else if (BN == 32) {
    if ((rc = make_tmap(&tb, B, K, N, 32, 64, 64))) return rc;
  } else {
    if ((rc = make_tmap(&tb, B, K, N, 64, 64, 128))) return rc;
  }
#define BP_GT(BN_, AM_, BM_, SW_)                                                  \
  if (BN == BN_ && a_mn == (AM_ == A_MNMAJOR) && b_mn == (BM_ == B_MNMAJOR))      \
    return launch_gemm<BN_, AM_, BM_, SW_>(g, ta, tb, s);
  BP_GT(32, A_KMAJOR, B_KMAJOR, 128)
  BP_GT(64, A_KMAJOR, B_KMAJOR, 128)
  BP_GT(128, A_KMAJOR, B_KMAJOR, 128)
  BP_GT(256, A_KMAJOR, B_KMAJOR, 128)
  BP_GT(32, A_MNMAJOR, B_MNMAJOR, 64)
  BP_GT(64, A_MNMAJOR, B_MNMAJOR, 128)
  BP_GT(256, A_MNMAJOR, B_MNMAJOR, 128)
  BP_GT(64, A_KMAJOR, B_MNMAJOR, 128)
  BP_GT(128, A_KMAJOR, B_MNMAJOR, 128)
  BP_GT(64, A_MNMAJOR, B_KMAJOR, 128)
#undef BP_GT
  set_error("gemm_test: combination not instantiated (N=%d a_mn=%d b_mn=%d)", N, a_mn, b_mn);
  return BP_ERR_UNSUPPORTED;
}

// Shifted-tap GEMM test entry: C[m][n] = sum_t sum_c A[m + off_t][c] B[n][t*C + c], A [R][C] K-major,
// B [N][taps*C]; window_mode 0 = one TMA box per tap, 1/2 = one window per channel block
// (descriptor base_offset 0 / (addr >> 7) & 7).  N in {32, 64}; C multiple of 64.
extern "C" int bp_gemm_shift_test(const void* A, const void* B, float* Cout, int R, int Cin, int N,
                                  int taps, const int* offs, int window_mode, void* trace,
                                  int trace_tiles, void* stream) {
  if (int e = init_driver()) return e;
  cudaStream_t s = (cudaStream_t)stream;
  if (Cin % 64 || taps < 1 || taps > kMaxShifts || !(N == 32 || N == 64)) {
    set_error("shift_test: bad args");
    return BP_ERR_ARG;
  }
  int mn = 0, mx = 0;
  for (int t = 0; t < taps; ++t) {
    mn = offs[t] < mn ? offs[t] : mn;
    mx = offs[t] > mx ? offs[t] : mx;
  }
  GemmArgs g = base_args();
  g.m_tiles = (R + 127) / 128;
  g.n_tiles = 1;
  g.a_cb = Cin / 64;
  g.num_kb = g.kb_per_split = taps * g.a_cb;
  for (int t = 0; t < taps; ++t) g.a_row_off[t] = offs[t];
  g.a_ntaps = taps;
  g.a_min_off = mn;
  g.a_win_rows = (128 + mx - mn + 7) & ~7;
  g.N = N;
  g.M = R;
  g.out_f32 = 1;
  g.out = Cout;
  g.r_img = N;
  g.trace = reinterpret_cast<unsigned long long*>(trace);
  g.trace_tiles = trace_tiles;
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_tmap(&ta, A, R, Cin, 64, window_mode ? g.a_win_rows : 128, 128))) return rc;
  if ((rc = make_tmap(&tb, B, N, (long long)taps * Cin, 64, N, 128))) return rc;
  if (N == 32) {
    if (window_mode == 0) return launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true, 0>(g, ta, tb, s);
    if (window_mode == 1) return launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true, 1>(g, ta, tb, s);
    return launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true, 2>(g, ta, tb, s);
  }
  if (window_mode == 0) return launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, true, 0>(g, ta, tb, s);
  if (window_mode == 1) return launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, true, 1>(g, ta, tb, s);
  return launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, true, 2>(g, ta, tb, s);
}

// debug: the next GEMM launch records per-tile role timestamps (%globaltimer ns) into
// buf[(cta * tiles + i) * 16 + event] (0/1 producer, 2/3 MMA, 4/5 epilogue, 6/7 u8 converter)
extern "C" int bp_gemm_trace_next(void* buf, int tiles, int skip) {
  g_trace_next = buf;
  g_trace_tiles = tiles;
  g_trace_skip = skip;
  return BP_OK;
}

extern "C" int bp_atari_set_wgrad_window(int on) {
  const int prev = wgrad_window() ? 1 : 0;
  if (on >= 0) g_wgrad_win = on ? 1 : 0;
  return prev;
}

extern "C" int bp_atari_set_conv1_u8(int on) {
  const int prev = conv1_u8_mode();
  if (on >= 0) g_conv1_u8 = on > 2 ? 2 : on;
  return prev;
}

extern "C" int64_t bp_atari_param_count(int num_actions, int use_lstm) {
  if (num_actions < 1 || num_actions > 31) return -1;
  int64_t off[P_COUNT + 1];
  param_offsets(num_actions, use_lstm, off);
  return off[P_COUNT];
}

extern "C" int bp_atari_param_offsets(int num_actions, int use_lstm, int64_t* offsets) {
  if (num_actions < 1 || num_actions > 31 || !offsets) {
    set_error("atari: num_actions must be in [1, 31]");
    return BP_ERR_ARG;
  }
  param_offsets(num_actions, use_lstm, offsets);
  return BP_OK;
}

extern "C" size_t bp_atari_workspace_bytes(int num_actions, int max_frames) {
  (void)num_actions;
  if (init_driver()) return 0;
  NetPlan P, Q;  // sized for either weight-gradient mode (bp_atari_set_wgrad_window)
  make_plan(max_frames, g_num_sms, &P, true);
  make_plan(max_frames, g_num_sms, &Q, false);
  return (P.total_floats > Q.total_floats ? P.total_floats : Q.total_floats) * sizeof(float);
}

static int check_net(const BpAtariNet* net, int n) {
  if (!net || n < 1 || n > net->max_frames || net->num_actions < 1 || net->num_actions > 31) {
    set_error("atari: bad net / frame count %d (max %d)", n, net ? net->max_frames : -1);
    return BP_ERR_ARG;
  }
  return init_driver();
}

extern "C" int bp_atari_pack_weights(const BpAtariNet* net, const float* params, void* stream) {
  if (int e = check_net(net, 1)) return e;
  int64_t off[P_COUNT + 1];
  param_offsets(net->num_actions, net->use_lstm, off);
  cast_bf16_kernel<<<296, 256, 0, (cudaStream_t)stream>>>(
      params, reinterpret_cast<__nv_bfloat16*>(net->wbf), off[P_COUNT]);
  return check_launch("cast_bf16_kernel");
}

// frames -> conv torso -> fc -> augmented core [n][576] (net->core)
// frames: u8 [n][4][84][84], or (plane_index != null) a plane store [num_planes][84][84]
// fc_splitk > 1 (small-batch inference): the fc GEMM writes fc_splitk f32 split-K partials of
// x3 . Wfc^T into the workspace instead of core[:, :512] (infer_heads_kernel finishes it)
__global__ void advance_seed_kernel(unsigned long long* seed_state);

static int torso_forward(const BpAtariNet* net, int n, const uint8_t* frames, const int32_t* plane_index,
                         int num_planes, const float* reward, const int64_t* last_action,
                         const float* params, const int64_t* off, cudaStream_t s, int fc_splitk = 1,
                         unsigned long long* seed_state = nullptr) {
  const int A = net->num_actions;
  const __nv_bfloat16* wbf = reinterpret_cast<const __nv_bfloat16*>(net->wbf);
  auto bf = [](void* p) { return reinterpret_cast<__nv_bfloat16*>(p); };
  int rc;
  // 1. frames -> space-to-depth bf16 (+ augmented core columns), heads operand
  // prep folded into conv1 (default): the heads pack and the core columns run in conv1's idle
  // warp 3 instead of a kernel of their own at the head of the chain (cfg1 step span 359.1 ->
  // 356.8 us, cfg3 1245.2 -> 1241.6 us; env BP_PREP_FOLD=0: the separate prep_kernel)
  static const bool prep_fold = [] {
    const char* e = std::getenv("BP_PREP_FOLD");
    return !(e && e[0] == '0');
  }();
  // (only when conv1 runs one CTA per SM: at small n its few CTAs would serialise the work --
  // k=1 inference: conv1 5.2 -> 21.3 us folded)
  if (int e = tma_init()) return e;  // (the SM count)
  const bool fold = conv1_u8() && prep_fold && (long long)n * 441 >= 128LL * g_num_sms;
  if (conv1_u8() && !fold) {  // conv1 converts the frames on chip (and writes X0 for the weight gradient)
    launch_pdl(prep_kernel, dim3(36 + (n * 8 + 511) / 512), dim3(512), 0, s, params + off[P_WP],
               params + off[P_BP], params + off[P_WV], params + off[P_BV], bf(net->whf), reward, last_action,
               bf(net->core), n, A, seed_state);
    if ((rc = check_launch("prep_kernel"))) return rc;
  } else if (!fold) {
    if (seed_state) {
      launch_pdl(advance_seed_kernel, dim3(1), dim3(1), 0, s, seed_state);
      if ((rc = check_launch("advance_seed_kernel"))) return rc;
    }
    frames_s2d_kernel<<<n * 21, 128, 0, s>>>(frames, plane_index, num_planes, bf(net->x0), reward, last_action,
                                             bf(net->core), A);
    if ((rc = check_launch("frames_s2d_kernel"))) return rc;
    pack_heads_kernel<<<36, 512, 0, s>>>(params + off[P_WP], params + off[P_BP], params + off[P_WV],
                                         params + off[P_BV], bf(net->whf), A);
    if ((rc = check_launch("pack_heads_kernel"))) return rc;
  }
  CUtensorMap ta, tb;
  // 2. conv1: X0 [n*441, 64] x W1 [32, 256] -> relu(./255 + b1) -> X1 (s2d-2 layout)
  //    u8 mode: the X0 window of every tile is built on chip from the u8 frames
  {
    const long long R = (long long)n * 441;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 4;
    const int offs[4] = {0, 1, 21, 22};
    for (int i = 0; i < 4; ++i) g.a_row_off[i] = offs[i];
    set_window(g, 4);
    if ((rc = make_tmap(&tb, wbf + off[P_W1], 32, 256, 64, 32, 128))) return rc;
    if (conv1_u8()) {
      ta = tb;  // (unused by the u8 producer)
      g.u8 = frames;
      g.u8_index = plane_index;
      g.u8_planes = num_planes;
      g.u8_rows = R;
      g.u8_x0_out = (net->flags & BP_NET_NO_X0) ? nullptr : bf(net->x0);
    } else if ((rc = make_tmap(&ta, net->x0, R, 64, 64, g.a_win_rows, 128))) {
      return rc;
    }
    g.N = 32;
    g.M = (int)R;
    g.alpha = 1.f / 255.f;
    g.bias = params + off[P_B1];
    g.relu = 1;
    g.out = net->x1;
    g.bits_out = reinterpret_cast<uint32_t*>(net->m1);
    g.gh = 21; g.gw = 21; g.vh = 20; g.vw = 20; g.sy = 2; g.sx = 2;
    g.r_img = 100 * 128; g.r_y = 10 * 128; g.r_x = 128; g.r_sub = 32;
    if (fold)
      g.prep = PrepArgs{params + off[P_WP], params + off[P_BP], params + off[P_WV], params + off[P_BV], bf(net->whf),
                        reward, last_action, bf(net->core), n, A, seed_state};
    if (conv1_u8_mode() == 2) {
      if ((rc = launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true, 1, 2, EPK_FWD>(g, ta, tb, s))) return rc;
    } else if (conv1_u8()) {
      if ((rc = launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true, 1, 1, EPK_FWD>(g, ta, tb, s))) return rc;
    } else if ((rc = launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true, 1, 0, EPK_FWD>(g, ta, tb, s))) {
      return rc;
    }
  }
  // 3. conv2: X1 [n*100, 128], 2x2 taps on the 10x10 grid -> X2 [n*81, 64]
  {
    const long long R = (long long)n * 100;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 8;
    g.a_cb = 2;
    const int offs[4] = {0, 1, 10, 11};
    for (int i = 0; i < 4; ++i) g.a_row_off[i] = offs[i];
    set_window(g, 4);
    if ((rc = make_tmap(&ta, net->x1, R, 128, 64, g.a_win_rows, 128))) return rc;
    if ((rc = make_tmap(&tb, wbf + off[P_W2], 64, 512, 64, 64, 128))) return rc;
    g.N = 64;
    g.M = (int)R;
    g.bias = params + off[P_B2];
    g.relu = 1;
    g.out = net->x2;
    g.bits_out = reinterpret_cast<uint32_t*>(net->m2);
    g.gh = 10; g.gw = 10; g.vh = 9; g.vw = 9;
    g.r_img = 81 * 64; g.r_y = 9 * 64; g.r_x = 64;
    if ((rc = launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, true, 1, 0, EPK_FWD>(g, ta, tb, s))) return rc;
  }
  // 4. conv3: X2 [n*81, 64], 3x3 taps on the 9x9 grid -> X3 [n, 3136] ((y, x, c) order)
  {
    const long long R = (long long)n * 81;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 9;
    for (int dy = 0; dy < 3; ++dy)
      for (int dx = 0; dx < 3; ++dx) g.a_row_off[dy * 3 + dx] = dy * 9 + dx;
    set_window(g, 9);
    if ((rc = make_tmap(&ta, net->x2, R, 64, 64, g.a_win_rows, 128))) return rc;
    if ((rc = make_tmap(&tb, wbf + off[P_W3], 64, 576, 64, 64, 128))) return rc;
    g.N = 64;
    g.M = (int)R;
    g.bias = params + off[P_B3];
    g.relu = 1;
    g.out = net->x3;
    g.bits_out = reinterpret_cast<uint32_t*>(net->m3);
    g.gh = 9; g.gw = 9; g.vh = 7; g.vw = 7;
    g.r_img = 3136; g.r_y = 7 * 64; g.r_x = 64;
    if ((rc = launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, true, 1, 0, EPK_FWD>(g, ta, tb, s))) return rc;
  }
  // 5. fc: X3 [n, 3136] x Wfc [512, 3136] -> core[:, :512] = relu(. + bfc)
  if (fc_splitk > 1) {  // latency-bound small batches: K split over more CTAs, f32 partials
    const int mt = (n + 127) / 128;
    if ((rc = make_tmap(&ta, net->x3, n, 3136, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, wbf + off[P_WFC], 512, 3136, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = mt;
    g.n_tiles = 8;
    g.splits = fc_splitk;
    g.num_kb = 49;
    g.kb_per_split = (49 + fc_splitk - 1) / fc_splitk;
    g.a_cb = 49;
    g.N = 512;
    g.M = n;
    g.out_f32 = 1;
    g.out = net->ws;
    g.split_stride = (long long)n * 512;
    g.r_img = 512;
    return launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s);
  }
  {
    // 128-column tiles when 64-column ones would need a second wave: half the re-reads of
    // X3 from L2 (the fc GEMM is L2->SM bandwidth-bound) and a single wave
    const int mt = (n + 127) / 128;
    const bool wide = mt * 8 > g_num_sms;
    if ((rc = make_tmap(&ta, net->x3, n, 3136, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, wbf + off[P_WFC], 512, 3136, 64, wide ? 128 : 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = mt;
    g.n_tiles = wide ? 4 : 8;
    g.num_kb = g.kb_per_split = 49;
    g.a_cb = 49;
    g.N = 512;
    g.M = n;
    g.bias = params + off[P_BFC];
    g.relu = 1;
    g.out = net->core;
    g.bits_out = reinterpret_cast<uint32_t*>(net->mc);
    g.r_img = kCoreW;
    if ((rc = wide ? launch_gemm<128, A_KMAJOR, B_KMAJOR, 128, false, 0, 0, EPK_FWD>(g, ta, tb, s)
                   : launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, false, 0, 0, EPK_FWD>(g, ta, tb, s)))
      return rc;
  }
  return BP_OK;
}

// heads: head_in [n, 576] ([core | 1 | 0]) x Whf [32, 576] -> logits [n, A], baseline [n]
// Small-batch inference tail (n <= kInferSmallN): one CTA per row finishes the split-K fc
// (fixed-order sum of the partials + bias, ReLU, the bf16 rounding core[:, :512] has on the
// GEMM path), appends the augmented columns prep wrote, and computes the A + 1 heads on CUDA
// cores (bf16 operands, f32 accumulation: the same operands as the heads GEMM, a different
// summation order) and the Gumbel-max action.  Replaces the fc epilogue + heads GEMM, whose
// latency chains (3.2 MB of fc weights through 8 CTAs; 9 serial K-blocks in one CTA) dominate
// small dynamic batches.
constexpr int kInferSmallN = 256;  // (measured: k = 1 / 32 / 256 gain, k = 1024 does not)
__global__ void __launch_bounds__(128) infer_heads_kernel(const float* __restrict__ part, int S, long long sstride,
                                                          const float* __restrict__ bfc,
                                                          const __nv_bfloat16* __restrict__ core,
                                                          const __nv_bfloat16* __restrict__ whf, int A,
                                                          float* __restrict__ logits, float* __restrict__ baseline,
                                                          int64_t* __restrict__ actions, unsigned long long seed,
                                                          const unsigned long long* __restrict__ seed_state,
                                                          int greedy) {
  pdl_wait();
  __shared__ float c[kCoreW];
  __shared__ float o[32];
  const int r = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int k = tid; k < 512; k += 128) {
    float acc = 0.f;
    for (int q = 0; q < S; ++q) acc += part[(size_t)q * sstride + (size_t)r * 512 + k];
    c[k] = __bfloat162float(__float2bfloat16_rn(fmaxf(acc + bfc[k], 0.f)));
  }
  for (int k = 512 + tid; k < kCoreW; k += 128) c[k] = __bfloat162float(core[(size_t)r * kCoreW + k]);
  __syncthreads();
  for (int a = warp; a <= A; a += 4) {
    float acc = 0.f;
    for (int k = lane; k < kCoreW; k += 32) acc = fmaf(c[k], __bfloat162float(whf[a * kCoreW + k]), acc);
#pragma unroll
    for (int sh = 16; sh >= 1; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
    if (lane == 0) o[a] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = j <= A ? o[j] : 0.f;
    for (int a = 0; a < A; ++a) logits[(size_t)r * A + a] = v[a];
    baseline[r] = o[A];
    if (actions)
      actions[r] = gumbel_argmax<32>(v, A, seed_state ? *seed_state : seed, (unsigned long long)r, greedy != 0);
  }
}

// fused action sampling of the heads epilogue (inference: bp_atari_forward_sample)
struct SampleSpec {
  int64_t* actions;
  unsigned long long seed;
  unsigned long long* seed_state;  // device-resident seed (graph replays): advanced per call
  int greedy;
};

// graph-replayable sampling: every call advances the device-resident seed (splitmix64 step)
__global__ void advance_seed_kernel(unsigned long long* seed_state) {
  pdl_trigger();  // the forward's first kernel may launch now (it waits for this one)
  pdl_wait();     // the previous call's sampler has read the seed
  advance_seed_dev(seed_state);
}


static int heads_forward(const BpAtariNet* net, int n, const void* head_in, float* logits, float* baseline,
                         cudaStream_t s, const SampleSpec* smp = nullptr) {
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_tmap(&ta, head_in, n, kCoreW, 64, 128, 128))) return rc;
  if ((rc = make_tmap(&tb, net->whf, 32, kCoreW, 64, 32, 128))) return rc;
  GemmArgs g = base_args();
  g.m_tiles = (n + 127) / 128;
  g.n_tiles = 1;
  g.num_kb = g.kb_per_split = kCoreW / 64;
  g.a_cb = kCoreW / 64;
  g.N = 32;
  g.M = n;
  g.heads = 1;
  g.A = net->num_actions;
  g.logits = logits;
  g.baseline = baseline;
  if (smp) {
    g.actions = smp->actions;
    g.sample_seed = smp->seed;
    g.seed_state = smp->seed_state;
    g.greedy = smp->greedy;
    return launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true, 0, 0, EPK_HEADS>(g, ta, tb, s);
  }
  return launch_gemm<32, A_KMAJOR, B_KMAJOR, 128, true>(g, ta, tb, s);
}

static int check_planes(const uint8_t* planes, const int32_t* plane_index, int num_planes) {
  if (!planes || (plane_index && num_planes < 1)) {
    set_error("atari: null frames / plane store, or num_planes < 1");
    return BP_ERR_ARG;
  }
  return BP_OK;
}

static int atari_forward(const BpAtariNet* net, int n, const uint8_t* frames, const int32_t* plane_index,
                         int num_planes, const float* reward, const int64_t* last_action, const float* params,
                         float* logits, float* baseline, void* stream, const SampleSpec* smp = nullptr) {
  if (int e = check_net(net, n)) return e;
  if (int e = check_planes(frames, plane_index, num_planes)) return e;
  if (net->use_lstm) {
    set_error("atari: LSTM net -> bp_atari_lstm_forward");
    return BP_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t off[P_COUNT + 1];
  param_offsets(net->num_actions, 0, off);
  int rc;
  unsigned long long* seed_state = smp ? smp->seed_state : nullptr;  // advanced by the torso's first kernel
  // small inference batches (no backward follows): split-K fc + CUDA-core heads and sampling
  const int mt = (n + 127) / 128;
  int S = 148 / (mt * 8);
  S = S > 7 ? 7 : S;
  if (smp && (net->flags & BP_NET_NO_X0) && n <= kInferSmallN && S >= 2 && small_infer() &&
      (size_t)S * n * 512 * sizeof(float) <= net->ws_bytes) {
    if ((rc = torso_forward(net, n, frames, plane_index, num_planes, reward, last_action, params, off, s, S,
                            seed_state)))
      return rc;
    launch_pdl(infer_heads_kernel, dim3(n), dim3(128), 0, s, reinterpret_cast<const float*>(net->ws), S,
               (long long)n * 512, params + off[P_BFC], reinterpret_cast<const __nv_bfloat16*>(net->core),
               reinterpret_cast<const __nv_bfloat16*>(net->whf), net->num_actions, logits, baseline, smp->actions,
               smp->seed, (const unsigned long long*)smp->seed_state, smp->greedy);
    return check_launch("infer_heads_kernel");
  }
  if ((rc = torso_forward(net, n, frames, plane_index, num_planes, reward, last_action, params, off, s, 1,
                          seed_state)))
    return rc;
  return heads_forward(net, n, net->core, logits, baseline, s, smp);
}

extern "C" int bp_atari_forward(const BpAtariNet* net, int n, const uint8_t* frames,
                                const float* reward, const int64_t* last_action, const float* params,
                                float* logits, float* baseline, void* stream) {
  return atari_forward(net, n, frames, nullptr, 0, reward, last_action, params, logits, baseline, stream);
}

extern "C" int bp_atari_forward_planes(const BpAtariNet* net, int n, const uint8_t* planes,
                                       const int32_t* plane_index, int num_planes, const float* reward,
                                       const int64_t* last_action, const float* params, float* logits,
                                       float* baseline, void* stream) {
  if (!plane_index) {
    set_error("atari: bp_atari_forward_planes needs a plane index");
    return BP_ERR_ARG;
  }
  return atari_forward(net, n, planes, plane_index, num_planes, reward, last_action, params, logits, baseline,
                       stream);
}

extern "C" int bp_atari_forward_sample(const BpAtariNet* net, int n, const uint8_t* frames,
                                       const int32_t* plane_index, int num_planes, const float* reward,
                                       const int64_t* last_action, const float* params, uint64_t seed,
                                       uint64_t* seed_state, int greedy, float* logits, float* baseline, int64_t* actions,
                                       void* stream) {
  if (!actions) {
    set_error("atari: bp_atari_forward_sample needs an actions buffer");
    return BP_ERR_ARG;
  }
  const SampleSpec smp{actions, (unsigned long long)seed, reinterpret_cast<unsigned long long*>(seed_state),
                       greedy};
  return atari_forward(net, n, frames, plane_index, plane_index ? num_planes : 0, reward, last_action, params,
                       logits, baseline, stream, &smp);
}

// G = [d_logits | d_baseline | 0] bf16, then the heads data-gradient:
//   dh_f32 == nullptr: d_fc = (G x Whf[:, :512]) * relu mask, colsum -> d bfc partials
//   dh_f32 != nullptr: dh_f32 [n][576] = G x Whf (unmasked, f32: the LSTM output gradient)
static int heads_backward(const BpAtariNet* net, int n, const float* d_logits, const float* d_baseline,
                          const NetPlan& P, float* ws, float* dh_f32, cudaStream_t s) {
  auto bf = [](void* p) { return reinterpret_cast<__nv_bfloat16*>(p); };
  int rc;
  launch_pdl(pack_g_kernel, dim3((n * 8 + 255) / 256), dim3(256), 0, s, d_logits, d_baseline, bf(net->g), n,
             net->num_actions);
  if ((rc = check_launch("pack_g_kernel"))) return rc;
  CUtensorMap ta, tb;
  if ((rc = make_tmap(&ta, net->g, n, 64, 64, 128, 128))) return rc;
  if ((rc = make_tmap(&tb, net->whf, 32, kCoreW, 64, 64, 128))) return rc;  // MN-major, rows >= 32 OOB = 0
  GemmArgs g = base_args();
  g.m_tiles = (n + 127) / 128;
  g.num_kb = g.kb_per_split = 1;
  g.M = n;
  if (dh_f32) {
    g.n_tiles = kCoreW / 64;
    g.N = kCoreW;
    g.out_f32 = 1;
    g.out = dh_f32;
    g.r_img = kCoreW;
  } else {
    g.n_tiles = 8;
    g.N = 512;
    g.mask_bits = reinterpret_cast<const uint32_t*>(net->mc);
    g.mask_ld = kCoreW;
    g.out = net->d_fc;
    g.r_img = 512;
    g.colsum = ws + P.cs_off[3];
    return launch_gemm<64, A_KMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_DGRAD>(g, ta, tb, s);
  }
  return launch_gemm<64, A_KMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s);
}

// d_fc -> conv torso data / weight gradients, heads weight gradient (A operand head_in),
// deterministic finalize of every partial into grads
// the u8 frame source of the forward (for the conv1 weight gradient without an X0 grid)
struct FrameSrc {
  const uint8_t* frames;
  const int32_t* plane_index;
  int num_planes;
};

// heads weight gradient: split-K partials of head_in^T . G (the finalize reduces them).
// beside > 0: a PDL successor of the LSTM's layer-1 backward recurrence on at most `beside`
// CTAs, waiting for it only at its end (its inputs are final before that recurrence starts)
static int heads_wgrad(const BpAtariNet* net, int n, const void* head_in, const NetPlan& P, float* ws,
                       cudaStream_t s, int beside) {
  const WgPlan& w = P.wg[3];
  CUtensorMap ta, tb;
  int r;
  if ((r = make_tmap(&ta, head_in, n, kCoreW, 64, 64, 128))) return r;
  if ((r = make_tmap(&tb, net->g, n, 64, 64, 64, 128))) return r;
  GemmArgs g = base_args();
  g.m_tiles = w.m_tiles;
  g.n_tiles = w.n_tiles;
  g.splits = w.splits;
  g.num_kb = w.num_kb;
  g.kb_per_split = w.kb_per;
  g.a_atoms_per_shift = kCoreW / 64;
  g.a_nshifts = 1;
  g.a_row_off[0] = 0;
  g.N = w.Npad;
  g.M = (int)w.Mpad;
  g.out_f32 = 1;
  g.out = ws + w.off;
  g.split_stride = w.Mpad * w.Npad;
  g.r_img = w.Npad;
  if (beside > 0) {
    g.max_ctas = beside;
    g.pdl_late = 1;
  }
  return launch_gemm<64, A_MNMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s);
}

static int torso_backward(const BpAtariNet* net, int n, const FrameSrc* src, const void* head_in, float* grads,
                          const int64_t* off,
                          const NetPlan& P, float* ws, cudaStream_t s, bool heads_wgrad_done = false) {
  const int A = net->num_actions;
  const __nv_bfloat16* wbf = reinterpret_cast<const __nv_bfloat16*>(net->wbf);
  int rc;
  CUtensorMap ta, tb;
  // fc dgrad: d_pre3 (conv3 9x9 grid) = (d_fc [n,512] x Wfc [512,3136]) * (X3 > 0); colsum -> d b3
  {
    if ((rc = make_tmap(&ta, net->d_fc, n, 512, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, wbf + off[P_WFC], 512, 3136, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (n + 127) / 128;
    g.n_tiles = 49;
    g.num_kb = g.kb_per_split = 8;
    g.a_cb = 8;
    g.N = 3136;
    g.M = n;
    g.mask_bits = reinterpret_cast<const uint32_t*>(net->m3);
    g.out = net->d_pre3;
    g.r_img = 81 * 64;
    g.cdiv = 64; g.cq = 7; g.cs1 = 9 * 64; g.cs2 = 64;
    g.colsum = wgrad_window() ? nullptr : ws + P.cs_off[2];  // window mode: bias from the wgrad ones atom
    if (wgrad_window()) {  // 128-column tiles (the last half empty): d_fc re-read 25x instead of 49x
      g.n_tiles = 25;
      if ((rc = launch_gemm<128, A_KMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_DGRAD>(g, ta, tb, s))) return rc;
    } else if ((rc = launch_gemm<64, A_KMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_DGRAD>(g, ta, tb, s))) {
      return rc;
    }
  }
  // fc weight gradient first (it only needs X3 and d_fc), transposed: D[k][o] = sum_n X3[n][k] d_fc[n][o] (M = 3136 features in 25
  // m-tiles, N = 512 in 128-column tiles: one wave of 100 tiles, X3 read 4x / d_fc 25x from L2),
  // stored transposed into grads[o][k] (per column, a warp's 32 rows are one contiguous run)
  {
    if ((rc = make_tmap(&ta, net->x3, n, 3136, 64, 64, 128))) return rc;
    if ((rc = make_tmap(&tb, net->d_fc, n, 512, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (3136 + 127) / 128;
    g.n_tiles = 4;
    g.num_kb = g.kb_per_split = (n + 63) / 64;
    g.a_atoms_per_shift = 49;
    g.a_nshifts = 1;
    g.N = 512;
    g.M = 3136;
    g.out_f32 = 1;
    g.out = grads + off[P_WFC];
    g.r_img = 1;
    g.cdiv = 1;
    g.cq = 1;
    g.cs1 = 3136;
    g.col_stride = 3136;
    if ((rc = launch_gemm<128, A_MNMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s))) return rc;
    // the fc weight gradient is final: the data-parallel learner may start its all-reduce
    if (net->fc_grad_ready && cudaEventRecord((cudaEvent_t)net->fc_grad_ready, s) != cudaSuccess) {
      set_error("atari backward: cudaEventRecord(fc_grad_ready) failed");
      return BP_ERR_LAUNCH;
    }
  }
  // conv3 dgrad: d_pre2 (conv2 10x10 grid) = sum_taps d_pre3[m - off] W3_tap^T * (X2 > 0)
  {
    const long long R = (long long)n * 81;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 9;
    for (int dy = 0; dy < 3; ++dy)
      for (int dx = 0; dx < 3; ++dx) g.a_row_off[dy * 3 + dx] = -(dy * 9 + dx);
    set_window(g, 9);
    if ((rc = make_tmap(&ta, net->d_pre3, R, 64, 64, g.a_win_rows, 128))) return rc;
    if ((rc = make_tmap(&tb, wbf + off[P_W3], 64, 576, 64, 64, 128))) return rc;
    g.b_kb_per_tap = 1;
    g.b_tap_stride = 64;
    g.N = 64;
    g.M = (int)R;
    g.mask_bits = reinterpret_cast<const uint32_t*>(net->m2);
    g.out = net->d_pre2;
    g.gh = 9; g.gw = 9; g.vh = 9; g.vw = 9;
    g.r_img = 100 * 64; g.r_y = 10 * 64; g.r_x = 64;
    g.colsum = wgrad_window() ? nullptr : ws + P.cs_off[1];  // db2 (window mode: from the conv2 wgrad)
    if ((rc = launch_gemm<64, A_KMAJOR, B_MNMAJOR, 128, true, 1, 0, EPK_DGRAD>(g, ta, tb, s))) return rc;
  }
  // conv2 dgrad: d_pre1 (conv1 21x21 grid) = sum_taps d_pre2[m - off] W2_tap^T * (X1 > 0), inverse s2d
  {
    const long long R = (long long)n * 100;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 4;
    const int offs[4] = {0, 1, 10, 11};
    for (int i = 0; i < 4; ++i) g.a_row_off[i] = -offs[i];
    set_window(g, 4);
    if ((rc = make_tmap(&ta, net->d_pre2, R, 64, 64, g.a_win_rows, 128))) return rc;
    if ((rc = make_tmap(&tb, wbf + off[P_W2], 64, 512, 64, 64, 128))) return rc;
    g.b_kb_per_tap = 1;
    g.b_tap_stride = 128;
    g.N = 128;
    g.M = (int)R;
    g.mask_bits = reinterpret_cast<const uint32_t*>(net->m1);
    g.out = net->d_pre1;
    g.gh = 10; g.gw = 10; g.vh = 10; g.vw = 10;
    g.r_img = 441 * 32; g.r_y = 2 * 21 * 32; g.r_x = 2 * 32;
    g.cdiv = 32; g.cq = 2; g.cs1 = 21 * 32; g.cs2 = 32;
    g.colsum = wgrad_window() ? nullptr : ws + P.cs_off[0];  // window mode: db1 from the conv1 wgrad
    if ((rc = launch_gemm<128, A_KMAJOR, B_MNMAJOR, 128, true, 1, 0, EPK_DGRAD>(g, ta, tb, s))) return rc;
  }
  // weight gradients
  auto wgrad = [&](int i, const void* X, long long xrows, int xcols, int atoms_per_shift, int nshifts,
                   const int* offs, const void* dY, int ncols) -> int {
    const WgPlan& w = P.wg[i];
    int r;
    if ((r = make_tmap(&ta, X, xrows, xcols, 64, 64, 128))) return r;
    GemmArgs g = base_args();
    g.m_tiles = w.m_tiles;
    g.n_tiles = w.n_tiles;
    g.splits = w.splits;
    g.num_kb = w.num_kb;
    g.kb_per_split = w.kb_per;
    g.a_atoms_per_shift = atoms_per_shift;
    g.a_nshifts = nshifts;
    for (int k = 0; k < nshifts; ++k) g.a_row_off[k] = offs[k];
    g.N = w.Npad;
    g.M = (int)w.Mpad;
    g.out_f32 = 1;
    g.out = ws + w.off;
    g.split_stride = w.Mpad * w.Npad;
    g.r_img = w.Npad;
    if (ncols == 32) {
      if ((r = make_tmap(&tb, dY, xrows, 32, 32, 64, 64))) return r;
      return launch_gemm<32, A_MNMAJOR, B_MNMAJOR, 64, false, 0, 0, EPK_F32>(g, ta, tb, s);
    }
    if ((r = make_tmap(&tb, dY, xrows, 64, 64, 64, 128))) return r;
    return launch_gemm<64, A_MNMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s);
  };
  // conv weight gradients, window kernel: X window + dY box per K-block feed every m-tile
  auto wgrad_win = [&](int i, const void* X, long long xrows, int xcols, int nshifts, const int* offs,
                       const void* dY, int ncols) -> int {
    const WgPlan& w = P.wg[i];
    WgArgs g;
    memset(&g, 0, sizeof(g));
    g.num_kb = w.num_kb;
    g.kb_per_split = w.kb_per;
    g.splits = w.splits;
    g.a_cb = xcols / 64;
    g.nshifts = nshifts;
    g.atoms_per_shift = xcols / 64;
    int mx = 0;
    for (int k = 0; k < nshifts; ++k) {
      g.row_off[k] = offs[k];
      mx = offs[k] > mx ? offs[k] : mx;
    }
    g.min_off = 0;
    g.win_rows = (64 + mx + 7) & ~7;
    g.Mpad = (int)w.Mpad;
    g.N = w.Npad;
    // the atom after the taps: bias rows (conv3; conv1 with BP_CONV1_ONES)
    g.ones_atom = i == 1 || (i == 0 && !conv1_ones()) ? -1 : nshifts * (xcols / 64);
    g.out = ws + w.off;
    if (i == 0 && !conv1_ones()) g.colsum = ws + P.cs_off[0];  // db1: the column-sum warp
    if (i == 1) g.colsum = ws + P.cs_off[1];                     // db2: the column-sum warp
    int r;
    if ((r = make_tmap(&ta, X, xrows, xcols, 64, g.win_rows, 128))) return r;
    if (ncols == 32) {
      if ((r = make_tmap(&tb, dY, xrows, 32, 32, 64, 64))) return r;
      return conv1_ones() ? launch_wgrad_win<32, 64, 3, 0, 1, 88>(g, ta, tb, s)
                          : launch_wgrad_win<32, 64, 2, 0, 1, 88>(g, ta, tb, s);
    }
    if ((r = make_tmap(&tb, dY, xrows, 64, 64, 64, 128))) return r;
    return i == 1 ? launch_wgrad_win<64, 128, 4, 0, 2, 80>(g, ta, tb, s)
                  : launch_wgrad_win<64, 128, 5, 0, 1, 88>(g, ta, tb, s);
  };
  {
    const int o1[4] = {0, 1, 21, 22};
    const int o2[4] = {0, 1, 10, 11};
    int o3[9];
    for (int dy = 0; dy < 3; ++dy)
      for (int dx = 0; dx < 3; ++dx) o3[dy * 3 + dx] = dy * 9 + dx;
    if (src && conv1_u8() && (net->flags & BP_NET_NO_X0)) {
      // conv1: windows converted on chip from the u8 frames (no X0 grid)
      const WgPlan& w = P.wg[0];
      WgArgs g;
      memset(&g, 0, sizeof(g));
      g.num_kb = w.num_kb;
      g.kb_per_split = w.kb_per;
      g.splits = w.splits;
      g.a_cb = 1;
      g.nshifts = 4;
      g.atoms_per_shift = 1;
      for (int k = 0; k < 4; ++k) g.row_off[k] = o1[k];
      g.min_off = 0;
      g.win_rows = (64 + 22 + 7) & ~7;
      g.Mpad = (int)w.Mpad;
      g.N = w.Npad;
      g.ones_atom = wgrad_window() && conv1_ones() ? 4 : -1;
      g.out = ws + w.off;
      if (wgrad_window() && !conv1_ones()) g.colsum = ws + P.cs_off[0];  // db1: the column-sum warp
      g.u8 = src->frames;
      g.u8_index = src->plane_index;
      g.u8_planes = src->num_planes;
      g.u8_rows = (long long)n * 441;
      if ((rc = make_tmap(&tb, net->d_pre1, (long long)n * 441, 32, 32, 64, 64))) return rc;
      if ((rc = wgrad_window() && conv1_ones() ? launch_wgrad_win<32, 64, 3, 1, 1, 88>(g, tb, tb, s)
                               : launch_wgrad_win<32, 64, 2, 1, 1, 88>(g, tb, tb, s)))
        return rc;
    } else if (wgrad_window()) {
      if ((rc = wgrad_win(0, net->x0, (long long)n * 441, 64, 4, o1, net->d_pre1, 32))) return rc;
    } else if ((rc = wgrad(0, net->x0, (long long)n * 441, 64, 1, 4, o1, net->d_pre1, 32))) {
      return rc;
    }
    if (wgrad_window()) {
      if ((rc = wgrad_win(1, net->x1, (long long)n * 100, 128, 4, o2, net->d_pre2, 64))) return rc;
      if ((rc = wgrad_win(2, net->x2, (long long)n * 81, 64, 9, o3, net->d_pre3, 64))) return rc;
    } else {
      if ((rc = wgrad(1, net->x1, (long long)n * 100, 128, 2, 4, o2, net->d_pre2, 64))) return rc;
      if ((rc = wgrad(2, net->x2, (long long)n * 81, 64, 1, 9, o3, net->d_pre3, 64))) return rc;
    }
    if (!heads_wgrad_done && (rc = heads_wgrad(net, n, head_in, P, ws, s, 0))) return rc;
  }
  // deterministic finalize: conv weight grads (transpose to [Cout][K]), heads, biases
  {
    FinArgs f;
    memset(&f, 0, sizeof(f));
    const int pw[3] = {P_W1, P_W2, P_W3};
    const int Mv[3] = {256, 512, 576};
    const int Nv[3] = {32, 64, 64};
    int k = 0;
    for (int i = 0; i < 3; ++i) {
      const WgPlan& w = P.wg[i];
      f.job[k++] = {ws + w.off, grads + off[pw[i]], 0, w.splits, Mv[i], Nv[i], w.Npad, w.Mpad,
                    i == 0 ? 1.f / 255.f : 1.f};
    }
    {
      const WgPlan& w = P.wg[3];
      f.job[k++] = {ws + w.off, nullptr, 2, w.splits, 513 + A + 1, A + 1, w.Npad, w.Mpad, 1.f};
    }
    // biases.  Window mode: db1 and db2 are the column-sum warp's per-CTA sums of the bf16 dY
    // boxes in the conv1 / conv2 weight-gradient kernels; db3 (and db1 with BP_CONV1_ONES) the
    // all-ones-atom rows of the conv3 (conv1) weight-gradient partials, split-reduced like the
    // weights.  Per-tap mode: from the data-gradient epilogue column sums: db1 from conv2 dgrad
    // (width 128 = 4 groups of 32), db2 from conv3 dgrad, db3 from fc dgrad (3136 = 49 x 64).
    // dbfc always from the heads dgrad.
    const int pb[4] = {P_B1, P_B2, P_B3, P_BFC};
    const int C[4] = {32, 64, 64, 512};
    const int ones_row[3] = {4 * 64, 0, 9 * 64};
    for (int i = 0; i < 4; ++i) {
      if ((i == 0 && wgrad_window() && !conv1_ones()) || (i == 1 && wgrad_window())) {
        // the conv1 / conv2 window wgrad's per-CTA dY column sums
        f.job[k++] = {ws + P.cs_off[i], grads + off[pb[i]], 1, P.wg[i].splits, 1, C[i], 0, 0, 1.f};
      } else if ((i == 2 || (i == 0 && conv1_ones())) && wgrad_window()) {
        const WgPlan& w = P.wg[i];
        f.job[k++] = {ws + w.off + (size_t)ones_row[i] * w.Npad, grads + off[pb[i]], 0, w.splits, 1, C[i],
                      w.Npad, w.Mpad, 1.f};
      } else {
        f.job[k++] = {ws + P.cs_off[i], grads + off[pb[i]], 1, P.cs_rows[i], P.cs_n[i] / C[i], C[i], 0, 0,
                      1.f};
      }
    }
    f.njobs = k;
    f.A = A;
    f.wp_grad = grads + off[P_WP];
    f.bp_grad = grads + off[P_BP];
    f.wv_grad = grads + off[P_WV];
    f.bv_grad = grads + off[P_BV];
    launch_pdl(finalize_kernel, dim3(4 * g_num_sms, k), dim3(256), 0, s, f);
    if ((rc = check_launch("finalize_kernel"))) return rc;
  }
  return BP_OK;
}

static int plan_for(const BpAtariNet* net, int n, NetPlan* P) {
  make_plan(n, g_num_sms, P, wgrad_window());
  if (P->total_floats * sizeof(float) > net->ws_bytes) {
    set_error("atari backward: workspace %zu < %zu bytes", net->ws_bytes, P->total_floats * sizeof(float));
    return BP_ERR_ARG;
  }
  return BP_OK;
}

static int atari_backward(const BpAtariNet* net, int n, const FrameSrc* src, const float* d_logits,
                          const float* d_baseline, float* grads, void* stream) {
  if (int e = check_net(net, n)) return e;
  if (!src && (net->flags & BP_NET_NO_X0) && conv1_u8()) {
    set_error("atari: this net keeps no X0 grid (BP_NET_NO_X0): use bp_atari_backward_frames");
    return BP_ERR_ARG;
  }
  if (net->use_lstm) {
    set_error("atari: LSTM net -> bp_atari_lstm_backward");
    return BP_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t off[P_COUNT + 1];
  param_offsets(net->num_actions, 0, off);
  NetPlan P;
  int rc;
  if ((rc = plan_for(net, n, &P))) return rc;
  float* ws = reinterpret_cast<float*>(net->ws);
  if ((rc = heads_backward(net, n, d_logits, d_baseline, P, ws, nullptr, s))) return rc;
  return torso_backward(net, n, src, net->core, grads, off, P, ws, s);
}

extern "C" int bp_atari_backward(const BpAtariNet* net, int n, const float* d_logits,
                                 const float* d_baseline, const float* reward,
                                 const int64_t* last_action, float* grads, void* stream) {
  (void)reward;
  (void)last_action;  // (their contribution to the heads gradient comes from the augmented core)
  return atari_backward(net, n, nullptr, d_logits, d_baseline, grads, stream);
}

extern "C" int bp_atari_backward_frames(const BpAtariNet* net, int n, const uint8_t* frames,
                                        const int32_t* plane_index, int num_planes, const float* d_logits,
                                        const float* d_baseline, float* grads, void* stream) {
  if (int e = check_planes(frames, plane_index, num_planes)) return e;
  const FrameSrc src{frames, plane_index, num_planes};
  return atari_backward(net, n, &src, d_logits, d_baseline, grads, stream);
}

// ============================================================ LSTM core
// input projection / weight-gradient operand: wih [G4][576] = [W_ih | b_ih + b_hh | 0], rows >= 4H zero
__global__ void pack_lstm_wih_kernel(const float* __restrict__ wih, const float* __restrict__ bih,
                                     const float* __restrict__ bhh, __nv_bfloat16* __restrict__ dst, int H,
                                     int G4) {
  // one block per output row, one bf16 pair per thread (coalesced row reads / writes).
  // Output row rp = j * 4 + gate holds torch row r = gate * H + j: the gate-interleaved G4
  // order of gx, dgates and the weight-gradient rows (an owner's 4 gates are contiguous)
  // PDL: parameters only -- starts early, waits for its predecessor at the end (as lstm_cl_pack)
  pdl_trigger();
  const int rp = blockIdx.x, k = 2 * threadIdx.x;
  const int r = rp < 4 * H ? (rp & 3) * H + (rp >> 2) : 4 * H;
  auto val = [&](int kk) {
    if (r >= 4 * H) return 0.f;
    return kk < H ? wih[(size_t)r * H + kk] : (kk == H ? bih[r] + bhh[r] : 0.f);
  };
  reinterpret_cast<__nv_bfloat162*>(dst + (size_t)rp * kCoreW)[threadIdx.x] =
      __floats2bfloat162_rn(val(k), val(k + 1));
  pdl_wait();
}

// weight-gradient GEMM outputs [G4][576] -> torch-layout grads of one layer
// (two split-K halves, `half` elements apart, summed in a fixed order)
#ifndef BP_LSTM_WG_SPLITS
#define BP_LSTM_WG_SPLITS 2
#endif
constexpr int kLstmWgSplits = BP_LSTM_WG_SPLITS;  // split-K of the LSTM weight-gradient GEMMs (4: no faster)

__global__ void lstm_scatter_kernel(const float* __restrict__ pih, const float* __restrict__ phh, size_t half,
                                    float* __restrict__ gwih, float* __restrict__ gwhh,
                                    float* __restrict__ gbih, float* __restrict__ gbhh, int H) {
  // one block per torch gate row r (= GEMM row rp = j * 4 + gate, gate-interleaved order),
  // threads over the hidden columns (coalesced)
  pdl_trigger();  // the next GEMM may set up (it waits for this kernel)
  pdl_wait();     // the weight-gradient partials
  const int r = blockIdx.x;
  const int rp = (r % H) * 4 + r / H;
  for (int k = threadIdx.x; k < H; k += blockDim.x) {
    const size_t o = (size_t)rp * kCoreW + k;
    float si = pih[o], sh = phh[o];
#pragma unroll
    for (int q = 1; q < kLstmWgSplits; ++q) {  // fixed order
      si += pih[o + q * half];
      sh += phh[o + q * half];
    }
    gwih[(size_t)r * H + k] = si;
    gwhh[(size_t)r * H + k] = sh;
  }
  if (threadIdx.x == 0) {
    const size_t o = (size_t)rp * kCoreW + H;
    float b = pih[o];
#pragma unroll
    for (int q = 1; q < kLstmWgSplits; ++q) b += pih[o + q * half];
    gbih[r] = b;
    gbhh[r] = b;
  }
}

// d_fc [n][512] bf16 = dcore[:, :512] * relu mask; bias-gradient partials per 32-row group
__global__ void __launch_bounds__(128) lstm_dfc_kernel(const float* __restrict__ dcore,
                                                       const uint32_t* __restrict__ mc,
                                                       __nv_bfloat16* __restrict__ d_fc,
                                                       float* __restrict__ colsum, int n) {
  // rows [32*grp, 32*grp + 32), one column per thread; the 32 loads are independent
  pdl_trigger();  // the torso backward's first GEMM may set up (it waits for this kernel)
  pdl_wait();     // the layer-0 input gradient
  const int grp = blockIdx.x, c = blockIdx.y * blockDim.x + threadIdx.x;
  float s = 0.f;
  const int rows = n - grp * 32 < 32 ? n - grp * 32 : 32;
  if (rows <= 0) {  // padding groups of the partial layout (the finalize reads their zeros)
    colsum[(size_t)grp * 512 + c] = 0.f;
    return;
  }
  float x[32];
  uint32_t w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {  // every load issued before the first use
    const size_t m = (size_t)grp * 32 + (i < rows ? i : 0), bit = m * kCoreW + c;
    x[i] = __ldg(dcore + m * kCoreW + c);
    w[i] = __ldg(mc + (bit >> 5)) >> (bit & 31);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < rows) {
      const float v = (w[i] & 1u) ? x[i] : 0.f;
      d_fc[((size_t)grp * 32 + i) * 512 + c] = __float2bfloat16_rn(v);
      s += v;
    }
  }
  colsum[(size_t)grp * 512 + c] = s;
}

// cooperative path: recurrent partial sums; cluster path: packed W_hh fragments of both layers
extern "C" size_t bp_lstm_partial_floats(int hidden) {
  const size_t coop = lstm_part_floats(hidden), cl = 2 * lstm_cl_frag_words();
  return coop > cl ? coop : cl;
}

// cluster recurrence when 16-CTA clusters are available (bp_lstm_set_mode overrides)
static bool lstm_use_cluster() {
  if ((g_lstm_mode & 15) == 1) return false;
  return lstm_cluster_batch() > 0;
}

extern "C" int bp_lstm_cluster_active(void) { return lstm_use_cluster() ? 1 : 0; }
extern "C" int bp_lstm_cluster_capacity(void) { return lstm_cluster_batch() / 8; }

static int lstm_g4(int H) { return (4 * H + 127) & ~127; }

static int check_lstm(const BpAtariNet* net, const BpLstmCore* core, int T1, int B) {
  if (int e = check_net(net, T1 * B)) return e;
  if (!net->use_lstm || !core || core->hidden != 513 + net->num_actions || T1 * B > core->max_rows) {
    set_error("lstm: net / core mismatch (use_lstm %d, hidden %d, rows %d of %d)", net->use_lstm,
              core ? core->hidden : -1, T1 * B, core ? core->max_rows : -1);
    return BP_ERR_ARG;
  }
  return BP_OK;
}

static int atari_lstm_forward(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                              const uint8_t* frames, const int32_t* plane_index, int num_planes,
                              const float* reward, const int64_t* last_action, const uint8_t* done,
                              const float* params, const float* h0, const float* c0, float* logits,
                              float* baseline, float* hN, float* cN, void* stream,
                              const SampleSpec* smp = nullptr) {
  if (int e = check_lstm(net, core, T1, B)) return e;
  if (int e = check_planes(frames, plane_index, num_planes)) return e;
  cudaStream_t s = (cudaStream_t)stream;
  const int n = T1 * B, H = core->hidden, G4 = lstm_g4(H);
  int64_t off[P_COUNT + 1];
  param_offsets(net->num_actions, 1, off);
  int rc;
  if ((rc = torso_forward(net, n, frames, plane_index, num_planes, reward, last_action, params, off, s, 1,
                          smp ? smp->seed_state : nullptr)))
    return rc;
  __nv_bfloat16* wih = reinterpret_cast<__nv_bfloat16*>(core->wih);
  const size_t wsz = (size_t)G4 * kCoreW;
  // layer l's input-weight operand; layer 1's packing (and its W_hh fragments below) run as
  // PDL successors of layer 0's recurrence, on the SMs its clusters leave free
  auto pack_wih = [&](int l) {
    const int pw = l ? P_WIH1 : P_WIH0, pb = l ? P_BIH1 : P_BIH0, pc = l ? P_BHH1 : P_BHH0;
    launch_pdl(pack_lstm_wih_kernel, dim3(G4), dim3(kCoreW / 2), 0, s, params + off[pw], params + off[pb],
               params + off[pc], wih + l * wsz, H, G4);
    return check_launch("pack_lstm_wih_kernel");
  };
  if ((rc = pack_wih(0))) return rc;
  auto bfp = [&](void* base, int l) {
    return reinterpret_cast<__nv_bfloat16*>(base) + (size_t)l * core->max_rows * kCoreW;
  };
  const bool cl = lstm_use_cluster();
  // layer 0's W_hh fragments: packed beside layer 0's W_ih operand (both read parameters only
  // and start at their predecessor's trigger) instead of between the gx GEMM and the recurrence
  if (cl && (rc = lstm_cl_pack(params + off[P_WHH0], H, reinterpret_cast<uint32_t*>(core->part), s))) return rc;
  for (int l = 0; l < 2; ++l) {
    if (l == 1) {
      if (cl && (rc = lstm_cl_pack(params + off[P_WHH1], H,
                                   reinterpret_cast<uint32_t*>(core->part) + lstm_cl_frag_words(), s)))
        return rc;
      if ((rc = pack_wih(1))) return rc;
    }
    // gx [n][G4] = x_aug [n][576] . wih^T (biases through the ones column)
    CUtensorMap ta, tb;
    const void* x = l ? (const void*)bfp(core->out, 0) : net->core;
    if ((rc = make_tmap(&ta, x, n, kCoreW, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, wih + l * wsz, G4, kCoreW, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (n + 127) / 128;
    g.n_tiles = G4 / 64;
    g.num_kb = g.kb_per_split = kCoreW / 64;
    g.a_cb = kCoreW / 64;
    g.N = G4;
    g.M = n;
    g.out_f32 = 1;
    g.out = core->gx;
    g.r_img = G4;
    if ((rc = launch_gemm<64, A_KMAJOR, B_KMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s))) return rc;
    const int pass = cl ? lstm_cluster_batch() : kLstmB;
    for (int b0 = 0; b0 < B; b0 += pass) {
      LstmFwdArgs a;
      a.H = H;
      a.B = B - b0 < pass ? B - b0 : pass;
      a.ldb = B;
      a.b0 = b0;
      a.T1 = T1;
      a.whh = params + off[l ? P_WHH1 : P_WHH0];
      a.gx = core->gx;
      a.gx_ld = G4;
      a.done = done;
      a.h0 = h0 + (size_t)l * B * H;
      a.c0 = c0 + (size_t)l * B * H;
      a.hx = core->hx;
      // per layer [max_rows][8H] f32: the cluster path's [rows][H][8] act8 records, or the
      // cooperative path's [rows][4H] gates in its first half
      a.gates = core->gates + (size_t)l * core->max_rows * 8 * H;
      a.act8 = a.gates;
      a.cseq = core->cseq + (size_t)l * core->max_rows * H;
      a.out_aug = bfp(core->out, l);
      a.hprev_aug = bfp(core->hprev, l);
      a.aug_ld = kCoreW;
      a.hN = hN + (size_t)l * B * H;
      a.cN = cN + (size_t)l * B * H;
      a.dbg = g_lstm_mode >> 4;
      a.wfrag = reinterpret_cast<const uint32_t*>(core->part) + (size_t)l * lstm_cl_frag_words();
      if ((rc = cl ? lstm_cl_launch_fwd(a, s) : lstm_launch_fwd(a, s))) return rc;
    }
  }
  return heads_forward(net, n, bfp(core->out, 1), logits, baseline, s, smp);
}

extern "C" int bp_atari_lstm_forward(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                                     const uint8_t* frames, const float* reward, const int64_t* last_action,
                                     const uint8_t* done, const float* params, const float* h0,
                                     const float* c0, float* logits, float* baseline, float* hN, float* cN,
                                     void* stream) {
  return atari_lstm_forward(net, core, T1, B, frames, nullptr, 0, reward, last_action, done, params, h0, c0,
                            logits, baseline, hN, cN, stream);
}

extern "C" int bp_atari_lstm_forward_planes(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                                            const uint8_t* planes, const int32_t* plane_index, int num_planes,
                                            const float* reward, const int64_t* last_action,
                                            const uint8_t* done, const float* params, const float* h0,
                                            const float* c0, float* logits, float* baseline, float* hN,
                                            float* cN, void* stream) {
  if (!plane_index) {
    set_error("atari: bp_atari_lstm_forward_planes needs a plane index");
    return BP_ERR_ARG;
  }
  return atari_lstm_forward(net, core, T1, B, planes, plane_index, num_planes, reward, last_action, done, params,
                            h0, c0, logits, baseline, hN, cN, stream);
}

extern "C" int bp_atari_lstm_forward_sample(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                                            const uint8_t* frames, const int32_t* plane_index, int num_planes,
                                            const float* reward, const int64_t* last_action,
                                            const uint8_t* done, const float* params, const float* h0,
                                            const float* c0, uint64_t seed, uint64_t* seed_state,
                                            int greedy, float* logits,
                                            float* baseline, float* hN, float* cN, int64_t* actions,
                                            void* stream) {
  if (!actions) {
    set_error("atari: bp_atari_lstm_forward_sample needs an actions buffer");
    return BP_ERR_ARG;
  }
  const SampleSpec smp{actions, (unsigned long long)seed, reinterpret_cast<unsigned long long*>(seed_state),
                       greedy};
  return atari_lstm_forward(net, core, T1, B, frames, plane_index, plane_index ? num_planes : 0, reward,
                            last_action, done, params, h0, c0, logits, baseline, hN, cN, stream, &smp);
}

extern "C" int bp_atari_lstm_backward(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                                      const float* d_logits, const float* d_baseline, const uint8_t* done,
                                      const float* params, const float* c0, float* grads, void* stream) {
  if (int e = check_lstm(net, core, T1, B)) return e;
  cudaStream_t s = (cudaStream_t)stream;
  const int n = T1 * B, H = core->hidden, G4 = lstm_g4(H);
  int64_t off[P_COUNT + 1];
  param_offsets(net->num_actions, 1, off);
  NetPlan P;
  int rc;
  if ((rc = plan_for(net, n, &P))) return rc;
  float* ws = reinterpret_cast<float*>(net->ws);
  auto bfp = [&](void* base, int l) {
    return reinterpret_cast<__nv_bfloat16*>(base) + (size_t)l * core->max_rows * kCoreW;
  };
  const __nv_bfloat16* wih = reinterpret_cast<const __nv_bfloat16*>(core->wih);
  const size_t wsz = (size_t)G4 * kCoreW;
  // d(out[1]) [n][576] f32 from the heads
  if ((rc = heads_backward(net, n, d_logits, d_baseline, P, ws, core->dh, s))) return rc;
  const bool cl = lstm_use_cluster();
  const int pass = cl ? lstm_cluster_batch() : kLstmB;
  auto dgates = [&](int l) {  // per layer: layer 1's weight gradients read it beside layer 0's recurrence
    return reinterpret_cast<__nv_bfloat16*>(core->dgates) + (size_t)l * core->max_rows * G4;
  };
  // the recurrence of layer l (gradient w.r.t. its output: dh_in) -> dgates(l)
  auto recur = [&](int l, const float* dh_in) -> int {
    for (int b0 = 0; b0 < B; b0 += pass) {
      LstmBwdArgs a;
      a.H = H;
      a.B = B - b0 < pass ? B - b0 : pass;
      a.ldb = B;
      a.b0 = b0;
      a.T1 = T1;
      a.whh = params + off[l ? P_WHH1 : P_WHH0];
      a.gates = core->gates + (size_t)l * core->max_rows * 8 * H;
      a.act8 = a.gates;
      a.cseq = core->cseq + (size_t)l * core->max_rows * H;
      a.c0 = c0 + (size_t)l * B * H;
      a.done = done;
      a.dh_out = dh_in;
      a.dh_ld = kCoreW;
      a.part = core->part;
      a.dgates = dgates(l);
      a.dg_ld = G4;
      a.wfrag = reinterpret_cast<const uint32_t*>(core->part) + (size_t)l * lstm_cl_frag_words() +
                lstm_cl_frag_dir_words();
      if (int r = cl ? lstm_cl_launch_bwd(a, s) : lstm_launch_bwd(a, s)) return r;
    }
    return BP_OK;
  };
  // weight gradients of layer l: D[r][k] = sum_rows dgates[row][r] * X[row][k], X = layer input /
  // previous state.  beside > 0: PDL successors of layer 0's recurrence on at most `beside` CTAs
  // each (the SMs its clusters leave free), waiting for it only at their end
  auto wgrads = [&](int l, int beside) -> int {
    CUtensorMap ta, tb;
    for (int w = 0; w < 2; ++w) {
      const void* X = w == 0 ? (l ? (const void*)bfp(core->out, 0) : net->core) : (const void*)bfp(core->hprev, l);
      if (int r = make_tmap(&ta, dgates(l), n, G4, 64, 64, 128)) return r;
      if (int r = make_tmap(&tb, X, n, kCoreW, 64, 64, 128)) return r;
      GemmArgs g = base_args();
      g.m_tiles = G4 / 128;
      g.n_tiles = kCoreW / 64;
      // split-K (the lstm_scatter_kernel sums the parts in a fixed order): 17 x 9 = 153 tiles
      // would need a second wave for 5 tiles on 148 SMs
      g.splits = kLstmWgSplits;
      g.num_kb = (n + 63) / 64;
      g.kb_per_split = (g.num_kb + kLstmWgSplits - 1) / kLstmWgSplits;
      g.a_atoms_per_shift = G4 / 64;
      g.a_nshifts = 1;
      g.N = kCoreW;
      g.M = G4;
      g.out_f32 = 1;
      g.out = core->wpart + (size_t)w * kLstmWgSplits * G4 * kCoreW;
      g.split_stride = (long long)G4 * kCoreW;
      g.r_img = kCoreW;
      if (beside > 0) {
        g.max_ctas = beside;
        g.pdl_late = 1;
      }
      if (int r = launch_gemm<64, A_MNMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s)) return r;
    }
    launch_pdl(lstm_scatter_kernel, dim3(4 * H), dim3(288), 0, s, (const float*)core->wpart,
               (const float*)(core->wpart + (size_t)kLstmWgSplits * G4 * kCoreW), (size_t)G4 * kCoreW,
                                            grads + off[l ? P_WIH1 : P_WIH0], grads + off[l ? P_WHH1 : P_WHH0],
                                            grads + off[l ? P_BIH1 : P_BIH0], grads + off[l ? P_BHH1 : P_BHH0], H);
    return check_launch("lstm_scatter_kernel");
  };
  // input gradient of layer l: dx [n][576] = dgates [n][G4] . wih [G4][576]
  auto dgrad = [&](int l, float* dx_out) -> int {
    CUtensorMap ta, tb;
    if (int r = make_tmap(&ta, dgates(l), n, G4, 64, 128, 128)) return r;
    if (int r = make_tmap(&tb, wih + l * wsz, G4, kCoreW, 64, 64, 128)) return r;
    GemmArgs g = base_args();
    g.m_tiles = (n + 127) / 128;
    g.n_tiles = kCoreW / 64;
    g.num_kb = g.kb_per_split = G4 / 64;
    g.a_cb = G4 / 64;
    g.N = kCoreW;
    g.M = n;
    g.out_f32 = 1;
    g.out = dx_out;
    g.r_img = kCoreW;
    return launch_gemm<64, A_KMAJOR, B_MNMAJOR, 128, false, 0, 0, EPK_F32>(g, ta, tb, s);
  };
  // layer 1, then layer 0's recurrence with layer 1's weight gradients beside it (cluster path:
  // the recurrence occupies ceil(B / 8) x 16 SMs); dh: d(out[1]) from the heads, dx: d(out[0])
  const int busy = cl ? ((pass < B ? pass : B) + 7) / 8 * 16 : g_num_sms;
  const int spare = (g_num_sms - busy) / 2;  // per weight-gradient GEMM (two run side by side)
  if ((rc = recur(1, core->dh))) return rc;
  // the heads weight gradient needs only G and layer 1's output: beside layer 1's recurrence
  const bool beside = cl && B <= pass && g_num_sms - busy >= 16;
  if (beside && (rc = heads_wgrad(net, n, bfp(core->out, 1), P, ws, s, g_num_sms - busy))) return rc;
  if ((rc = dgrad(1, core->dx))) return rc;
  if ((rc = recur(0, core->dx))) return rc;
  if ((rc = wgrads(1, cl && B <= pass && spare >= 8 ? spare : 0))) return rc;
  if ((rc = dgrad(0, core->dh))) return rc;
  if ((rc = wgrads(0, 0))) return rc;
  // layer-0 input gradient (core->dh) -> d_fc (relu mask) + bias partials for dbfc
  launch_pdl(lstm_dfc_kernel, dim3(P.cs_rows[3], 4), dim3(128), 0, s, (const float*)core->dh,
             reinterpret_cast<const uint32_t*>(net->mc), reinterpret_cast<__nv_bfloat16*>(net->d_fc),
             ws + P.cs_off[3], n);
  if ((rc = check_launch("lstm_dfc_kernel"))) return rc;
  return torso_backward(net, n, nullptr, bfp(core->out, 1), grads, off, P, ws, s, beside);
}

// ============================================================ action sampling
namespace bp {
// same draw as the fused heads epilogue (gumbel_argmax, common.cuh) for any A
__global__ void sample_actions_kernel(const float* __restrict__ logits, int n, int A, uint64_t seed,
                                      int greedy, int64_t* __restrict__ actions) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float* row = logits + (size_t)r * A;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  float best = -INFINITY;
  int arg = 0;
  for (int j0 = 0; j0 < A; j0 += 4) {
    uint4 w = make_uint4(0u, 0u, 0u, 0u);
    if (!greedy) w = philox4x32_10(make_uint4((uint32_t)r, 0u, (uint32_t)(j0 >> 2), 0u), key);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      if (j < A) {
        const float v = row[j];
        const float x = greedy ? v : v + gumbel_of(ws[q]);
        if (x > best) {
          best = x;
          arg = j;
        }
      }
    }
  }
  actions[r] = arg;
}
}  // namespace bp

extern "C" int bp_sample_actions_f32(const float* logits, int n, int A, uint64_t seed, int greedy,
                                     int64_t* actions, void* stream) {
  if (n < 0 || A < 1 || !logits || !actions) {
    bp::set_error("sample_actions: bad args");
    return BP_ERR_ARG;
  }
  if (n == 0) return BP_OK;
  bp::sample_actions_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(logits, n, A, seed,
                                                                               greedy, actions);
  return bp::check_launch("sample_actions_kernel");
}
