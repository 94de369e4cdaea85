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
// Master parameters (f32, flat, see bp_atari_param_offsets) keep the upstream
// torch layouts (state_dict compatible); bp_atari_pack_weights gathers them into
// the bf16 GEMM operand copies and the weight-gradient finalize scatters back.
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "umma_gemm.cuh"

namespace bp {

// ============================================================ param layout
enum {
  P_W1, P_B1, P_W2, P_B2, P_W3, P_B3, P_WFC, P_BFC, P_WP, P_BP, P_WV, P_BV, P_COUNT
};

static void param_offsets(int A, int64_t* off) {
  const int64_t core = 512 + 1 + A;
  const int64_t sizes[P_COUNT] = {256 * 32, 32, 512 * 64, 64, 576 * 64, 64, 3136 * 512, 512,
                                  A * core, A, core, 1};
  int64_t o = 0;
  for (int i = 0; i < P_COUNT; ++i) {
    off[i] = o;
    o += sizes[i];
  }
  off[P_COUNT] = o;
}

// ============================================================ tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int g_num_sms = 0;

static int init_driver() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

// bf16 row-major [rows][cols]; box {box_cols (inner), box_rows}
static int make_tmap(CUtensorMap* m, const void* ptr, long long rows, long long cols, int box_cols,
                     int box_rows, int swz) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld box=%dx%d", (int)r, rows, cols,
              box_cols, box_rows);
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
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
  return g;
}

template <int BN, int AM, int BM, int BSWZ>
static int launch_gemm(const GemmArgs& g, const CUtensorMap& ta, const CUtensorMap& tb, cudaStream_t s) {
  using Cfg = GemmCfg<BN, AM, BM, BSWZ>;
  auto kern = umma_gemm_kernel<BN, AM, BM, BSWZ>;
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
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  kern<<<grid, kGemmThreads, Cfg::SMEM, s>>>(g, ta, tb);
  return check_launch("umma_gemm_kernel");
}

static int splits_for(int tiles_mn, int num_kb) {
  int sp = (g_num_sms + tiles_mn - 1) / tiles_mn;
  if (sp > num_kb) sp = num_kb;
  return sp < 1 ? 1 : sp;
}

// ============================================================ support kernels

// u8 frames [N,4,84,84] -> X0 [N*21*21, 64] bf16, channel = ci*16 + ry*4 + rx
__global__ void __launch_bounds__(128) frames_s2d_kernel(const uint8_t* __restrict__ frames,
                                                         __nv_bfloat16* __restrict__ x0) {
  __shared__ __align__(16) uint8_t slab[4][4][84];
  const int img = blockIdx.x / 21, Y = blockIdx.x % 21;
  for (int w = threadIdx.x; w < 16 * 21; w += 128) {
    const int row = w / 21, col = w % 21;  // row = ci*4 + ry
    const int ci = row >> 2, ry = row & 3;
    const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(
        frames + (((size_t)img * 4 + ci) * 84 + (4 * Y + ry)) * 84) + col);
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

// G [N][64] bf16 = [d_logits (A) | d_baseline | 0 ...]
__global__ void pack_g_kernel(const float* __restrict__ dlog, const float* __restrict__ dbase,
                              __nv_bfloat16* __restrict__ G, int n, int A) {
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

// ---- torch-layout <-> shifted-GEMM K index.  Master parameters keep the
// upstream torch layouts (conv: [Cout][Cin][kh][kw], fc: [512][3136] with
// features in (c, y, x) order); the GEMMs use K = (tap, input channel).
//   L=1 conv1: k = (dy*2+dx)*64 + ci*16 + ry*4 + rx,  ky = 4dy+ry, kx = 4dx+rx
//   L=2 conv2: k = (dy*2+dx)*128 + (py*2+px)*32 + c,  ky = 2dy+py, kx = 2dx+px
//   L=3 conv3: k = (dy*3+dx)*64 + c
//   L=4 fc   : k = (y*7+x)*64 + c  -> torch feature c*49 + y*7 + x
BP_DEVICE long long torch_w_index(int L, int co, int k) {
  if (L == 1) {
    const int tap = k >> 6, c = k & 63, dy = tap >> 1, dx = tap & 1;
    const int ci = c >> 4, ry = (c >> 2) & 3, rx = c & 3;
    return (((long long)co * 4 + ci) * 8 + 4 * dy + ry) * 8 + 4 * dx + rx;
  } else if (L == 2) {
    const int tap = k >> 7, cc = k & 127, dy = tap >> 1, dx = tap & 1;
    const int q = cc >> 5, c = cc & 31, py = q >> 1, px = q & 1;
    return (((long long)co * 32 + c) * 4 + 2 * dy + py) * 4 + 2 * dx + px;
  } else if (L == 3) {
    const int tap = k >> 6, c = k & 63, dy = tap / 3, dx = tap % 3;
    return (((long long)co * 64 + c) * 3 + dy) * 3 + dx;
  } else {
    const int pos = k >> 6, c = k & 63;
    return (long long)co * 3136 + c * 49 + pos;
  }
}

struct PackJob {
  const float* src;   // torch-layout weight
  __nv_bfloat16* dst;
  int kind;           // 0 fwd [Cout][K]; 1 conv dgrad [Cin][taps*Cout]; 2 fc dgrad [3136][512];
                      // 3 heads fwd Whf[32][512]; 4 heads dgrad Whd[512][64]
  int L, cout, K, cin, taps;
};
struct PackArgs {
  PackJob job[10];
  int njobs;
  const float* wp;
  const float* wv;
  int A, core;
};

__global__ void pack_weights_kernel(const __grid_constant__ PackArgs a) {
  const PackJob& j = a.job[blockIdx.y];
  const long long total = j.kind == 3 ? 32 * 512 : j.kind == 4 ? 512 * 64 : (long long)j.cout * j.K;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    float v;
    if (j.kind == 0) {
      const int co = (int)(i / j.K), k = (int)(i % j.K);
      v = j.src[torch_w_index(j.L, co, k)];
    } else if (j.kind == 1) {
      const int row = j.taps * j.cout;
      const int cin = (int)(i / row), r = (int)(i % row);
      const int tap = r / j.cout, co = r % j.cout;
      v = j.src[torch_w_index(j.L, co, tap * j.cin + cin)];
    } else if (j.kind == 2) {
      const int f = (int)(i / 512), o = (int)(i % 512);
      v = j.src[torch_w_index(4, o, f)];
    } else if (j.kind == 3) {  // Whf[aa][k], aa < 32, k < 512
      const int aa = (int)(i / 512), k = (int)(i % 512);
      v = aa < a.A ? a.wp[(size_t)aa * a.core + k] : (aa == a.A ? a.wv[k] : 0.f);
    } else {  // Whd[k][aa], k < 512, aa < 64
      const int k = (int)(i / 64), aa = (int)(i % 64);
      v = aa < a.A ? a.wp[(size_t)aa * a.core + k] : (aa == a.A ? a.wv[k] : 0.f);
    }
    j.dst[i] = __float2bfloat16_rn(v);
  }
}

// ---- column sums (bias gradients): src bf16 [rows][C] -> partial[cta][C]
struct ColsumJob {
  const __nv_bfloat16* src;
  long long rows;
  int C;
  float* partial;  // [ctas][C]
};
struct ColsumArgs {
  ColsumJob job[4];
  int ctas;  // per job
};

__global__ void __launch_bounds__(256) colsum_kernel(const __grid_constant__ ColsumArgs a) {
  const ColsumJob& j = a.job[blockIdx.y];
  const int groups = j.C / 8;          // 8 columns per thread
  const int rlanes = 256 / groups;     // rows in flight
  const int cg = threadIdx.x % groups, rl = threadIdx.x / groups;
  const long long per = (j.rows + a.ctas - 1) / a.ctas;
  const long long r0 = (long long)blockIdx.x * per, r1 = min(j.rows, r0 + per);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (rl < rlanes) {
    for (long long r = r0 + rl; r < r1; r += rlanes) {
      const uint4 w = __ldcs(reinterpret_cast<const uint4*>(j.src + r * j.C + cg * 8));
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&w);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += __bfloat162float(h[k]);
    }
  }
  __shared__ float red[256][9];
#pragma unroll
  for (int k = 0; k < 8; ++k) red[threadIdx.x][k] = acc[k];
  __syncthreads();
  for (int c = threadIdx.x; c < j.C; c += 256) {
    const int g = c / 8, k = c % 8;
    float s = 0.f;
    for (int l = 0; l < rlanes; ++l) s += red[l * groups + g][k];
    j.partial[(size_t)blockIdx.x * j.C + c] = s;
  }
}

// ---- heads auxiliary gradients: bias, reward column, one-hot columns.
// out partial[cta][(A+1)*(A+2)]: for a in [0, A]: [bias, reward, onehot_0..onehot_{A-1}]
__global__ void __launch_bounds__(512) heads_aux_kernel(const float* __restrict__ dlog,
                                                        const float* __restrict__ dbase,
                                                        const float* __restrict__ reward,
                                                        const int64_t* __restrict__ last_action,
                                                        int n, int A, float* __restrict__ partial) {
  const int nout = (A + 1) * (A + 2);
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    const int a = o / (A + 2), c = o % (A + 2);
    float s = 0.f;
    for (int r = r0; r < r1; ++r) {
      const float gv = a < A ? dlog[(size_t)r * A + a] : dbase[r];
      if (c == 0) s += gv;
      else if (c == 1) s += gv * fminf(fmaxf(reward[r], -1.f), 1.f);
      else if (last_action[r] == c - 2) s += gv;
    }
    partial[(size_t)blockIdx.x * nout + o] = s;
  }
}

// ---- finalize: deterministic reductions of every partial buffer into the f32 grads
struct FinJob {
  const float* partial;
  float* dst;
  int kind;        // 0 split-K [splits][Mpad][N] -> torch-layout dst; 1 colsum [ctas][C]; 2 heads-wgrad; 3 heads-aux
  int L;           // kind 0: layer for torch_w_index
  int splits;      // kind 0/2: splits, kind 1/3: ctas
  int M, N, Npad;  // kind 0/2: valid rows / cols, partial row length; kind 1/3: N = width
  long long Mpad;
  float alpha;
};
struct FinArgs {
  FinJob job[12];
  int njobs;
  int A, core;
  float* wp_grad;  // heads routing
  float* bp_grad;
  float* wv_grad;
  float* bv_grad;
};

__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ FinArgs a) {
  const FinJob& j = a.job[blockIdx.y];
  const long long total = (j.kind == 0 || j.kind == 2) ? (long long)j.M * j.N : j.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    if (j.kind == 0 || j.kind == 2) {
      const long long m = i / j.N, n = i % j.N;
      for (int sp = 0; sp < j.splits; ++sp) s += j.partial[((long long)sp * j.Mpad + m) * j.Npad + n];
      s *= j.alpha;
      if (j.kind == 0) {
        j.dst[torch_w_index(j.L, (int)n, (int)m)] = s;
      } else {  // heads wgrad: D[k][aa] -> dWp[aa][k] / dWv[k]
        if (n < a.A) a.wp_grad[n * a.core + m] = s;
        else if (n == a.A) a.wv_grad[m] = s;
      }
    } else {
      for (int c = 0; c < j.splits; ++c) s += j.partial[(long long)c * j.N + i];
      if (j.kind == 1) {
        j.dst[i] = s;
      } else {  // heads aux: o = aa*(A+2) + c
        const int aa = (int)(i / (a.A + 2)), c = (int)(i % (a.A + 2));
        float* row = aa < a.A ? a.wp_grad + (size_t)aa * a.core : a.wv_grad;
        if (c == 0) {
          if (aa < a.A) a.bp_grad[aa] = s;
          else a.bv_grad[0] = s;
        } else if (c == 1) {
          row[512] = s;
        } else {
          row[513 + (c - 2)] = s;
        }
      }
    }
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
  WgPlan wg[5];  // conv1, conv2, conv3, fc, heads
  size_t colsum_off[4];
  int colsum_ctas;
  size_t aux_off;
  int aux_ctas;
  size_t total_floats;
};

static void make_plan(int n, int A, int sms, NetPlan* P) {
  const long long rows[5] = {(long long)n * 441, (long long)n * 100, (long long)n * 81, n, n};
  const int M[5] = {256, 512, 576, 3136, 512};
  const int BNs[5] = {32, 64, 64, 256, 64};
  const int Ns[5] = {32, 64, 64, 512, 64};
  size_t off = 0;
  for (int i = 0; i < 5; ++i) {
    WgPlan& w = P->wg[i];
    w.m_tiles = (M[i] + 127) / 128;
    w.n_tiles = Ns[i] / BNs[i];
    w.num_kb = (int)((rows[i] + 63) / 64);
    int sp = (sms + w.m_tiles * w.n_tiles - 1) / (w.m_tiles * w.n_tiles);
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
  P->colsum_ctas = 2 * sms;
  const int C[4] = {32, 64, 64, 512};
  for (int i = 0; i < 4; ++i) {
    P->colsum_off[i] = off;
    off += ((size_t)P->colsum_ctas * C[i] + 63) & ~size_t(63);
  }
  P->aux_ctas = 64;
  P->aux_off = off;
  off += ((size_t)P->aux_ctas * (A + 1) * (A + 2) + 63) & ~size_t(63);
  P->total_floats = off;
}

}  // namespace bp

// ============================================================ C ABI
using namespace bp;

// Raw engine entry for unit tests: C[M][N] f32 = A . B^T with
//   a_mn = 0: A stored [M][K] (K-major), 1: A stored [K][M] (MN-major)
//   b_mn = 0: B stored [N][K],           1: B stored [K][N]
// M % 128 == 0 (a_mn=0) or M % 64 == 0 (a_mn=1); K % 64 == 0; N in {32, 64, 128, 256} or a
// multiple of 256 (K-major B) / of 64 (MN-major B).
extern "C" int bp_gemm_bf16_test(const void* A, const void* B, float* C, int M, int N, int K,
                                 int a_mn, int b_mn, int splits, void* stream) {
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
  g.out_f32 = 1;
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
  BP_GT(64, A_MNMAJOR, B_KMAJOR, 128)
#undef BP_GT
  set_error("gemm_test: combination not instantiated (N=%d a_mn=%d b_mn=%d)", N, a_mn, b_mn);
  return BP_ERR_UNSUPPORTED;
}

extern "C" int64_t bp_atari_param_count(int num_actions, int use_lstm) {
  if (num_actions < 1 || num_actions > 31 || use_lstm) return -1;
  int64_t off[P_COUNT + 1];
  param_offsets(num_actions, off);
  return off[P_COUNT];
}

extern "C" int bp_atari_param_offsets(int num_actions, int use_lstm, int64_t* offsets) {
  if (num_actions < 1 || num_actions > 31 || use_lstm || !offsets) {
    set_error("atari: num_actions must be in [1, 31] (LSTM core: separate entry points)");
    return BP_ERR_ARG;
  }
  param_offsets(num_actions, offsets);
  return BP_OK;
}

extern "C" size_t bp_atari_workspace_bytes(int num_actions, int max_frames) {
  if (init_driver()) return 0;
  NetPlan P;
  make_plan(max_frames, num_actions, g_num_sms, &P);
  return P.total_floats * sizeof(float);
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
  const int A = net->num_actions, core = 512 + 1 + A;
  int64_t off[P_COUNT + 1];
  param_offsets(A, off);
  PackArgs a;
  memset(&a, 0, sizeof(a));
  auto bf = [](void* p) { return reinterpret_cast<__nv_bfloat16*>(p); };
  int k = 0;
  // forward B operands [N][K] from master [K][N]  (2D transpose: P=K, Q=N, R=1)
  a.job[k++] = {params + off[P_W1], bf(net->w1f), 0, 1, 32, 256, 64, 4};
  a.job[k++] = {params + off[P_W2], bf(net->w2f), 0, 2, 64, 512, 128, 4};
  a.job[k++] = {params + off[P_W3], bf(net->w3f), 0, 3, 64, 576, 64, 9};
  a.job[k++] = {params + off[P_WFC], bf(net->wfcf), 0, 4, 512, 3136, 3136, 1};
  a.job[k++] = {params + off[P_W2], bf(net->w2d), 1, 2, 64, 512, 128, 4};
  a.job[k++] = {params + off[P_W3], bf(net->w3d), 1, 3, 64, 576, 64, 9};
  a.job[k++] = {params + off[P_WFC], bf(net->wfcd), 2, 4, 512, 3136, 3136, 1};
  a.job[k++] = {nullptr, bf(net->whf), 3, 0, 0, 0, 0, 0};
  a.job[k++] = {nullptr, bf(net->whd), 4, 0, 0, 0, 0, 0};
  a.njobs = k;
  a.wp = params + off[P_WP];
  a.wv = params + off[P_WV];
  a.A = A;
  a.core = core;
  pack_weights_kernel<<<dim3(148, k), 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch("pack_weights_kernel");
}

extern "C" int bp_atari_forward(const BpAtariNet* net, int n, const uint8_t* frames,
                                const float* reward, const int64_t* last_action, const float* params,
                                float* logits, float* baseline, void* stream) {
  if (int e = check_net(net, n)) return e;
  cudaStream_t s = (cudaStream_t)stream;
  const int A = net->num_actions, core = 512 + 1 + A;
  int64_t off[P_COUNT + 1];
  param_offsets(A, off);
  int rc;
  // 1. frames -> space-to-depth bf16
  frames_s2d_kernel<<<n * 21, 128, 0, s>>>(frames, reinterpret_cast<__nv_bfloat16*>(net->x0));
  if ((rc = check_launch("frames_s2d_kernel"))) return rc;
  CUtensorMap ta, tb;
  // 2. conv1: X0 [n*441, 64] x w1f [32, 256] -> relu(./255 + b1) -> X1 (s2d-2 layout)
  {
    const long long R = (long long)n * 441;
    if ((rc = make_tmap(&ta, net->x0, R, 64, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->w1f, 32, 256, 64, 32, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 4;
    g.a_cb = 1;
    const int offs[4] = {0, 1, 21, 22};
    for (int i = 0; i < 4; ++i) g.a_row_off[i] = offs[i];
    g.N = 32;
    g.M = (int)R;
    g.alpha = 1.f / 255.f;
    g.bias = params + off[P_B1];
    g.relu = 1;
    g.out = net->x1;
    g.gh = 21; g.gw = 21; g.vh = 20; g.vw = 20; g.sy = 2; g.sx = 2;
    g.r_img = 100 * 128; g.r_y = 10 * 128; g.r_x = 128; g.r_sub = 32;
    if ((rc = launch_gemm<32, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 3. conv2: X1 [n*100, 128], 2x2 taps on the 10x10 grid -> X2 [n*81, 64]
  {
    const long long R = (long long)n * 100;
    if ((rc = make_tmap(&ta, net->x1, R, 128, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->w2f, 64, 512, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 8;
    g.a_cb = 2;
    const int offs[4] = {0, 1, 10, 11};
    for (int i = 0; i < 4; ++i) g.a_row_off[i] = offs[i];
    g.N = 64;
    g.M = (int)R;
    g.bias = params + off[P_B2];
    g.relu = 1;
    g.out = net->x2;
    g.gh = 10; g.gw = 10; g.vh = 9; g.vw = 9;
    g.r_img = 81 * 64; g.r_y = 9 * 64; g.r_x = 64;
    if ((rc = launch_gemm<64, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 4. conv3: X2 [n*81, 64], 3x3 taps on the 9x9 grid -> X3 [n, 3136] ((y, x, c) order)
  {
    const long long R = (long long)n * 81;
    if ((rc = make_tmap(&ta, net->x2, R, 64, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->w3f, 64, 576, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 9;
    g.a_cb = 1;
    for (int dy = 0; dy < 3; ++dy)
      for (int dx = 0; dx < 3; ++dx) g.a_row_off[dy * 3 + dx] = dy * 9 + dx;
    g.N = 64;
    g.M = (int)R;
    g.bias = params + off[P_B3];
    g.relu = 1;
    g.out = net->x3;
    g.gh = 9; g.gw = 9; g.vh = 7; g.vw = 7;
    g.r_img = 3136; g.r_y = 7 * 64; g.r_x = 64;
    if ((rc = launch_gemm<64, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 5. fc: X3 [n, 3136] x wfcf [512, 3136] -> H = relu(. + bfc) [n, 512]
  {
    if ((rc = make_tmap(&ta, net->x3, n, 3136, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->wfcf, 512, 3136, 64, 256, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (n + 127) / 128;
    g.n_tiles = 2;
    g.num_kb = g.kb_per_split = 49;
    g.a_cb = 49;
    g.N = 512;
    g.M = n;
    g.bias = params + off[P_BFC];
    g.relu = 1;
    g.out = net->h;
    g.r_img = 512;
    if ((rc = launch_gemm<256, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 6. heads: H [n, 512] x whf [32, 512] -> logits [n, A], baseline [n]
  {
    if ((rc = make_tmap(&ta, net->h, n, 512, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->whf, 32, 512, 64, 32, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (n + 127) / 128;
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 8;
    g.a_cb = 8;
    g.N = 32;
    g.M = n;
    g.heads = 1;
    g.A = A;
    g.core = core;
    g.wp = params + off[P_WP];
    g.bp = params + off[P_BP];
    g.wv = params + off[P_WV];
    g.bv = params + off[P_BV];
    g.reward = reward;
    g.last_action = last_action;
    g.logits = logits;
    g.baseline = baseline;
    if ((rc = launch_gemm<32, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  return BP_OK;
}

extern "C" int bp_atari_backward(const BpAtariNet* net, int n, const float* d_logits,
                                 const float* d_baseline, const float* reward,
                                 const int64_t* last_action, float* grads, void* stream) {
  if (int e = check_net(net, n)) return e;
  cudaStream_t s = (cudaStream_t)stream;
  const int A = net->num_actions, core = 512 + 1 + A;
  int64_t off[P_COUNT + 1];
  param_offsets(A, off);
  NetPlan P;
  make_plan(n, A, g_num_sms, &P);
  if (P.total_floats * sizeof(float) > net->ws_bytes) {
    set_error("atari backward: workspace %zu < %zu bytes", net->ws_bytes, P.total_floats * sizeof(float));
    return BP_ERR_ARG;
  }
  float* ws = reinterpret_cast<float*>(net->ws);
  auto bf = [](void* p) { return reinterpret_cast<__nv_bfloat16*>(p); };
  int rc;
  CUtensorMap ta, tb;
  // 1. G = [d_logits | d_baseline | 0] bf16
  pack_g_kernel<<<(n * 8 + 255) / 256, 256, 0, s>>>(d_logits, d_baseline, bf(net->g), n, A);
  if ((rc = check_launch("pack_g_kernel"))) return rc;
  // 2. heads dgrad: d_fc = (G [n,64] x whd [512,64]^T) * (H > 0)
  {
    if ((rc = make_tmap(&ta, net->g, n, 64, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->whd, 512, 64, 64, 256, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (n + 127) / 128;
    g.n_tiles = 2;
    g.num_kb = g.kb_per_split = 1;
    g.N = 512;
    g.M = n;
    g.mask = bf(net->h);
    g.out = net->d_fc;
    g.r_img = 512;
    if ((rc = launch_gemm<256, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 3. fc dgrad: d_pre3 (conv3 9x9 grid) = (d_fc [n,512] x wfcd [3136,512]^T) * (X3 > 0)
  {
    if ((rc = make_tmap(&ta, net->d_fc, n, 512, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->wfcd, 3136, 512, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (n + 127) / 128;
    g.n_tiles = 49;
    g.num_kb = g.kb_per_split = 8;
    g.a_cb = 8;
    g.N = 3136;
    g.M = n;
    g.mask = bf(net->x3);
    g.out = net->d_pre3;
    g.r_img = 81 * 64;
    g.cdiv = 64; g.cq = 7; g.cs1 = 9 * 64; g.cs2 = 64;
    if ((rc = launch_gemm<64, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 4. conv3 dgrad: d_pre2 (conv2 10x10 grid) = sum_taps d_pre3[m - off] w3d * (X2 > 0)
  {
    const long long R = (long long)n * 81;
    if ((rc = make_tmap(&ta, net->d_pre3, R, 64, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->w3d, 64, 576, 64, 64, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 9;
    for (int dy = 0; dy < 3; ++dy)
      for (int dx = 0; dx < 3; ++dx) g.a_row_off[dy * 3 + dx] = -(dy * 9 + dx);
    g.N = 64;
    g.M = (int)R;
    g.mask = bf(net->x2);
    g.out = net->d_pre2;
    g.gh = 9; g.gw = 9; g.vh = 9; g.vw = 9;
    g.r_img = 100 * 64; g.r_y = 10 * 64; g.r_x = 64;
    if ((rc = launch_gemm<64, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 5. conv2 dgrad: d_pre1 (conv1 21x21 grid) = sum_taps d_pre2[m - off] w2d * (X1 > 0), inverse s2d
  {
    const long long R = (long long)n * 100;
    if ((rc = make_tmap(&ta, net->d_pre2, R, 64, 64, 128, 128))) return rc;
    if ((rc = make_tmap(&tb, net->w2d, 128, 256, 64, 128, 128))) return rc;
    GemmArgs g = base_args();
    g.m_tiles = (int)((R + 127) / 128);
    g.n_tiles = 1;
    g.num_kb = g.kb_per_split = 4;
    const int offs[4] = {0, 1, 10, 11};
    for (int i = 0; i < 4; ++i) g.a_row_off[i] = -offs[i];
    g.N = 128;
    g.M = (int)R;
    g.mask = bf(net->x1);
    g.out = net->d_pre1;
    g.gh = 10; g.gw = 10; g.vh = 10; g.vw = 10;
    g.r_img = 441 * 32; g.r_y = 2 * 21 * 32; g.r_x = 2 * 32;
    g.cdiv = 32; g.cq = 2; g.cs1 = 21 * 32; g.cs2 = 32;
    if ((rc = launch_gemm<128, A_KMAJOR, B_KMAJOR, 128>(g, ta, tb, s))) return rc;
  }
  // 6. weight gradients: D[(tap, cin)][cout] = sum_rows X[row + off_tap][cin] dY[row][cout]
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
      return launch_gemm<32, A_MNMAJOR, B_MNMAJOR, 64>(g, ta, tb, s);
    } else if (ncols == 64) {
      if ((r = make_tmap(&tb, dY, xrows, 64, 64, 64, 128))) return r;
      return launch_gemm<64, A_MNMAJOR, B_MNMAJOR, 128>(g, ta, tb, s);
    } else {
      if ((r = make_tmap(&tb, dY, xrows, 512, 64, 64, 128))) return r;
      return launch_gemm<256, A_MNMAJOR, B_MNMAJOR, 128>(g, ta, tb, s);
    }
  };
  {
    const int o1[4] = {0, 1, 21, 22};
    if ((rc = wgrad(0, net->x0, (long long)n * 441, 64, 1, 4, o1, net->d_pre1, 32))) return rc;
    const int o2[4] = {0, 1, 10, 11};
    if ((rc = wgrad(1, net->x1, (long long)n * 100, 128, 2, 4, o2, net->d_pre2, 64))) return rc;
    int o3[9];
    for (int dy = 0; dy < 3; ++dy)
      for (int dx = 0; dx < 3; ++dx) o3[dy * 3 + dx] = dy * 9 + dx;
    if ((rc = wgrad(2, net->x2, (long long)n * 81, 64, 1, 9, o3, net->d_pre3, 64))) return rc;
    const int o0[1] = {0};
    if ((rc = wgrad(3, net->x3, n, 3136, 49, 1, o0, net->d_fc, 512))) return rc;
    if ((rc = wgrad(4, net->h, n, 512, 8, 1, o0, net->g, 64))) return rc;
  }
  // 7. bias gradients (column sums) + heads auxiliary gradients
  {
    ColsumArgs c;
    memset(&c, 0, sizeof(c));
    c.ctas = P.colsum_ctas;
    c.job[0] = {bf(net->d_pre1), (long long)n * 441, 32, ws + P.colsum_off[0]};
    c.job[1] = {bf(net->d_pre2), (long long)n * 100, 64, ws + P.colsum_off[1]};
    c.job[2] = {bf(net->d_pre3), (long long)n * 81, 64, ws + P.colsum_off[2]};
    c.job[3] = {bf(net->d_fc), (long long)n, 512, ws + P.colsum_off[3]};
    colsum_kernel<<<dim3(c.ctas, 4), 256, 0, s>>>(c);
    if ((rc = check_launch("colsum_kernel"))) return rc;
    heads_aux_kernel<<<P.aux_ctas, 512, 0, s>>>(d_logits, d_baseline, reward, last_action, n, A,
                                                 ws + P.aux_off);
    if ((rc = check_launch("heads_aux_kernel"))) return rc;
  }
  // 8. deterministic finalize into the f32 gradient buffer
  {
    FinArgs f;
    memset(&f, 0, sizeof(f));
    const int pw[4] = {P_W1, P_W2, P_W3, P_WFC};
    const int Mv[4] = {256, 512, 576, 3136};
    const int Nv[4] = {32, 64, 64, 512};
    int k = 0;
    for (int i = 0; i < 4; ++i) {
      const WgPlan& w = P.wg[i];
      f.job[k++] = {ws + w.off, grads + off[pw[i]], 0, i + 1, w.splits, Mv[i], Nv[i], w.Npad, w.Mpad,
                    i == 0 ? 1.f / 255.f : 1.f};
    }
    {
      const WgPlan& w = P.wg[4];
      f.job[k++] = {ws + w.off, nullptr, 2, 0, w.splits, 512, A + 1, w.Npad, w.Mpad, 1.f};
    }
    const int pb[4] = {P_B1, P_B2, P_B3, P_BFC};
    for (int i = 0; i < 4; ++i)
      f.job[k++] = {ws + P.colsum_off[i], grads + off[pb[i]], 1, 0, P.colsum_ctas, 0, Nv[i], 0, 0, 1.f};
    f.job[k++] = {ws + P.aux_off, nullptr, 3, 0, P.aux_ctas, 0, (A + 1) * (A + 2), 0, 0, 1.f};
    f.njobs = k;
    f.A = A;
    f.core = core;
    f.wp_grad = grads + off[P_WP];
    f.bp_grad = grads + off[P_BP];
    f.wv_grad = grads + off[P_WV];
    f.bv_grad = grads + off[P_BV];
    finalize_kernel<<<dim3(64, k), 256, 0, s>>>(f);
    if ((rc = check_launch("finalize_kernel"))) return rc;
  }
  return BP_OK;
}

// ============================================================ action sampling
namespace bp {
BP_DEVICE uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void sample_actions_kernel(const float* __restrict__ logits, int n, int A, uint64_t seed,
                                      int greedy, int64_t* __restrict__ actions) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  float best = -INFINITY;
  int arg = 0;
  for (int j = 0; j < A; ++j) {
    float v = logits[(size_t)r * A + j];
    if (!greedy) {
      const uint64_t h = mix64(seed ^ mix64(((uint64_t)r << 8) | (uint64_t)j));
      const float u = ((float)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);  // (0, 1)
      v += -logf(-logf(u));  // Gumbel(0, 1)
    }
    if (v > best) {
      best = v;
      arg = j;
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
