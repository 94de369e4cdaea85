// Recurrent part of the AtariNet LSTM core: upstream nn.LSTM(H, H, 2) stepped one
// time row at a time with done resets (core_state = notdone_t * core_state before
// step t; TorchBeast monobeast.AtariNet.forward).  The batched input projections
// (x_t W_ih^T + b_ih + b_hh for all rows at once) and the weight / input gradients
// are tcgen05 GEMMs in network.cu; only the serial h_{t-1} -> h_t chain is here.
//
// Persistent cooperative kernels, one per layer and direction, one grid barrier per
// time step.  CTA c owns hidden units [4c, 4c+4) -> the 16 gate rows {gate*H + j}.
//   forward : the CTA's 16 rows of W_hh stay in shared memory (f32, k-major).  Each
//             step it copies h_{t-1} of all units (exchange buffer [H][32], L2) into
//             shared memory with the reset applied, computes its 16 x 32 pre-gate tile
//             (8 warps split K, 4x4 register tiles, fixed-order cross-warp sum), and
//             the thread owning (unit, batch) updates c in a register and publishes h_t.
//   backward: the same 16 rows.  Each step the CTA multiplies its own gate gradients
//             dz_{t+1} (16 x 32, shared memory) into a partial W_hh^T dz for every unit
//             ([32][H] partial per CTA, L2), then after the barrier sums the partials of
//             all CTAs for its own units in a fixed order (deterministic) and forms dz_t.
// All recurrent arithmetic is f32.
#include <cooperative_groups.h>

#include "common.cuh"
#include "lstm.h"

namespace cg = cooperative_groups;

namespace bp {

constexpr int kLstmThreads = 256;
constexpr int kRows = 4 * kLstmU;  // 16 gate rows per CTA

BP_DEVICE float sigm(float x) { return 1.f / (1.f + __expf(-x)); }

static __host__ __device__ int lstm_kp(int H) { return (H + 31) & ~31; }
static __host__ __device__ int lstm_hp(int H) { return (H + 3) & ~3; }

int g_lstm_mode = 0;

int lstm_grid(int H) { return (H + kLstmU - 1) / kLstmU; }
size_t lstm_part_floats(int H) { return (size_t)2 * lstm_grid(H) * kLstmB * lstm_hp(H); }

// --------------------------------------------------------------------------- forward
// optional per-step %globaltimer trace of CTA 0 (diagnostics: bp_lstm_trace)
__device__ unsigned long long* g_lstm_trace = nullptr;

BP_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kLstmThreads, 1) lstm_fwd_kernel(const LstmFwdArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  __shared__ uint64_t hbar;
  const int H = a.H, B = a.B, H4 = 4 * H;
  const int KP = lstm_kp(H), KS = KP / 8;
  const int u0 = blockIdx.x * kLstmU;
  const int nu = min(kLstmU, H - u0);
  float* wt = sm;                      // [KP][16]  W_hh rows (gate*4 + u), k-major
  float* ht = wt + KP * kRows;         // [KP][32]  h_{t-1} (reset applied to the sums), k-major
  float* red = ht + KP * kLstmB;       // [8][16][32] per-warp partial pre-gates
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long* trace = (blockIdx.x == 0 && tid == 0) ? g_lstm_trace : nullptr;
  if (tid == 0) {
    mbar_init(&hbar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < KP * kRows; i += kLstmThreads) {
    const int k = i / kRows, r = i % kRows;
    const int gate = r / kLstmU, u = r % kLstmU;
    wt[i] = (u < nu && k < H) ? a.whh[(size_t)(gate * H + u0 + u) * H + k] : 0.f;
  }
  for (int i = H * kLstmB + tid; i < KP * kLstmB; i += kLstmThreads) ht[i] = 0.f;
  // h0 (transposed to [k][b]; batch columns >= B zero)
  for (int i = tid; i < H * kLstmB; i += kLstmThreads) {
    const int k = i / kLstmB, b = i % kLstmB;
    ht[i] = b < B ? a.h0[(size_t)(a.b0 + b) * H + k] : 0.f;
  }
  const int ou = tid / kLstmB, ob = tid % kLstmB;
  const bool owner = tid < kLstmU * kLstmB && ou < nu && ob < B;
  const int j = u0 + ou;
  float c = 0.f, hown = 0.f;
  // the owner's per-step inputs are loaded one step ahead (off the critical path)
  float gxn[4] = {0.f, 0.f, 0.f, 0.f};
  bool donen = false;
  if (owner) {
    c = a.c0[(size_t)(a.b0 + ob) * H + j];
    hown = a.h0[(size_t)(a.b0 + ob) * H + j];
    const size_t row = (size_t)a.b0 + ob;
#pragma unroll
    for (int gate = 0; gate < 4; ++gate) gxn[gate] = a.gx[row * a.gx_ld + j * 4 + gate];
    donen = a.done[row];
  }
  const int rg = lane >> 3, bg = lane & 7;
  uint32_t hphase = 0;
  __syncthreads();
  for (int t = 0; t < a.T1; ++t) {
    const size_t trow = (size_t)t * a.ldb + a.b0;
    if (trace) trace[t * 4 + 0] = gtimer();
    if (t > 0) {  // h_{t-1} of every unit: one bulk copy of the exchange buffer
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        fence_proxy_async_smem();
        mbar_expect_tx(&hbar, (uint32_t)(H * kLstmB * sizeof(float)));
        bulk_g2s(ht, a.hx + (size_t)((t - 1) & 1) * H * kLstmB, (uint32_t)(H * kLstmB * sizeof(float)), &hbar);
      }
      mbar_wait_parity(&hbar, hphase);
      hphase ^= 1;
    }
    if (trace) trace[t * 4 + 1] = gtimer();
    {
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
      const float* wp = wt + (size_t)warp * KS * kRows + rg * 4;
      const float* hp = ht + (size_t)warp * KS * kLstmB + bg * 4;
#pragma unroll 4
      for (int k = 0; k < KS; ++k) {
        const float4 w4 = *reinterpret_cast<const float4*>(wp + k * kRows);
        const float4 h4 = *reinterpret_cast<const float4*>(hp + k * kLstmB);
        const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
        const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(wv[i], hv[q], acc[i][q]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        *reinterpret_cast<float4*>(red + ((size_t)warp * kRows + rg * 4 + i) * kLstmB + bg * 4) =
            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
    __syncthreads();
    if (trace) trace[t * 4 + 2] = gtimer();
    if (owner) {
      const size_t row = trow + ob;
      // reset: W_hh (notdone_t * h_{t-1}) = notdone_t * (W_hh h_{t-1})
      const float nd = donen ? 0.f : 1.f;
      float z[4];
#pragma unroll
      for (int gate = 0; gate < 4; ++gate) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[((size_t)w * kRows + gate * kLstmU + ou) * kLstmB + ob];
        z[gate] = nd * s + gxn[gate];
      }
      if (t + 1 < a.T1) {  // next step's inputs
        const size_t nrow = row + a.ldb;
#pragma unroll
        for (int gate = 0; gate < 4; ++gate) gxn[gate] = a.gx[nrow * a.gx_ld + j * 4 + gate];
        donen = a.done[nrow];
      }
      a.hprev_aug[row * a.aug_ld + j] = __float2bfloat16_rn(nd * hown);
      const float ig = sigm(z[0]), fg = sigm(z[1]), gg = tanhf(z[2]), og = sigm(z[3]);
      c = fg * (nd * c) + ig * gg;
      const float h = og * tanhf(c);
      float* act = a.gates + row * H4;
      act[j] = ig;
      act[H + j] = fg;
      act[2 * H + j] = gg;
      act[3 * H + j] = og;
      a.cseq[row * H + j] = c;
      __stcg(a.hx + (size_t)(t & 1) * H * kLstmB + (size_t)j * kLstmB + ob, h);
      a.out_aug[row * a.aug_ld + j] = __float2bfloat16_rn(h);
      hown = h;
      if (t == a.T1 - 1) {
        a.hN[(size_t)(a.b0 + ob) * H + j] = h;
        a.cN[(size_t)(a.b0 + ob) * H + j] = c;
      }
    }
    if (blockIdx.x == 0 && tid < B) {  // bias (ones) column of both augmented sequences
      const size_t row = trow + tid;
      a.out_aug[row * a.aug_ld + H] = __float2bfloat16_rn(1.f);
      a.hprev_aug[row * a.aug_ld + H] = __float2bfloat16_rn(1.f);
    }
    if (trace) trace[t * 4 + 3] = gtimer();
    grid.sync();
  }
}

// --------------------------------------------------------------------------- backward
__global__ void __launch_bounds__(kLstmThreads, 1) lstm_bwd_kernel(const LstmBwdArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int H = a.H, B = a.B, H4 = 4 * H, HP = lstm_hp(H), G = gridDim.x;
  const int u0 = blockIdx.x * kLstmU;
  const int nu = min(kLstmU, H - u0);
  float* w = sm;                     // [16][HP]  W_hh rows (gate*4 + u), row-major
  float* zs = w + kRows * HP;        // [16][32]  own dz_{t+1}
  float4* red = reinterpret_cast<float4*>(zs + kRows * kLstmB);  // [8][32] float4
  const int tid = threadIdx.x;
  unsigned long long* trace = (blockIdx.x == 0 && tid == 0) ? g_lstm_trace : nullptr;
  if (trace) trace += (size_t)4 * a.T1;
  for (int i = tid; i < kRows * HP; i += kLstmThreads) {
    const int r = i / HP, k = i % HP;
    const int gate = r / kLstmU, u = r % kLstmU;
    w[i] = (u < nu && k < H) ? a.whh[(size_t)(gate * H + u0 + u) * H + k] : 0.f;
  }
  for (int i = tid; i < kRows * kLstmB; i += kLstmThreads) zs[i] = 0.f;
  const int ou = tid / kLstmB, ob = tid % kLstmB;
  const bool owner = tid < kLstmU * kLstmB && ou < nu && ob < B;
  const int j = u0 + ou;
  const int nq = HP / 4;
  const int rb = tid % kLstmB, grp = tid / kLstmB;  // reduction role: batch column, CTA group
  float dcf = 0.f;
  __syncthreads();
  for (int t = a.T1 - 1; t >= 0; --t) {
    const size_t trow = (size_t)t * a.ldb + a.b0;
    if (trace) trace[t * 4 + 0] = gtimer();
    // the owner's inputs for this step: issued first, consumed after the exchange
    float dho = 0.f, ig = 0.f, fg = 0.f, gg = 0.f, og = 0.f, c = 0.f, cprev = 0.f, nd = 0.f, ndn = 0.f;
    if (owner) {
      const size_t row = trow + ob;
      dho = a.dh_out[row * a.dh_ld + j];
      const float* act = a.gates + row * H4;
      ig = act[j];
      fg = act[H + j];
      gg = act[2 * H + j];
      og = act[3 * H + j];
      c = a.cseq[row * H + j];
      nd = a.done[row] ? 0.f : 1.f;
      cprev = t == 0 ? a.c0[(size_t)(a.b0 + ob) * H + j] : a.cseq[(row - a.ldb) * H + j];
      if (t + 1 < a.T1) ndn = a.done[row + a.ldb] ? 0.f : 1.f;
    }
    float dh_rec = 0.f;
    if (t + 1 < a.T1) {
      float* part = a.part + (size_t)((t + 1) & 1) * G * kLstmB * HP;
      // partial[b][k] = sum over own rows r of dz_{t+1}[r][b] * W_hh[r][k], all k
      float* mine = part + (size_t)blockIdx.x * kLstmB * HP;
      for (int tile = tid; tile < nq * 8; tile += kLstmThreads) {
        const int jq = tile % nq, bq = tile / nq;
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          const float4 w4 = *reinterpret_cast<const float4*>(w + (size_t)r * HP + jq * 4);
          const float4 z4 = *reinterpret_cast<const float4*>(zs + r * kLstmB + bq * 4);
          const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
          const float zv[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(zv[i], wv[q], acc[i][q]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          __stcg(reinterpret_cast<float4*>(mine + (size_t)(bq * 4 + i) * HP + jq * 4),
                 make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]));
      }
      if (trace) trace[t * 4 + 1] = gtimer();
      grid.sync();
      if (trace) trace[t * 4 + 2] = gtimer();
      {  // fixed-order reduction over CTAs for the own 4 units: thread (b, group); all loads
         // of a thread are issued before the sum (one L2 round trip)
        constexpr int kMaxPer = (kLstmKmax / kLstmU + 7) / 8;
        float4 v[kMaxPer];
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
          const int cta = grp + 8 * q;
          v[q] = cta < G ? __ldcg(reinterpret_cast<const float4*>(part + ((size_t)cta * kLstmB + rb) * HP + u0))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
          s.x += v[q].x;
          s.y += v[q].y;
          s.z += v[q].z;
          s.w += v[q].w;
        }
        red[grp * kLstmB + rb] = s;
      }
      __syncthreads();
      if (owner) {
#pragma unroll
        for (int g = 0; g < 8; ++g) dh_rec += (&red[g * kLstmB + ob].x)[ou];
      }
    }
    if (owner) {
      const size_t row = trow + ob;
      const float dh = dho + ndn * dh_rec;
      const float tc = tanhf(c);
      cprev *= nd;
      const float dc = dh * og * (1.f - tc * tc) + ndn * dcf;
      const float dz[4] = {dc * gg * ig * (1.f - ig), dc * cprev * fg * (1.f - fg), dc * ig * (1.f - gg * gg),
                           dh * tc * og * (1.f - og)};
      dcf = dc * fg;
      __nv_bfloat16* dg = a.dgates + row * a.dg_ld;
#pragma unroll
      for (int gate = 0; gate < 4; ++gate) {
        zs[(gate * kLstmU + ou) * kLstmB + ob] = dz[gate];
        dg[j * 4 + gate] = __float2bfloat16_rn(dz[gate]);
      }
    }
    __syncthreads();
    if (trace) trace[t * 4 + 3] = gtimer();
  }
}

static size_t fwd_smem(int H) { return sizeof(float) * ((size_t)lstm_kp(H) * (kRows + kLstmB) + 8 * kRows * kLstmB); }
static size_t bwd_smem(int H) { return sizeof(float) * ((size_t)kRows * lstm_hp(H) + kRows * kLstmB + 8 * kLstmB * 4); }

template <typename Args>
static int coop_launch(const void* fn, const Args& a, size_t smem, const char* name, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    set_error("%s smem %zu: %s", name, smem, cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  const int grid = lstm_grid(a.H);
  int per_sm = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kLstmThreads, smem);
  if (per_sm * sms < grid) {
    set_error("%s: %d CTAs cannot be co-resident (%d per SM x %d SMs)", name, grid, per_sm, sms);
    return BP_ERR_UNSUPPORTED;
  }
  void* args[] = {const_cast<Args*>(&a)};
  e = cudaLaunchCooperativeKernel(fn, grid, kLstmThreads, args, smem, s);
  if (e != cudaSuccess) {
    set_error("%s launch: %s", name, cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  return check_launch(name);
}

static int check_args(int H, int B, int T1) {
  if (H < 1 || H > kLstmKmax || B < 1 || B > kLstmB || T1 < 1) {
    set_error("lstm: H=%d (<= %d), B chunk=%d (<= %d), T1=%d", H, kLstmKmax, B, kLstmB, T1);
    return BP_ERR_ARG;
  }
  return BP_OK;
}

int lstm_launch_fwd(const LstmFwdArgs& a, cudaStream_t s) {
  if (int e = check_args(a.H, a.B, a.T1)) return e;
  return coop_launch((const void*)lstm_fwd_kernel, a, fwd_smem(a.H), "lstm_fwd_kernel", s);
}

extern "C" int bp_lstm_set_mode(int mode) {
  if (mode >= 16) {  // diagnostics: cluster path with debug bits (mode >> 4)
    g_lstm_mode = mode;
    return BP_OK;
  }
  if (mode < 0 || mode > 2) {
    set_error("lstm mode %d (0 auto, 1 cooperative, 2 cluster)", mode);
    return BP_ERR_ARG;
  }
  if (mode == 2 && lstm_cluster_batch() == 0) {
    set_error("lstm: 16-CTA clusters unavailable on this device");
    return BP_ERR_UNSUPPORTED;
  }
  g_lstm_mode = mode;
  return BP_OK;
}

extern "C" int bp_lstm_trace(void* buf) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  cudaError_t e = cudaMemcpyToSymbol(g_lstm_trace, &p, sizeof(p));
  if (e == cudaSuccess && lstm_cl_set_trace(buf) != BP_OK) e = cudaErrorUnknown;
  if (e != cudaSuccess) {
    set_error("lstm trace: %s", cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

int lstm_launch_bwd(const LstmBwdArgs& a, cudaStream_t s) {
  if (int e = check_args(a.H, a.B, a.T1)) return e;
  return coop_launch((const void*)lstm_bwd_kernel, a, bwd_smem(a.H), "lstm_bwd_kernel", s);
}

}  // namespace bp
