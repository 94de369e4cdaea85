// Global-norm clip + RMSProp, replacing SharedModel.apply_gradients
// (pipeline.py:247-251) = clip_global_norm (model.py:224-233) + rmsprop_step
// (model.py:236-268).  Two HBM-bound passes over flat fp32 buffers:
//   1. bp_sumsq_f32        : sum g^2 -> device double (deterministic two-level reduce)
//   2. bp_rmsprop_clip_f32 : reads the norm on device (no host sync), clips and
//                            updates p / square_avg in place (float4 vectorised).
#include "common.cuh"

namespace bp {

constexpr int kOptThreads = 256;
#ifndef BP_SUMSQ_BLOCKS
#define BP_SUMSQ_BLOCKS (2 * 148)  // A/B vs 4 and 8 x 148: within noise
#endif
constexpr int kSumsqBlocks = BP_SUMSQ_BLOCKS;

__global__ void __launch_bounds__(kOptThreads) sumsq_kernel(const float* __restrict__ x, int64_t n,
                                                            double* __restrict__ out,
                                                            double* __restrict__ partials,
                                                            unsigned* __restrict__ counter) {
  pdl_trigger();  // the update may launch once every block has started; it waits for this kernel
  pdl_wait();
  const int64_t tid = (int64_t)blockIdx.x * kOptThreads + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kOptThreads;
  float acc = 0.f;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = tid; i < n4; i += stride) {
      const float4 v = __ldcs(x4 + i);
      acc = fmaf(v.x, v.x, acc);
      acc = fmaf(v.y, v.y, acc);
      acc = fmaf(v.z, v.z, acc);
      acc = fmaf(v.w, v.w, acc);
    }
    for (int64_t i = (n4 << 2) + tid; i < n; i += stride) acc = fmaf(x[i], x[i], acc);
  } else {
    for (int64_t i = tid; i < n; i += stride) acc = fmaf(x[i], x[i], acc);
  }
  double d = warp_sum((double)acc);
  __shared__ double red[kOptThreads / 32];
  __shared__ bool is_last;
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int k = 0; k < kOptThreads / 32; ++k) s += red[k];
    partials[blockIdx.x] = s;
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last) {  // the last block reduces the partials: fixed strided split + fixed tree
    __threadfence();
    double s = 0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += kOptThreads) s += ((volatile double*)partials)[k];
    s = warp_sum(s);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int k = 0; k < kOptThreads / 32; ++k) t += red[k];
      *out = t;
      *counter = 0u;
    }
  }
}

struct ClipScale {
  float scale;
  bool ok;
};

BP_DEVICE ClipScale clip_scale(const double* sumsq, float max_norm, int mode) {
  const double ss = *sumsq;
  ClipScale c{1.f, isfinite(ss) != 0};
  const double norm = sqrt(ss);
  if (mode == 0) {  // beastpipe model.py:229-232
    if (max_norm > 0.f && norm > (double)max_norm) c.scale = (float)((double)max_norm / norm);
  } else if (mode == 1) {  // torch clip_grad_norm_
    const double coef = (double)max_norm / (norm + 1e-6);
    c.scale = (float)(coef < 1.0 ? coef : 1.0);
  }
  return c;
}

BP_DEVICE float rms_one(float& p, float g, float& s, float lr, float alpha, float eps) {
  s = alpha * s + (1.f - alpha) * g * g;
  const float denom = sqrtf(s) + eps;
  const float step = denom != 0.f ? g / denom : 0.f;  // model.py:261-262
  p = p - lr * step;
  return g;
}

__global__ void __launch_bounds__(kOptThreads)
    rmsprop_kernel(float* __restrict__ p, float* __restrict__ g, float* __restrict__ s, int64_t n,
                   const double* __restrict__ sumsq, float max_norm, int mode, float lr_host,
                   const float* __restrict__ lr_dev, float alpha, float eps, int write_grads,
                   float* __restrict__ norm_out, __nv_bfloat16* __restrict__ mirror,
                   unsigned* status, const double* __restrict__ reject_loss) {
  pdl_wait();
  ClipScale cs = clip_scale(sumsq, max_norm, mode);
  // the step's total loss is non-finite (a NaN loss, or a batch violation poisoned it):
  // reject like a non-finite gradient, without a second status bit (the loss kernel set one)
  const bool loss_ok = reject_loss == nullptr || isfinite(*reject_loss);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (norm_out) *norm_out = (float)sqrt(*sumsq);
    if (!cs.ok && loss_ok) set_status(status, BP_STATUS_NONFINITE_GRAD);
  }
  cs.ok = cs.ok && loss_ok;
  if (!cs.ok) return;  // reject the step, params untouched (model.py:251-252)
  const float lr = lr_dev ? *lr_dev : lr_host;
  const float sc = cs.scale;
  const int64_t tid = (int64_t)blockIdx.x * kOptThreads + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kOptThreads;
  const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                     reinterpret_cast<uintptr_t>(s)) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(mirror) & 7u) == 0;
  int64_t start = 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    float4* p4 = reinterpret_cast<float4*>(p);
    float4* g4 = reinterpret_cast<float4*>(g);
    float4* s4 = reinterpret_cast<float4*>(s);
    for (int64_t i = tid; i < n4; i += stride) {
      float4 pv = p4[i], sv = s4[i];
      float4 gv = __ldcs(g4 + i);
      gv.x *= sc; gv.y *= sc; gv.z *= sc; gv.w *= sc;
      rms_one(pv.x, gv.x, sv.x, lr, alpha, eps);
      rms_one(pv.y, gv.y, sv.y, lr, alpha, eps);
      rms_one(pv.z, gv.z, sv.z, lr, alpha, eps);
      rms_one(pv.w, gv.w, sv.w, lr, alpha, eps);
      p4[i] = pv;
      s4[i] = sv;
      if (write_grads) g4[i] = gv;
      if (mirror) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(pv.x, pv.y), hi = __floats2bfloat162_rn(pv.z, pv.w);
        reinterpret_cast<uint2*>(mirror)[i] =
            make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
      }
    }
    start = n4 << 2;
  }
  for (int64_t i = start + tid; i < n; i += stride) {
    float pv = p[i], sv = s[i];
    const float gv = g[i] * sc;
    rms_one(pv, gv, sv, lr, alpha, eps);
    p[i] = pv;
    s[i] = sv;
    if (write_grads) g[i] = gv;
    if (mirror) mirror[i] = __float2bfloat16_rn(pv);
  }
}

// stats read-back buffer: [losses 4 x f64 | status u32 | pad u32 | done tb x u8 | returns tb x f32
// at byte offset 40 + tb (byte stores when that is not 4-byte aligned)]; one element per thread
constexpr int kStatsHead = 40;
__global__ void __launch_bounds__(1024) pack_stats_kernel(const double* __restrict__ losses,
                                                         const uint8_t* __restrict__ done,
                                                         const float* __restrict__ ret, int tb,
                                                         unsigned* __restrict__ status,
                                                         const double* __restrict__ sumsq,
                                                         unsigned* __restrict__ seq_state,
                                                         uint8_t* __restrict__ out) {
  pdl_wait();
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (i0 < 4) reinterpret_cast<double*>(out)[i0] = losses[i0];
  if (i0 == 4) {  // the step's status word: read back, then cleared for the next step
    unsigned st = 0u;
    if (status) {
      st = *status;
      *status = 0u;
    }
    // the optimiser's verdict, derived from the same inputs it uses (rmsprop_kernel: a
    // non-finite norm with a finite total loss), so this pack may run beside the update
    if (sumsq && !isfinite(*sumsq) && isfinite(losses[3])) st |= BP_STATUS_NONFINITE_GRAD;
    reinterpret_cast<unsigned*>(out)[8] = st;
  }
  for (int i = i0; i < tb; i += gridDim.x * blockDim.x) {  // (few blocks: one system fence each)
    out[kStatsHead + i] = done[i] ? 1 : 0;
    if (ret) {
    uint8_t* o = out + kStatsHead + tb;
    if ((tb & 3) == 0) {
      reinterpret_cast<float*>(o)[i] = ret[i];
    } else {
      const uint32_t v = __float_as_uint(ret[i]);
      o[4 * i] = (uint8_t)v;
      o[4 * i + 1] = (uint8_t)(v >> 8);
      o[4 * i + 2] = (uint8_t)(v >> 16);
      o[4 * i + 3] = (uint8_t)(v >> 24);
    }
    }
  }
  // completion word (seq_state != null): the last block to finish publishes the pack's
  // sequence number in word 9 after every block's writes are visible system-wide, so a host
  // thread can spin on the pinned buffer instead of synchronising on an event
  // ONE system-scope fence per pack, by thread 0 of the last block.  Fences are cumulative:
  // each block's barrier + gpu-scope fence orders its writes before its counter increment,
  // and the last block's system fence orders everything it has observed before the sequence
  // store (the split-K semaphore pattern).  A system fence waits for a flush round trip
  // through PCIe: ~1 us idle, but 10-20 us while a pinned H2D copy (the next batch's infeed)
  // saturates the link -- a fence per thread made this kernel 34 us there, one fence 12 us.
  if (seq_state) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&seq_state[0], 1u) == gridDim.x - 1) {
        seq_state[0] = 0u;
        const unsigned s = seq_state[1] + 1u;
        seq_state[1] = s;
        __threadfence_system();
        *reinterpret_cast<volatile unsigned*>(out + 36) = s;
      }
    }
  }
}

}  // namespace bp

using namespace bp;

extern "C" int bp_pack_stats(const double* losses, const uint8_t* done, const float* episode_return, int tb,
                             unsigned* status, const double* sumsq, unsigned* seq_state, void* out,
                             void* stream) {
  if (!losses || !done || !out || tb < 0) {
    set_error("pack_stats: bad args");
    return BP_ERR_ARG;
  }
  const int n = tb > 5 ? tb : 5;
  const int blocks = (n + 8191) / 8192;  // 1024 threads x <= 8 elements per block
  launch_pdl(pack_stats_kernel, dim3(blocks), dim3(1024), 0, (cudaStream_t)stream, losses, done,
             episode_return, tb, status, sumsq, seq_state, reinterpret_cast<uint8_t*>(out));
  return check_launch("pack_stats_kernel");
}

extern "C" size_t bp_sumsq_workspace_bytes(int64_t n) {
  (void)n;
  return 256 + kSumsqBlocks * sizeof(double);
}

extern "C" int bp_sumsq_f32(const float* x, int64_t n, double* sumsq, void* workspace, void* stream) {
  if (n < 0 || !sumsq || !workspace) {
    set_error("sumsq: bad args");
    return BP_ERR_ARG;
  }
  unsigned* counter = reinterpret_cast<unsigned*>(workspace);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + 256);
  int64_t want = (n / 4 + kOptThreads - 1) / kOptThreads;
  int grid = (int)(want < 1 ? 1 : (want > kSumsqBlocks ? kSumsqBlocks : want));
  launch_pdl(sumsq_kernel, dim3(grid), dim3(kOptThreads), 0, (cudaStream_t)stream, x, n, sumsq, partials, counter);
  return check_launch("sumsq_kernel");
}

extern "C" int bp_rmsprop_clip_f32(float* params, float* grads, float* square_avg, int64_t n,
                                   const double* sumsq, float max_norm, int clip_mode, float lr,
                                   const float* lr_dev, float alpha, float eps,
                                   int write_clipped_grads, float* norm_out, void* bf16_mirror,
                                   unsigned* status, const double* reject_if_nonfinite, void* stream) {
  if (n < 0 || !params || !grads || !square_avg || !sumsq || clip_mode < 0 || clip_mode > 2) {
    set_error("rmsprop_clip: bad args");
    return BP_ERR_ARG;
  }
  int64_t want = (n / 4 + kOptThreads - 1) / kOptThreads;
  int grid = (int)(want < 1 ? 1 : (want > 8 * 148 ? 8 * 148 : want));
  launch_pdl(rmsprop_kernel, dim3(grid), dim3(kOptThreads), 0, (cudaStream_t)stream, params, grads, square_avg, n,
             sumsq, max_norm, clip_mode, lr, lr_dev, alpha, eps, write_clipped_grads, norm_out,
             reinterpret_cast<__nv_bfloat16*>(bf16_mirror), status, reject_if_nonfinite);
  return check_launch("rmsprop_kernel");
}
