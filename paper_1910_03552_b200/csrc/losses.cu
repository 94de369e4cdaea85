// The north-star loss helpers as fused reduction kernels with their backward:
//   compute_policy_gradient_loss(logits, actions, advantages) = sum_i -log pi_i(a_i) adv_i
//   compute_baseline_loss(advantages)                         = 0.5 sum adv^2
//   compute_entropy_loss(logits)                              = sum_i sum_j pi_ij log pi_ij
// [upstream torchbeast monobeast.py, not vendored].  The in-tree arithmetic they restate is
// beastpipe losses_from_targets (vtrace.py:169-221: pg :194, baseline :195, entropy :196 via
// model.py:212-215) and its exact gradients (d_logits :208-214).
//
// Each forward is ONE HBM-bound pass (logits read once, row in registers / L1): one thread per
// row, f64 per-thread sums, warp and block trees, then the last block reduces the per-block
// partials in a fixed order -- deterministic, no atomics on the value.  Each backward is one
// elementwise pass that reads the upstream scalar gradient from device memory (no host sync).
#include "common.cuh"

namespace bp {

constexpr int kLossThreads = 256;
constexpr int kLossMaxBlocks = 2 * 148;

enum { LK_BASELINE = 0, LK_ENTROPY = 1, LK_PG = 2 };

struct RowLse {
  float m, lse;  // row max, log-sum-exp
};

BP_DEVICE RowLse row_lse(const float* __restrict__ x, int A) {
  float m = -INFINITY;
  for (int j = 0; j < A; ++j) m = fmaxf(m, x[j]);
  float s = 0.f;
  for (int j = 0; j < A; ++j) s += __expf(x[j] - m);
  return RowLse{m, m + __logf(s)};
}

template <int KIND>
__global__ void __launch_bounds__(kLossThreads)
    loss_fwd_kernel(const float* __restrict__ logits, const int64_t* __restrict__ actions,
                    const float* __restrict__ adv, long long rows, int A, double* __restrict__ partials,
                    unsigned* __restrict__ counter, float* __restrict__ out, double* __restrict__ out64,
                    unsigned* __restrict__ status) {
  pdl_wait();
  double acc = 0.0;
  unsigned bad = 0u;
  for (long long i = (long long)blockIdx.x * kLossThreads + threadIdx.x; i < rows;
       i += (long long)gridDim.x * kLossThreads) {
    if constexpr (KIND == LK_BASELINE) {
      const float a = adv[i];
      acc += 0.5 * (double)a * (double)a;
    } else {
      const float* x = logits + i * A;
      const RowLse r = row_lse(x, A);
      if constexpr (KIND == LK_ENTROPY) {
        float s = 0.f;  // sum_j pi_j log pi_j of this row
        for (int j = 0; j < A; ++j) {
          const float lp = x[j] - r.lse;
          s += __expf(lp) * lp;
        }
        acc += (double)s;
      } else {
        const int64_t a = actions[i];
        int aa = (int)a;
        if (a < 0 || a >= A) {  // F.nll_loss rejects out-of-range targets
          bad |= BP_STATUS_ACTION_RANGE;
          aa = 0;
        }
        acc -= (double)(x[aa] - r.lse) * (double)adv[i];
      }
    }
  }
  if (!isfinite(acc)) bad |= BP_STATUS_NONFINITE_LOSS;
  set_status(status, bad);
  acc = warp_sum(acc);
  __shared__ double red[kLossThreads / 32];
  __shared__ bool is_last;
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < kLossThreads / 32; ++k) s += red[k];
    partials[blockIdx.x] = s;
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) s += ((volatile double*)partials)[k];  // fixed order
    *out = (float)s;
    if (out64) *out64 = s;
    *counter = 0u;  // workspace left zeroed (graph-replay safe)
  }
}

// d_logits / d_advantages = grad_out * d(loss)/d(input); grad_out is the autograd scalar
template <int KIND>
__global__ void __launch_bounds__(kLossThreads)
    loss_bwd_kernel(const float* __restrict__ logits, const int64_t* __restrict__ actions,
                    const float* __restrict__ adv, long long rows, int A, const float* __restrict__ grad_out,
                    float* __restrict__ d_in) {
  pdl_wait();
  const float g = *grad_out;
  for (long long i = (long long)blockIdx.x * kLossThreads + threadIdx.x; i < rows;
       i += (long long)gridDim.x * kLossThreads) {
    if constexpr (KIND == LK_BASELINE) {
      d_in[i] = g * adv[i];  // d/dadv 0.5 adv^2
    } else {
      const float* x = logits + i * A;
      float* d = d_in + i * A;
      const RowLse r = row_lse(x, A);
      if constexpr (KIND == LK_ENTROPY) {
        // d/dx_j sum_k p_k lp_k = p_j (lp_j - sum_k p_k lp_k)  (= p_j (lp_j + H), model.py:212-215)
        float s = 0.f;
        for (int j = 0; j < A; ++j) {
          const float lp = x[j] - r.lse;
          s += __expf(lp) * lp;
        }
        for (int j = 0; j < A; ++j) {
          const float lp = x[j] - r.lse;
          d[j] = g * __expf(lp) * (lp - s);
        }
      } else {
        // d/dx_j -lp_a adv = adv (p_j - [j == a])  (advantages are detached upstream)
        const int64_t a = actions[i];
        const float ga = g * adv[i];
        for (int j = 0; j < A; ++j) d[j] = ga * (__expf(x[j] - r.lse) - (j == a ? 1.f : 0.f));
      }
    }
  }
}

static int loss_grid(long long rows) {
  const long long want = (rows + kLossThreads - 1) / kLossThreads;
  return (int)(want < 1 ? 1 : (want > kLossMaxBlocks ? kLossMaxBlocks : want));
}

static int loss_fwd(int kind, const float* logits, const int64_t* actions, const float* adv, long long rows,
                    int A, float* out, double* out64, void* workspace, unsigned* status, void* stream) {
  if (rows < 0 || !out || !workspace || (kind != LK_BASELINE && (!logits || A < 1)) ||
      (kind != LK_ENTROPY && !adv) || (kind == LK_PG && !actions)) {
    set_error("loss helper: bad args (rows %lld, A %d)", rows, A);
    return BP_ERR_ARG;
  }
  unsigned* counter = reinterpret_cast<unsigned*>(workspace);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + 256);
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid(loss_grid(rows)), block(kLossThreads);
  if (kind == LK_BASELINE)
    launch_pdl(loss_fwd_kernel<LK_BASELINE>, grid, block, 0, s, logits, actions, adv, rows, A, partials, counter,
               out, out64, status);
  else if (kind == LK_ENTROPY)
    launch_pdl(loss_fwd_kernel<LK_ENTROPY>, grid, block, 0, s, logits, actions, adv, rows, A, partials, counter,
               out, out64, status);
  else
    launch_pdl(loss_fwd_kernel<LK_PG>, grid, block, 0, s, logits, actions, adv, rows, A, partials, counter, out,
               out64, status);
  return check_launch("loss_fwd_kernel");
}

static int loss_bwd(int kind, const float* logits, const int64_t* actions, const float* adv, long long rows,
                    int A, const float* grad_out, float* d_in, void* stream) {
  if (rows < 0 || !grad_out || !d_in || (kind != LK_BASELINE && (!logits || A < 1)) ||
      (kind != LK_ENTROPY && !adv) || (kind == LK_PG && !actions)) {
    set_error("loss helper backward: bad args (rows %lld, A %d)", rows, A);
    return BP_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  long long want = (rows + kLossThreads - 1) / kLossThreads;
  const dim3 grid((unsigned)(want < 1 ? 1 : (want > 8 * 148 ? 8 * 148 : want))), block(kLossThreads);
  if (kind == LK_BASELINE)
    launch_pdl(loss_bwd_kernel<LK_BASELINE>, grid, block, 0, s, logits, actions, adv, rows, A, grad_out, d_in);
  else if (kind == LK_ENTROPY)
    launch_pdl(loss_bwd_kernel<LK_ENTROPY>, grid, block, 0, s, logits, actions, adv, rows, A, grad_out, d_in);
  else
    launch_pdl(loss_bwd_kernel<LK_PG>, grid, block, 0, s, logits, actions, adv, rows, A, grad_out, d_in);
  return check_launch("loss_bwd_kernel");
}

}  // namespace bp

using namespace bp;

extern "C" size_t bp_loss_workspace_bytes(void) { return 256 + kLossMaxBlocks * sizeof(double); }

extern "C" int bp_pg_loss_f32(const float* logits, const int64_t* actions, const float* advantages, long long rows,
                              int A, float* out, double* out64, void* workspace, unsigned* status, void* stream) {
  return loss_fwd(LK_PG, logits, actions, advantages, rows, A, out, out64, workspace, status, stream);
}
extern "C" int bp_baseline_loss_f32(const float* advantages, long long n, float* out, double* out64,
                                    void* workspace, void* stream) {
  return loss_fwd(LK_BASELINE, nullptr, nullptr, advantages, n, 1, out, out64, workspace, nullptr, stream);
}
extern "C" int bp_entropy_loss_f32(const float* logits, long long rows, int A, float* out, double* out64,
                                   void* workspace, unsigned* status, void* stream) {
  return loss_fwd(LK_ENTROPY, logits, nullptr, nullptr, rows, A, out, out64, workspace, status, stream);
}
extern "C" int bp_pg_loss_bwd_f32(const float* logits, const int64_t* actions, const float* advantages,
                                  long long rows, int A, const float* grad_out, float* d_logits, void* stream) {
  return loss_bwd(LK_PG, logits, actions, advantages, rows, A, grad_out, d_logits, stream);
}
extern "C" int bp_baseline_loss_bwd_f32(const float* advantages, long long n, const float* grad_out,
                                        float* d_advantages, void* stream) {
  return loss_bwd(LK_BASELINE, nullptr, nullptr, advantages, n, 1, grad_out, d_advantages, stream);
}
extern "C" int bp_entropy_loss_bwd_f32(const float* logits, long long rows, int A, const float* grad_out,
                                       float* d_logits, void* stream) {
  return loss_bwd(LK_ENTROPY, logits, nullptr, nullptr, rows, A, grad_out, d_logits, stream);
}
