// Fused V-trace kernels for sm_100a.
//
// One kernel family, three modes:
//   MODE_LOGITS : vtrace.from_logits            (action_log_rhos + vtrace_targets,
//                                                 beastpipe vtrace.py:51-128)
//   MODE_IW     : vtrace.from_importance_weights (vtrace_targets, vtrace.py:94-128)
//   MODE_LOSS   : fused learner loss              (compute_losses, vtrace.py:224-255:
//                                                 V-trace + losses_from_targets :169-221)
//
// Layout: all tensors time-major (T, B[, A]).  A CTA owns a tile of BT batch
// columns for ALL T rows (columns are independent; the scan runs along T).
//
//   phase 1  row-parallel, streamed over T in chunks of TC = 128/BT time rows:
//            warp 0 issues one TMA bulk copy (cp.async.bulk + mbarrier) per
//            contiguous (time row, BT*A) logits span into a 2-4 stage smem ring
//            (cp.async fallback when spans are not 16B multiples); one thread
//            per (t, b) row computes both log-softmaxes (row in registers for
//            A = 6 / 18), gathers the action, and parks log_rho / discount /
//            reward / value in smem scan arrays.
//   phase 2  parallel delta / c precompute, then the serial reverse scan
//            acc = delta_t + gamma_t c_t acc (BT threads, FMA chain only),
//            then parallel vs / pg_advantage outputs.
//   phase 3  (MODE_LOSS) loss partial sums -> deterministic last-block reduce;
//            second streamed pass over the learner logits (L2-resident, already
//            prefetched under phase 2) computes d_logits in smem and writes them
//            back with TMA bulk stores.
#include <cstdio>
#include <cstdarg>
#include <algorithm>

#include "common.cuh"

namespace bp {

int vt3_launch(bool loss, const float* beh, const float* tgt, const int64_t* act, const void* disc_or_done,
               const float* rew, const float* val, const float* boot, int T, int B, int A,
               float clip_rho, float clip_pg_rho, float clip_c, float discount, float pg_cost,
               float baseline_cost, float entropy_cost, int reward_clip, float* vs, float* pg,
               float* log_rhos, float* beh_logp, float* tgt_logp, float* clipped_rhos, float* d_logits,
               float* d_baseline, double* losses, void* workspace, size_t ws_bytes, unsigned* status,
               cudaStream_t s);


enum { MODE_LOGITS = 0, MODE_IW = 1, MODE_LOSS = 2 };

constexpr int kThreads = 128;  // == (t, b) rows per chunk
constexpr int kMaxStages = 4;
constexpr int kCpAsyncStages = 3;
constexpr int kMaxA = 48;
constexpr int kMaxTB = 2048;  // T * BT bound for the smem scan arrays
constexpr size_t kSmemBudget = 100 * 1024;  // -> 2 CTAs / SM

struct VtArgs {
  const float* beh;      // (T,B,A)
  const float* tgt;      // (T,B,A) target / learner logits
  const int64_t* act;    // (T,B)
  const float* disc;     // (T,B)           MODE_LOGITS / MODE_IW
  const uint8_t* done;   // (T,B) done[1:]  MODE_LOSS
  const float* rew;      // (T,B)
  const float* val;      // (T,B) values, or (T+1,B) baseline in MODE_LOSS
  const float* boot;     // (B)             (MODE_LOSS: val + T*B)
  const float* lr_in;    // (T,B)           MODE_IW
  int T, B, A;
  float clip_rho, clip_pg_rho, clip_c;
  float discount, pg_cost, baseline_cost, entropy_cost;
  int reward_clip;
  float* vs;
  float* pg;
  float* log_rhos;
  float* beh_logp;
  float* tgt_logp;
  float* clipped_rhos;
  float* d_logits;
  float* d_baseline;
  double* losses;
  double* partials;  // gridDim.x * 3
  unsigned* counter;
  unsigned* status;
};

__host__ __device__ inline int round_up4(int x) { return (x + 3) & ~3; }

struct SmemPlan {
  int TC, RS, nst;       // time rows per chunk, smem row stride (floats), pipeline stages
  size_t stage_floats;   // per stage, both tensors
  size_t scan_off;       // float offset of the scan arrays
  int n_scan;            // number of T*BT arrays
  size_t bytes;
};

__host__ __device__ inline SmemPlan make_plan(int mode, int BT, int T, int A, bool bulk) {
  SmemPlan p;
  p.TC = kThreads / BT;
  p.RS = round_up4(BT * A);
  const int ntens = (mode == MODE_IW) ? 0 : 2;
  p.stage_floats = (size_t)ntens * p.TC * p.RS;
  p.n_scan = (mode == MODE_LOSS) ? 10 : 6;
  const size_t scan_floats = (size_t)p.n_scan * T * BT + BT;
  if (bulk) {
    p.nst = kMaxStages;
    while (p.nst > 2 && (p.nst * p.stage_floats + scan_floats) * sizeof(float) > kSmemBudget) --p.nst;
  } else {
    p.nst = kCpAsyncStages;
  }
  p.scan_off = p.nst * p.stage_floats;
  p.bytes = (p.scan_off + scan_floats) * sizeof(float);
  return p;
}

// cp.async fallback (unaligned spans / tiny tiles): all threads copy 4 or 16 bytes each
template <bool VEC>
BP_DEVICE void issue_chunk_cpasync(float* stage, const float* src, int RS, int t0, int nt, int b0,
                                   int bw, int B, int A) {
  const int span = bw * A;
  if constexpr (VEC) {
    const int pieces = span >> 2;
    const int total = nt * pieces;
    for (int i = threadIdx.x; i < total; i += kThreads) {
      const int tr = i / pieces;
      const int p = i - tr * pieces;
      cp_async16(stage + tr * RS + 4 * p, src + ((size_t)(t0 + tr) * B + b0) * A + 4 * p);
    }
  } else {
    const int total = nt * span;
    for (int i = threadIdx.x; i < total; i += kThreads) {
      const int tr = i / span;
      const int p = i - tr * span;
      cp_async4(stage + tr * RS + p, src + ((size_t)(t0 + tr) * B + b0) * A + p);
    }
  }
}

struct RowSoftmax {
  float lse;     // log sum exp (max-shifted: m + log s)
  float xa;      // logit of the action
  float ent;     // entropy (only when requested)
  bool finite;
};

// log-softmax statistics of one row x[0..A); AT > 0: A known at compile time
// (row held in registers, vector LDS), AT == 0: runtime A.
template <int AT, bool ENT>
BP_DEVICE RowSoftmax row_softmax(const float* x, int A, int a) {
  RowSoftmax r;
  float m = -INFINITY, sx = 0.f, s = 0.f, sxe = 0.f;
  if constexpr (AT > 0) {
    float v[AT];
    if constexpr (AT % 2 == 0) {
#pragma unroll
      for (int i = 0; i < AT / 2; ++i) {
        const float2 t = reinterpret_cast<const float2*>(x)[i];
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < AT; ++i) v[i] = x[i];
    }
#pragma unroll
    for (int i = 0; i < AT; ++i) {
      m = fmaxf(m, v[i]);
      sx += v[i];
    }
#pragma unroll
    for (int i = 0; i < AT; ++i) {
      const float z = v[i] - m;
      const float e = fast_exp(z);
      s += e;
      if constexpr (ENT) sxe = fmaf(e, z, sxe);
    }
  } else {
    for (int j = 0; j < A; ++j) {
      const float v = x[j];
      m = fmaxf(m, v);
      sx += v;
    }
    for (int j = 0; j < A; ++j) {
      const float z = x[j] - m;
      const float e = fast_exp(z);
      s += e;
      if constexpr (ENT) sxe = fmaf(e, z, sxe);
    }
  }
  const float ls = fast_log(s);
  r.lse = m + ls;
  r.xa = x[a];
  r.ent = ENT ? (ls - sxe / s) : 0.f;
  r.finite = isfinite(sx) && isfinite(r.lse) && (!ENT || isfinite(r.ent));
  return r;
}

template <int AT>
BP_DEVICE void dlogits_row(float* x, int A, int a, float lse, float H, float pa, float ec) {
  // d = pg_cost*adv*(pi - onehot) + ent_cost*pi*(log pi + H)   (vtrace.py:207-210)
  if constexpr (AT > 0) {
#pragma unroll
    for (int j = 0; j < AT; ++j) {
      const float lp = x[j] - lse;
      const float p = fast_exp(lp);
      x[j] = pa * (p - (j == a ? 1.f : 0.f)) + ec * p * (lp + H);
    }
  } else {
    for (int j = 0; j < A; ++j) {
      const float lp = x[j] - lse;
      const float p = fast_exp(lp);
      x[j] = pa * (p - (j == a ? 1.f : 0.f)) + ec * p * (lp + H);
    }
  }
}

template <int BT, bool BULK, bool VEC, int MODE, int AT>
__global__ void __launch_bounds__(kThreads) vtrace_kernel(VtArgs g) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  const int T = g.T, B = g.B, A = (AT > 0) ? AT : g.A;
  const int b0 = blockIdx.x * BT;
  const int bw = min(BT, B - b0);
  const SmemPlan plan = make_plan(MODE, BT, T, A, BULK);
  const int TC = plan.TC, RS = plan.RS, nst = plan.nst;
  const int TB = T * BT;
  float* scan = smem + plan.scan_off;
  float* s_lr = scan;              // log_rho -> pg rho clip
  float* s_disc = scan + TB;
  float* s_rew = scan + 2 * TB;
  float* s_val = scan + 3 * TB;
  float* s_delta = scan + 4 * TB;  // delta -> vs - V
  float* s_dc = scan + 5 * TB;     // gamma*c -> pg advantage
  float* s_lse = scan + 6 * TB;    // MODE_LOSS: learner log Z
  float* s_ent = scan + 7 * TB;    //            entropy
  float* s_tlp = scan + 8 * TB;    //            learner log pi(a)
  int* s_act = reinterpret_cast<int*>(scan + 9 * TB);
  int64_t* s_act64 = reinterpret_cast<int64_t*>(s_delta);  // phase-1 staging in slots 4-5
  float* s_boot = scan + plan.n_scan * TB;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int tl = tid / BT;  // time row within chunk
  const int bl = tid % BT;  // column within tile
  const uint32_t span_bytes = (uint32_t)(bw * A * sizeof(float));
  unsigned bad = 0;

  if constexpr (BULK) {
    if (tid == 0) {
      for (int s = 0; s < nst; ++s) mbar_init(&full_bar[s], 1);
      fence_mbar_init();
    }
  }
  if (tid < bw) {
    const float bv = g.boot[b0 + tid];
    s_boot[tid] = bv;
    if (!isfinite(bv)) bad |= BP_STATUS_NONFINITE_IN;
  }
  __syncthreads();

  const int nchunks = (T + TC - 1) / TC;
  // chunk q < nchunks: phase-1 logits (beh + tgt); q >= nchunks: phase-3 learner logits
  auto issue = [&](int q) {
    const bool p3 = q >= nchunks;
    const int c = p3 ? q - nchunks : q;
    if constexpr (BULK) {
      if (warp == 0 && c < nchunks && (!p3 || MODE == MODE_LOSS)) {
        float* st = smem + (size_t)(q % nst) * plan.stage_floats;
        const int t0 = c * TC, nt = min(TC, T - t0);
        const int ntens = p3 ? 1 : 2;
        if (p3) {
          bulk_wait_read_1();  // the stage's d_logits stores (all but the newest group) have read smem
          __syncwarp();
        }
        if (lane == 0) mbar_expect_tx(&full_bar[q % nst], span_bytes * nt * ntens);
        __syncwarp();
        for (int r = lane; r < nt * ntens; r += 32) {
          const int k = r / nt, tr = r - k * nt;
          const float* src = (p3 || k == 1) ? g.tgt : g.beh;
          bulk_g2s(st + k * TC * RS + tr * RS, src + ((size_t)(t0 + tr) * B + b0) * A, span_bytes,
                   &full_bar[q % nst]);
        }
      }
    } else {
      if (c < nchunks && (!p3 || MODE == MODE_LOSS)) {
        float* st = smem + (size_t)(q % nst) * plan.stage_floats;
        const int t0 = c * TC, nt = min(TC, T - t0);
        if (p3) {
          issue_chunk_cpasync<VEC>(st, g.tgt, RS, t0, nt, b0, bw, B, A);
        } else {
          issue_chunk_cpasync<VEC>(st, g.beh, RS, t0, nt, b0, bw, B, A);
          issue_chunk_cpasync<VEC>(st + TC * RS, g.tgt, RS, t0, nt, b0, bw, B, A);
        }
      }
      cp_async_commit();
    }
  };
  auto wait_chunk = [&](int q) {
    if constexpr (BULK) {
      mbar_wait_parity(&full_bar[q % nst], (uint32_t)((q / nst) & 1));
    } else {
      cp_async_wait<kCpAsyncStages - 1>();
      __syncthreads();
    }
  };

  // ----------------------------------------------------------------- phase 1
  if constexpr (MODE != MODE_IW) {
    // Small (T, BT) inputs of the whole tile are prefetched once, up front, with
    // cp.async straight into the smem scan arrays (thread i owns elements i + 128k,
    // exactly the rows it processes below).  In the cp.async path they join
    // chunk 0's commit group.
    for (int i = tid; i < TB; i += kThreads) {
      const int t = i / BT, b = i % BT;
      if (b < bw) {
        const size_t idx = (size_t)t * B + b0 + b;
        cp_async8(s_act64 + i, g.act + idx);
        cp_async4(s_rew + i, g.rew + idx);
        cp_async4(s_val + i, g.val + idx);
        if constexpr (MODE != MODE_LOSS) cp_async4(s_disc + i, g.disc + idx);
      }
    }
    if constexpr (MODE == MODE_LOSS) {
#pragma unroll 4
      for (int i = tid; i < TB; i += kThreads) {
        const int t = i / BT, b = i % BT;
        if (b < bw) s_disc[i] = __ldg(g.done + (size_t)t * B + b0 + b) ? 0.f : g.discount;
      }
    }
    if constexpr (BULK) cp_async_commit();
    for (int q = 0; q < nst - 1; ++q) issue(q);
    for (int c = 0; c < nchunks; ++c) {
      issue(c + nst - 1);
      const int t = c * TC + tl;
      const bool live = (t < T) && (bl < bw);
      const size_t idx = (size_t)t * B + b0 + bl;
      const int si = t * BT + bl;
      if constexpr (BULK) {
        if (c == 0) cp_async_wait<0>();
      }
      wait_chunk(c);
      if (live) {
        const int64_t a64 = s_act64[si];
        float rv = s_rew[si];
        const float vv = s_val[si], dv = s_disc[si];
        const float* st = smem + (size_t)(c % nst) * plan.stage_floats;
        int a = (int)a64;
        if (a64 < 0 || a64 >= A) {
          bad |= BP_STATUS_ACTION_RANGE;
          a = 0;
        }
        const RowSoftmax rb = row_softmax<AT, false>(st + tl * RS + bl * A, A, a);
        const RowSoftmax rt = row_softmax<AT, MODE == MODE_LOSS>(st + TC * RS + tl * RS + bl * A, A, a);
        const float blp = rb.xa - rb.lse;
        const float tlp = rt.xa - rt.lse;
        const float lr = tlp - blp;
        const float raw_rv = rv;  // finiteness is checked before the clip (fminf drops a NaN)
        if constexpr (MODE == MODE_LOSS) {
          // discount = (float)gamma * ~done, exact (set in the prefetch above)
          if (g.reward_clip) {
            rv = fminf(fmaxf(rv, -1.f), 1.f);
            s_rew[si] = rv;
          }
        } else {
          if (dv < 0.f) bad |= BP_STATUS_NEG_DISCOUNT;
        }
        if constexpr (MODE == MODE_LOSS) {
          // learner step: a non-finite batch field (reward, behaviour logits) is a schema
          // violation (validate_batch, rollout.py:189-192); the learner's own outputs are not
          if (!(rb.finite && isfinite(raw_rv))) bad |= BP_STATUS_BATCH_NONFINITE;
          if (!(rt.finite && isfinite(lr) && isfinite(vv) && isfinite(dv))) bad |= BP_STATUS_NONFINITE_IN;
        } else if (!(rb.finite && rt.finite && isfinite(lr) && isfinite(rv) && isfinite(vv) && isfinite(dv))) {
          bad |= BP_STATUS_NONFINITE_IN;
        }
        s_lr[si] = lr;
        if constexpr (MODE == MODE_LOSS) {
          s_lse[si] = rt.lse;
          s_ent[si] = rt.ent;
          s_tlp[si] = tlp;
          s_act[si] = a;
        } else {
          if (g.log_rhos) g.log_rhos[idx] = lr;
          if (g.beh_logp) g.beh_logp[idx] = blp;
          if (g.tgt_logp) g.tgt_logp[idx] = tlp;
        }
      }
      __syncthreads();  // stage (c % nst) may be refilled next iteration
    }
    // (in MODE_LOSS the loop tail above already issued the first nst-1 phase-3
    //  chunks of learner logits, so they stream in under phase 2)
  } else {
    // MODE_IW: only (T,B) inputs -- straight coalesced loads into smem
    for (int i = tid; i < TB; i += kThreads) {
      const int t = i / BT, b = i % BT;
      if (b < bw) {
        const size_t idx = (size_t)t * B + b0 + b;
        const float lr = g.lr_in[idx], dv = g.disc[idx], rv = g.rew[idx], vv = g.val[idx];
        if (dv < 0.f) bad |= BP_STATUS_NEG_DISCOUNT;
        if (!(isfinite(lr) && isfinite(dv) && isfinite(rv) && isfinite(vv)))
          bad |= BP_STATUS_NONFINITE_IN;
        s_lr[i] = lr;
        s_disc[i] = dv;
        s_rew[i] = rv;
        s_val[i] = vv;
      }
    }
    __syncthreads();
  }

  // ----------------------------------------------------------------- phase 2
  // 2a: delta_t = min(rho_bar, rho)(r + gamma V_{t+1} - V), gamma*c  (vtrace.py:113-117)
  for (int i = tid; i < TB; i += kThreads) {
    const int t = i / BT, b = i % BT;
    if (b < bw) {
      const float rho = fast_exp(s_lr[i]);
      const float cr = fminf(g.clip_rho, rho);
      const float cc = fminf(g.clip_c, rho);
      const float vnext = (t + 1 < T) ? s_val[i + BT] : s_boot[b];
      const float dsc = s_disc[i];
      s_delta[i] = cr * (s_rew[i] + dsc * vnext - s_val[i]);
      s_dc[i] = dsc * cc;
      s_lr[i] = fminf(g.clip_pg_rho, rho);
      if constexpr (MODE != MODE_LOGITS) {
        if (g.clipped_rhos) g.clipped_rhos[(size_t)t * B + b0 + b] = cr;
      }
    }
  }
  __syncthreads();
  // 2b: serial reverse scan, one thread per column (vtrace.py:119-123)
  if (tid < bw) {
    float acc = 0.f;
    int i = (T - 1) * BT + tid;
#pragma unroll 8
    for (int t = T - 1; t >= 0; --t, i -= BT) {
      acc = fmaf(s_dc[i], acc, s_delta[i]);
      s_delta[i] = acc;
    }
  }
  __syncthreads();
  // 2c: vs = acc + V; pg = clip_pg(rho)(r + gamma vs_{t+1} - V) (vtrace.py:124-127)
  double pg_sum = 0.0, base_sum = 0.0, ent_sum = 0.0;
  for (int i = tid; i < TB; i += kThreads) {
    const int t = i / BT, b = i % BT;
    if (b < bw) {
      const float v = s_val[i];
      const float vsv = s_delta[i] + v;
      const float vs_next = (t + 1 < T) ? (s_delta[i + BT] + s_val[i + BT]) : s_boot[b];
      const float pgv = s_lr[i] * (s_rew[i] + s_disc[i] * vs_next - v);
      const size_t idx = (size_t)t * B + b0 + b;
      if (g.vs) g.vs[idx] = vsv;
      if (g.pg) g.pg[idx] = pgv;
      if constexpr (MODE == MODE_LOSS) {
        s_dc[i] = pgv;  // keep for d_logits
        const float dvs = vsv - v;
        pg_sum -= (double)pgv * (double)s_tlp[i];
        base_sum += 0.5 * (double)dvs * (double)dvs;
        ent_sum -= (double)s_ent[i];
        g.d_baseline[idx] = g.baseline_cost * (v - vsv);
      }
    }
  }

  if constexpr (MODE == MODE_LOSS) {
    if (tid < bw) g.d_baseline[(size_t)T * B + b0 + tid] = 0.f;  // bootstrap row: stop-grad
    // ------------------------------------------------------- phase 3a: loss sums
    __shared__ double red[3][kThreads / 32];
    __shared__ bool is_last;
    // any violation in this CTA poisons the loss sums: the total becomes NaN, which rejects
    // the optimiser step on every data-parallel rank after the loss all-reduce
    if (__syncthreads_or(bad != 0u) && tid == 0) pg_sum = __longlong_as_double(0x7ff8000000000000LL);
    pg_sum = warp_sum(pg_sum);
    base_sum = warp_sum(base_sum);
    ent_sum = warp_sum(ent_sum);
    if (lane == 0) {
      red[0][warp] = pg_sum;
      red[1][warp] = base_sum;
      red[2][warp] = ent_sum;
    }
    __syncthreads();  // also orders s_dc (pg advantages) for phase 3b
    if (tid == 0) {
      double a0 = 0, a1 = 0, a2 = 0;
      for (int k = 0; k < kThreads / 32; ++k) {
        a0 += red[0][k];
        a1 += red[1][k];
        a2 += red[2][k];
      }
      g.partials[3 * blockIdx.x + 0] = a0;
      g.partials[3 * blockIdx.x + 1] = a1;
      g.partials[3 * blockIdx.x + 2] = a2;
      __threadfence();
      const unsigned prev = atomicAdd(g.counter, 1u);
      is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last && tid == 0) {
      __threadfence();
      double a0 = 0, a1 = 0, a2 = 0;
      for (int k = 0; k < (int)gridDim.x; ++k) {  // fixed order: deterministic
        a0 += ((volatile double*)g.partials)[3 * k + 0];
        a1 += ((volatile double*)g.partials)[3 * k + 1];
        a2 += ((volatile double*)g.partials)[3 * k + 2];
      }
      const double total = (double)g.pg_cost * a0 + (double)g.baseline_cost * a1 +
                           (double)g.entropy_cost * a2;
      g.losses[0] = a0;
      g.losses[1] = a1;
      g.losses[2] = a2;
      g.losses[3] = total;
      if (!isfinite(total)) bad |= BP_STATUS_NONFINITE_LOSS;
      *g.counter = 0u;  // leave the workspace zeroed (graph-replay safe)
    }

    // ------------------------------------------------------- phase 3b: d_logits
    for (int c = 0; c < nchunks; ++c) {
      const int q = nchunks + c;
      if constexpr (!BULK) issue(q + nst - 1);
      wait_chunk(q);
      float* st = smem + (size_t)(q % nst) * plan.stage_floats;
      const int t0 = c * TC, nt = min(TC, T - t0);
      const int t = t0 + tl;
      if (t < T && bl < bw) {
        const int si = t * BT + bl;
        dlogits_row<AT>(st + tl * RS + bl * A, A, s_act[si], s_lse[si], s_ent[si],
                        g.pg_cost * s_dc[si], g.entropy_cost);
      }
      if constexpr (BULK) {
        fence_proxy_async_smem();
        __syncthreads();
        if (warp == 0) {
          for (int r = lane; r < nt; r += 32)
            bulk_s2g(g.d_logits + ((size_t)(t0 + r) * B + b0) * A, st + r * RS, span_bytes);
          bulk_commit();
        }
        // refill the stage whose stores were issued one iteration ago
        issue(q + nst - 1);
      } else {
        __syncthreads();
        const int span = bw * A;
        if constexpr (VEC) {
          const int pieces = span >> 2, total = nt * pieces;
          for (int i = tid; i < total; i += kThreads) {
            const int tr = i / pieces, p = i - tr * pieces;
            const float4 v = *reinterpret_cast<const float4*>(st + tr * RS + 4 * p);
            st_cs4(reinterpret_cast<float4*>(g.d_logits + ((size_t)(t0 + tr) * B + b0) * A + 4 * p), v);
          }
        } else {
          const int total = nt * span;
          for (int i = tid; i < total; i += kThreads) {
            const int tr = i / span, p = i - tr * span;
            st_cs(g.d_logits + ((size_t)(t0 + tr) * B + b0) * A + p, st[tr * RS + p]);
          }
        }
        __syncthreads();
      }
    }
    if constexpr (BULK) {
      if (warp == 0) bulk_wait_all();
    }
  }
  set_status(g.status, bad);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int pick_bt(int B, int T) {
  int bt = 16;
  while (bt > 1 && (B + bt - 1) / bt < 2 * 148) bt >>= 1;
  if (bt == 2) bt = 1;
  while (bt > 1 && T * bt > kMaxTB) bt >>= 1;
  return bt;
}

template <int BT, bool BULK, bool VEC, int MODE, int AT>
static int launch_cfg(const VtArgs& a, cudaStream_t s) {
  const SmemPlan plan = make_plan(MODE, BT, a.T, a.A, BULK);
  auto kern = vtrace_kernel<BT, BULK, VEC, MODE, AT>;
  if (plan.bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)plan.bytes);
    if (e != cudaSuccess) {
      set_error("vtrace: smem attribute (%zu bytes): %s", plan.bytes, cudaGetErrorString(e));
      return BP_ERR_LAUNCH;
    }
  }
  const int grid = (a.B + BT - 1) / BT;
  kern<<<grid, kThreads, plan.bytes, s>>>(a);
  return check_launch("vtrace_kernel");
}

template <int BT, int MODE, int AT>
static int launch_path(const VtArgs& a, cudaStream_t s, bool vec_ok) {
  // bulk (TMA 1D) path: every per-time-row span is 16B aligned and a multiple of 16 bytes
  const bool spans16 = ((BT * a.A) % 4 == 0) && ((a.B * a.A) % 4 == 0);
  if (MODE != MODE_IW && vec_ok && spans16) return launch_cfg<BT, true, true, MODE, AT>(a, s);
  if (vec_ok && spans16) return launch_cfg<BT, false, true, MODE, AT>(a, s);
  return launch_cfg<BT, false, false, MODE, AT>(a, s);
}

template <int BT, int MODE>
static int launch_a(const VtArgs& a, cudaStream_t s, bool vec_ok) {
  if (MODE == MODE_IW) return launch_path<BT, MODE, 1>(a, s, false);
  if (a.A == 6) return launch_path<BT, MODE, 6>(a, s, vec_ok);
  if (a.A == 18) return launch_path<BT, MODE, 18>(a, s, vec_ok);
  return launch_path<BT, MODE, 0>(a, s, vec_ok);
}

template <int MODE>
static int launch_mode(const VtArgs& a, cudaStream_t s, bool vec_ok) {
  switch (pick_bt(a.B, a.T)) {
    case 16: return launch_a<16, MODE>(a, s, vec_ok);
    case 8: return launch_a<8, MODE>(a, s, vec_ok);
    case 4: return launch_a<4, MODE>(a, s, vec_ok);
    case 1: return launch_a<1, MODE>(a, s, vec_ok);
  }
  return BP_ERR_UNSUPPORTED;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static int check_dims(int T, int B, int A, bool need_a) {
  if (T < 1 || B < 1 || (need_a && A < 1)) {
    set_error("vtrace: bad dims T=%d B=%d A=%d", T, B, A);
    return BP_ERR_ARG;
  }
  if (need_a && A > kMaxA) {
    set_error("vtrace: num_actions %d > %d unsupported", A, kMaxA);
    return BP_ERR_UNSUPPORTED;
  }
  if (T > kMaxTB) {
    set_error("vtrace: unroll length %d > %d unsupported", T, kMaxTB);
    return BP_ERR_UNSUPPORTED;
  }
  return BP_OK;
}

}  // namespace bp

using namespace bp;

extern "C" int bp_vtrace_from_logits_f32(const float* behavior_logits, const float* target_logits,
                                         const int64_t* actions, const float* discounts,
                                         const float* rewards, const float* values,
                                         const float* bootstrap_value, int T, int B, int A,
                                         float clip_rho, float clip_pg_rho, float clip_c,
                                         float* vs, float* pg_advantages, float* log_rhos,
                                         float* behavior_logp, float* target_logp,
                                         unsigned* status, void* stream) {
  if (int e = check_dims(T, B, A, true)) return e;
  if (!(clip_rho > 0.f && clip_pg_rho > 0.f && clip_c > 0.f)) {
    set_error("vtrace: clip thresholds must be > 0");
    return BP_ERR_ARG;
  }
  VtArgs a{};
  a.beh = behavior_logits;
  a.tgt = target_logits;
  a.act = actions;
  a.disc = discounts;
  a.rew = rewards;
  a.val = values;
  a.boot = bootstrap_value;
  a.T = T;
  a.B = B;
  a.A = A;
  a.clip_rho = clip_rho;
  a.clip_pg_rho = clip_pg_rho;
  a.clip_c = clip_c;
  a.vs = vs;
  a.pg = pg_advantages;
  a.log_rhos = log_rhos;
  a.beh_logp = behavior_logp;
  a.tgt_logp = target_logp;
  a.status = status;
  // bandwidth regime: tile-resident kernel (vtrace_tile.cu); other shapes: the generic kernel
  const int rc = vt3_launch(false, behavior_logits, target_logits, actions, discounts, rewards, values,
                            bootstrap_value, T, B, A, clip_rho, clip_pg_rho, clip_c, 0.f, 0.f, 0.f, 0.f, 0,
                            vs, pg_advantages, log_rhos, behavior_logp, target_logp, nullptr, nullptr,
                            nullptr, nullptr, nullptr, 0, status, (cudaStream_t)stream);
  if (rc != BP_ERR_UNSUPPORTED) return rc;
  return launch_mode<MODE_LOGITS>(a, (cudaStream_t)stream,
                                  aligned16(behavior_logits) && aligned16(target_logits));
}

extern "C" int bp_vtrace_from_importance_weights_f32(const float* log_rhos, const float* discounts,
                                                     const float* rewards, const float* values,
                                                     const float* bootstrap_value, int T, int B,
                                                     float clip_rho, float clip_pg_rho,
                                                     float clip_c, float* vs, float* pg_advantages,
                                                     float* clipped_rhos, unsigned* status,
                                                     void* stream) {
  if (int e = check_dims(T, B, 1, false)) return e;
  if (!(clip_rho > 0.f && clip_pg_rho > 0.f && clip_c > 0.f)) {
    set_error("vtrace: clip thresholds must be > 0");
    return BP_ERR_ARG;
  }
  VtArgs a{};
  a.lr_in = log_rhos;
  a.disc = discounts;
  a.rew = rewards;
  a.val = values;
  a.boot = bootstrap_value;
  a.T = T;
  a.B = B;
  a.A = 1;
  a.clip_rho = clip_rho;
  a.clip_pg_rho = clip_pg_rho;
  a.clip_c = clip_c;
  a.vs = vs;
  a.pg = pg_advantages;
  a.clipped_rhos = clipped_rhos;
  a.status = status;
  return launch_mode<MODE_IW>(a, (cudaStream_t)stream, false);
}

extern "C" size_t bp_learner_loss_workspace_bytes(int T, int B, int A) {
  (void)A;
  const int bt = pick_bt(B, T);
  const size_t grid = (size_t)(B + bt - 1) / bt;
  const size_t grid2 = (size_t)(B + 1) / 2;  // tile-resident kernel: <= B / 2 tiles (2-column tiles)
  return 256 + (grid > grid2 ? grid : grid2) * 3 * sizeof(double);
}

extern "C" int bp_learner_loss_f32(const float* learner_logits, const float* learner_baseline,
                                   const float* behavior_logits, const int64_t* actions,
                                   const float* rewards, const uint8_t* done, int T, int B, int A,
                                   float discount, float clip_rho, float clip_pg_rho, float clip_c,
                                   float pg_cost, float baseline_cost, float entropy_cost,
                                   int reward_clip, float* d_logits, float* d_baseline, float* vs,
                                   float* pg_advantages, float* clipped_rhos, double* losses,
                                   void* workspace, unsigned* status, void* stream) {
  if (int e = check_dims(T, B, A, true)) return e;
  if (!(clip_rho > 0.f && clip_pg_rho > 0.f && clip_c > 0.f) || !(discount > 0.f && discount <= 1.f)) {
    set_error("learner_loss: bad config (discount %g, clips %g %g %g)", discount, clip_rho,
              clip_pg_rho, clip_c);
    return BP_ERR_ARG;
  }
  if (!d_logits || !d_baseline || !losses || !workspace) {
    set_error("learner_loss: null output/workspace");
    return BP_ERR_ARG;
  }
  VtArgs a{};
  a.beh = behavior_logits;
  a.tgt = learner_logits;
  a.act = actions;
  a.done = done;
  a.rew = rewards;
  a.val = learner_baseline;
  a.boot = learner_baseline + (size_t)T * B;
  a.T = T;
  a.B = B;
  a.A = A;
  a.clip_rho = clip_rho;
  a.clip_pg_rho = clip_pg_rho;
  a.clip_c = clip_c;
  a.discount = discount;
  a.pg_cost = pg_cost;
  a.baseline_cost = baseline_cost;
  a.entropy_cost = entropy_cost;
  a.reward_clip = reward_clip;
  a.vs = vs;
  a.pg = pg_advantages;
  a.clipped_rhos = clipped_rhos;
  a.d_logits = d_logits;
  a.d_baseline = d_baseline;
  a.losses = losses;
  a.counter = reinterpret_cast<unsigned*>(workspace);
  a.partials = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + 256);
  a.status = status;
  {
    int rc = vt3_launch(true, behavior_logits, learner_logits, actions, done, rewards, learner_baseline,
                        learner_baseline + (size_t)T * B, T, B, A, clip_rho, clip_pg_rho, clip_c,
                        discount, pg_cost, baseline_cost, entropy_cost, reward_clip, vs, pg_advantages,
                        nullptr, nullptr, nullptr, clipped_rhos, d_logits, d_baseline, losses, workspace,
                        bp_learner_loss_workspace_bytes(T, B, A), status, (cudaStream_t)stream);
    if (rc != BP_ERR_UNSUPPORTED) return rc;
  }
  const bool vec = aligned16(learner_logits) && aligned16(behavior_logits) && aligned16(d_logits);
  return launch_mode<MODE_LOSS>(a, (cudaStream_t)stream, vec);
}
