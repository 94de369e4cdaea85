// Tile-resident persistent V-trace kernels (B % 4 == 0, T <= 256, A in {6, 18}).
//
// Same math as vtrace.cu (MODE_LOGITS = from_logits, MODE_LOSS = fused
// learner loss; beastpipe vtrace.py:51-128 / :169-255), laid out for HBM throughput
// at the learner's batch sizes:
//   * a tile is BT batch columns x all T rows (BT = 4; 8 for large B); persistent CTAs
//     (as many as fit per SM) walk the tiles round-robin, each with two tile slots in
//     shared memory: while a tile is computed, the next tile's behaviour and target
//     logits stream into the other slot (2D TMA boxes of 16 time rows, one mbarrier per
//     row chunk) and its small (T, B) inputs load into registers
//   * one thread per (t, b) row, no producer/consumer hand-off: it waits only for its
//     own row chunk, computes both log-softmaxes with the row in registers, the exact
//     action gather, rho / delta / c, and parks the scan inputs in smem
//   * one warp per column runs the reverse discounted scan as a suffix scan of affine
//     maps (exact zero-discount cut), then every row thread emits vs / pg_advantages
//   * MODE_LOSS: the learner-logit tile is still resident, so d_logits are computed from
//     smem and stored straight from registers - the learner logits cross HBM once
//   * loss sums: f64 per-CTA partials, last-CTA fixed-order reduce (deterministic)
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"
#include "tma_host.h"

namespace bp {
namespace vt3 {

constexpr int kChunk = 16;    // time rows per TMA box / mbarrier
constexpr int kMaxT = 256;    // one thread per (t, b) row: T * BT <= 1024
constexpr int kMaxChunks = kMaxT / kChunk;

struct Args {
  int T, B, nchunks, ntiles;
  float clip_rho, clip_pg_rho, clip_c, discount, pg_cost, baseline_cost, entropy_cost;
  int reward_clip;
  const int64_t* act;
  const float* rew;
  const float* val;   // (T, B) values; MODE_LOSS: (T+1, B) baseline
  const float* boot;  // (B)
  const float* disc;  // MODE_LOGITS
  const uint8_t* done;  // MODE_LOSS: (T, B) done[1:]
  float* vs;
  float* pg;
  float* log_rhos;
  float* beh_logp;
  float* tgt_logp;
  float* clipped_rhos;  // MODE_LOSS (nullable)
  float* d_baseline;
  double* losses;
  double* partials;
  unsigned* counter;
  unsigned* status;
};

struct Maps {
  CUtensorMap beh, tgt, dlog;
};

__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }

// two tile slots (behaviour + target logits each), one set of scan arrays, barriers
// two tile slots (behaviour + target logits each), two sets of scan arrays, barriers
struct Plan {
  size_t half, slot, scan, delta, dc, bars, total;
};
__host__ __device__ inline Plan plan(int T, int A, int kBT) {
  Plan p;
  const int nch = (T + kChunk - 1) / kChunk;
  p.half = al128((size_t)nch * kChunk * kBT * A * 4);
  p.slot = 2 * p.half;
  p.scan = 2 * al128((size_t)T * kBT * 4);
  p.delta = 2 * p.slot;
  p.dc = p.delta + al128((size_t)T * kBT * 4);
  p.bars = p.delta + 2 * p.scan;
  p.total = p.bars + (2 * kMaxChunks + 2) * 8;
  return p;
}

BP_DEVICE void tma_store_2d(const CUtensorMap* m, const void* src, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(sm100::smem_addr(src)), "r"(x), "r"(y)
      : "memory");
}

// mbarrier wait without a suspend-time hint (pure polling)
BP_DEVICE void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra S_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}

// named barrier over the compute warps only (the producer warp never joins it)
BP_DEVICE void comp_sync(int n) { asm volatile("bar.sync 1, %0;\n" ::"r"(n) : "memory"); }

// log-sum-exp, gathered logit and (ENT) entropy of one row, row held in registers
template <int A, bool ENT>
BP_DEVICE void row_stats(const float* x, int a, float& lse, float& xa, float& ent, bool& fin) {
  constexpr float kLog2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;
  float v[A];
#pragma unroll
  for (int i = 0; i < A / 2; ++i) {
    const float2 t = reinterpret_cast<const float2*>(x)[i];
    v[2 * i] = t.x;
    v[2 * i + 1] = t.y;
  }
  float m = v[0], mn = v[0];
#pragma unroll
  for (int i = 1; i < A; ++i) {
    m = fmaxf(m, v[i]);
    mn = fminf(mn, v[i]);
  }
  const float ml = m * kLog2e;
  float s = 0.f, sxe = 0.f;
#pragma unroll
  for (int i = 0; i < A; ++i) {
    const float e = ex2_approx(fmaf(v[i], kLog2e, -ml));
    s += e;
    if constexpr (ENT) sxe = fmaf(e, v[i] - m, sxe);
  }
  const float ls = lg2_approx(s) * kLn2;
  lse = m + ls;
  xa = x[a];
  ent = ENT ? ls - sxe / s : 0.f;
  // NaN / +inf poison lse; -inf anywhere shows in the row minimum
  fin = isfinite(mn) && isfinite(lse) && (!ENT || isfinite(ent));
}

// the per-row (T, B) inputs of one tile, loaded into registers one tile ahead
struct RowIn {
  int64_t a;
  float r, v, vn, d;
};

// volatile asm loads: issued where written (the compiler may not sink them to their first
// use in the next tile, which would expose the HBM latency the prefetch is there to hide)
BP_DEVICE float ldnc_f32(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];\n" : "=f"(v) : "l"(p));
  return v;
}
BP_DEVICE int64_t ldnc_s64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.nc.s64 %0, [%1];\n" : "=l"(v) : "l"(p));
  return v;
}
BP_DEVICE uint32_t ldnc_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.nc.u8 %0, [%1];\n" : "=h"(v) : "l"(p));
  return v;
}

#ifndef BP_VT3_VOLATILE
#define BP_VT3_VOLATILE 0
#endif
constexpr bool kVolatileLoads = BP_VT3_VOLATILE;

template <bool LOSS>
BP_DEVICE RowIn load_row(const Args& g, int tile, int kBT, int t, int b) {
  RowIn x{0, 0.f, 0.f, 0.f, 0.f};
  if (t < g.T && tile < g.ntiles) {
    const int B = g.B;
    const size_t idx = (size_t)t * B + tile * kBT + b;
    if constexpr (kVolatileLoads) {
      x.a = ldnc_s64(g.act + idx);
      x.r = ldnc_f32(g.rew + idx);
      x.v = ldnc_f32(g.val + idx);
      x.vn = ldnc_f32((t + 1 < g.T) ? g.val + idx + B : g.boot + tile * kBT + b);
      if constexpr (LOSS)
        x.d = ldnc_u8(g.done + idx) ? 0.f : g.discount;  // exact: float32(gamma) or 0
      else
        x.d = ldnc_f32(g.disc + idx);
    } else {
      x.a = __ldg(g.act + idx);
      x.r = __ldg(g.rew + idx);
      x.v = __ldg(g.val + idx);
      x.vn = __ldg((t + 1 < g.T) ? g.val + idx + B : g.boot + tile * kBT + b);
      if constexpr (LOSS)
        x.d = __ldg(g.done + idx) ? 0.f : g.discount;  // exact: float32(gamma) or 0
      else
        x.d = __ldg(g.disc + idx);
    }
  }
  return x;
}

template <int A, int kBT, bool LOSS>
__global__ void __launch_bounds__(1024) vt3_kernel(const __grid_constant__ Args g,
                                                   const __grid_constant__ Maps mp) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // persistent grid (every CTA resident at once): the next kernel (the learner's G pack) may
  // launch now; it waits for this kernel before reading its outputs
  pdl_trigger();
  pdl_wait();
  constexpr int RS = kBT * A;  // floats per tile row
  const int T = g.T, B = g.B, nch = g.nchunks;
  const Plan P = plan(T, A, kBT);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.bars);  // [2][kMaxChunks]
  uint64_t* freed = full + 2 * kMaxChunks;                        // [2]
  const int tid = threadIdx.x;
  // MODE_LOSS adds a producer warp (the last one) that owns the TMA traffic, so that no
  // compute thread waits for a d_logits store to drain before its slot is refilled; in
  // MODE_LOGITS thread 0 issues the loads between tiles
  constexpr bool kProducer = LOSS;
  const int ncomp = kProducer ? blockDim.x - 32 : blockDim.x;
  const uint32_t chunk_bytes = (uint32_t)(2 * kChunk * RS * 4);
  auto issue = [&](int tile, int slot) {
    float* sb = reinterpret_cast<float*>(smem + slot * P.slot);
    float* st = reinterpret_cast<float*>(smem + slot * P.slot + P.half);
    for (int c = 0; c < nch; ++c) {
      uint64_t* bar = &full[slot * kMaxChunks + c];
      mbar_expect_tx(bar, chunk_bytes);
      sm100::tma_load_2d(sb + c * kChunk * RS, &mp.beh, bar, tile * RS, c * kChunk);
      sm100::tma_load_2d(st + c * kChunk * RS, &mp.tgt, bar, tile * RS, c * kChunk);
    }
  };
  if (tid == 0) {
    for (int c = 0; c < 2 * kMaxChunks; ++c) mbar_init(&full[c], 1);
    for (int c = 0; c < 2; ++c) mbar_init(&freed[c], ncomp / 32);
    fence_mbar_init();
    sm100::tma_prefetch_desc(&mp.beh);
    sm100::tma_prefetch_desc(&mp.tgt);
    // MODE_LOGITS: the second tile is issued at the top of the first iteration; MODE_LOSS:
    // the producer warp issues both first tiles
    if (!kProducer && (int)blockIdx.x < g.ntiles) issue(blockIdx.x, 0);
  }
  __syncthreads();  // barrier inits visible before anyone waits

  unsigned bad = 0;
  double pg_sum = 0.0, base_sum = 0.0, ent_sum = 0.0;
  if (kProducer && tid >= ncomp) {
    // ------------------------------------------------------------ producer warp
    // Refills a slot with a whole tile (both logit tensors, all T rows) once the compute
    // warps release it and the TMA store of the d_logits they wrote over it has read it.
    // The whole warp runs the loop (a divergent warp must not reach the CTA barriers of
    // the loss reduction); lane 0 issues and waits on the bulk traffic.
    const bool lead = tid == ncomp;
    int k = 0;
    if (lead)
      for (int tile = blockIdx.x; tile < g.ntiles && k < 2; tile += gridDim.x, ++k) issue(tile, k);
    k = 0;
    for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++k) {
      const int slot = k & 1;
      mbar_wait_parity(&freed[slot], (k >> 1) & 1);
      if (lead) {
        const float* st = reinterpret_cast<const float*>(smem + slot * P.slot + P.half);
        for (int c = 0; c < nch; ++c) tma_store_2d(&mp.dlog, st + c * kChunk * RS, tile * RS, c * kChunk);
        bulk_commit();
        bulk_wait_read_all();
        const int next2 = tile + 2 * gridDim.x;
        if (next2 < g.ntiles) issue(next2, slot);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ compute warps
    const int t = tid / kBT, b = tid % kBT;
    const bool live = t < T;
    RowIn cur = load_row<LOSS>(g, blockIdx.x, kBT, t, b);
    int k = 0;
    for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++k) {
      const int slot = k & 1;
      if (!kProducer && tid == 0 && tile + (int)gridDim.x < g.ntiles) issue(tile + gridDim.x, slot ^ 1);
      const RowIn nxt = load_row<LOSS>(g, tile + gridDim.x, kBT, t, b);
      float* s_beh = reinterpret_cast<float*>(smem + slot * P.slot);
      float* s_tgt = reinterpret_cast<float*>(smem + slot * P.slot + P.half);
      float* s_delta = reinterpret_cast<float*>(smem + P.delta + slot * P.scan);
      float* s_dc = reinterpret_cast<float*>(smem + P.dc + slot * P.scan);
      const int b0 = tile * kBT;
      const size_t idx = (size_t)t * B + b0 + b;
      float rv = cur.r;
      const float vv = cur.v, vnext = cur.vn, dv = cur.d;
      float lt = 0.f, et = 0.f, tlp = 0.f, pgr = 0.f;
      int a = 0;
      if (live) {
        a = (int)cur.a;
        if (cur.a < 0 || cur.a >= A) {
          bad |= BP_STATUS_ACTION_RANGE;
          a = 0;
        }
        if (LOSS && g.reward_clip) rv = fminf(fmaxf(rv, -1.f), 1.f);
        mbar_wait_parity(&full[slot * kMaxChunks + t / kChunk], (k >> 1) & 1);
        float lb, xb, eb, xt;
        bool fb, ft;
        row_stats<A, false>(s_beh + tid * A, a, lb, xb, eb, fb);
        row_stats<A, LOSS>(s_tgt + tid * A, a, lt, xt, et, ft);
        const float blp = xb - lb;
        tlp = xt - lt;
        const float lr = tlp - blp;
        const float rho = fast_exp(lr);
        const float cr = fminf(g.clip_rho, rho);
        pgr = fminf(g.clip_pg_rho, rho);
        if constexpr (LOSS) {
          if (g.clipped_rhos) g.clipped_rhos[idx] = cr;
        }
        s_delta[tid] = cr * (rv + dv * vnext - vv);
        s_dc[tid] = dv * fminf(g.clip_c, rho);
        if constexpr (!LOSS) {
          if (dv < 0.f) bad |= BP_STATUS_NEG_DISCOUNT;
          if (g.log_rhos) g.log_rhos[idx] = lr;
          if (g.beh_logp) g.beh_logp[idx] = blp;
          if (g.tgt_logp) g.tgt_logp[idx] = tlp;
        }
        if constexpr (LOSS) {
          // learner step: a non-finite batch field (reward, behaviour logits) is a schema
          // violation (validate_batch, rollout.py:189-192); the learner's own outputs are not
          if (!(fb && isfinite(cur.r))) bad |= BP_STATUS_BATCH_NONFINITE;  // (before the clip)
          if (!(ft && isfinite(lr) && isfinite(vv) && isfinite(vnext) && isfinite(dv)))
            bad |= BP_STATUS_NONFINITE_IN;
        } else if (!(fb && ft && isfinite(lr) && isfinite(rv) && isfinite(vv) && isfinite(vnext) && isfinite(dv))) {
          bad |= BP_STATUS_NONFINITE_IN;
        }
      }
      comp_sync(ncomp);
      // Warp-parallel reverse scan, one warp per column: acc_t = delta_t + (gamma_t c_t)
      // acc_{t+1}, acc_T = 0.  Each lane composes the affine maps x -> a + b x of its
      // contiguous segment, a 5-step shuffle suffix scan gives the value entering each
      // segment, and a local sweep writes acc_t.  A zero discount makes b == 0 exactly, so
      // the dependence on later steps is cut exactly as in the sequential recursion
      // (vtrace.py:121-123).
      {
        const int w = tid >> 5, lane = tid & 31;
        if (w < kBT) {
          const int kk = (T + 31) >> 5;
          const int t0 = lane * kk, t1 = min(T, t0 + kk);
          float ga = 0.f, gb = 1.f;
          for (int u = t1 - 1; u >= t0; --u) {
            const float d = s_delta[u * kBT + w], c = s_dc[u * kBT + w];
            ga = fmaf(c, ga, d);
            gb = c * gb;
          }
          float sa = ga, sb = gb;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const float na = __shfl_down_sync(0xffffffffu, sa, off);
            const float nb = __shfl_down_sync(0xffffffffu, sb, off);
            if (lane + off < 32) {
              sa = fmaf(sb, na, sa);
              sb = sb * nb;
            }
          }
          float acc = __shfl_down_sync(0xffffffffu, sa, 1);
          if (lane == 31) acc = 0.f;
          for (int u = t1 - 1; u >= t0; --u) {
            const int i = u * kBT + w;
            acc = fmaf(s_dc[i], acc, s_delta[i]);
            s_delta[i] = acc;
          }
        }
      }
      comp_sync(ncomp);
      if (live) {
        const float vsv = s_delta[tid] + vv;
        const float vs_next = (t + 1 < T ? s_delta[tid + kBT] : 0.f) + vnext;
        const float pgv = pgr * (rv + dv * vs_next - vv);
        if (g.vs) g.vs[idx] = vsv;
        if (g.pg) g.pg[idx] = pgv;
        if constexpr (LOSS) {
          const float dvs = vsv - vv;
          pg_sum -= (double)pgv * (double)tlp;
          base_sum += 0.5 * (double)dvs * (double)dvs;
          ent_sum -= (double)et;
          g.d_baseline[idx] = g.baseline_cost * (vv - vsv);
          // d_logits in place over the resident learner-logit row (the producer stores it)
          const float pa = g.pg_cost * pgv, ec = g.entropy_cost;
          float* x = s_tgt + tid * A;
#pragma unroll
          for (int j = 0; j < A; ++j) {
            const float lp = x[j] - lt;
            const float p = fast_exp(lp);
            x[j] = pa * (p - (j == a ? 1.f : 0.f)) + ec * p * (lp + et);
          }
        }
      }
      if constexpr (kProducer) {
        if (tid < kBT) g.d_baseline[(size_t)T * B + b0 + tid] = 0.f;
        fence_proxy_async_smem();  // generic-proxy smem writes -> the producer's TMA store
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive_cta(&freed[slot]);  // this warp is done with the slot
      } else {
        __syncthreads();  // every warp is done with this slot and the scan arrays
      }
      cur = nxt;
    }
  }

  if constexpr (LOSS) {
    // deterministic loss sums: warp trees -> fixed-order CTA sum -> last CTA reduces
    __shared__ double red[3][32];
    __shared__ bool is_last;
    const int lane = tid & 31, w = tid >> 5, nw = (blockDim.x + 31) >> 5;
    // any violation in this CTA poisons the loss sums: the total becomes NaN, which rejects
    // the optimiser step on every data-parallel rank after the loss all-reduce
    if (__syncthreads_or(bad != 0u) && tid == 0) pg_sum = __longlong_as_double(0x7ff8000000000000LL);
    pg_sum = warp_sum(pg_sum);
    base_sum = warp_sum(base_sum);
    ent_sum = warp_sum(ent_sum);
    if (lane == 0) {
      red[0][w] = pg_sum;
      red[1][w] = base_sum;
      red[2][w] = ent_sum;
    }
    __syncthreads();
    if (tid == 0) {
      double a0 = 0, a1 = 0, a2 = 0;
      for (int q = 0; q < nw; ++q) {
        a0 += red[0][q];
        a1 += red[1][q];
        a2 += red[2][q];
      }
      g.partials[3 * blockIdx.x + 0] = a0;
      g.partials[3 * blockIdx.x + 1] = a1;
      g.partials[3 * blockIdx.x + 2] = a2;
      __threadfence();
      is_last = atomicAdd(g.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last) {
      __threadfence();
      double a0 = 0, a1 = 0, a2 = 0;
      const volatile double* pp = g.partials;
      for (int q = tid; q < (int)gridDim.x; q += blockDim.x) {
        a0 += pp[3 * q + 0];
        a1 += pp[3 * q + 1];
        a2 += pp[3 * q + 2];
      }
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      a2 = warp_sum(a2);
      __syncthreads();  // red[] reuse
      if (lane == 0) {
        red[0][w] = a0;
        red[1][w] = a1;
        red[2][w] = a2;
      }
      __syncthreads();
      if (tid == 0) {
        double s0 = 0, s1 = 0, s2 = 0;
        for (int q = 0; q < nw; ++q) {
          s0 += red[0][q];
          s1 += red[1][q];
          s2 += red[2][q];
        }
        const double total = (double)g.pg_cost * s0 + (double)g.baseline_cost * s1 +
                             (double)g.entropy_cost * s2;
        g.losses[0] = s0;
        g.losses[1] = s1;
        g.losses[2] = s2;
        g.losses[3] = total;
        if (!isfinite(total)) bad |= BP_STATUS_NONFINITE_LOSS;
        *g.counter = 0u;
      }
    }
  }
  if (kProducer && tid == ncomp) bulk_wait_all();  // d_logits stores complete before exit
  set_status(g.status, bad);
}

}  // namespace vt3

// ---------------------------------------------------------------------------- host
// BP_ERR_UNSUPPORTED when the shape is outside this kernel's regime; the caller then uses
// the generic kernel (vtrace.cu).
int vt3_launch(bool loss, const float* beh, const float* tgt, const int64_t* act, const void* disc_or_done,
               const float* rew, const float* val, const float* boot, int T, int B, int A,
               float clip_rho, float clip_pg_rho, float clip_c, float discount, float pg_cost,
               float baseline_cost, float entropy_cost, int reward_clip, float* vs, float* pg,
               float* log_rhos, float* beh_logp, float* tgt_logp, float* clipped_rhos, float* d_logits,
               float* d_baseline, double* losses, void* workspace, size_t ws_bytes, unsigned* status,
               cudaStream_t s) {
  using namespace vt3;
  static const int bt_env = [] {
    const char* e = std::getenv("BP_VT3_BT");
    return e ? std::atoi(e) : 0;
  }();
  // columns per tile: BT * A * 4 bytes per TMA box row must be a multiple of 16
  // from_logits at large B streams best with 8-column tiles (fewer, longer TMA rows; T=80 A=18
  // B=4096: 13.2 vs 13.8 us with 4-column tiles, B=16384: 40.6 vs 43.9 us); the loss mode is
  // the same at 4 or 8 columns (24.2 / 24.8 us at B=4096, tools/vt3_sweep.py)
  // small B (the per-GPU learner batch) is latency-bound: 2-column tiles double the CTAs
  int kBT = bt_env ? bt_env : (!loss && B >= 4096 && B % 8 == 0) ? 8 : (B <= 256 && B % 2 == 0) ? 2 : 4;
  if (!(kBT == 2 || kBT == 4 || kBT == 8) || T * kBT > 992) kBT = 4;
  if (!(A == 6 || A == 18) || B % kBT || T > kMaxT || T * kBT > 992) return BP_ERR_UNSUPPORTED;
  const uintptr_t al = reinterpret_cast<uintptr_t>(beh) | reinterpret_cast<uintptr_t>(tgt) |
                       (loss ? reinterpret_cast<uintptr_t>(d_logits) : 0);
  if (al & 15u) return BP_ERR_UNSUPPORTED;
  if (int e = tma_init()) return e;
  Maps m;
  int rc;
  if ((rc = tma_make_2d(&m.beh, beh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, (long long)B * A, kBT * A, kChunk, 0)))
    return rc;
  if ((rc = tma_make_2d(&m.tgt, tgt, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, (long long)B * A, kBT * A, kChunk, 0)))
    return rc;
  if (loss) {
    if ((rc = tma_make_2d(&m.dlog, d_logits, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, (long long)B * A, kBT * A,
                          kChunk, 0)))
      return rc;
  } else {
    m.dlog = m.beh;
  }
  Args g{};
  g.T = T;
  g.B = B;
  g.nchunks = (T + kChunk - 1) / kChunk;
  g.ntiles = B / kBT;
  g.clip_rho = clip_rho;
  g.clip_pg_rho = clip_pg_rho;
  g.clip_c = clip_c;
  g.discount = discount;
  g.pg_cost = pg_cost;
  g.baseline_cost = baseline_cost;
  g.entropy_cost = entropy_cost;
  g.reward_clip = reward_clip;
  g.act = act;
  g.rew = rew;
  g.val = val;
  g.boot = boot;
  g.disc = loss ? nullptr : reinterpret_cast<const float*>(disc_or_done);
  g.done = loss ? reinterpret_cast<const uint8_t*>(disc_or_done) : nullptr;
  g.vs = vs;
  g.pg = pg;
  g.log_rhos = log_rhos;
  g.beh_logp = beh_logp;
  g.tgt_logp = tgt_logp;
  g.clipped_rhos = clipped_rhos;
  g.d_baseline = d_baseline;
  g.losses = losses;
  g.status = status;
  static const int blocks_env = [] {
    const char* e = std::getenv("BP_VT3_CTAS_PER_SM");
    return e ? std::atoi(e) : 0;
  }();
  const Plan P = plan(T, A, kBT);
  // compute threads: one per (t, b) row, >= one warp per column; MODE_LOSS: + producer warp
  const int threads = (T * kBT > 32 * kBT ? ((T * kBT + 31) / 32) * 32 : 32 * kBT) + (loss ? 32 : 0);
  if (loss && !workspace) return BP_ERR_UNSUPPORTED;
  g.counter = loss ? reinterpret_cast<unsigned*>(workspace) : nullptr;
  g.partials = loss ? reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + 256) : nullptr;
  // persistent grid: every CTA that fits at once (smem holds two tile slots per CTA)
#define BP_VT3(AT_, LOSS_)                                                                        \
  {                                                                                               \
    auto k = kBT == 2 ? vt3_kernel<AT_, 2, LOSS_> : kBT == 8 ? vt3_kernel<AT_, 8, LOSS_> : vt3_kernel<AT_, 4, LOSS_>; \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.total); \
    int per_sm = 0;                                                                               \
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, P.total); \
    if (e != cudaSuccess || per_sm < 1) {                                                         \
      set_error("vt3 occupancy: %s", cudaGetErrorString(e));                                      \
      return BP_ERR_LAUNCH;                                                                       \
    }                                                                                             \
    if (blocks_env > 0 && blocks_env < per_sm) per_sm = blocks_env;                               \
    const int grid = g.ntiles < per_sm * tma_num_sms() ? g.ntiles : per_sm * tma_num_sms();       \
    if (loss && ws_bytes < 256 + (size_t)grid * 3 * sizeof(double)) return BP_ERR_UNSUPPORTED;    \
    launch_pdl(k, dim3(grid), dim3(threads), P.total, s, g, m);                                  \
    return check_launch("vt3_kernel");                                                            \
  }
  if (A == 6) {
    if (loss) BP_VT3(6, true) else BP_VT3(6, false)
  } else {
    if (loss) BP_VT3(18, true) else BP_VT3(18, false)
  }
#undef BP_VT3
}

}  // namespace bp
