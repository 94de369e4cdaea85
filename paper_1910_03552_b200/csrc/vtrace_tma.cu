// Persistent producer/consumer V-trace kernels for the bandwidth regime (B >= 512).
//
// Same math as vtrace.cu (MODE_LOGITS = from_logits, MODE_LOSS = fused learner loss,
// beastpipe vtrace.py:51-128 / :169-255), restructured for HBM throughput:
//   * grid = min(tiles, 2 x #SMs) persistent CTAs; a tile = BT batch columns x all T rows
//   * warp 4 is a dedicated TMA producer: per tile it loads the small (T, BT) inputs
//     (actions, rewards, values, discounts / done) as 2D TMA boxes into one of two
//     double-buffered input sets, then streams the logits as one 2D TMA box per
//     tensor per chunk of TC time rows into a 4-stage ring; it runs ahead across
//     tiles, so the next tile's bytes stream in under this tile's scan
//   * warps 0-3 consume: one (t, b) row per thread per chunk, release ring stages
//     through mbarriers (no CTA-wide barriers in the stream), reverse scan per column,
//     and in MODE_LOSS write d_logits with 2D TMA tensor stores
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tma_host.h"

namespace bp {
namespace vt2 {

constexpr int kCons = 128;             // consumer threads
constexpr int kThreads = kCons + 32;   // + producer warp
constexpr int kNst = 4;                // ring stages
constexpr int kMaxT = 256;             // TMA box rows

struct Args {
  int T, B, A, BT, TC, ntiles, nchunks, loss;
  float clip_rho, clip_pg_rho, clip_c, discount, pg_cost, baseline_cost, entropy_cost;
  int reward_clip;
  const float* boot;  // (B) bootstrap values (MODE_LOSS: baseline + T*B)
  const uint8_t* done;  // MODE_LOSS: (T, B) done[1:]
  float* vs;
  float* pg;
  float* log_rhos;
  float* beh_logp;
  float* tgt_logp;
  float* d_baseline;
  double* losses;
  double* partials;
  unsigned* counter;
  unsigned* status;
};

struct Maps {
  CUtensorMap beh, tgt, act, rew, val, disc, dlog;
};

__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }

// shared-memory carve-up (bytes), identical on host and device
struct Plan {
  size_t stage_bytes, ring, in_set, in_act, in_rew, in_val, in_disc, in_done, work, w_lr, w_delta,
      w_dc, w_lse, w_ent, w_tlp, w_act, boot, bars, total;
};
__host__ __device__ inline Plan plan(int T, int BT, int A, int TC, bool loss) {
  Plan p;
  const size_t tb = (size_t)T * BT;
  p.stage_bytes = al128((size_t)2 * TC * BT * A * 4);
  p.ring = 0;
  size_t o = p.stage_bytes * kNst;
  // one input set (x2)
  p.in_act = 0;
  p.in_rew = al128(tb * 8);
  p.in_val = p.in_rew + al128(tb * 4);
  p.in_disc = p.in_val + al128(tb * 4);
  p.in_done = p.in_disc + al128(tb * 4);
  p.in_set = p.in_done + al128((size_t)T * 16);
  p.work = o + 2 * p.in_set;
  p.w_lr = 0;
  p.w_delta = al128(tb * 4);
  p.w_dc = p.w_delta + al128(tb * 4);
  p.w_lse = p.w_dc + al128(tb * 4);
  p.w_ent = p.w_lse + (loss ? al128(tb * 4) : 0);
  p.w_tlp = p.w_ent + (loss ? al128(tb * 4) : 0);
  p.w_act = p.w_tlp + (loss ? al128(tb * 4) : 0);
  p.boot = p.w_act + (loss ? al128(tb * 4) : 0);
  p.bars = p.work + p.boot + al128((size_t)BT * 4);
  p.total = p.bars + 256;
  return p;
}

BP_DEVICE void cons_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

BP_DEVICE void tma_store_2d(const CUtensorMap* m, const void* src, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(sm100::smem_addr(src)), "r"(x), "r"(y)
      : "memory");
}

template <int AT, bool ENT>
BP_DEVICE void row_stats(const float* x, int a, float& lse, float& xa, float& ent, bool& fin) {
  constexpr float kLog2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;
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
  float m = v[0], mn = v[0];
#pragma unroll
  for (int i = 1; i < AT; ++i) {
    m = fmaxf(m, v[i]);
    mn = fminf(mn, v[i]);
  }
  // sum 2^(x log2e - m log2e): one FFMA + one MUFU.EX2 per element
  const float ml = m * kLog2e;
  float s = 0.f, sxe = 0.f;
#pragma unroll
  for (int i = 0; i < AT; ++i) {
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

template <int BT, int AT, bool LOSS>
__global__ void __launch_bounds__(kThreads) vt2_kernel(const __grid_constant__ Args g,
                                                       const __grid_constant__ Maps mp) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int A = AT;
  constexpr int TC = kCons / BT;
  constexpr int RS = BT * A;  // floats per smem row
  const int T = g.T, B = g.B;
  const Plan P = plan(T, BT, A, TC, LOSS);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.bars);
  uint64_t* empty = full + kNst;
  uint64_t* sfull = empty + kNst;  // [2]
  uint64_t* sfree = sfull + 2;     // [2]
  const int tid = threadIdx.x;
  const int nchunks = g.nchunks;

  if (tid == kCons) {
    for (int s = 0; s < kNst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons / 32);  // one arrival per consumer warp
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sfull[s], LOSS ? 2 : 1);  // LOSS: + the producer warp's discount conversion
      mbar_init(&sfree[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= kCons) {
    // ------------------------------------------------------------ producer warp
    // The whole warp runs the loop (warp-uniform state); lane 0 issues the TMA traffic,
    // and in MODE_LOSS all lanes turn the tile's done flags into exact discounts.
    const int lane = tid - kCons;
    if (lane == 0) {
      sm100::tma_prefetch_desc(&mp.beh);
      sm100::tma_prefetch_desc(&mp.tgt);
    }
    uint32_t q = 0;
    int st = 0;
    const uint32_t small_bytes = (uint32_t)(T * BT * 8 + 2 * T * BT * 4 + (LOSS ? 0 : T * BT * 4));
    const uint32_t chunk2 = (uint32_t)(2 * TC * RS * 4), chunk1 = (uint32_t)(TC * RS * 4);
    for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++st) {
      const int b0 = tile * BT;
      const int set = st & 1;
      uint8_t* in = smem + P.work - 2 * P.in_set + set * P.in_set;
      mbar_wait_parity(&sfree[set], (((uint32_t)st >> 1) & 1u) ^ 1u);
      if (lane == 0) {
        mbar_expect_tx(&sfull[set], small_bytes);
        sm100::tma_load_2d(in + P.in_act, &mp.act, &sfull[set], b0, 0);
        sm100::tma_load_2d(in + P.in_rew, &mp.rew, &sfull[set], b0, 0);
        sm100::tma_load_2d(in + P.in_val, &mp.val, &sfull[set], b0, 0);
        if constexpr (!LOSS) sm100::tma_load_2d(in + P.in_disc, &mp.disc, &sfull[set], b0, 0);
      }
      if constexpr (LOSS) {  // discount = (float)gamma * ~done, exact
        float4* s_disc4 = reinterpret_cast<float4*>(in + P.in_disc);
        const float gm = g.discount;
        if ((B & 3) == 0 && b0 + 4 <= B) {
          // the 4 flags of a time row are one aligned u32: issue all loads, then convert
          uint32_t w[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int t = lane + 32 * k;
            w[k] = t < T ? __ldg(reinterpret_cast<const uint32_t*>(g.done + (size_t)t * B + b0)) : 0u;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int t = lane + 32 * k;
            if (t < T)
              s_disc4[t] = make_float4((w[k] & 0xffu) ? 0.f : gm, (w[k] & 0xff00u) ? 0.f : gm,
                                       (w[k] & 0xff0000u) ? 0.f : gm, (w[k] & 0xff000000u) ? 0.f : gm);
          }
        } else {
          float* s_disc = reinterpret_cast<float*>(s_disc4);
          for (int i = lane; i < T * BT; i += 32) {
            const int t = i / BT, b = i % BT;
            s_disc[i] = (b0 + b < B && g.done[(size_t)t * B + b0 + b]) ? 0.f : gm;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&sfull[set]);
      }
      for (int c = 0; c < nchunks; ++c, ++q) {
        const int s = q % kNst;
        mbar_wait_parity(&empty[s], ((q / kNst) & 1u) ^ 1u);
        if (lane == 0) {
          mbar_expect_tx(&full[s], chunk2);
          uint8_t* stg = smem + P.ring + s * P.stage_bytes;
          sm100::tma_load_2d(stg, &mp.beh, &full[s], b0 * A, c * TC);
          sm100::tma_load_2d(stg + TC * RS * 4, &mp.tgt, &full[s], b0 * A, c * TC);
        }
        __syncwarp();
      }
      if constexpr (LOSS) {
        for (int c = 0; c < nchunks; ++c, ++q) {
          const int s = q % kNst;
          mbar_wait_parity(&empty[s], ((q / kNst) & 1u) ^ 1u);
          if (lane == 0) {
            mbar_expect_tx(&full[s], chunk1);
            sm100::tma_load_2d(smem + P.ring + s * P.stage_bytes, &mp.tgt, &full[s], b0 * A, c * TC);
          }
          __syncwarp();
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumer warps
  const int tl = tid / BT, bl = tid % BT;
  float* wk = reinterpret_cast<float*>(smem + P.work);
  float* s_lr = reinterpret_cast<float*>(smem + P.work + P.w_lr);
  float* s_delta = reinterpret_cast<float*>(smem + P.work + P.w_delta);
  float* s_dc = reinterpret_cast<float*>(smem + P.work + P.w_dc);
  float* s_lse = reinterpret_cast<float*>(smem + P.work + P.w_lse);
  float* s_ent = reinterpret_cast<float*>(smem + P.work + P.w_ent);
  float* s_tlp = reinterpret_cast<float*>(smem + P.work + P.w_tlp);
  int* s_act = reinterpret_cast<int*>(smem + P.work + P.w_act);
  float* s_boot = reinterpret_cast<float*>(smem + P.work + P.boot);
  (void)wk;
  unsigned bad = 0;
  double pg_sum = 0.0, base_sum = 0.0, ent_sum = 0.0;
  uint32_t q = 0;
  int st = 0;
  const int TB = T * BT;
  for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++st) {
    const int b0 = tile * BT;
    const int bw = min(BT, B - b0);
    const int set = st & 1;
    uint8_t* in = smem + P.work - 2 * P.in_set + set * P.in_set;
    const int64_t* s_act64 = reinterpret_cast<const int64_t*>(in + P.in_act);
    float* s_rew = reinterpret_cast<float*>(in + P.in_rew);
    float* s_val = reinterpret_cast<float*>(in + P.in_val);
    float* s_disc = reinterpret_cast<float*>(in + P.in_disc);
    if (tid < bw) {
      const float bv = g.boot[b0 + tid];
      s_boot[tid] = bv;
      if (!isfinite(bv)) bad |= BP_STATUS_NONFINITE_IN;
    }
    mbar_wait_parity(&sfull[set], ((uint32_t)st >> 1) & 1u);
    // ---------------------------------------------------------------- phase 1
    for (int c = 0; c < nchunks; ++c, ++q) {
      const int s = q % kNst;
      mbar_wait_parity(&full[s], (q / kNst) & 1u);
      const int t = c * TC + tl;
      if (t < T && bl < bw) {
        const float* stg = reinterpret_cast<const float*>(smem + P.ring + s * P.stage_bytes);
        const int si = t * BT + bl;
        const int64_t a64 = s_act64[si];
        int a = (int)a64;
        if (a64 < 0 || a64 >= A) {
          bad |= BP_STATUS_ACTION_RANGE;
          a = 0;
        }
        float lb, xb, eb, lt, xt, et;
        bool fb, ft;
        row_stats<AT, false>(stg + tl * RS + bl * A, a, lb, xb, eb, fb);
        row_stats<AT, LOSS>(stg + TC * RS + tl * RS + bl * A, a, lt, xt, et, ft);
        const float blp = xb - lb, tlp = xt - lt, lr = tlp - blp;
        float rv = s_rew[si];
        const float vv = s_val[si], dv = s_disc[si];
        if constexpr (LOSS) {
          if (g.reward_clip) {
            rv = fminf(fmaxf(rv, -1.f), 1.f);
            s_rew[si] = rv;
          }
          s_lse[si] = lt;
          s_ent[si] = et;
          s_tlp[si] = tlp;
          s_act[si] = a;
        } else {
          if (dv < 0.f) bad |= BP_STATUS_NEG_DISCOUNT;
          const size_t idx = (size_t)t * B + b0 + bl;
          if (g.log_rhos) g.log_rhos[idx] = lr;
          if (g.beh_logp) g.beh_logp[idx] = blp;
          if (g.tgt_logp) g.tgt_logp[idx] = tlp;
        }
        if (!(fb && ft && isfinite(lr) && isfinite(rv) && isfinite(vv) && isfinite(dv)))
          bad |= BP_STATUS_NONFINITE_IN;
        s_lr[si] = lr;
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive_cta(&empty[s]);  // this warp is done with the stage
    }
    cons_sync();  // phase-1 scan-array writes visible to all consumer warps
    // ---------------------------------------------------------------- phase 2
    for (int i = tid; i < TB; i += kCons) {
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
      }
    }
    cons_sync();
    // Warp-parallel reverse scan (one warp per column, BT == 4 consumer warps):
    // acc_t = f_t(acc_{t+1}) with f_t(x) = delta_t + (gamma_t c_t) x, acc_T = 0.  Each
    // lane composes its segment of ceil(T/32) steps, a 5-step shuffle suffix-scan of the
    // affine maps (a, b): x -> a + b x gives the value entering each segment, and a short
    // local sweep writes acc_t.  A zero discount makes b == 0 exactly, so dependence on
    // later steps is cut exactly as in the sequential recursion (vtrace.py:121-123).
    {
      const int w = tid >> 5, lane = tid & 31;
      if (w < bw) {
        const int k = (T + 31) >> 5;
        const int t0 = lane * k, t1 = min(T, t0 + k);
        float ga = 0.f, gb = 1.f;  // identity
        for (int t = t1 - 1; t >= t0; --t) {
          const float d = s_delta[t * BT + w], c = s_dc[t * BT + w];
          ga = fmaf(c, ga, d);
          gb = c * gb;
        }
        float sa = ga, sb = gb;  // inclusive suffix composition S_l = G_l o ... o G_31
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float na = __shfl_down_sync(0xffffffffu, sa, off);
          const float nb = __shfl_down_sync(0xffffffffu, sb, off);
          if (lane + off < 32) {
            sa = fmaf(sb, na, sa);
            sb = sb * nb;
          }
        }
        float acc = __shfl_down_sync(0xffffffffu, sa, 1);  // H_l(0) = S_{l+1}.a
        if (lane == 31) acc = 0.f;
        for (int t = t1 - 1; t >= t0; --t) {
          const int i = t * BT + w;
          acc = fmaf(s_dc[i], acc, s_delta[i]);
          s_delta[i] = acc;
        }
      }
    }
    cons_sync();
    for (int i = tid; i < TB; i += kCons) {
      const int t = i / BT, b = i % BT;
      if (b < bw) {
        const float v = s_val[i];
        const float vsv = s_delta[i] + v;
        const float vs_next = (t + 1 < T) ? (s_delta[i + BT] + s_val[i + BT]) : s_boot[b];
        const float pgv = s_lr[i] * (s_rew[i] + s_disc[i] * vs_next - v);
        const size_t idx = (size_t)t * B + b0 + b;
        if (g.vs) g.vs[idx] = vsv;
        if (g.pg) g.pg[idx] = pgv;
        if constexpr (LOSS) {
          s_dc[i] = pgv;
          const float dvs = vsv - v;
          pg_sum -= (double)pgv * (double)s_tlp[i];
          base_sum += 0.5 * (double)dvs * (double)dvs;
          ent_sum -= (double)s_ent[i];
          g.d_baseline[idx] = g.baseline_cost * (v - vsv);
        }
      }
    }
    if constexpr (LOSS) {
      if (tid < bw) g.d_baseline[(size_t)T * B + b0 + tid] = 0.f;
      cons_sync();
      // ---------------------------------------------------------- phase 3: d_logits
      int pending = -1;  // stage whose TMA store may still be reading smem (released one chunk later)
      for (int c = 0; c < nchunks; ++c, ++q) {
        const int s = q % kNst;
        mbar_wait_parity(&full[s], (q / kNst) & 1u);
        float* stg = reinterpret_cast<float*>(smem + P.ring + s * P.stage_bytes);
        const int t = c * TC + tl;
        if (t < T && bl < bw) {
          const int si = t * BT + bl;
          const float lse = s_lse[si], H = s_ent[si], pa = g.pg_cost * s_dc[si], ec = g.entropy_cost;
          const int a = s_act[si];
          float* x = stg + tl * RS + bl * A;
#pragma unroll
          for (int j = 0; j < A; ++j) {
            const float lp = x[j] - lse;
            const float p = fast_exp(lp);
            x[j] = pa * (p - (j == a ? 1.f : 0.f)) + ec * p * (lp + H);
          }
        }
        fence_proxy_async_smem();
        cons_sync();
        if (tid == 0) {
          tma_store_2d(&mp.dlog, stg, b0 * A, c * TC);  // clipped at the tensor edges
          bulk_commit();
          if (pending >= 0) {
            bulk_wait_read_1();  // every store but the newest has read its stage
            mbar_arrive_cnt(&empty[pending], kCons / 32);
          }
          pending = s;
        }
      }
      if (tid == 0 && pending >= 0) {
        bulk_wait_read_all();
        mbar_arrive_cnt(&empty[pending], kCons / 32);
      }
    }
    cons_sync();
    if (tid == 0) mbar_arrive_cta(&sfree[set]);
  }
  if constexpr (LOSS) {
    if (tid == 0) bulk_wait_all();  // d_logits stores complete before exit
  }

  if constexpr (LOSS) {
    __shared__ double red[3][kCons / 32];
    __shared__ bool is_last;
    const int lane = tid & 31, w = tid >> 5;
    pg_sum = warp_sum(pg_sum);
    base_sum = warp_sum(base_sum);
    ent_sum = warp_sum(ent_sum);
    if (lane == 0) {
      red[0][w] = pg_sum;
      red[1][w] = base_sum;
      red[2][w] = ent_sum;
    }
    cons_sync();
    if (tid == 0) {
      double a0 = 0, a1 = 0, a2 = 0;
      for (int k = 0; k < kCons / 32; ++k) {
        a0 += red[0][k];
        a1 += red[1][k];
        a2 += red[2][k];
      }
      g.partials[3 * blockIdx.x + 0] = a0;
      g.partials[3 * blockIdx.x + 1] = a1;
      g.partials[3 * blockIdx.x + 2] = a2;
      __threadfence();
      is_last = atomicAdd(g.counter, 1u) == gridDim.x - 1;
    }
    cons_sync();
    if (is_last && tid == 0) {
      __threadfence();
      double a0 = 0, a1 = 0, a2 = 0;
      for (int k = 0; k < (int)gridDim.x; ++k) {
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
      *g.counter = 0u;
    }
  }
  set_status(g.status, bad);
}

}  // namespace vt2

// ---------------------------------------------------------------------------- host
// Returns BP_ERR_UNSUPPORTED when the shape is outside this kernel's regime (the
// caller then uses the generic kernel in vtrace.cu).
int vt2_launch(bool loss, const float* beh, const float* tgt, const int64_t* act, const void* disc_or_done,
               const float* rew, const float* val, const float* boot, int T, int B, int A,
               float clip_rho, float clip_pg_rho, float clip_c, float discount, float pg_cost,
               float baseline_cost, float entropy_cost, int reward_clip, float* vs, float* pg,
               float* log_rhos, float* beh_logp, float* tgt_logp, float* d_logits, float* d_baseline,
               double* losses, void* workspace, size_t ws_bytes, unsigned* status, cudaStream_t s) {
  using namespace vt2;
  constexpr int BT = 4;  // == number of consumer warps (one warp per column in the scan)
  if (!(A == 6 || A == 18) || B < 512 || T > kMaxT || (B * A) % 4 || (BT * A) % 4)
    return BP_ERR_UNSUPPORTED;
  const uintptr_t al = reinterpret_cast<uintptr_t>(beh) | reinterpret_cast<uintptr_t>(tgt) |
                       reinterpret_cast<uintptr_t>(act) | reinterpret_cast<uintptr_t>(rew) |
                       reinterpret_cast<uintptr_t>(val) | reinterpret_cast<uintptr_t>(disc_or_done) |
                       (loss ? reinterpret_cast<uintptr_t>(d_logits) : 0);
  if (al & 15u) return BP_ERR_UNSUPPORTED;
  if (int e = tma_init()) return e;
  const int TC = kCons / BT;
  Maps m;
  int rc;
  if ((rc = tma_make_2d(&m.beh, beh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, (long long)B * A, BT * A, TC, 0)))
    return rc;
  if ((rc = tma_make_2d(&m.tgt, tgt, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, (long long)B * A, BT * A, TC, 0)))
    return rc;
  if ((rc = tma_make_2d(&m.act, act, CU_TENSOR_MAP_DATA_TYPE_INT64, 8, T, B, BT, T, 0))) return rc;
  if ((rc = tma_make_2d(&m.rew, rew, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, BT, T, 0))) return rc;
  if ((rc = tma_make_2d(&m.val, val, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, BT, T, 0))) return rc;
  if (loss) {
    m.disc = m.rew;  // done flags are read by the producer warp directly (Args::done)
    if ((rc = tma_make_2d(&m.dlog, d_logits, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, (long long)B * A, BT * A,
                          TC, 0)))
      return rc;
  } else {
    if ((rc = tma_make_2d(&m.disc, disc_or_done, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, BT, T, 0))) return rc;
    m.dlog = m.beh;
  }
  Args g{};
  g.T = T;
  g.B = B;
  g.A = A;
  g.BT = BT;
  g.TC = TC;
  g.ntiles = (B + BT - 1) / BT;
  g.nchunks = (T + TC - 1) / TC;
  g.loss = loss;
  g.clip_rho = clip_rho;
  g.clip_pg_rho = clip_pg_rho;
  g.clip_c = clip_c;
  g.discount = discount;
  g.pg_cost = pg_cost;
  g.baseline_cost = baseline_cost;
  g.entropy_cost = entropy_cost;
  g.reward_clip = reward_clip;
  g.boot = boot;
  g.done = loss ? reinterpret_cast<const uint8_t*>(disc_or_done) : nullptr;
  g.vs = vs;
  g.pg = pg;
  g.log_rhos = log_rhos;
  g.beh_logp = beh_logp;
  g.tgt_logp = tgt_logp;
  g.d_baseline = d_baseline;
  g.losses = losses;
  g.status = status;
  const int grid = g.ntiles < 2 * tma_num_sms() ? g.ntiles : 2 * tma_num_sms();
  if (loss) {
    if (!workspace || ws_bytes < 256 + (size_t)grid * 3 * sizeof(double)) return BP_ERR_UNSUPPORTED;
    g.counter = reinterpret_cast<unsigned*>(workspace);
    g.partials = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + 256);
  }
  const Plan P = plan(T, BT, A, TC, loss);
#define BP_VT2(AT_, LOSS_)                                                                        \
  {                                                                                               \
    auto k = vt2_kernel<BT, AT_, LOSS_>;                                                          \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.total); \
    if (e != cudaSuccess) {                                                                       \
      set_error("vt2 smem attr: %s", cudaGetErrorString(e));                                      \
      return BP_ERR_LAUNCH;                                                                       \
    }                                                                                             \
    k<<<grid, kThreads, P.total, s>>>(g, m);                                                      \
    return check_launch("vt2_kernel");                                                            \
  }
  if (A == 6) {
    if (loss) BP_VT2(6, true) else BP_VT2(6, false)
  } else {
    if (loss) BP_VT2(18, true) else BP_VT2(18, false)
  }
#undef BP_VT2
}

}  // namespace bp
