// LSTM recurrence on thread-block clusters (the fast path; lstm.cu holds the
// grid-cooperative fallback).  Same contract as lstm.cu: upstream nn.LSTM(H, H, 2)
// stepped per time row with done resets, input projections precomputed by tcgen05 GEMMs.
//
// One cluster of 16 CTAs per group of 8 batch columns.  CTA r of a cluster owns hidden
// units [34r, 34r+34) -> 136 gate rows {gate*H + j} (padded to 144 = 9 MMA row tiles).
// W_hh never leaves the register file: at kernel start every warp loads its share of
// the CTA's W_hh slice as bf16 mma.sync A-fragments (~108 registers per thread), so a
// time step is
//   forward : 12 warps x 3 (row-tile, K-quarter) items of m16n8k16 MMAs against h_{t-1}
//             (bf16, from shared memory via ldmatrix), a fixed-order sum of the K-quarters,
//             the cell update (f32, c in a register) by the thread owning (unit, batch),
//             and a bulk DSMEM copy of the CTA's 34 new h values per column to all 16 CTAs,
//             signalled on the receivers' mbarriers.
//   backward: partial W_hh^T dz over the CTA's own 136 rows for all H units (A-fragments
//             of W_hh^T), each owner's share sent by bulk DSMEM copy to the CTA owning those
//             units, then a fixed-order sum of the 16 partials (deterministic) and the
//             gate-gradient math.
// Operands of the recurrent MMAs are bf16 (W_hh, h_{t-1}, dz) with f32 accumulation --
// the same precision class as every other GEMM of the network; the cell state, gates and
// all element-wise math are f32 (MUFU tanh).  No grid-wide barrier, no L2 round trip on
// the recurrent critical path.
#include "common.cuh"
#include "lstm.h"
#include "tma_host.h"

namespace bp {

namespace {

constexpr int CS = 16;              // CTAs per cluster
constexpr int NB = 8;               // batch columns per cluster (MMA N)
constexpr int UC = 34;              // hidden units per CTA (16 * 34 = 544 >= H)
constexpr int RR = 4 * UC;          // 136 gate rows per CTA
constexpr int MT = 9;               // row tiles of 16 (144 rows)
constexpr int KST = 34;             // K steps of 16 over 544 hidden units
constexpr int RS = 152;             // dz row stride (bf16), RS/2 % 32 == 12
constexpr int WARPS = 12;
constexpr int THREADS = WARPS * 32;
constexpr int ITEMS = 3;            // work items per warp
constexpr int KSMAX = 9;            // K steps per item

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  return l | (h << 16);
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// four 8x8 bf16 matrices; lane l supplies the row address of matrix l/8, row l%8
__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// four transposed 8x8 bf16 matrices (B operand stored [k][n]); lane l supplies the address of
// row l % 8 of matrix l / 8
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                                  uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(saddr), "r"(rank));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// MUFU.TANH (max relative error ~2^-11, below the bf16 W_hh operand rounding of this path)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigm(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }

// W_hh element of local gate row R (= gate * UC + u) of CTA `rank`, hidden column k
__device__ __forceinline__ float w_local(const float* whh, int H, int rank, int R, int k) {
  if (R >= RR || k >= H) return 0.f;
  const int gate = R / UC, u = R % UC;
  const int j = rank * UC + u;
  if (j >= H) return 0.f;
  return whh[(size_t)(gate * H + j) * H + k];
}

__device__ unsigned long long* g_cl_trace = nullptr;  // diagnostics (bp_lstm_trace)

// SM cycle counter (one SM records: consistent; %globaltimer is too coarse for sub-us phases)
__device__ __forceinline__ unsigned long long gtimer() { return (unsigned long long)clock64(); }

constexpr int KH = CS * UC;         // 544 hidden rows of the transposed recurrent operand
constexpr uint32_t FWD_SLICE = UC * NB * 2;           // bytes of one CTA's h slice ([unit][batch])
constexpr uint32_t BWD_SLICE = UC * NB * 4;           // bytes of one CTA's partial for one owner
constexpr int OWNERS = UC * NB;                       // 272 owner threads (warps 0..8)

struct FwdSmem {
  float rec[2][NB][UC][8];               // step records {i, f, g, o, c, -} by step parity: the
                                         // box of one 4D TMA store (act8, [rows][H][8])
  __nv_bfloat16 hT[2][KH][NB];           // MMA operand h_{t-1}, transposed [unit][batch], by step
                                         // parity: every CTA's slice lands here directly (one
                                         // contiguous 544 B block per source), no unpack
  __nv_bfloat16 out[UC][NB];             // this CTA's new h slice [unit][batch]
  float red[4][MT * 16][NB];             // per K-quarter partial pre-gates
  uint64_t bar[2];                       // incoming-slice barriers, by step parity
};

struct BwdSmem {
  float recv[2][CS][UC][NB];             // [parity][source CTA][unit][batch] partial W^T dz
  float part[2][CS][UC][NB];             // outgoing partials, by step parity and owner CTA
  __nv_bfloat16 dz[NB][RS];              // own dz, [batch][local gate row]
  uint64_t bar[2];
};

// shared::cta -> shared::cluster bulk copy completing on the destination CTA's mbarrier
// 4D tensor store of a step-record box (smem -> global, bulk async-group of the issuing thread)
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, uint32_t src, int x, int y, int z, int w) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}

__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "r"(src), "r"(bytes), "r"(bar)
      : "memory");
}

}  // namespace

int lstm_cl_set_trace(void* buf) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  return cudaMemcpyToSymbol(g_cl_trace, &p, sizeof(p)) == cudaSuccess ? BP_OK : BP_ERR_LAUNCH;
}

// --------------------------------------------------------------------------- forward
// Per step: MMAs -> owners (cell update into staging, own h slice) -> 16 lanes send the
// slice to all 16 CTAs with bulk DSMEM copies completing on each receiver's mbarrier;
// while the slices travel, all threads write the step's outputs to global memory
// (coalesced, off the critical path) -> wait for the 16 incoming slices -> unpack.  The
// dataflow orders buffer reuse (a CTA cannot send step t+2 before it has received every
// CTA's step t+1, which each CTA sends only after it consumed step t), so there is no
// cluster-wide barrier inside the loop.
__global__ void __launch_bounds__(THREADS, 1) lstm_cl_fwd_kernel(const __grid_constant__ LstmFwdArgs a,
                                                                  const __grid_constant__ CUtensorMap tm_rec) {
  extern __shared__ __align__(128) unsigned char smraw[];
  FwdSmem& S = *reinterpret_cast<FwdSmem*>(smraw);
  const int H = a.H;
  const int rank = (int)cluster_rank();
  const int cb = (blockIdx.x / CS) * NB;  // first batch column of this cluster (within the pass)
  const int u0 = rank * UC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tig = lane & 3;
  unsigned long long* trace = (blockIdx.x == 0 && tid == 0) ? g_cl_trace : nullptr;
  if (trace) trace[4 * a.T1 * 2] = gtimer();

  // ---- A fragments of this warp's items (rows mt*16.., K-steps of quarter kq), pre-packed
  //      by lstm_cl_pack in per-lane order: coalesced 4-byte loads
  uint32_t af[ITEMS][KSMAX][4];
  {
    const uint32_t* fp = a.wfrag + (size_t)(rank * WARPS + warp) * (ITEMS * KSMAX * 4 * 32) + lane;
#pragma unroll
    for (int s = 0; s < ITEMS; ++s)
#pragma unroll
      for (int q = 0; q < KSMAX; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) af[s][q][r] = __ldg(fp + ((s * KSMAX + q) * 4 + r) * 32);
  }
  // ---- h0 of this cluster's columns (all units); padding zero
  for (int i = tid; i < KH * NB; i += THREADS) {
    const int k = i / NB, b = i % NB;
    const int col = cb + b;
    float v = 0.f;
    if (k < H && col < a.B) v = a.h0[(size_t)(a.b0 + col) * H + k];
    S.hT[0][k][b] = __float2bfloat16_rn(v);
  }
  for (int i = tid; i < UC * NB; i += THREADS) (&S.out[0][0])[i] = __float2bfloat16_rn(0.f);
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  // ---- owner role: thread (unit, batch) keeps c in a register
  const int ou = tid / NB, ob = tid % NB;
  const int j = u0 + ou;
  const int col = cb + ob;
  const bool owner = tid < OWNERS && j < H && col < a.B;
  float c = 0.f, hown = 0.f, gxn[4] = {0.f, 0.f, 0.f, 0.f};
  __nv_bfloat16 hb_out = __float2bfloat16_rn(0.f), hb_prev = hb_out;  // this step's bf16 sequence values
  bool donen = false;
  if (owner) {
    const size_t row = (size_t)a.b0 + col;
    c = a.c0[row * H + j];
    hown = a.h0[row * H + j];
#pragma unroll
    {  // gate-interleaved gx columns (j * 4 + gate): one 16-byte load
      const float4 v = *reinterpret_cast<const float4*>(a.gx + row * a.gx_ld + (size_t)j * 4);
      gxn[0] = v.x; gxn[1] = v.y; gxn[2] = v.z; gxn[3] = v.w;
    }
    donen = a.done[row];
  }
  uint32_t phase[2] = {0u, 0u};
  // ldmatrix.trans row address: lane l -> hidden row 16 ks + l (matrices: k-step ks rows 0-7,
  // 8-15, k-step ks + 1 rows 0-7, 8-15), 16 B per row
  const uint32_t ld_base = smem_u32(&S.hT[0][lane][0]);
  const int ncols = a.B - cb < NB ? a.B - cb : NB;
  cluster_sync_all();  // every CTA running, barriers initialised, before any DSMEM traffic
  // every CTA resident: a PDL-launched successor that does not read this kernel's output (the
  // next layer's weight packing, lstm_cl_pack / pack_lstm_wih) may start on the free SMs now
  pdl_trigger();
  if (trace) trace[4 * a.T1 * 2 + 1] = gtimer();
  // the step records {i, f, g, o, c} leave through one 4D TMA store per step (issued by thread
  // STORE_TID, asynchronous: no global-store instructions on the recurrent critical path); the
  // bf16 sequences (h_t, notdone_t h_{t-1}) are stored by the owners directly
  constexpr int STORE_TID = 32;
  if (tid == STORE_TID) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_rec)) : "memory");
  for (int t = 0; t < a.T1; ++t) {
    const int p = t & 1;
    if (trace) trace[t * 4 + 0] = gtimer();
    // ---- recurrent pre-gates W_hh h_{t-1}: 3 independent accumulator chains per warp
    {
      float acc[ITEMS][4];
#pragma unroll
      for (int s = 0; s < ITEMS; ++s) acc[s][0] = acc[s][1] = acc[s][2] = acc[s][3] = 0.f;
#pragma unroll
      for (int q = 0; q < KSMAX; q += 2) {
#pragma unroll
        for (int s = 0; s < ITEMS; ++s) {
          const int item = warp + WARPS * s;
          const int kq = item / MT;
          const int ks = kq * 9 + q;
          if (ks < KST && !(a.dbg & 2)) {
            uint32_t b0, b1, b2, b3;  // k-steps ks and ks + 1
            ldmatrix_x4_trans(ld_base + (uint32_t)((t & 1) * KH * NB * 2 + ks * 256), b0, b1, b2, b3);
            mma16816(acc[s], af[s][q], b0, b1);
            if (q + 1 < KSMAX && ks + 1 < KST) mma16816(acc[s], af[s][q + 1], b2, b3);
          }
        }
      }
#pragma unroll
      for (int s = 0; s < ITEMS; ++s) {
        const int item = warp + WARPS * s;
        const int mt = item % MT, kq = item / MT;
        *reinterpret_cast<float2*>(&S.red[kq][mt * 16 + g][2 * tig]) = make_float2(acc[s][0], acc[s][1]);
        *reinterpret_cast<float2*>(&S.red[kq][mt * 16 + g + 8][2 * tig]) = make_float2(acc[s][2], acc[s][3]);
      }
    }
    if (tid < CS) bulk_wait_read_all();  // the previous step's slice copies have read S.out
    if (tid == STORE_TID) bulk_wait_read_1();  // step t-2's record store has read S.rec[p]
    __syncthreads();
    if (trace) trace[t * 4 + 1] = gtimer();
    if (owner) {
      const size_t row = (size_t)t * a.ldb + a.b0 + col;
      const float nd = donen ? 0.f : 1.f;  // W (notdone h) = notdone (W h)
      float z[4];
#pragma unroll
      for (int gate = 0; gate < 4; ++gate) {
        const int R = gate * UC + ou;
        z[gate] = nd * ((S.red[0][R][ob] + S.red[1][R][ob]) + (S.red[2][R][ob] + S.red[3][R][ob])) + gxn[gate];
      }
      const float ig = sigm(z[0]), fg = sigm(z[1]), gg = tanh_fast(z[2]), og = sigm(z[3]);
      c = fg * (nd * c) + ig * gg;
      const float h = og * tanh_fast(c);
      const __nv_bfloat16 hb = __float2bfloat16_rn(h);
      S.out[ou][ob] = hb;
      if (!(a.dbg & 1)) {
        *reinterpret_cast<float4*>(&S.rec[p][ob][ou][0]) = make_float4(ig, fg, gg, og);
        S.rec[p][ob][ou][4] = c;
        fence_proxy_async_smem();  // generic writes -> the TMA store (async proxy)
      }
      hb_out = hb;
      hb_prev = __float2bfloat16_rn(nd * hown);
      hown = h;
      if (t == a.T1 - 1) {
        a.hN[(size_t)(a.b0 + col) * H + j] = h;
        a.cN[(size_t)(a.b0 + col) * H + j] = c;
      }
    }
    if (rank == 0 && tid < ncols && !(a.dbg & 1)) {  // bias (ones) column of both augmented rows
      const size_t row = (size_t)t * a.ldb + a.b0 + cb + tid;
      a.out_aug[row * a.aug_ld + H] = __float2bfloat16_rn(1.f);
      a.hprev_aug[row * a.aug_ld + H] = __float2bfloat16_rn(1.f);
    }
    __syncthreads();
    if (tid == STORE_TID && !(a.dbg & 1)) {
      tma_store_4d(&tm_rec, smem_u32(&S.rec[p][0][0][0]), 0, u0, a.b0 + cb, t);
      bulk_commit();
    }
    if (trace) trace[t * 4 + 2] = gtimer();
    const bool exch = t + 1 < a.T1;
    // ---- exchange: own slice -> every CTA's in[p][rank] (bulk DSMEM copies, one per lane)
    if (exch && warp == 0) {
      if (lane == 0) mbar_expect_tx(&S.bar[p], CS * FWD_SLICE);
      if (lane < CS) {
        fence_proxy_async_smem();
        bulk_s2cluster(mapa(smem_u32(&S.hT[(t + 1) & 1][rank * UC][0]), (uint32_t)lane), smem_u32(&S.out[0][0]),
                       FWD_SLICE, mapa(smem_u32(&S.bar[p]), (uint32_t)lane));
        bulk_commit();
      }
    }
    // the bf16 sequences: stored while the slices travel (off the owner -> exchange path);
    // the next step's inputs are prefetched here too -- issued before the owners' proxy fence
    // (MEMBAR) they would have stalled it until they returned
    if (owner) {
      const size_t row = (size_t)t * a.ldb + a.b0 + col;
      if (!(a.dbg & 1)) {
        a.out_aug[row * a.aug_ld + j] = hb_out;
        a.hprev_aug[row * a.aug_ld + j] = hb_prev;
      }
      if (t + 1 < a.T1) {
        const size_t nrow = row + a.ldb;
#pragma unroll
        for (int gate = 0; gate < 4; ++gate) gxn[gate] = a.gx[nrow * a.gx_ld + (size_t)j * 4 + gate];
        donen = a.done[nrow];
      }
    }
    if (!exch) break;
    mbar_wait_parity(&S.bar[p], phase[p]);
    phase[p] ^= 1u;
    // (the slices landed in hT[(t + 1) & 1]: each thread's own wait orders its reads of them;
    //  S.red / S.out / S.rec reuse is ordered by the barriers of the next step)
    if (trace) trace[t * 4 + 3] = gtimer();
  }
  if (tid < CS) bulk_wait_read_all();
  if (tid == STORE_TID) bulk_wait_all();  // the record stores are complete before the CTA exits
  cluster_sync_all();  // no CTA leaves while a peer may still read / write its shared memory
}

// --------------------------------------------------------------------------- backward
__global__ void __launch_bounds__(THREADS, 1) lstm_cl_bwd_kernel(const LstmBwdArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  BwdSmem& S = *reinterpret_cast<BwdSmem*>(smraw);
  const int H = a.H;
  const int rank = (int)cluster_rank();
  const int cb = (blockIdx.x / CS) * NB;
  const int u0 = rank * UC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tig = lane & 3;

  // ---- A fragments of W_hh^T (rows = hidden column j, K = own gate rows), pre-packed
  uint32_t af[ITEMS][KSMAX][4];
  {
    const uint32_t* fp = a.wfrag + (size_t)(rank * WARPS + warp) * (ITEMS * KSMAX * 4 * 32) + lane;
#pragma unroll
    for (int s = 0; s < ITEMS; ++s)
#pragma unroll
      for (int q = 0; q < KSMAX; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) af[s][q][r] = __ldg(fp + ((s * KSMAX + q) * 4 + r) * 32);
  }
  unsigned long long* trace = (blockIdx.x == 0 && tid == 0) ? g_cl_trace : nullptr;
  if (trace) trace += (size_t)4 * a.T1;
  for (int i = tid; i < NB * RS; i += THREADS) (&S.dz[0][0])[i] = __float2bfloat16_rn(0.f);
  for (int i = tid; i < 2 * CS * UC * NB; i += THREADS) (&S.part[0][0][0][0])[i] = 0.f;
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  const int ou = tid / NB, ob = tid % NB;
  const int j = u0 + ou;
  const int col = cb + ob;
  const bool owner = tid < UC * NB && j < H && col < a.B;
  float dcf = 0.f;
  uint32_t phase[2] = {0u, 0u};
  // ldmatrix row address: matrix m = lane / 8 -> (k-step +m/2, k half m%2), row n = lane % 8
  const uint32_t ld_base = smem_u32(&S.dz[lane & 7][((lane >> 3) & 1) * 8 + (lane >> 4) * 16]);
  cluster_sync_all();
  pdl_trigger();  // every CTA resident: the previous layer's weight gradients may start beside

  // the owner's inputs of step tt, prefetched one step ahead (issued after the previous
  // step's owner math, so no global load sits in front of the recurrent MMAs)
  float dho = 0.f, ig = 0.f, fg = 0.f, gg = 0.f, og = 0.f, cc = 0.f, cprev = 0.f, nd = 0.f, ndn = 0.f;
  auto load_step = [&](int tt) {
    if (!owner) return;
    const size_t row = (size_t)tt * a.ldb + a.b0 + col;
    dho = a.dh_out[row * a.dh_ld + j];
    const float* rec = a.act8 + (row * H + j) * 8;
    const float4 gv = *reinterpret_cast<const float4*>(rec);
    ig = gv.x;
    fg = gv.y;
    gg = gv.z;
    og = gv.w;
    cc = rec[4];
    nd = a.done[row] ? 0.f : 1.f;
    cprev = tt == 0 ? a.c0[(size_t)(a.b0 + col) * H + j] : a.act8[((row - a.ldb) * H + j) * 8 + 4];
    ndn = tt + 1 < a.T1 ? (a.done[row + a.ldb] ? 0.f : 1.f) : 0.f;
  };
  load_step(a.T1 - 1);

  for (int t = a.T1 - 1; t >= 0; --t) {
    const size_t trow = (size_t)t * a.ldb + a.b0;
    if (trace) trace[t * 4 + 0] = gtimer();
    float dh_rec = 0.f;
    if (t + 1 < a.T1) {
      const int p = t & 1;
      // partial[j][b] = sum over own rows r of W_hh[r][j] dz_{t+1}[r][b], staged by owner CTA of j
      {
        float acc[ITEMS][4];
#pragma unroll
        for (int s = 0; s < ITEMS; ++s) acc[s][0] = acc[s][1] = acc[s][2] = acc[s][3] = 0.f;
#pragma unroll
        for (int q = 0; q < KSMAX; q += 2) {
          uint32_t b0, b1, b2, b3;  // k-steps q and q + 1
          ldmatrix_x4(ld_base + (uint32_t)q * 32u, b0, b1, b2, b3);
#pragma unroll
          for (int s = 0; s < ITEMS; ++s) {
            if (warp + WARPS * s < KST) {
              mma16816(acc[s], af[s][q], b0, b1);
              if (q + 1 < KSMAX) mma16816(acc[s], af[s][q + 1], b2, b3);
            }
          }
        }
        // (S.part[p] was last read by the copies of step t + 2: waited for at the end of t + 1)
#pragma unroll
        for (int s = 0; s < ITEMS; ++s) {
          const int mt = warp + WARPS * s;
          if (mt < KST) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              const int jj = mt * 16 + g + 8 * half;
              if (jj < H)
                *reinterpret_cast<float2*>(&S.part[p][jj / UC][jj % UC][2 * tig]) =
                    make_float2(acc[s][2 * half], acc[s][2 * half + 1]);
            }
          }
        }
      }
      __syncthreads();
      if (trace) trace[t * 4 + 1] = gtimer();
      if (warp == 0) {
        if (lane == 0) mbar_expect_tx(&S.bar[p], CS * BWD_SLICE);
        if (lane < CS) {
          fence_proxy_async_smem();
          bulk_s2cluster(mapa(smem_u32(&S.recv[p][rank][0][0]), (uint32_t)lane), smem_u32(&S.part[p][lane][0][0]),
                         BWD_SLICE, mapa(smem_u32(&S.bar[p]), (uint32_t)lane));
          bulk_commit();
        }
      }
      mbar_wait_parity(&S.bar[p], phase[p]);
      phase[p] ^= 1u;
      if (trace) trace[t * 4 + 2] = gtimer();
      if (owner) {
#pragma unroll
        for (int src = 0; src < CS; ++src) dh_rec += S.recv[p][src][ou][ob];
      }
    }
    if (owner) {
      const size_t row = trow + col;
      const float dh = dho + ndn * dh_rec;
      const float tc = tanh_fast(cc);
      cprev *= nd;
      const float dc = dh * og * (1.f - tc * tc) + ndn * dcf;
      const float dz[4] = {dc * gg * ig * (1.f - ig), dc * cprev * fg * (1.f - fg), dc * ig * (1.f - gg * gg),
                           dh * tc * og * (1.f - og)};
      dcf = dc * fg;
      // gate-interleaved dgates columns (j * 4 + gate): one 8-byte store
      uint32_t zp[2];
#pragma unroll
      for (int gate = 0; gate < 4; ++gate) {
        const __nv_bfloat16 zb = __float2bfloat16_rn(dz[gate]);
        S.dz[ob][gate * UC + ou] = zb;
        const uint32_t bits = __bfloat16_as_ushort(zb);
        if (gate & 1) zp[gate >> 1] |= bits << 16;
        else zp[gate >> 1] = bits;
      }
      *reinterpret_cast<uint2*>(a.dgates + row * a.dg_ld + (size_t)j * 4) = make_uint2(zp[0], zp[1]);
      if (t > 0) load_step(t - 1);
    }
    if (tid < CS) bulk_wait_read_1();  // step t+1's copies have read S.part[p ^ 1] (reused by t - 1)
    __syncthreads();
    if (trace) trace[t * 4 + 3] = gtimer();
  }
  if (tid < CS) bulk_wait_read_all();
  cluster_sync_all();
}

// --------------------------------------------------------------------------- fragment pack
// W_hh (f32, torch layout) -> per-lane bf16 mma.sync A-fragments of both recurrent kernels:
// frag[dir][rank][warp][item][kstep][reg][lane] (u32 = 2 bf16), dir 0 forward (rows = own
// gate rows, K = hidden), dir 1 backward (rows = hidden, K = own gate rows).  Run once per
// weight update; the kernels then load their ~108 fragment registers with coalesced loads.
// PDL: reads only the parameters, so it starts early (beside the previous layer's recurrence)
// and waits for its predecessor only at the end -- completion stays transitive for the chain
__global__ void lstm_cl_pack_kernel(const float* __restrict__ whh, int H, uint32_t* __restrict__ frag) {
  pdl_trigger();
  constexpr int PER_WARP = ITEMS * KSMAX * 4 * 32;
  constexpr int PER_DIR = CS * WARPS * PER_WARP;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * PER_DIR; i += gridDim.x * blockDim.x) {
    const int dir = i / PER_DIR;
    int rem = i % PER_DIR;
    const int rank = rem / (WARPS * PER_WARP);
    rem %= WARPS * PER_WARP;
    const int warp = rem / PER_WARP;
    rem %= PER_WARP;
    const int s = rem / (KSMAX * 128), q = (rem / 128) % KSMAX, r = (rem / 32) % 4, lane = rem % 32;
    const int g = lane >> 2, tig = lane & 3;
    float v0 = 0.f, v1 = 0.f;
    if (dir == 0) {
      const int item = warp + WARPS * s;
      const int mt = item % MT, kq = item / MT;
      const int ks = kq * 9 + q;
      if (ks < KST) {
        const int row = mt * 16 + g + ((r & 1) ? 8 : 0), c0 = ks * 16 + 2 * tig + ((r & 2) ? 8 : 0);
        v0 = w_local(whh, H, rank, row, c0);
        v1 = w_local(whh, H, rank, row, c0 + 1);
      }
    } else {
      const int mt = warp + WARPS * s;
      if (mt < KST) {
        const int jrow = mt * 16 + g + ((r & 1) ? 8 : 0), k0 = q * 16 + 2 * tig + ((r & 2) ? 8 : 0);
        v0 = w_local(whh, H, rank, k0, jrow);
        v1 = w_local(whh, H, rank, k0 + 1, jrow);
      }
    }
    frag[i] = pack2(v0, v1);
  }
  pdl_wait();
}

size_t lstm_cl_frag_words() { return (size_t)2 * CS * WARPS * ITEMS * KSMAX * 4 * 32; }
size_t lstm_cl_frag_dir_words() { return (size_t)CS * WARPS * ITEMS * KSMAX * 4 * 32; }

int lstm_cl_pack(const float* whh, int H, uint32_t* frag, cudaStream_t s) {
  // one word per thread: the per-word index math and scattered W_hh reads are latency-bound
  launch_pdl(lstm_cl_pack_kernel, dim3((unsigned)((lstm_cl_frag_words() + 255) / 256)), dim3(256), 0, s, whh, H,
             frag);
  return check_launch("lstm_cl_pack_kernel");
}

// --------------------------------------------------------------------------- launch
static int g_cluster_ok = -1;  // -1 unknown, 0 unavailable, else max active clusters

template <typename Args>
static int cl_launch(const void* fn, const Args& a, size_t smem, const char* name, cudaStream_t s,
                     const CUtensorMap* tm = nullptr) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) {
    set_error("%s attributes: %s", name, cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  const int nclus = (a.B + NB - 1) / NB;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclus * CS);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<Args*>(&a), const_cast<CUtensorMap*>(tm)};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) {
    set_error("%s launch: %s", name, cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  return check_launch(name);
}

// number of 8-column clusters that can run at once (0: 16-CTA clusters unavailable)
int lstm_cluster_capacity() {
  if (g_cluster_ok >= 0) return g_cluster_ok;
  const void* fns[2] = {(const void*)lstm_cl_fwd_kernel, (const void*)lstm_cl_bwd_kernel};
  const size_t sm[2] = {sizeof(FwdSmem), sizeof(BwdSmem)};
  int cap = 1 << 30;
  for (int i = 0; i < 2; ++i) {
    if (cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm[i]) != cudaSuccess ||
        cudaFuncSetAttribute(fns[i], cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      g_cluster_ok = 0;
      return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = sm[i];
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fns[i], &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cap = n < cap ? n : cap;
  }
  g_cluster_ok = cap;
  return cap;
}

int lstm_cluster_batch() { return lstm_cluster_capacity() * NB; }

int lstm_cl_launch_fwd(const LstmFwdArgs& a, cudaStream_t s) {
  if (a.H > CS * UC || a.H < 1 || a.B < 1 || a.B > lstm_cluster_batch()) {
    set_error("lstm cluster: H=%d (<= %d), B pass %d (<= %d)", a.H, CS * UC, a.B, lstm_cluster_batch());
    return BP_ERR_ARG;
  }
  // act8 [T1][ldb][H][8] f32; one box = the CTA's UC units x the cluster's NB batch columns of a step
  CUtensorMap tm;
  const long long dims[4] = {8, a.H, a.ldb, a.T1};
  const long long strides[3] = {32, 32LL * a.H, 32LL * a.H * a.ldb};
  const int box[4] = {8, UC, NB, 1};
  if (int e = tma_make_f32(&tm, a.act8, 4, dims, strides, box)) return e;
  return cl_launch((const void*)lstm_cl_fwd_kernel, a, sizeof(FwdSmem), "lstm_cl_fwd_kernel", s, &tm);
}

int lstm_cl_launch_bwd(const LstmBwdArgs& a, cudaStream_t s) {
  if (a.H > CS * UC || a.H < 1 || a.B < 1 || a.B > lstm_cluster_batch()) {
    set_error("lstm cluster: H=%d (<= %d), B pass %d (<= %d)", a.H, CS * UC, a.B, lstm_cluster_batch());
    return BP_ERR_ARG;
  }
  return cl_launch((const void*)lstm_cl_bwd_kernel, a, sizeof(BwdSmem), "lstm_cl_bwd_kernel", s);
}

}  // namespace bp
