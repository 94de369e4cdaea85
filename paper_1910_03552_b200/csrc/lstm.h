// Internal interface of the LSTM recurrent kernels (lstm.cu) used by network.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bp {

constexpr int kLstmU = 4;       // hidden units per CTA (4 gate rows each -> 16 W_hh rows)
constexpr int kLstmB = 32;      // batch columns per recurrent pass (host loops over chunks)
constexpr int kLstmKmax = 576;  // max hidden size (A <= 31 -> H = 513 + A <= 544)

// Rows of every per-row tensor are t * ldb + b0 + b (time-major, full batch ldb).
struct LstmFwdArgs {
  int H, B, ldb, b0, T1;
  const float* whh;           // [4H][H] f32 (torch weight_hh)
  const float* gx;            // [rows][gx_ld] x W_ih^T + b_ih + b_hh (gate order i, f, g, o)
  int gx_ld;
  const uint8_t* done;        // [rows] (bool storage): state reset before step t
  const float* h0;            // [ldb][H]
  const float* c0;            // [ldb][H]
  float* hx;                  // [2][H][kLstmB] exchange (per chunk)
  float* gates;               // cooperative path: [rows][4H] activated i, f, g, o
  float* cseq;                // cooperative path: [rows][H]
  float* act8;                // cluster path: [rows][H][8] f32 {i, f, g, o, c, -, -, -}
  __nv_bfloat16* out_aug;     // [rows][aug_ld]: [h_t | 1 | 0]
  __nv_bfloat16* hprev_aug;   // [rows][aug_ld]: [notdone_t * h_{t-1} | 1 | 0]
  int aug_ld;
  float* hN;                  // [ldb][H]
  float* cN;                  // [ldb][H]
  int dbg;                    // diagnostics: bit 0 skip the step-output stores, bit 1 skip MMAs
  const uint32_t* wfrag;      // cluster path: packed forward A-fragments (lstm_cl_pack)
};

struct LstmBwdArgs {
  int H, B, ldb, b0, T1;
  const float* whh;
  const float* gates;         // cooperative path (as LstmFwdArgs)
  const float* cseq;
  const float* act8;          // cluster path (as LstmFwdArgs)
  const float* c0;
  const uint8_t* done;
  const float* dh_out;        // [rows][dh_ld] gradient w.r.t. the layer output h_t
  int dh_ld;
  float* part;                // [2][grid][kLstmB][Hp] recurrent partial sums
  __nv_bfloat16* dgates;      // [rows][dg_ld] pre-activation gate gradients
  int dg_ld;
  const uint32_t* wfrag;      // cluster path: packed backward A-fragments (lstm_cl_pack)
};

int lstm_grid(int H);
// cluster path (lstm_cluster.cu): columns per pass (0 = 16-CTA clusters unavailable)
int lstm_cluster_batch();
int lstm_cl_launch_fwd(const LstmFwdArgs& a, cudaStream_t s);
int lstm_cl_launch_bwd(const LstmBwdArgs& a, cudaStream_t s);
int lstm_cl_set_trace(void* buf);
// W_hh -> packed bf16 A-fragments of both cluster kernels (forward block, then backward)
size_t lstm_cl_frag_words();
size_t lstm_cl_frag_dir_words();
int lstm_cl_pack(const float* whh, int H, uint32_t* frag, cudaStream_t s);
// 0 auto (cluster path when available), 1 cooperative grid path, 2 cluster path
extern int g_lstm_mode;
int lstm_launch_fwd(const LstmFwdArgs& a, cudaStream_t s);
int lstm_launch_bwd(const LstmBwdArgs& a, cudaStream_t s);
size_t lstm_part_floats(int H);

}  // namespace bp
