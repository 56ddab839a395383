// tc_mlp.cuh -- fused multi-layer forward of the actor / critic MLPs on the tensor cores (sm_100a).
//
// One launch runs every hidden layer (and the actor's head layer) of up to MLP_MAXN network passes.
// A unit is (pass, 128-row block).  Layer 0 reads its input rows by TMA; every hidden layer's
// epilogue (bias + ReLU) writes its bf16 output into a shared-memory buffer in exactly the
// 128-byte-swizzled K-major layout the next layer's tcgen05.mma consumes, so hidden activations
// never make a round trip through L2 between layers.  Activations and packed ReLU masks go to HBM
// only for the passes whose backward needs them (TMA bulk stores straight from that buffer).
// Heads: critic -> N = 1 row dot fused into the last hidden epilogue; actor -> an N = 16k MMA on the
// last hidden buffer followed by the SAC / TD3 head epilogue (heads.cuh).
//
// Units are processed in groups ("super-units"): the passes of a group run back to back on the same
// 128-row block in one CTA.  A critic group may end with the fused loss epilogue (SURVEY.md §8(a)
// a4-a6; the same arithmetic as critic_loss_kernel): Bellman target y, g_q, the loss statistics
// partial of the block, and the critic-head backward dZ_L = g_q w_out 1[A_L > 0] for both critics,
// written through the shared buffer by TMA.  The last CTA reduces the statistics partials in block
// order into the step totals and snapshots the step counters for the optimizer.
#pragma once

#include "gemm.cuh"

namespace spz {

constexpr int MLP_MAXN = 6;  // passes per launch
constexpr int MLP_MAXL = 4;  // hidden layers
constexpr int MLP_MAXG = 2;  // group kinds per launch

struct MlpPass {
  const void* X;  // input rows [rows x k0] (bf16, pitch ldx)
  int ldx;
  int rows;
  int row0;  // actor head: local actor-pass row of this pass's row 0
  const void* W[MLP_MAXL + 1];  // bf16 weight shadows [out x in], pitch ldw
  int ldw[MLP_MAXL + 1];
  const float* bias[MLP_MAXL + 1];
  void* act[MLP_MAXL];        // bf16 hidden outputs [rows x h] (pitch h), or null (not stored)
  uint32_t* mask[MLP_MAXL];   // packed ReLU masks [rows x mask_ld] u32, or null
  const float* dot_w;         // critic head: q[m] = sum_n relu(z[m, n]) dot_w[n] + dot_b[0]
  const float* dot_b;
  float* dot_out;
};

// A group kind: passes p[pass[0..n)] run on the same row block, for every row block of rows rows.
// loss: 0 none; 1 loss rows (passes = q1, q2, q1', q2' on [s|a] / [s2|a']); 2 actor rows
// (passes = q1, q2 on [s|a~]).
struct MlpGroup {
  int n, loss, rows;
  int pass[4];
};

struct MlpLoss {
  const float *r, *d, *logp2, *logp, *log_alpha;
  const int64_t* step_p;  // step counters (step, t_c, t_a, t_al)
  const float* w[2];      // critic head weights (fp32 master)
  void* dZ[2];            // dZ_L of each critic [2 Bl x h] bf16: loss rows 0.., actor rows Bl..
  float *gq1, *gq2, *y;
  __nv_bfloat16* gq16[2];  // bf16 loss-row g_q, pitch 8 (tensor-core head gradients), may be null
  double* partials;       // [groups x NSTAT] statistics partials (one per super-unit)
  double* totals;
  int64_t* ctr_snap;
  float* la_snap;
  float* bc_snap;
  unsigned* ticket;
  float gamma, invB, beta1, beta2;
  int Bl, td3, delay;
};

struct MlpArgs {
  int n_pass;
  int L;       // hidden layers
  int h;       // hidden width (64, 128 or 256)
  int k0;      // input width (multiple of 64; zero-padded columns)
  int head_n;  // actor head width (2m SAC, m TD3); 0 = critic (row-dot head)
  int head_epi;  // EPI_SAC_HEAD / EPI_TD3_HEAD (actor)
  int mask_ld;
  HeadEpi head;
  MlpPass p[MLP_MAXN];
  // grouping: if n_group == 0 every pass is its own group
  int n_group;
  MlpGroup grp[MLP_MAXG];
  MlpLoss loss;  // used when a group has loss != 0
};

bool tc_mlp_supported(const MlpArgs& a);
cudaError_t tc_mlp_fwd(const MlpArgs& a, cudaStream_t st);
// Diagnostics: per-(CTA, unit, layer) timestamps of the fused kernel (see tc_mlp.cu).
cudaError_t mlp_trace(int on, unsigned long long* out, int n);

}  // namespace spz
