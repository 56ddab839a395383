// tc_actor_bwd.cuh -- fused actor backward on the tensor cores (sm_100a), SURVEY.md §8(a) a6 (the
// actor rows' input gradient through the critics) + a7 (actor head backward, eq. H, and the dgrad
// down the actor's hidden stack) in one launch.
//
// Per 128-row block of the s-rows:
//   S1  g_a  = sum_i dZ1_i W0_i[:, o:o+m]      critics' first-layer input gradient, action columns only
//              (K = h per critic, both critics into one TMEM accumulator; B = W0 read MN-major from
//               column o, so no transposed copy exists)
//   E1  dH   = eq. H (SAC: [g_mu | g_l] with g_lp = alpha / B; TD3: g_a (1 - a^2)) -> HBM (the head's
//              weight gradient operand) and shared memory (the next MMA's A operand)
//   S2  dA_L = dH W_head                        (K = nout <= 64)
//   E2  dZ_{L-1} = dA_L * 1[z_{L-1} > 0]        packed ReLU masks of the forward; -> HBM (TMA store) + SMEM
//   S3  dA_l = dZ_l W_l, l = L-1 .. 1           weight slabs streamed MN-major through the stage ring
//   E3  dZ_{l-1} = dA_l * 1[z_{l-1} > 0]
// Hidden gradients stay in shared memory between layers (the A operand of the next MMA), like the
// fused forward (tc_mlp.cuh).
#pragma once

#include "gemm.cuh"
#include "tc_mlp.cuh"

namespace spz {

struct ActorBwdArgs {
  int Bl, o, m, h, L, nout, td3, ncrit;
  int ldw0c;                       // pitch of the critics' layer-0 weight shadows (elements)
  int ldh;                         // dH pitch (elements)
  int mask_ld;                     // words per mask row
  const void* dZ1[2];              // critics' layer-0 dZ of the actor rows [Bl x h] (pitch h), bf16
  const void* W0c[2];              // critics' layer-0 weight shadows [h x ldw0c], bf16
  const void* Wa[MLP_MAXL + 1];    // actor weight shadows [out_l x ldwa_l], bf16
  int ldwa[MLP_MAXL + 1];
  const uint32_t* mask[MLP_MAXL];  // actor ReLU masks of the s-rows [Bl x mask_ld] per hidden layer
  void* dZa[MLP_MAXL];             // outputs dZ_l [Bl x h] (pitch h), bf16
  void* dH;                        // output [Bl x ldh], bf16
  const float *u, *a, *eps, *sig, *l;  // head cache of the s-rows, action-major [m x Bl]
  const float* log_alpha;
  float invB, lo, hi;
};

bool tc_actor_bwd_supported(const ActorBwdArgs& a);
cudaError_t tc_actor_bwd(const ActorBwdArgs& a, cudaStream_t st);

}  // namespace spz
