// learner.cu -- the update step: buffers, the per-batch launch plan, CUDA-graph replay, C API.
//
// One step is a fixed chain of device kernels with no host
// round-trip: gather -> actor forward on [s2; s] -> head -> target critics -> online
// critics -> Bellman target + losses -> critic backward -> actor backward ->
// statistics -> fused Adam + Polyak -> counter advance.  The chain is captured once
// per batch size into a CUDA graph and replayed n_steps times; the step counter and
// the ring fill live in device memory so the replay needs no host updates.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>

#include "comm.h"
#include "gemm.cuh"
#include "internal.h"
#include "kernels.cuh"
#include "tc_mlp.cuh"
#include "tc_gemm.cuh"
#include "tc_actor_bwd.cuh"

namespace spz {

// NET_V / NET_VT: SAC v1's state-value network and its Polyak target (reading #24)
enum NetId { NET_ACTOR = 0, NET_Q1 = 1, NET_Q2 = 2, NET_Q1T = 3, NET_Q2T = 4, NET_ACTORT = 5, NET_V = 6, NET_VT = 7, N_NETS = 8 };

struct NetLayout {
  int nl = 0;
  int in[8] = {}, out[8] = {};
  int64_t w[8] = {}, b[8] = {};  // master offsets relative to the net base
  int ld[8] = {};                // shadow row stride (elements, multiple of 8 -> 16-byte rows)
  int64_t sw[8] = {};            // shadow offsets relative to the net shadow base
  int64_t np = 0, ns = 0;
};

// kpad: row pitch granule of the layer-0 weight shadow (64 on the tensor-core path: 128-byte rows, so
// the first layer's TMA boxes are whole rows and its contraction runs over the zero-padded width)
static NetLayout make_layout(int in, int h, int L, int out, int kpad) {
  NetLayout n;
  n.nl = L + 1;
  int64_t p = 0, s = 0;
  for (int l = 0; l <= L; ++l) {
    n.in[l] = l == 0 ? in : h;
    n.out[l] = l == L ? out : h;
    n.w[l] = p;
    p += (int64_t)n.in[l] * n.out[l];
    n.b[l] = p;
    p += n.out[l];
    n.ld[l] = (int)round_up(n.in[l], l == 0 ? kpad : 8);
    n.sw[l] = s;
    s += round_up((int64_t)n.out[l] * n.ld[l], 64);
  }
  n.np = p;
  n.ns = s;
  return n;
}

struct Op {
  const char* cls;
  std::function<cudaError_t(cudaStream_t)> fn;
  int launches = 1;  // kernels this op launches
};

// diagnostics: SPZ_DZ_SPLIT=1 writes dZ_L in critic_dz_kernel at every width (h <= 256: in the loss kernel)
static bool dz_split_env() {
  const char* e = std::getenv("SPZ_DZ_SPLIT");
  return e && e[0] == '1';
}

// copies the read-back block into host-mapped memory (spz_update_async)
__global__ void publish_kernel(const unsigned long long* __restrict__ src, unsigned long long* dst, int words) {
  pdl_wait();  // (launched programmatically behind the update's last kernel where SPZ_PUBLISH_PDL is on)
  for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  // no system-scope fence: the host reads the slot only after the event recorded behind this kernel completed
  // (stream order makes the kernel's writes to mapped host memory visible by then)
}
static bool publish_pdl_env() {
  const char* e = std::getenv("SPZ_PUBLISH_PDL");
  return !(e && std::atoi(e) == 0);
}

// diagnostics: SPZ_ACTOR_BWD_UNFUSED=1 runs the actor backward as separate GEMM / head launches
static bool actor_bwd_unfused_env() {
  const char* e = std::getenv("SPZ_ACTOR_BWD_UNFUSED");
  return e && e[0] == '1';
}

// diagnostics: SPZ_FP32_SIMT=1 runs the FP32 precision path on the SIMT kernel instead of 3xTF32
static bool defer_totals_off_env() {
  const char* e = std::getenv("SPZ_DEFER_TOTALS");
  return e && std::atoi(e) == 0;
}
static bool wgrad_pre_off_env() {
  const char* e = std::getenv("SPZ_WGRAD_PRE");
  return e && std::atoi(e) == 0;
}
static bool fp32_simt_env() {
  static const bool on = [] {
    const char* e = std::getenv("SPZ_FP32_SIMT");
    return e && e[0] == '1';
  }();
  return on;
}

// One backend per precision: bf16 -> tcgen05 kind::f16, FP32 -> 3xTF32 tcgen05 (the SIMT kernel only under
// the explicit SPZ_FP32_SIMT=1 diagnostic).  The plan checks every GEMM against these kernels when it is
// built and fails with SPZ_EUNSUPPORTED instead of dispatching anywhere else (gemm_supported below).
template <typename T>
static bool gemm_supported(const GemmArgs& a) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) return tc_gemm_supported(a);
  else return fp32_simt_env() || tc_gemm_tf32_supported(a);
}

template <typename T>
static cudaError_t run_gemm(const GemmArgs& a, cudaStream_t st) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) return tc_gemm_bf16(a, st);
  else return fp32_simt_env() ? gemm_simt<T>(a, st) : tc_gemm_tf32x3(a, st);
}

}  // namespace spz

using namespace spz;

struct spz_learner {
  spz_config cfg{};
  spz_replay* ring = nullptr;
  int device = 0;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  bool td3 = false, bf16 = false;
  bool ddpg = false;  // TD3 kernels with the twin critic tied to the first (spz.h)
  bool v1 = false;    // SAC v1: state-value network V (+ target), no target critics (spz.h, reading #24)
  int o = 0, m = 0, h = 0, L = 0;
  size_t esz = 4;
  int64_t max_local = 0;  // rows handled by this rank at max_batch
  int64_t row0_max = 0;

  NetLayout net[N_NETS];
  bool has_net[N_NETS] = {};
  int64_t pbase[N_NETS] = {}, sbase[N_NETS] = {};
  int64_t p_log_alpha = 0, P_total = 0, S_total = 0;
  float *P = nullptr, *Mo = nullptr, *Vo = nullptr;
  void* S = nullptr;
  int64_t* counters = nullptr;  // step, t_critic, t_actor, t_alpha
  int* d_flag = nullptr;
  cudaEvent_t ev_read = nullptr;  // recorded after every enqueued update: ring pushes wait on it
  uint64_t seen_pack_gen = 0;     // ring->pack_gen at this learner's last wait on ev_pack
  // spz_update_async keeps up to two updates in flight; each owns a pinned slot for its read-back
  // device read-back block: the step statistics, counters and non-finite flag, contiguous so one copy
  // returns them
  struct ReadBack {
    StatsOut stats;
    int64_t ctr[8];
    int flag;
    int pad[3];
  };
  ReadBack* d_rb = nullptr;
  struct HostSlot {
    ReadBack rb;
  };
  HostSlot* h_slots = nullptr;    // pinned, host-mapped [2]
  unsigned long long* d_slots = nullptr;  // device view of h_slots (publish_kernel writes it)
  cudaEvent_t ev_slot[2] = {nullptr, nullptr};
  int inflight[2] = {0, 0}, n_inflight = 0, next_slot = 0;  // slot queue, oldest first
  int64_t host_step = 0;          // global step after every enqueued update (valid while n_inflight > 0)
  int plan_track_gen = 0;         // ring->track_gen the plan's gather was built for
  bool ctr_cached = false;  // h_counters[0..3] / h_flag mirror the device (set by read_counters; cleared while
                            // steps are enqueued): spz_update skips the leading device round trip
  StatsOut* d_stats = nullptr;
  StatsOut* h_stats = nullptr;  // pinned
  int* h_flag = nullptr;        // pinned
  int64_t* h_counters = nullptr;  // pinned

  // activations (T unless noted); sized for max_local rows
  void *Xa = nullptr, *Xc = nullptr, *dH = nullptr;
  int lda = 0, ldc = 0, ldh = 0;
  void* Aact[8] = {};
  void* dZa[8] = {};
  void* Aon[2][8] = {};
  void* Atg[2][8] = {};
  void* dZc[2][8] = {};
  uint32_t* mask_a[8] = {};     // packed ReLU masks of the actor hidden layers [2B x mw]
  uint32_t* mask_c[2][8] = {};  // ... and of the online critics' hidden layers
  int mw = 0;                   // mask words per row
  int qp = 1;                   // q partial slots per row (fused row dot over 256-column tiles)
  float* H = nullptr;
  float *q_on[2] = {}, *q_tg[2] = {}, *gq[2] = {}, *dXc[2] = {};
  // SAC v1 value network: activations / masks / gradients of the s rows, target activations (GEMM path)
  void *Av[8] = {}, *AvT[8] = {}, *dZv[8] = {};
  uint32_t* mask_v[8] = {};
  float *v_on = nullptr, *v_tg = nullptr, *gv = nullptr;
  __nv_bfloat16* gv16 = nullptr;
  __nv_bfloat16* gq16[2] = {};  // bf16 loss-row g_q, pitch 8 (tensor-core head gradients)
  float *logp = nullptr, *logp2 = nullptr, *r = nullptr, *d = nullptr, *y = nullptr;
  HeadCache cache{};
  int32_t* idx = nullptr;
  double* stat_partials = nullptr;
  int max_stat_blocks = 0;
  float* G = nullptr;  // gradient partials
  int64_t G_total = 0;
  AdamSegment* d_segs = nullptr;
  int max_segs = 0;
  ShadowEntry* d_shadow = nullptr;
  int n_shadow = 0;
  // row-sharded group (world_size > 1) and actor/critic split roles
  bool split = false;  // role != ALL: this learner runs one half of the Jacobi step
  int gsize = 1;       // ranks sharing this learner's role (row-sharded group)
  Comm comm;           // all ranks (exchange between the role groups)
  Comm gcomm;          // this role's group (gradient allreduce); == comm when not split
  ShadowEntry* d_shadow_recv = nullptr;  // shadows of the networks this role receives
  int n_shadow_recv = 0;
  float* Gred = nullptr;     // contiguous gradients of every trained tensor (+ log alpha slot)
  int64_t Gred_total = 0;
  double* statsum = nullptr;  // this rank's (then the group's) loss statistic totals

  // plan
  int64_t plan_B = -1;
  std::vector<Op> ops[2];  // [0] = plain step, [1] = TD3 delayed step (SAC uses [0] only)
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  cudaGraphExec_t exec_pub[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // + read-back publish to host slot [s]
  int n_adam_segs = 0;
  uint64_t sync_version = 0;
  uint64_t* h_sync = nullptr;  // pinned: the publication's seq / header words (spz_sync_actor)
  int* h_gate = nullptr;       // mapped: spz_learner_profile's release word
  int* d_gate = nullptr;
  unsigned* tickets = nullptr;  // last-block counter of the loss kernel
  unsigned* sched = nullptr;    // dynamic GEMM tile schedules: [counter, finished CTAs] per launch that uses one
  int64_t* ctr_snap = nullptr;  // counters as read at the start of the step (loss kernel -> Adam)
  std::vector<void*> allocs;
  struct DebugBuf { std::string name; void* ptr; size_t bytes; int esz; };
  std::vector<DebugBuf> debug;

  ~spz_learner();
};

namespace spz {

static spz_status dalloc(spz_learner* Lr, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (cudaMalloc(p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(SPZ_ENOMEM, "spz_learner_create: cannot allocate " + std::to_string(bytes) + " device bytes");
  }
  Lr->allocs.push_back(*p);
  // ordered on the learner's own (non-blocking) stream: the legacy default stream is not
  if (cudaMemsetAsync(*p, 0, bytes, Lr->own_stream) != cudaSuccess) return fail(SPZ_ECUDA, "cudaMemsetAsync failed");
  return SPZ_OK;
}


// Elements per float4 Adam segment (<= 4 x ADAM_NT; 0: scalar segments only).  SPZ_ADAM_VEC overrides.
static int adam_vec_seg() {
  if (const char* e = std::getenv("SPZ_ADAM_VEC")) return std::max(0, std::min(4 * ADAM_NT, std::atoi(e) / 4 * 4));
  return 4 * ADAM_NT;
}

// Split-K count of the merged weight-gradient GEMM.  Cost model per split count S (microseconds):
// waves of output tiles (128 x 256 each) over the SMs x (rows each tile contracts + a fixed per-tile
// cost of ~256 rows: epilogue + partial store) x ~7 ns per row (2*128*256 flops at ~9.3 TF/s per SM),
// plus the split partials' HBM traffic (written here, read by Adam: 8 B per parameter per split at
// ~6.5 TB/s).  The cheapest S wins, the smaller on a tie.  (The old fill rule S = floor(SMs / tiles)
// fell to S = 1 at 88 tiles -- HUM SAC v1 -- leaving 40% of the SMs idle over K = 65536.)  Never above
// the count at the largest batch, for which the partials are allocated.
static int wgrad_splits_at(const spz_learner* Lr, int64_t Bl, int sms) {
  const bool actor_on = Lr->cfg.role != SPZ_ROLE_CRITIC, critic_on = Lr->cfg.role != SPZ_ROLE_ACTOR;
  int64_t tiles = 0;
  auto net_tiles = [&](const NetLayout& n, int layers) {
    for (int l = 0; l < layers; ++l) tiles += cdiv(n.out[l], 128) * cdiv(n.in[l], 256);
  };
  if (critic_on) net_tiles(Lr->net[NET_Q1], Lr->net[NET_Q1].nl), net_tiles(Lr->net[NET_Q2], Lr->net[NET_Q2].nl);
  if (critic_on && Lr->v1) net_tiles(Lr->net[NET_V], Lr->net[NET_V].nl);
  if (actor_on) net_tiles(Lr->net[NET_ACTOR], Lr->net[NET_ACTOR].nl);
  tiles = std::max<int64_t>(1, tiles);
  int64_t params = 0;
  for (int id : {NET_Q1, NET_Q2, NET_V, NET_ACTOR}) {
    if (!Lr->has_net[id]) continue;
    const bool on = id == NET_ACTOR ? actor_on : critic_on;
    if (on) params += Lr->net[id].np;
  }
  const int smax = (int)std::max<int64_t>(1, std::min<int64_t>(32, Bl / 256));
  if (const char* e = std::getenv("SPZ_WGRAD_SC"))  // diagnostics: fixed split count
    if (std::atoi(e) > 0) return std::min(std::atoi(e), smax);
  int best = 1;
  double best_cost = 0.0;
  for (int S = 1; S <= smax; ++S) {
    const double waves = (double)cdiv(tiles * S, (int64_t)sms);
    const double cost = waves * ((double)cdiv(Bl, S) + 256.0) * 7e-3 + (double)S * params * 8.0 / 6.5e6;
    if (S == 1 || cost < best_cost) best = S, best_cost = cost;
  }
  return best;
}
static int wgrad_splits(const spz_learner* Lr, int64_t Bl) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::min(wgrad_splits_at(Lr, Bl, sms), wgrad_splits_at(Lr, Lr->max_local, sms));
}
static int64_t wgrad_rows(int64_t Bl, int s) { return round_up(cdiv(Bl, s), 128); }
// Split-K of the actor's weight gradients (bf16 path) behind the fused actor backward.  That kernel runs one CTA
// per 128 rows (B / 128 < SMs), and the weight-gradient launch behind it computes the critic / value tiles on the
// SMs it leaves idle, before its grid-dependency wait (dynamic tile schedule); the actor tiles are its tail, so
// they are cut finer than the critics' (shorter tiles after the wait, more partials for Adam to sum): 16 splits,
// measured at WLK (98.0 us per update against 100.2 with the critics' 9; 12: 98.4, 20: 99.2, 26: 100.5), never
// fewer than the critics' and never below 256 rows per split.  Behind the unfused actor backward (a GEMM over
// every SM) the critics' count (ANT: 279.6 us against 281.2 with 16).  SPZ_WGRAD_SA=<S> overrides (0: the
// critics' count).
static int actor_wgrad_splits_at(const spz_learner* Lr, int64_t Bl, int sms, bool fused) {
  const int Sw = wgrad_splits_at(Lr, Bl, sms);
  if (!Lr->bf16 || !fused) return Sw;
  const int smax = (int)std::max<int64_t>(1, std::min<int64_t>(32, Bl / 256));
  int want = 16;
  if (const char* e = std::getenv("SPZ_WGRAD_SA")) want = std::atoi(e);
  return want <= 0 ? Sw : std::max(Sw, std::min(want, smax));
}
static int actor_wgrad_splits(const spz_learner* Lr, int64_t Bl, bool fused) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // never above the count at the largest batch (the fused kernel's only possible size), for which the partials
  // are allocated
  return std::min(actor_wgrad_splits_at(Lr, Bl, sms, fused), actor_wgrad_splits_at(Lr, Lr->max_local, sms, Lr->cfg.hidden <= 256));
}
static int64_t actor_wgrad_rows(int64_t Bl, int s) { return round_up(cdiv(Bl, s), 64); }
static int bias_splits(int64_t Bl) { return (int)std::max<int64_t>(1, std::min<int64_t>(128, cdiv(Bl, 128))); }

// Gradient partial regions (one per trained tensor), laid out at create time for the
// largest split counts.
struct TensorSlot {
  int net, layer;
  bool weight;
  int64_t numel;
  int64_t g_off;
  int max_partials;
};

static std::vector<TensorSlot> trained_tensors(spz_learner* Lr) {
  std::vector<TensorSlot> v;
  const bool actor_on = Lr->cfg.role != SPZ_ROLE_CRITIC, critic_on = Lr->cfg.role != SPZ_ROLE_ACTOR;
  const int Sb = bias_splits(Lr->max_local);
  auto add_net = [&](int id) {
    const NetLayout& n = Lr->net[id];
    const int Sw = id == NET_ACTOR ? actor_wgrad_splits(Lr, Lr->max_local, Lr->cfg.hidden <= 256)
                                   : wgrad_splits(Lr, Lr->max_local);
    for (int l = 0; l < n.nl; ++l) {
      const bool head_vec = (id == NET_Q1 || id == NET_Q2 || id == NET_V) && l == n.nl - 1;  // N = 1 head: column sums
      // weight partials keep a 16-byte row pitch (TMA stores): out x round_up(in, 4)
      v.push_back({id, l, true, (int64_t)n.out[l] * (head_vec ? n.in[l] : round_up(n.in[l], 4)), 0,
                   head_vec ? std::max(Sb, Sw) : Sw});
      v.push_back({id, l, false, (int64_t)n.out[l], 0, std::max(Sb, Sw)});
    }
  };
  if (critic_on) {
    add_net(NET_Q1);
    add_net(NET_Q2);
    if (Lr->v1) add_net(NET_V);
  }
  if (actor_on) add_net(NET_ACTOR);
  int64_t off = 0;
  for (auto& t : v) {
    t.g_off = off;
    off += round_up(t.numel * t.max_partials, 64);
  }
  Lr->G_total = off + 64;  // + log alpha gradient slot at the end
  return v;
}

template <typename T>
static spz_status build_plan(spz_learner* Lr, int64_t B);
spz_status refresh_shadows(spz_learner* Lr);

}  // namespace spz

spz_learner::~spz_learner() {
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  if (own_stream) cudaStreamSynchronize(own_stream);
  if (ev_read) {
    if (ring) {
      std::lock_guard<std::mutex> lk(ring->mu);
      auto& v = ring->readers;
      v.erase(std::remove(v.begin(), v.end(), ev_read), v.end());
    }
    cudaEventDestroy(ev_read);
  }
  if (gcomm.handle && gcomm.handle != comm.handle) comm_destroy(&gcomm);
  comm_destroy(&comm);
  for (auto& e : exec)
    if (e) cudaGraphExecDestroy(e);
  for (auto& ev : exec_pub)
    for (auto& e : ev)
      if (e) cudaGraphExecDestroy(e);
  for (void* p : allocs) cudaFree(p);
  if (h_stats) cudaFreeHost(h_stats);
  if (h_slots) cudaFreeHost(h_slots);
  for (auto& e : ev_slot)
    if (e) cudaEventDestroy(e);
  if (h_flag) cudaFreeHost(h_flag);
  if (h_counters) cudaFreeHost(h_counters);
  if (h_sync) cudaFreeHost(h_sync);
  if (h_gate) cudaFreeHost(h_gate);
  if (own_stream) cudaStreamDestroy(own_stream);
  if (prev >= 0) cudaSetDevice(prev);
}

namespace spz {

// ----------------------------------------------------------------------------- plan
template <typename T>
static spz_status build_plan(spz_learner* Lr, int64_t B) {
  for (auto& v : Lr->ops) v.clear();
  for (auto& e : Lr->exec)
    if (e) {
      cudaGraphExecDestroy(e);
      e = nullptr;
    }
  for (auto& ev : Lr->exec_pub)
    for (auto& e : ev)
      if (e) {
        cudaGraphExecDestroy(e);
        e = nullptr;
      }
  // rows of this rank: contiguous share of the global batch inside its group (spz_plan_rank, DESIGN.md
  // reading #17); with split roles the critic group is ranks [0, n_critic) and the actor group the rest
  spz_plan plan;
  SPZ_TRY(spz_plan_rank(&Lr->cfg, B, &plan));
  const int Bl = (int)plan.rows;
  const int64_t row0 = plan.row0;
  const int o = Lr->o, m = Lr->m, h = Lr->h, L = Lr->L;
  const bool td3 = Lr->td3;
  const bool v1 = Lr->v1;
  const float invB = (float)(1.0 / (double)B);
  T* S = static_cast<T*>(Lr->S);
  float* P = Lr->P;
  const int lda = Lr->lda, ldc = Lr->ldc, ldh = Lr->ldh;
  const uint64_t seed = Lr->cfg.seed;
  const float lo = (float)Lr->cfg.log_std_min, hi = (float)Lr->cfg.log_std_max;
  const int delay = std::max(1, Lr->cfg.td3_policy_delay);
  const int Sw = wgrad_splits(Lr, Bl), Sb = bias_splits(Bl);
  const int64_t rows_w = wgrad_rows(Bl, Sw), rows_b = cdiv(Bl, Sb);
  // actor weight gradients: their own split-K behind the fused actor backward (set in a7)
  int64_t rows_a = rows_w;
  int Sa = Sw;
  auto Wp = [&](int id, int l) -> const T* { return S + Lr->sbase[id] + Lr->net[id].sw[l]; };
  auto bp = [&](int id, int l) -> const float* { return P + Lr->pbase[id] + Lr->net[id].b[l]; };
  auto ldw = [&](int id, int l) { return Lr->net[id].ld[l]; };
  auto Ta = [&](void* p, int64_t row, int ld) -> T* { return static_cast<T*>(p) + row * ld; };

  std::vector<TensorSlot> slots = trained_tensors(Lr);
  auto slot_of = [&](int id, int l, bool w) -> TensorSlot& {
    for (auto& s : slots)
      if (s.net == id && s.layer == l && s.weight == w) return s;
    return slots[0];
  };

  for (int variant = 0; variant < (td3 ? 2 : 1); ++variant) {
    std::vector<Op>& ops = Lr->ops[variant];
    const bool actor_step = !td3 || variant == 1;  // TD3: actor work only on delayed steps
    // roles: the critic side needs the actor only on s2 (a', log pi'); the actor side
    // needs the critics only on [s | a~] (Q(s, a~) and dQ/da~)
    const bool do_critic = Lr->cfg.role != SPZ_ROLE_ACTOR;
    const bool do_actor = Lr->cfg.role != SPZ_ROLE_CRITIC && actor_step;
    std::vector<GemmGroup> wgrads;
    std::vector<ColsumJob> colsums;
    auto empty_gemm = [](const GemmArgs& a) {
      for (int i = 0; i < a.n_groups; ++i)
        if (a.g[i].M > 0 && a.g[i].N > 0) return false;
      return true;
    };
    std::string unsupported;  // first GEMM the tensor-core kernels do not take (-> SPZ_EUNSUPPORTED)
    auto gemm = [&](const char* cls, GemmArgs a) {
      if (empty_gemm(a)) return;  // e.g. the TD3 actor role on a non-delayed step
      if (!gemm_supported<T>(a) && unsupported.empty())
        unsupported = std::string(cls) + " (M " + std::to_string(a.g[0].M) + ", N " + std::to_string(a.N) + ", K " +
                      std::to_string(a.K) + ", epilogue " + std::to_string(a.epi) + ")";
      ops.push_back({cls, [a](cudaStream_t st) { return run_gemm<T>(a, st); }});
    };
    auto mk = [&](int K, int epi, int amn, int bmn) {
      GemmArgs a{};
      a.K = K;
      a.epi = epi;
      a.a_mn = amn;
      a.b_mn = bmn;
      a.splits = 1;
      a.k_per_split = K;
      return a;
    };
    auto add = [&](GemmArgs& a, const void* A, int ldA, const void* Bm, int ldB, void* C, int ldC, int M, int N,
                   const float* bias = nullptr, const void* aux = nullptr, int ldAux = 0) -> GemmGroup& {
      GemmGroup& g = a.g[a.n_groups++];
      g = GemmGroup{};
      g.A = A;
      g.lda = ldA;
      g.B = Bm;
      g.ldb = ldB;
      g.C = C;
      g.ldc = ldC;
      g.M = M;
      g.N = N;
      g.bias = bias;
      g.aux = aux;
      g.ldaux = ldAux;
      a.N = std::max(a.N, N);
      return g;
    };
    // fused epilogues (row dot, actor heads, packed ReLU masks) exist only in the tcgen05 kernel
    auto tc_ok = [&](const GemmArgs& a) { return std::is_same<T, __nv_bfloat16>::value && tc_gemm_supported(a); };
    const bool bits = std::is_same<T, __nv_bfloat16>::value && tc_gemm_available();
    // bias (and critic-head) gradients come out of the weight-gradient GEMM (EPI_WGRAD_BIAS) on the
    // tensor-core path; the FP32 path sums columns (colsum_multi_kernel)
    const bool fuse_bias = bits;
    const int mw = Lr->mw;
    HeadEpi he{};
    he.m = m;
    he.o = o;
    he.Bl = Bl;
    he.ldx = ldc;
    he.row0 = row0;
    he.seed = seed;
    he.step_p = Lr->counters;
    he.lo = lo;
    he.hi = hi;
    he.noise = (float)Lr->cfg.td3_noise;
    he.clipc = (float)Lr->cfg.td3_noise_clip;
    he.Xc = Lr->Xc;
    he.u = Lr->cache.u;
    he.a = Lr->cache.a;
    he.eps = Lr->cache.eps;
    he.sig = Lr->cache.sig;
    he.l = Lr->cache.l;
    he.logp = Lr->logp;
    he.logp2 = Lr->logp2;

    // ---- a1 + a2: Philox indices + gather
    {
      const float* rec = Lr->ring->rec;
      const int R = Lr->ring->R;
      const int64_t* fill = Lr->ring->d_fill;  // written in stream order by the ring's pushes
      const int64_t* stp = Lr->counters;
      T *Xa = static_cast<T*>(Lr->Xa), *Xc = static_cast<T*>(Lr->Xc);
      float *rr = Lr->r, *dd = Lr->d;
      int32_t* idx = Lr->idx;
      uint32_t* tags = Lr->ring->tags;
      // two record buffers per block (the next group's copies in flight while one is stored) where they fit
      const size_t smem1 = (size_t)GATHER_ROWS * R * sizeof(float);  // <= 227 KB (checked by spz_replay_create)
      const int nbuf = 2 * smem1 <= 200 * 1024 ? 2 : 1;
      const size_t smem = nbuf * smem1;
      if (smem > 48 * 1024)
        SPZ_CUDA_TRY(cudaFuncSetAttribute(gather_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int nsm_g = 148, dev_g = 0;
      cudaGetDevice(&dev_g);
      cudaDeviceGetAttribute(&nsm_g, cudaDevAttrMultiProcessorCount, dev_g);
      // grid-stride: at most 4 blocks per SM (one group each at WLK; 3-7 pipelined groups at HUM / TD3)
      const unsigned ngrid = (unsigned)std::min<int64_t>(cdiv(Bl, GATHER_ROWS), 4 * (int64_t)nsm_g);
      ops.push_back({"gather", [=](cudaStream_t st) {
                       launch_pdl(gather_kernel<T>, dim3(ngrid), dim3(256), smem, st,
                           rec, R, o, m, fill, seed, stp, row0, Bl, Xa, lda, Xc, ldc, rr, dd, idx, tags, nbuf);
                       return cudaGetLastError();
                     }});
    }
    // ---- a3: actor forward.  SAC: online actor on [s2; s] (M = 2Bl).
    //      TD3: target actor on s2 (rows 0..Bl) every step, online actor on s on delayed steps
    //      (two groups of one launch per layer).
    {
      const NetLayout& an = Lr->net[NET_ACTOR];
      struct Pass { int id; int64_t row; int M; };
      std::vector<Pass> passes;
      if (v1) {
        passes.push_back({NET_ACTOR, Bl, Bl});  // SAC v1: the policy on s only (no a', role ALL)
      } else if (!td3) {
        if (do_critic && do_actor) passes.push_back({NET_ACTOR, 0, 2 * Bl});
        else if (do_critic) passes.push_back({NET_ACTOR, 0, Bl});
        else if (do_actor) passes.push_back({NET_ACTOR, Bl, Bl});
      } else {
        if (do_critic) passes.push_back({NET_ACTORT, 0, Bl});
        if (do_actor) passes.push_back({NET_ACTOR, Bl, Bl});
      }
      // fused multi-layer forward (hidden activations stay in SMEM between layers): one launch for
      // every hidden layer and the head; s2 rows store nothing, s rows their activations + masks
      bool fused = false;
      if (bits && !passes.empty()) {
        MlpArgs ma{};
        ma.L = L;
        ma.h = h;
        ma.k0 = lda;
        ma.head_n = an.out[L];
        ma.head_epi = td3 ? EPI_TD3_HEAD : EPI_SAC_HEAD;
        ma.mask_ld = mw;
        ma.head = he;
        for (const Pass& ps : passes) {
          // split an [s2; s] pass at Bl: the s2 half needs no backward state
          for (int half = 0; half < 2; ++half) {
            const int64_t r0 = ps.row + (half ? Bl : 0);
            if (r0 >= ps.row + ps.M) continue;
            const int rows = (int)std::min<int64_t>(Bl, ps.row + ps.M - r0);
            const bool srows = r0 >= Bl;  // s rows: the actor loss backpropagates through them
            MlpPass& q = ma.p[ma.n_pass++];
            q.X = Ta(Lr->Xa, r0, lda);
            q.ldx = lda;
            q.rows = rows;
            q.row0 = (int)r0;
            for (int l = 0; l <= L; ++l) {
              q.W[l] = Wp(ps.id, l);
              q.ldw[l] = ldw(ps.id, l);
              q.bias[l] = bp(ps.id, l);
            }
            for (int l = 0; l < L && srows; ++l) {
              q.act[l] = Ta(Lr->Aact[l], r0, h);
              q.mask[l] = Lr->mask_a[l] + r0 * mw;
            }
          }
        }
        if (tc_mlp_supported(ma)) {
          fused = true;
          ops.push_back({"actor_fwd_mlp", [ma](cudaStream_t st) { return tc_mlp_fwd(ma, st); }});
        }
      }
      for (int l = 0; l < L && !passes.empty() && !fused; ++l) {
        GemmArgs a = mk(l == 0 ? lda : an.in[l], EPI_BIAS_RELU, 0, 0);  // layer 0: over the zero-padded width
        for (const Pass& ps : passes) {
          GemmGroup& g = add(a, l == 0 ? (const void*)Ta(Lr->Xa, ps.row, lda) : (const void*)Ta(Lr->Aact[l - 1], ps.row, h),
                             l == 0 ? lda : h, Wp(ps.id, l), ldw(ps.id, l), Ta(Lr->Aact[l], ps.row, h), h, ps.M, h, bp(ps.id, l));
          if (bits && ps.id == NET_ACTOR) {
            g.mask_out = Lr->mask_a[l] + ps.row * mw;
            g.mask_ld = mw;
          }
        }
        if (bits && !tc_ok(a)) return fail(SPZ_EUNSUPPORTED, "internal: actor forward not supported by the tcgen05 kernel");
        gemm("actor_fwd_gemm", a);
      }
      // head layer: fused squashed-Gaussian (SAC) / tanh + smoothing (TD3) epilogue when possible
      // (TD3 actor role on a non-delayed step: no actor work at all)
      if (!passes.empty() && !fused) {
      GemmArgs a = mk(h, td3 ? EPI_TD3_HEAD : EPI_SAC_HEAD, 0, 0);
      a.head = he;
      for (const Pass& ps : passes) {
        GemmGroup& g = add(a, Ta(Lr->Aact[L - 1], ps.row, h), h, Wp(ps.id, L), ldw(ps.id, L), Lr->H + ps.row * ldh,
                           ldh, ps.M, an.out[L], bp(ps.id, L));
        g.row0 = (int)ps.row;
      }
      if (tc_ok(a)) {
        gemm("actor_head_gemm", a);
      } else {
        a.epi = EPI_BIAS_F32;
        gemm("actor_head_gemm", a);
        float* Hh = Lr->H;
        const int Mh = (int)(passes.back().row + passes.back().M);  // rows [0, Mh) of the actor pass
        const HeadEpi hh = he;
        const int t3 = td3;
        ops.push_back({"actor_head", [=](cudaStream_t st) {
                         if (t3) return launch_pdl(td3_head_fwd_kernel<T>, dim3((unsigned)cdiv(Mh, 128)), dim3(128), 0, st, Hh, ldh, hh, Mh);
                         return launch_pdl(sac_head_fwd_kernel<T>, dim3((unsigned)cdiv(Mh, 128)), dim3(128), 0, st, Hh, ldh, hh, Mh);
                       }});
      }
      }
    }
    // ---- SAC v1 (reading #24): the target value V'(s2) and the online value V(s) (activations + masks
    //      of the s rows for its backward), one fused launch over the actor's input rows [s2; s]
    if (v1) {
      const NetLayout& vn = Lr->net[NET_V];
      bool vfused = false;
      if (bits) {
        MlpArgs ma{};
        ma.L = L;
        ma.h = h;
        ma.k0 = lda;
        ma.mask_ld = mw;
        for (int pi = 0; pi < 2; ++pi) {
          const int id = pi == 0 ? NET_VT : NET_V;
          MlpPass& q = ma.p[ma.n_pass++];
          q.X = Ta(Lr->Xa, pi == 0 ? 0 : Bl, lda);
          q.ldx = lda;
          q.rows = Bl;
          for (int l = 0; l < L; ++l) {
            q.W[l] = Wp(id, l);
            q.ldw[l] = vn.ld[l];
            q.bias[l] = bp(id, l);
            if (pi == 1) {
              q.act[l] = Lr->Av[l];
              q.mask[l] = Lr->mask_v[l];
            }
          }
          q.bias[L] = bp(id, L);
          q.dot_w = P + Lr->pbase[id] + vn.w[L];
          q.dot_b = bp(id, L);
          q.dot_out = pi == 0 ? Lr->v_tg : Lr->v_on;
        }
        if (tc_mlp_supported(ma)) {
          vfused = true;
          ops.push_back({"value_fwd_mlp", [ma](cudaStream_t st) { return tc_mlp_fwd(ma, st); }});
        }
      }
      for (int l = 0; l < L && !vfused; ++l) {
        GemmArgs a = mk(l == 0 ? lda : h, EPI_BIAS_RELU, 0, 0);
        for (int pi = 0; pi < 2; ++pi) {
          const int id = pi == 0 ? NET_VT : NET_V;
          void* const* act = pi == 0 ? Lr->AvT : Lr->Av;
          GemmGroup& g = add(a, l == 0 ? (const void*)Ta(Lr->Xa, pi == 0 ? 0 : Bl, lda) : (const void*)act[l - 1],
                             l == 0 ? lda : h, Wp(id, l), vn.ld[l], act[l], h, Bl, h, bp(id, l));
          if (bits && pi == 1) {
            g.mask_out = Lr->mask_v[l];
            g.mask_ld = mw;
          }
          if (l == L - 1) {
            g.dot_w = P + Lr->pbase[id] + vn.w[L];
            g.dot_b = bp(id, L);
            g.dot_out = pi == 0 ? Lr->v_tg : Lr->v_on;
            g.dot_pstride = (h > 256 && h <= 1024) ? Lr->max_local : 0;
          }
        }
        if (bits && !tc_ok(a) && l < L - 1) return fail(SPZ_EUNSUPPORTED, "internal: value forward not supported by the tcgen05 kernel");
        if (l == L - 1 && !tc_ok(a)) {
          for (int i = 0; i < a.n_groups; ++i) a.g[i].dot_out = nullptr;
          gemm("value_fwd_gemm", a);
          RowdotArgs ra{};
          ra.M = Bl;
          ra.h = h;
          ra.ld = h;
          for (int pi = 0; pi < 2; ++pi) {
            const int id = pi == 0 ? NET_VT : NET_V;
            ra.g[pi].A = pi == 0 ? Lr->AvT[L - 1] : Lr->Av[L - 1];
            ra.g[pi].w = P + Lr->pbase[id] + vn.w[L];
            ra.g[pi].b = bp(id, L);
            ra.g[pi].q = pi == 0 ? Lr->v_tg : Lr->v_on;
          }
          const int M = Bl;
          ops.push_back({"value_head", [ra, M](cudaStream_t st) {
                           return launch_pdl(rowdot_kernel<T>, dim3((unsigned)cdiv((int64_t)M * 32, 256), 2), dim3(256), 0, st, ra);
                         }});
        } else {
          gemm("value_fwd_gemm", a);
        }
      }
    }
    // ---- a4: target critics on [s2 | a'] (M = Bl) and a5: online critics on [s | a ; s | a~]
    //      (M = 2Bl), all four in one launch per layer; the N = 1 head is a row dot fused into
    //      the last hidden layer's epilogue when the row fits one tile.
    const NetLayout& cn = Lr->net[NET_Q1];
    // online-critic rows [on0, on0 + Mon): loss rows [0, Bl) on the critic side, actor rows [Bl, 2Bl)
    const int on0 = do_critic ? 0 : Bl;
    const int Mon = (do_critic ? Bl : 0) + (do_actor ? Bl : 0);
    // TD3's actor loss uses Q1 alone (reading #18): Q2 never sees the actor rows (forward, dZ_L, dgrad)
    const bool fuse_loss_env = [] {
      const char* fl = std::getenv("SPZ_FUSE_CRITIC_LOSS");
      return fl && std::atoi(fl) == 1;
    }();
    const bool q2_skip_actor = td3 && !fuse_loss_env;
    const int Mon2 = q2_skip_actor ? (do_critic ? Bl : 0) : Mon;  // online rows of Q2
    bool cfused = false, lfused = false;  // fused critic forward / fused critic loss
    if (bits && (do_critic || do_actor)) {
      // fused multi-layer critic forward: online loss rows (activations + masks stored), online
      // actor rows (masks only: no critic weight gradient over them), target rows (nothing stored)
      MlpArgs ma{};
      ma.L = L;
      ma.h = h;
      ma.k0 = ldc;
      ma.mask_ld = mw;
      for (int kind = 0; kind < 3; ++kind) {
        if (kind == 0 && !do_critic) continue;
        if (kind == 1 && !do_actor) continue;
        if (kind == 2 && (!do_critic || v1)) continue;  // SAC v1 bootstraps V', not target critics
        for (int i = 0; i < 2; ++i) {
          if (kind == 1 && i == 1 && q2_skip_actor) continue;
          const int id = kind == 2 ? NET_Q1T + i : NET_Q1 + i;
          const int64_t xr = kind * (int64_t)Bl;          // row in Xc
          const int64_t ar = kind == 2 ? 0 : kind * (int64_t)Bl;  // row in the per-critic buffers
          MlpPass& q = ma.p[ma.n_pass++];
          q.X = Ta(Lr->Xc, xr, ldc);
          q.ldx = ldc;
          q.rows = Bl;
          for (int l = 0; l < L; ++l) {
            q.W[l] = Wp(id, l);
            q.ldw[l] = cn.ld[l];
            q.bias[l] = bp(id, l);
            if (kind == 0) q.act[l] = Ta(Lr->Aon[i][l], ar, h);
            if (kind != 2) q.mask[l] = Lr->mask_c[i][l] + ar * mw;
          }
          q.bias[L] = bp(id, L);
          q.dot_w = P + Lr->pbase[id] + Lr->net[id].w[L];
          q.dot_b = bp(id, L);
          q.dot_out = (kind == 2 ? Lr->q_tg[i] : Lr->q_on[i]) + ar;
        }
      }
      // optionally (SPZ_FUSE_CRITIC_LOSS=1) the Bellman target, losses, g_q, statistics and
      // critic-head backward run in the same launch: loss rows as one group (q1, q2, q1', q2' per
      // row block), actor rows as another (q1, q2).  Parity-tested, but off by default: at WLK the
      // serial 4-pass groups (one per CTA) cost more than the separate critic_loss kernel
      // (118.2 vs 114.7 us/update) because a unit's layer-1 weight delivery dominates its time.
      const char* fl = std::getenv("SPZ_FUSE_CRITIC_LOSS");
      if (fl && std::atoi(fl) == 1 && !v1) {
        int idx[3][2], n = 0;
        for (int kind = 0; kind < 3; ++kind)
          for (int i = 0; i < 2; ++i) {
            const bool present = kind == 1 ? do_actor : do_critic;
            idx[kind][i] = present ? n++ : -1;
          }
        if (do_critic) {
          MlpGroup& gr = ma.grp[ma.n_group++];
          gr.n = 4;
          gr.loss = 1;
          gr.rows = Bl;
          gr.pass[0] = idx[0][0], gr.pass[1] = idx[0][1], gr.pass[2] = idx[2][0], gr.pass[3] = idx[2][1];
        }
        if (do_actor) {
          MlpGroup& gr = ma.grp[ma.n_group++];
          gr.n = 2;
          gr.loss = 2;
          gr.rows = Bl;
          gr.pass[0] = idx[1][0], gr.pass[1] = idx[1][1];
        }
        MlpLoss& ls = ma.loss;
        ls.r = Lr->r;
        ls.d = Lr->d;
        ls.logp2 = Lr->logp2;
        ls.logp = Lr->logp;
        ls.log_alpha = P + Lr->p_log_alpha;
        ls.step_p = Lr->counters;
        for (int i = 0; i < 2; ++i) {
          ls.w[i] = P + Lr->pbase[NET_Q1 + i] + cn.w[L];
          ls.dZ[i] = Lr->dZc[i][L - 1];
          ls.gq16[i] = fuse_bias ? Lr->gq16[i] : nullptr;
        }
        ls.gq1 = Lr->gq[0];
        ls.gq2 = Lr->gq[1];
        ls.y = Lr->y;
        ls.partials = Lr->stat_partials;
        ls.totals = Lr->statsum;
        ls.ctr_snap = Lr->ctr_snap;
        ls.la_snap = reinterpret_cast<float*>(Lr->ctr_snap + 4);
        ls.bc_snap = reinterpret_cast<float*>(Lr->ctr_snap + 5);
        ls.ticket = Lr->tickets;
        ls.gamma = (float)Lr->cfg.gamma;
        ls.invB = invB;
        ls.beta1 = (float)Lr->cfg.beta1;
        ls.beta2 = (float)Lr->cfg.beta2;
        ls.Bl = Bl;
        ls.td3 = td3;
        ls.delay = delay;
      }
      if (tc_mlp_supported(ma)) {
        cfused = true;
        lfused = ma.n_group > 0;
        ops.push_back({"critic_fwd_mlp", [ma](cudaStream_t st) { return tc_mlp_fwd(ma, st); }});
      }
    }
    int qparts = 1;  // q partials the loss kernel sums (fused row dot of a wide last hidden layer)
    if (!cfused) {
      for (int l = 0; l < L; ++l) {
        GemmArgs a = mk(l == 0 ? ldc : cn.in[l], EPI_BIAS_RELU, 0, 0);  // layer 0: over the zero-padded width
        for (int pass = 0; pass < 2; ++pass) {
          const bool tgt = pass == 1;
          if (tgt && (!do_critic || v1)) continue;
          if (!tgt && Mon == 0) continue;
          const int r0c = tgt ? 2 * Bl : on0;  // row in Xc
          const int ra = tgt ? 0 : on0;        // row in the activation buffers
          for (int i = 0; i < 2; ++i) {
            const int id = tgt ? NET_Q1T + i : NET_Q1 + i;
            void* dst = Ta(tgt ? Lr->Atg[i][l] : Lr->Aon[i][l], ra, h);
            const void* src = l == 0 ? (const void*)Ta(Lr->Xc, r0c, ldc)
                                     : (const void*)Ta(tgt ? Lr->Atg[i][l - 1] : Lr->Aon[i][l - 1], ra, h);
            GemmGroup& g = add(a, src, l == 0 ? ldc : h, Wp(id, l), cn.ld[l], dst, h, tgt ? Bl : (i ? Mon2 : Mon), h, bp(id, l));
            if (bits && !tgt) {
              g.mask_out = Lr->mask_c[i][l] + (int64_t)ra * mw;
              g.mask_ld = mw;
            }
            if (l == L - 1) {
              g.dot_w = P + Lr->pbase[id] + Lr->net[id].w[L];
              g.dot_b = bp(id, L);
              g.dot_out = (tgt ? Lr->q_tg[i] : Lr->q_on[i]) + ra;
              g.dot_pstride = (h > 256 && h <= 1024) ? (tgt ? 1 : 2) * Lr->max_local : 0;  // per-256-column-tile partials (summed by critic_loss)
            }
          }
        }
        if (bits && !empty_gemm(a) && !tc_ok(a) && l < L - 1)
          return fail(SPZ_EUNSUPPORTED, "internal: critic forward not supported by the tcgen05 kernel");
        if (l == L - 1 && !empty_gemm(a) && !tc_ok(a)) {
          for (int i = 0; i < a.n_groups; ++i) a.g[i].dot_out = nullptr;
          gemm("critic_fwd_gemm", a);
          for (int pass = 0; pass < 2; ++pass) {
            const bool tgt = pass == 1;
            if ((tgt && (!do_critic || v1)) || (!tgt && Mon == 0)) continue;
            const int M = tgt ? Bl : Mon;
            const int rr0 = tgt ? 0 : on0;
            RowdotArgs ra{};
            ra.M = M;
            ra.h = h;
            ra.ld = h;
            for (int i = 0; i < 2; ++i) {
              const int id = tgt ? NET_Q1T + i : NET_Q1 + i;
              ra.g[i].A = Ta(tgt ? Lr->Atg[i][L - 1] : Lr->Aon[i][L - 1], rr0, h);
              ra.g[i].w = P + Lr->pbase[id] + Lr->net[id].w[L];
              ra.g[i].b = bp(id, L);
              ra.g[i].q = (tgt ? Lr->q_tg[i] : Lr->q_on[i]) + rr0;
            }
            ops.push_back({"critic_head", [ra, M](cudaStream_t st) {
                             return launch_pdl(rowdot_kernel<T>, dim3((unsigned)cdiv((int64_t)M * 32, 256), 2), dim3(256), 0, st, ra);
                           }});
          }
        } else {
          gemm("critic_fwd_gemm", a);
          if (l == L - 1 && h > 256) qparts = (int)cdiv(h, 256);  // <= 4 (wider rows take the rowdot path)
        }
      }
    }
    // ---- a4/a5: Bellman target, losses, head gradients, this rank's loss totals; a6 head backward
    // dZ_L written by the loss kernel itself (one row per warp) at h <= 256 up to 16K local rows (WLK
    // 109.1 -> 108.2 us); larger batches do better with the separate critic_dz_kernel (ANT 319.5 -> 315.4 us)
    const bool dz_in_loss = h <= 256 && Bl <= 16384 && !dz_split_env();  // (then qparts == 1: the kernel assumes it)
    const bool defer_totals = !(Lr->gsize > 1 || Lr->cfg.comm_mode == 2) && !lfused && !defer_totals_off_env();
    // diagnostics: SPZ_DIAG_LOSS=<rpw>,<blocks per SM> for the dZ-writing variant (rpw 1 or 2)
    int diag_rpw = 1, diag_cap = 4;
    if (const char* dl = std::getenv("SPZ_DIAG_LOSS")) std::sscanf(dl, "%d,%d", &diag_rpw, &diag_cap);
    const int loss_rpw = dz_in_loss ? (diag_rpw == 2 ? 2 : 1) : 4;
    int nsm_l = 148, dev_l = 0;
    cudaGetDevice(&dev_l);
    cudaDeviceGetAttribute(&nsm_l, cudaDevAttrMultiProcessorCount, dev_l);
    // grid cap: 2 blocks per SM for the statistics-only variant (HUM 138 -> 118 us, ANT 311 -> 306 us per
    // update); 4 per SM for the dZ-writing variant -- every block resident at once (64 registers x 256
    // threads), each walking 1-2 row blocks: WLK 105.2 -> 103.0 us per update against 8 per SM (two waves)
    const int nblk = (int)std::min<int64_t>(cdiv(Bl, LOSS_WARPS * loss_rpw), (dz_in_loss ? diag_cap : 2) * (int64_t)nsm_l);
    {
      LossArgs la{};
      la.qp = qparts;
      if (const char* dc = std::getenv("SPZ_DIAG_LOSS_CUT")) la.diag = std::atoi(dc);  // diagnostics only
      // the grid-wide reduction of the statistics partials (a ticket and the last block's pass: ~5 us on the
      // WLK critical path) moves into the optimizer, which needs the totals first, before its dependency wait;
      // a row-sharded group all-reduces the totals first, so there the loss kernel keeps it (SPZ_DEFER_TOTALS=0:
      // always here)
      la.defer_totals = defer_totals ? 1 : 0;
      la.bad2 = Lr->tickets + 200;  // two words past the ticket counters (<= 1 + 19 in use)
      la.q2_no_actor = q2_skip_actor;
      la.v1 = v1;
      la.qps_tg = Lr->max_local;
      la.qps_on = 2 * Lr->max_local;
      la.qt1 = Lr->q_tg[0];
      la.qt2 = Lr->q_tg[1];
      la.q1 = Lr->q_on[0];
      la.q2 = Lr->q_on[1];
      la.logp2 = Lr->logp2;
      la.logp = Lr->logp;
      la.r = Lr->r;
      la.d = Lr->d;
      la.log_alpha = P + Lr->p_log_alpha;
      la.step_p = Lr->counters;
      la.gq1 = Lr->gq[0];
      la.gq2 = Lr->gq[1];
      la.y = Lr->y;
      la.partials = Lr->stat_partials;
      la.totals = Lr->statsum;
      la.ticket = Lr->tickets;
      la.ctr_snap = Lr->ctr_snap;
      la.la_snap = reinterpret_cast<float*>(Lr->ctr_snap + 4);
      la.bc_snap = reinterpret_cast<float*>(Lr->ctr_snap + 5);
      la.beta1 = (float)Lr->cfg.beta1;
      la.beta2 = (float)Lr->cfg.beta2;
      la.mask_ld = mw;
      for (int i = 0; i < 2; ++i) {
        la.mask[i] = bits ? Lr->mask_c[i][L - 1] : nullptr;
        la.A[i] = Lr->Aon[i][L - 1];
        la.w[i] = P + Lr->pbase[NET_Q1 + i] + cn.w[L];
        la.dZ[i] = Lr->dZc[i][L - 1];
        la.gq16[i] = fuse_bias ? Lr->gq16[i] : nullptr;
      }
      la.gamma = (float)Lr->cfg.gamma;
      la.invB = invB;
      la.Bl = Bl;
      la.td3 = td3;
      la.delay = delay;
      la.loss_rows = do_critic;
      la.actor_rows = do_actor;
      la.h = h;
      la.ld = h;
      if (v1) {  // the bootstrap reads V'(s2); the actor rows also yield g_V
        la.qt1 = la.qt2 = Lr->v_tg;
        la.vo = Lr->v_on;
        la.vps = Lr->max_local;
        la.gv = Lr->gv;
        la.gv16 = fuse_bias ? Lr->gv16 : nullptr;
      }
      // h <= 256: dZ_L written by the loss kernel (one row per warp); wider rows: critic_dz_kernel
      const bool dz_sep = !dz_in_loss && (do_critic || do_actor);
      if (!lfused) {  // (the fused critic forward with loss groups computes all of this itself)
        if (!dz_in_loss && la.qp == 1)
          ops.push_back({"critic_loss", [la, nblk](cudaStream_t st) {
                           return launch_pdl(critic_loss_kernel<T, false, 4, true>, dim3(nblk), dim3(LOSS_NT), 0, st, la);
                         }});
        else if (!dz_in_loss)
          ops.push_back({"critic_loss", [la, nblk](cudaStream_t st) {
                           return launch_pdl(critic_loss_kernel<T, false, 4>, dim3(nblk), dim3(LOSS_NT), 0, st, la);
                         }});
        else if (loss_rpw == 2)
          ops.push_back({"critic_loss", [la, nblk](cudaStream_t st) {
                           return launch_pdl(critic_loss_kernel<T, true, 2>, dim3(nblk), dim3(LOSS_NT), 0, st, la);
                         }});
        else
          ops.push_back({"critic_loss", [la, nblk](cudaStream_t st) {
                           return launch_pdl(critic_loss_kernel<T, true, 1>, dim3(nblk), dim3(LOSS_NT), 0, st, la);
                         }});
      }
      if (dz_sep && !lfused) {
        DzArgs da{};
        for (int i = 0; i < 2; ++i) {
          da.gq[i] = la.gq1 == nullptr ? nullptr : (i ? la.gq2 : la.gq1);
          da.mask[i] = la.mask[i];
          da.A[i] = la.A[i];
          da.w[i] = la.w[i];
          da.dZ[i] = la.dZ[i];
        }
        da.r0 = do_critic ? 0 : Bl;
        da.rows = (int64_t)(do_critic ? Bl : 0) + (do_actor ? Bl : 0);
        da.q2_end = q2_skip_actor ? (int64_t)Bl : da.r0 + da.rows;
        da.hv = h / 8;
        da.ld = h;
        da.mask_ld = mw;
        const int64_t nthr = da.rows * da.hv;
        ops.push_back({"critic_head_dz", [da, nthr](cudaStream_t st) {
                         return launch_pdl(critic_dz_kernel<T>, dim3((unsigned)cdiv(nthr, 256)), dim3(256), 0, st, da);
                       }});
      }
      if (v1) {
        // V's head backward dZ_L = g_V w_V 1[z_L > 0] (the second slot mirrors the first and writes nothing)
        DzArgs da{};
        for (int i = 0; i < 2; ++i) {
          da.gq[i] = Lr->gv;
          da.mask[i] = bits ? Lr->mask_v[L - 1] : nullptr;
          da.A[i] = Lr->Av[L - 1];
          da.w[i] = P + Lr->pbase[NET_V] + Lr->net[NET_V].w[L];
          da.dZ[i] = Lr->dZv[L - 1];
        }
        da.r0 = 0;
        da.rows = Bl;
        da.q2_end = 0;
        da.hv = h / 8;
        da.ld = h;
        da.mask_ld = mw;
        const int64_t nthr = da.rows * da.hv;
        ops.push_back({"value_dz", [da, nthr](cudaStream_t st) {
                         return launch_pdl(critic_dz_kernel<T>, dim3((unsigned)cdiv(nthr, 256)), dim3(256), 0, st, da);
                       }});
      }
    }
    // ---- a6 (actor rows) + a7: one fused launch on the tensor-core path (tc_actor_bwd.cuh): critic
    //      input gradient of the action columns, head backward (eq. H), dgrad down the actor stack
    ActorBwdArgs ab{};
    bool abwd_fused = false;
    if (bits && do_actor && !actor_bwd_unfused_env()) {
      const NetLayout& an = Lr->net[NET_ACTOR];
      ab.Bl = (int)Bl;
      ab.o = o;
      ab.m = m;
      ab.h = h;
      ab.L = L;
      ab.nout = an.out[L];
      ab.td3 = td3;
      ab.ncrit = td3 ? 1 : 2;
      ab.ldw0c = cn.ld[0];
      ab.ldh = ldh;
      ab.mask_ld = mw;
      for (int i = 0; i < 2; ++i) {
        ab.dZ1[i] = Ta(Lr->dZc[i][0], Bl, h);
        ab.W0c[i] = Wp(NET_Q1 + i, 0);
      }
      for (int l = 0; l <= L; ++l) {
        ab.Wa[l] = Wp(NET_ACTOR, l);
        ab.ldwa[l] = an.ld[l];
      }
      for (int l = 0; l < L; ++l) {
        ab.mask[l] = Lr->mask_a[l] + (int64_t)Bl * mw;
        ab.dZa[l] = Lr->dZa[l];
      }
      ab.dH = Lr->dH;
      ab.u = Lr->cache.u;
      ab.a = Lr->cache.a;
      ab.eps = Lr->cache.eps;
      ab.sig = Lr->cache.sig;
      ab.l = Lr->cache.l;
      ab.log_alpha = P + Lr->p_log_alpha;
      ab.invB = invB;
      ab.lo = lo;
      ab.hi = hi;
      abwd_fused = tc_actor_bwd_supported(ab);
      if (abwd_fused) {
        const int sa = actor_wgrad_splits(Lr, Bl, true);
        if (sa != Sw) {
          rows_a = actor_wgrad_rows(Bl, sa);
          Sa = (int)cdiv(Bl, rows_a);
        }
      }
    }
    // ---- a6: critic backward
    {
      // dgrad through hidden layers l = L-1 .. 1 (the online rows [on0, on0 + Mon))
      for (int l = L - 1; l >= 1; --l) {
        GemmArgs a = mk(h, bits ? EPI_MASK_BITS : EPI_MASK, 0, 1);
        for (int i = 0; i < 2; ++i) {
          if (bits)
            add(a, Ta(Lr->dZc[i][l], on0, h), h, Wp(NET_Q1 + i, l), cn.ld[l], Ta(Lr->dZc[i][l - 1], on0, h), h, i ? Mon2 : Mon, h,
                nullptr, Lr->mask_c[i][l - 1] + (int64_t)on0 * mw, mw);
          else
            add(a, Ta(Lr->dZc[i][l], on0, h), h, Wp(NET_Q1 + i, l), cn.ld[l], Ta(Lr->dZc[i][l - 1], on0, h), h, i ? Mon2 : Mon, h,
                nullptr, Ta(Lr->Aon[i][l - 1], on0, h), h);
        }
        if (v1) {  // the value network's dgrad rides in the same launch (its B s rows)
          const NetLayout& vn = Lr->net[NET_V];
          if (bits)
            add(a, Lr->dZv[l], h, Wp(NET_V, l), vn.ld[l], Lr->dZv[l - 1], h, Bl, h, nullptr, Lr->mask_v[l - 1], mw);
          else
            add(a, Lr->dZv[l], h, Wp(NET_V, l), vn.ld[l], Lr->dZv[l - 1], h, Bl, h, nullptr, Lr->Av[l - 1], h);
        }
        if (bits && !empty_gemm(a) && !tc_ok(a)) return fail(SPZ_EUNSUPPORTED, "internal: critic dgrad not supported by the tcgen05 kernel");
        gemm("critic_dgrad_gemm", a);
      }
      // input dgrad for the actor rows (only the action columns are consumed)
      if (do_actor && !abwd_fused) {
        GemmArgs a = mk(h, EPI_F32, 0, 1);
        for (int i = 0; i < (td3 ? 1 : 2); ++i)
          add(a, Ta(Lr->dZc[i][0], Bl, h), h, Wp(NET_Q1 + i, 0), cn.ld[0], Lr->dXc[i], ldc, Bl, o + m);
        gemm("critic_input_dgrad_gemm", a);
      }
      // wgrad (B loss rows) and bias column sums are collected and launched with the actor's below
      for (int i = 0; i < (do_critic ? 2 : 0); ++i)
        for (int l = 0; l < L; ++l) {
          GemmGroup g{};
          g.A = Lr->dZc[i][l];
          g.lda = h;
          g.B = l == 0 ? Lr->Xc : Lr->Aon[i][l - 1];
          g.ldb = l == 0 ? ldc : h;
          g.C = Lr->G + slot_of(NET_Q1 + i, l, true).g_off;
          g.ldc = (int)round_up(cn.in[l], 4);
          g.M = h;
          g.N = cn.in[l];
          g.split_stride = (int64_t)h * g.ldc;
          if (fuse_bias) {
            g.colsum_out = Lr->G + slot_of(NET_Q1 + i, l, false).g_off;
            g.colsum_stride = h;
          }
          wgrads.push_back(g);
        }
      for (int i = 0; i < (do_critic ? 2 : 0); ++i) {
        if (fuse_bias) {
          // critic head: dw_L = g_q^T A_{L-1}, db_L = sum g_q, with g_q (bf16) as a one-row A operand
          GemmGroup g{};
          g.A = Lr->gq16[i];
          g.lda = 8;
          g.B = Lr->Aon[i][L - 1];
          g.ldb = h;
          g.C = Lr->G + slot_of(NET_Q1 + i, L, true).g_off;
          g.ldc = h;
          g.M = 1;
          g.N = h;
          g.split_stride = h;
          g.colsum_out = Lr->G + slot_of(NET_Q1 + i, L, false).g_off;
          g.colsum_stride = 1;
          wgrads.push_back(g);
          continue;
        }
        for (int l = 0; l < L; ++l)
          colsums.push_back({Lr->dZc[i][l], nullptr, Lr->G + slot_of(NET_Q1 + i, l, false).g_off, h, h, Bl, 0});
        colsums.push_back({Lr->Aon[i][L - 1], Lr->gq[i], Lr->G + slot_of(NET_Q1 + i, L, true).g_off, h, h, Bl, 0});
        colsums.push_back({Lr->gq[i], nullptr, Lr->G + slot_of(NET_Q1 + i, L, false).g_off, 1, 1, Bl, 1});
      }
    }
    // ---- SAC v1: value network wgrad over its B s rows (dZ_l^T A_{l-1}; head: g_V^T A_{L-1})
    if (v1) {
      const NetLayout& vn = Lr->net[NET_V];
      for (int l = 0; l < L; ++l) {
        GemmGroup g{};
        g.A = Lr->dZv[l];
        g.lda = h;
        g.B = l == 0 ? (const void*)Ta(Lr->Xa, Bl, lda) : (const void*)Lr->Av[l - 1];
        g.ldb = l == 0 ? lda : h;
        g.C = Lr->G + slot_of(NET_V, l, true).g_off;
        g.ldc = (int)round_up(vn.in[l], 4);
        g.M = h;
        g.N = vn.in[l];
        g.split_stride = (int64_t)h * g.ldc;
        if (fuse_bias) {
          g.colsum_out = Lr->G + slot_of(NET_V, l, false).g_off;
          g.colsum_stride = h;
        }
        wgrads.push_back(g);
      }
      if (fuse_bias) {
        GemmGroup g{};
        g.A = Lr->gv16;
        g.lda = 8;
        g.B = Lr->Av[L - 1];
        g.ldb = h;
        g.C = Lr->G + slot_of(NET_V, L, true).g_off;
        g.ldc = h;
        g.M = 1;
        g.N = h;
        g.split_stride = h;
        g.colsum_out = Lr->G + slot_of(NET_V, L, false).g_off;
        g.colsum_stride = 1;
        wgrads.push_back(g);
      } else {
        for (int l = 0; l < L; ++l)
          colsums.push_back({Lr->dZv[l], nullptr, Lr->G + slot_of(NET_V, l, false).g_off, h, h, Bl, 0});
        colsums.push_back({Lr->Av[L - 1], Lr->gv, Lr->G + slot_of(NET_V, L, true).g_off, h, h, Bl, 0});
        colsums.push_back({Lr->gv, nullptr, Lr->G + slot_of(NET_V, L, false).g_off, 1, 1, Bl, 1});
      }
    }
    // weight gradients collected so far (critics, value net) read nothing the actor backward writes
    size_t n_pre_wgrads = wgrads.size();
    // ---- a7: actor backward (s-rows Bl..2Bl of the actor activations)
    if (do_actor) {
      const NetLayout& an = Lr->net[NET_ACTOR];
      const int nout = an.out[L];  // 2m (SAC) or m (TD3)
      T* dH = static_cast<T*>(Lr->dH);
      if (abwd_fused) {
        ops.push_back({"actor_bwd_fused", [ab](cudaStream_t st) { return tc_actor_bwd(ab, st); }});
      } else {
        float *x1 = Lr->dXc[0], *x2 = Lr->dXc[1];
        HeadCache cache = Lr->cache;
        const float* la = P + Lr->p_log_alpha;
        if (!td3) {
          ops.push_back({"actor_head_bwd", [=](cudaStream_t st) {
                           launch_pdl(sac_head_bwd_kernel<T>, dim3((unsigned)cdiv((int64_t)Bl * m, 256)), dim3(256), 0, st, 
                               x1, x2, ldc, o, m, Bl, cache, la, invB, lo, hi, dH, ldh);
                           return cudaGetLastError();
                         }});
        } else {
          ops.push_back({"actor_head_bwd", [=](cudaStream_t st) {
                           launch_pdl(td3_head_bwd_kernel<T>, dim3((unsigned)cdiv((int64_t)Bl * m, 256)), dim3(256), 0, st, 
                               x1, ldc, o, m, Bl, cache.a, dH, ldh);
                           return cudaGetLastError();
                         }});
        }
      }
      // dgrad: dZ_{L-1} = (dH W_out) * 1[A_{L-1} > 0], then down the hidden stack
      for (int l = L; l >= 1 && !abwd_fused; --l) {
        GemmArgs a = mk(an.out[l], bits ? EPI_MASK_BITS : EPI_MASK, 0, 1);
        if (bits)
          add(a, l == L ? (const void*)dH : (const void*)Lr->dZa[l], l == L ? ldh : h, Wp(NET_ACTOR, l), an.ld[l],
              Lr->dZa[l - 1], h, Bl, h, nullptr, Lr->mask_a[l - 1] + (int64_t)Bl * mw, mw);
        else
          add(a, l == L ? (const void*)dH : (const void*)Lr->dZa[l], l == L ? ldh : h, Wp(NET_ACTOR, l), an.ld[l],
              Lr->dZa[l - 1], h, Bl, h, nullptr, Ta(Lr->Aact[l - 1], Bl, h), h);
        if (bits && !tc_ok(a)) return fail(SPZ_EUNSUPPORTED, "internal: actor dgrad not supported by the tcgen05 kernel");
        gemm("actor_dgrad_gemm", a);
      }
      // wgrad: dW_l = dZ_l^T A_{l-1} over the Bl s-rows (dZ_L = dH)
      for (int l = 0; l <= L; ++l) {
        GemmGroup g{};
        g.A = l == L ? (const void*)dH : (const void*)Lr->dZa[l];
        g.lda = l == L ? ldh : h;
        g.B = l == 0 ? (const void*)Ta(Lr->Xa, Bl, lda) : (const void*)Ta(Lr->Aact[l - 1], Bl, h);
        g.ldb = l == 0 ? lda : h;
        g.C = Lr->G + slot_of(NET_ACTOR, l, true).g_off;
        g.ldc = (int)round_up(an.in[l], 4);
        g.M = an.out[l];
        g.N = an.in[l];
        g.split_stride = (int64_t)an.out[l] * g.ldc;
        if (fuse_bias) {
          g.colsum_out = Lr->G + slot_of(NET_ACTOR, l, false).g_off;
          g.colsum_stride = an.out[l];
        }
        if (Sa != Sw) {
          g.splits = Sa;
          g.k_per_split = (int)rows_a;
        }
        wgrads.push_back(g);
      }
      for (int l = 0; l <= L && !fuse_bias; ++l)
        colsums.push_back({l == L ? (const void*)dH : (const void*)Lr->dZa[l], nullptr,
                           Lr->G + slot_of(NET_ACTOR, l, false).g_off, l == L ? ldh : h, an.out[l], Bl, 0});
      (void)nout;
    }
    // ---- every weight gradient (split-K over the batch, <= 8 tensors per launch) and every bias
    //      gradient (one column-sum launch)
    // diagnostics only (results are wrong): SPZ_DIAG_MUTATE="drop_wgrad=i" / "drop_bias=i" drops the i-th
    // weight / bias gradient job, "tau0" freezes the targets -- the parity tests must fail under each
    if (const char* mu = std::getenv("SPZ_DIAG_MUTATE")) {
      const std::string ms(mu);
      auto idx_of = [&](const char* key) -> int {
        const size_t p = ms.find(key);
        return p == std::string::npos ? -1 : std::atoi(ms.c_str() + p + std::strlen(key));
      };
      const int dw = idx_of("drop_wgrad="), dbi = idx_of("drop_bias=");
      if (dw >= 0 && dw < (int)wgrads.size()) {
        wgrads.erase(wgrads.begin() + dw);
        if ((size_t)dw < n_pre_wgrads) --n_pre_wgrads;
      }
      if (dbi >= 0) {
        if (fuse_bias && dbi < (int)wgrads.size()) wgrads[dbi].colsum_out = nullptr;
        else if (!fuse_bias && dbi < (int)colsums.size()) colsums.erase(colsums.begin() + dbi);
      }
    }
    {
      GemmArgs a = mk(Bl, fuse_bias ? EPI_WGRAD_BIAS : EPI_F32, 1, 1);
      a.splits = Sw;
      a.k_per_split = (int)rows_w;
      // Behind an actor-backward kernel (PDL), the first launch computes the critic / value weight gradients --
      // whose inputs that kernel does not write -- before its grid-dependency wait, on a dynamic tile schedule:
      // its CTAs that start on the SMs the actor backward leaves idle take those tiles first (SPZ_WGRAD_PRE=0:
      // static schedule, everything after the wait)
      bool pre = false;
      if (!ops.empty() && n_pre_wgrads > 0 && bits && !wgrad_pre_off_env()) {
        static const char* const actor_ops[] = {"actor_bwd_fused", "actor_dgrad_gemm", "actor_head_bwd"};
        for (const char* c : actor_ops)
          if (std::strcmp(ops.back().cls, c) == 0) pre = true;
      }
      if (pre) {
        a.sched = Lr->sched + 2 * variant;
        a.n_pre_groups = (int)std::min<size_t>(n_pre_wgrads, MAX_GROUPS);
      }
      for (const GemmGroup& g : wgrads) {
        if (a.n_groups == MAX_GROUPS) {
          gemm("wgrad_gemm", a);
          a.n_groups = 0;
          a.N = 0;
          a.sched = nullptr;  // later launches: static schedule, wait first
          a.n_pre_groups = 0;
        }
        a.g[a.n_groups++] = g;
        a.N = std::max(a.N, g.N);
      }
      if (a.n_groups) gemm("wgrad_gemm", a);
      for (size_t c0 = 0; c0 < colsums.size(); c0 += MAX_COLSUM_JOBS) {
        ColsumArgs ca{};
        ca.rps = (int)rows_b;
        for (size_t c = c0; c < colsums.size() && c < c0 + MAX_COLSUM_JOBS; ++c) ca.j[ca.n_jobs++] = colsums[c];
        ops.push_back({"bias_grad", [ca, Sb](cudaStream_t st) {
                         return launch_pdl(colsum_multi_kernel<T>, dim3(Sb, ca.n_jobs), dim3(CS_TX * CS_TY), 0, st, ca);
                       }});
      }
    }
    // row-sharded groups reduce their split partials into one contiguous buffer and all-reduce it
    // together with the loss totals before the (identical) optimizer step on every rank
    const bool sharded = Lr->gsize > 1 || Lr->cfg.comm_mode == 2;
    // ---- a9: fused Adam + Polyak (+ shadow refresh) over every trained tensor
    {
      std::vector<AdamTensor> tens;
      std::vector<AdamSegment> segs;
      for (auto& s : slots) {
        // TD3, non-delayed step: the actor is not updated -- no segments for it (their blocks would only load
        // its optimizer state: 35 MB per step at the TD3 config); row-sharded groups keep one buffer layout
        if (td3 && !actor_step && s.net == NET_ACTOR && !sharded) continue;
        const NetLayout& n = Lr->net[s.net];
        AdamTensor t{};
        t.p_off = Lr->pbase[s.net] + (s.weight ? n.w[s.layer] : n.b[s.layer]);
        const bool head_vec = (s.net == NET_Q1 || s.net == NET_Q2 || s.net == NET_V) && s.layer == n.nl - 1;
        t.numel = s.weight ? (int64_t)n.out[s.layer] * n.in[s.layer] : n.out[s.layer];
        t.partials = Lr->G + s.g_off;
        t.n_partials = (s.weight && !head_vec) || fuse_bias ? (s.net == NET_ACTOR ? Sa : Sw) : Sb;
        t.pld = s.weight ? (head_vec ? n.in[s.layer] : (int)round_up(n.in[s.layer], 4)) : 1;
        t.pstride = s.weight ? (int64_t)n.out[s.layer] * t.pld : n.out[s.layer];
        t.opt = s.net == NET_ACTOR ? 1 : 0;
        t.cols = s.weight ? n.in[s.layer] : 0;
        t.ld = n.ld[s.layer];
        t.s_off = s.weight ? Lr->sbase[s.net] + n.sw[s.layer] : -1;
        int tid = s.net == NET_Q1 ? NET_Q1T : s.net == NET_Q2 ? NET_Q2T : s.net == NET_V ? NET_VT : (td3 ? NET_ACTORT : -1);
        if (tid >= 0 && !Lr->has_net[tid]) tid = -1;  // SAC v1: no target critics
        t.t_off = tid >= 0 ? Lr->pbase[tid] + (s.weight ? n.w[s.layer] : n.b[s.layer]) : -1;
        t.ts_off = (tid >= 0 && s.weight) ? Lr->sbase[tid] + n.sw[s.layer] : -1;
        tens.push_back(t);
      }
      if (!td3 && Lr->cfg.alpha_auto && Lr->cfg.role != SPZ_ROLE_CRITIC) {
        AdamTensor t{};
        t.p_off = Lr->p_log_alpha;
        t.numel = 1;
        t.partials = Lr->G + Lr->G_total - 64;
        t.n_partials = 1;
        t.opt = 2;
        t.s_off = t.t_off = t.ts_off = -1;
        tens.push_back(t);
      }
      // red_off: position of each tensor in the contiguous gradient buffer (sharded mode)
      {
        int64_t off = 0;
        for (auto& t : tens) {
          t.red_off = off;
          off += round_up(t.numel, 16);
        }
      }
      // float4 segments (4 consecutive elements per thread) where every access of the tensor is 16-byte aligned
      // (8-byte for the bf16 shadow) and 4 consecutive elements share one row; SPZ_ADAM_VEC=0 disables them
      const int vec_seg = adam_vec_seg();
      auto vec_ok = [&](const AdamTensor& t) {
        if (vec_seg == 0 || t.opt == 2 || t.numel % 4 || t.p_off % 4 || (t.t_off >= 0 && t.t_off % 4)) return false;
        if (reinterpret_cast<uintptr_t>(t.partials) % 16 || t.pstride % 4) return false;
        if (t.cols > 0) {
          if (t.cols % 4 || t.pld % 4 || t.ld % 4 || t.s_off % 4 || (t.ts_off >= 0 && t.ts_off % 4)) return false;
        } else if (t.pld != 1) {
          return false;
        }
        return true;
      };
      auto segments = [&](const std::vector<AdamTensor>& ts) {
        std::vector<AdamSegment> v;
        for (const AdamTensor& t : ts) {
          const bool vc = vec_ok(t);
          const int64_t seg = vc ? vec_seg : ADAM_SEG;
          for (int64_t st = 0; st < t.numel; st += seg) {
            AdamSegment sg{};
            sg.t = t;
            sg.start = st;
            sg.count = (int32_t)std::min<int64_t>(seg, t.numel - st);
            sg.vec = vc ? 1 : 0;
            v.push_back(sg);
          }
        }
        return v;
      };
      segs = segments(tens);
      if (segs.empty()) {  // (the TD3 actor role on a non-delayed step) one empty block: statistics and counters
        AdamSegment sg{};
        sg.t.s_off = sg.t.t_off = sg.t.ts_off = -1;
        segs.push_back(sg);
      }
      const int nsegs = (int)segs.size();
      if (4 * (nsegs + 1) > Lr->max_segs) return fail(SPZ_EINVAL, "internal: Adam table overflow");
      const size_t sb = segs.size() * sizeof(AdamSegment);
      AdamSegment* ds = Lr->d_segs + variant * (Lr->max_segs / 4);
      if (sharded) {
        // table 1 (partials -> Gred) is `segs`; table 2 (Gred -> Adam) replaces the partial sources
        AdamSegment* ds2 = Lr->d_segs + (2 + variant) * (Lr->max_segs / 4);
        std::vector<AdamTensor> tens2 = tens;
        for (auto& t : tens2) {
          if (t.opt == 2) continue;  // log alpha: gradient computed from the all-reduced totals
          t.partials = Lr->Gred + t.red_off;
          t.n_partials = 1;
          t.pld = t.cols > 0 ? t.cols : 1;  // dense
          t.pstride = t.numel;
        }
        const std::vector<AdamSegment> segs2 = segments(tens2);
        SPZ_CUDA_TRY(cudaMemcpyAsync(ds2, segs2.data(), sb, cudaMemcpyHostToDevice, Lr->stream));
        SPZ_CUDA_TRY(cudaMemcpyAsync(ds, segs.data(), sb, cudaMemcpyHostToDevice, Lr->stream));
        SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
        float* Gr = Lr->Gred;
        const unsigned nsg = (unsigned)segs.size();
        ops.push_back({"grad_reduce", [=](cudaStream_t st) {
                         return launch_pdl(reduce_partials_kernel, dim3(nsg), dim3(ADAM_NT), 0, st, (const AdamSegment*)ds, Gr);
                       }});
        if (Lr->cfg.comm_mode == 0 || Lr->cfg.comm_mode == 2) {
          const Comm cm = Lr->gcomm;
          const size_t n = (size_t)Lr->Gred_total;
          double* ss = Lr->statsum;
          ops.push_back({"allreduce", [=](cudaStream_t st) {
                           cudaError_t e = comm_allreduce_sum(cm, Gr, n, false, st);
                           if (e != cudaSuccess) return e;
                           return comm_allreduce_sum(cm, ss, NSTAT, true, st);
                         }, 0});
        }
        ds = ds2;
      } else {
        SPZ_CUDA_TRY(cudaMemcpyAsync(ds, segs.data(), sb, cudaMemcpyHostToDevice, Lr->stream));
        SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
      }
      AdamHyper hp{};
      hp.lr[0] = (float)Lr->cfg.lr_critic;
      hp.lr[1] = (float)Lr->cfg.lr_actor;
      hp.lr[2] = (float)Lr->cfg.lr_alpha;
      hp.beta1 = (float)Lr->cfg.beta1;
      hp.beta2 = (float)Lr->cfg.beta2;
      hp.eps = (float)Lr->cfg.adam_eps;
      hp.tau = (float)Lr->cfg.tau;
      if (const char* mu = std::getenv("SPZ_DIAG_MUTATE"))
        if (std::string(mu).find("tau0") != std::string::npos) hp.tau = 0.f;  // diagnostics only
      hp.td3 = td3;
      hp.delay = delay;
      hp.totals = Lr->statsum;
      if (defer_totals) {
        hp.stat_partials = Lr->stat_partials;
        hp.n_stat_blocks = nblk;
        hp.bad2 = Lr->tickets + 200;
      }
      hp.log_alpha = reinterpret_cast<const float*>(Lr->ctr_snap + 4);
      hp.stats = Lr->d_stats;
      hp.target_entropy = Lr->cfg.target_entropy;
      hp.B = (double)B;
      hp.snap = Lr->ctr_snap;
      hp.bc = reinterpret_cast<const float*>(Lr->ctr_snap + 5);
      hp.alpha_auto = Lr->cfg.alpha_auto;
      hp.diag_nowork = std::getenv("SPZ_DIAG_ADAM_NOWORK") != nullptr;  // diagnostics only (results are wrong)
      {  // the totals / snapshot may be read before the dependency wait only if the op right before Adam is a
         // kernel that waits before it triggers and is not their writer (e.g. not the loss kernel itself: the TD3
         // actor role on a non-delayed step goes loss -> Adam), or the non-PDL allreduce
        static const char* const safe[] = {"wgrad_gemm", "bias_grad", "actor_bwd_fused", "actor_dgrad_gemm", "actor_head_bwd",
                                           "critic_dgrad_gemm", "critic_input_dgrad_gemm", "allreduce"};
        hp.prewait = 0;
        if (!ops.empty())
          for (const char* c : safe)
            if (std::strcmp(ops.back().cls, c) == 0) hp.prewait = 1;
      }
      hp.critic_on = Lr->cfg.role != SPZ_ROLE_ACTOR;
      hp.actor_on = Lr->cfg.role != SPZ_ROLE_CRITIC;
      float *Pm = Lr->P, *Mm = Lr->Mo, *Vm = Lr->Vo;
      int64_t* ctr = Lr->counters;
      int* fl = Lr->d_flag;
      const unsigned nseg = (unsigned)segs.size();
      // one round of split-partial loads where the grid is at most two blocks per SM and some tensor has more
      // than 8 splits (SPZ_ADAM_WIDE=0 / 1 forces)
      int max_parts = 0;
      for (const AdamSegment& sg : segs) max_parts = std::max(max_parts, (int)sg.t.n_partials);
      int nsm_a = 148, dev_a = 0;
      cudaGetDevice(&dev_a);
      cudaDeviceGetAttribute(&nsm_a, cudaDevAttrMultiProcessorCount, dev_a);
      bool wide = (int)nseg <= 2 * nsm_a && max_parts > SPZ_ADAM_CH4;
      if (const char* aw = std::getenv("SPZ_ADAM_WIDE")) wide = std::atoi(aw) == 1;
      ops.push_back({"adam_polyak", [=](cudaStream_t st) {
                       if (wide)
                         return launch_pdl(adam_polyak_kernel<T, true>, dim3(nseg), dim3(ADAM_NT), 0, st, (const AdamSegment*)ds, hp, Pm,
                                           Mm, Vm, S, ctr, fl);
                       return launch_pdl(adam_polyak_kernel<T, false>, dim3(nseg), dim3(ADAM_NT), 0, st, (const AdamSegment*)ds, hp, Pm,
                                         Mm, Vm, S, ctr, fl);
                     }});
    }
    // ---- a10: split roles exchange the updated parameters at the step boundary:
    //      phi_{k+1} (+ log alpha, TD3 phi') from the actor leader, theta_{k+1} from the critic leader
    if (Lr->split && Lr->cfg.world_size > 1 && Lr->cfg.comm_mode == 0) {
      const Comm cm = Lr->comm;
      const int nc = plan.actor_root, c0 = plan.critic_root;
      float* pa = P + Lr->pbase[NET_ACTOR];
      const size_t na = (size_t)Lr->net[NET_ACTOR].np;
      float* pat = Lr->has_net[NET_ACTORT] ? P + Lr->pbase[NET_ACTORT] : nullptr;
      float* pla = P + Lr->p_log_alpha;
      float* pq = P + Lr->pbase[NET_Q1];
      const size_t nq = (size_t)(Lr->pbase[NET_Q2] + Lr->net[NET_Q2].np - Lr->pbase[NET_Q1]);
      const ShadowEntry* sh = Lr->d_shadow_recv;
      const int nsh = Lr->n_shadow_recv;
      ops.push_back({"exchange", [=](cudaStream_t st) {
                       cudaError_t e = comm_broadcast_f32(cm, pa, na, nc, st);
                       if (e == cudaSuccess) e = comm_broadcast_f32(cm, pla, 1, nc, st);
                       if (e == cudaSuccess && pat) e = comm_broadcast_f32(cm, pat, na, nc, st);
                       if (e == cudaSuccess) e = comm_broadcast_f32(cm, pq, nq, c0, st);
                       if (e != cudaSuccess) return e;
                       return launch_pdl(shadow_refresh_kernel<T>, dim3(64, nsh), dim3(256), 0, st, sh, nsh, (const float*)P, S);
                     }, 1});
    }
    if (!unsupported.empty()) {
      for (auto& v : Lr->ops) v.clear();
      return fail(SPZ_EUNSUPPORTED, std::string("spz_update: GEMM ") + unsupported + " is not supported by the " +
                                        (Lr->bf16 ? "bf16 tcgen05" : "3xTF32 tcgen05") + " kernels (no other backend)");
    }
  }
  // diagnostics only: SPZ_DIAG_NOOP_OPS=k appends k empty PDL kernels to the step (kernel-boundary cost)
  if (const char* nn = std::getenv("SPZ_DIAG_NOOP_OPS")) {
    const int k = std::atoi(nn);
    for (auto& v : Lr->ops)
      if (!v.empty())
        for (int i = 0; i < k; ++i)
          v.push_back({"noop", [](cudaStream_t st) { return launch_pdl(noop_kernel, dim3(148), dim3(128), 0, st, 0); }});
  }
  // diagnostics only (results are wrong): SPZ_DIAG_SKIP_OPS="cls1,cls2" drops those op classes so a
  // timing run shows their marginal cost inside the graph replay
  if (const char* skip = std::getenv("SPZ_DIAG_SKIP_OPS")) {
    for (auto& v : Lr->ops)
      v.erase(std::remove_if(v.begin(), v.end(),
                             [skip](const Op& op) {
                               const std::string list = std::string(",") + skip + ",";
                               return list.find(std::string(",") + op.cls + ",") != std::string::npos;
                             }),
              v.end());
  }
  Lr->plan_track_gen = Lr->ring->track_gen;
  Lr->plan_B = B;
  return SPZ_OK;
}

static cudaError_t enqueue_publish(spz_learner* Lr, int slot, cudaStream_t st) {
  constexpr int W = (int)(sizeof(spz_learner::ReadBack) / 8);
  unsigned long long* dst = Lr->d_slots + (size_t)slot * (sizeof(spz_learner::HostSlot) / 8);
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(Lr->d_rb);
  if (publish_pdl_env()) return launch_pdl(publish_kernel, dim3(1), dim3(32), 0, st, src, dst, W);
  publish_kernel<<<1, 32, 0, st>>>(src, dst, W);
  return cudaGetLastError();
}

static spz_status run_ops(spz_learner* Lr, int variant, cudaStream_t st) {
  for (auto& op : Lr->ops[variant]) {
    cudaError_t e = op.fn(st);
    if (e != cudaSuccess) return fail(SPZ_ECUDA, std::string("kernel ") + op.cls + ": " + cudaGetErrorString(e));
  }
  return SPZ_OK;
}

static cudaError_t enqueue_publish(spz_learner* Lr, int slot, cudaStream_t st);
// One step of `variant` as a CUDA graph; pub_slot >= 0: the graph ends with the read-back publish into host slot
// pub_slot (a programmatically launched node behind the optimizer: no stream operation between consecutive
// updates, where a separate launch cost ~4 us per step of the end-to-end loop)
static spz_status ensure_graph(spz_learner* Lr, int variant, int pub_slot = -1) {
  cudaGraphExec_t& ex = pub_slot < 0 ? Lr->exec[variant] : Lr->exec_pub[variant][pub_slot];
  if (ex) return SPZ_OK;
  cudaStream_t cs;
  SPZ_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  SPZ_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  spz_status s = run_ops(Lr, variant, cs);
  if (s == SPZ_OK && pub_slot >= 0) {
    const cudaError_t pe = enqueue_publish(Lr, pub_slot, cs);
    if (pe != cudaSuccess) s = fail(SPZ_ECUDA, std::string("publish: ") + cudaGetErrorString(pe));
  }
  cudaError_t e = cudaStreamEndCapture(cs, &g);
  cudaStreamDestroy(cs);
  if (s != SPZ_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  if (e != cudaSuccess) return fail(SPZ_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(SPZ_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  return SPZ_OK;
}

static spz_status prepare(spz_learner* Lr, int64_t batch) {
  if (batch < 1 || batch > Lr->cfg.max_batch)
    return fail(SPZ_EINVAL, "batch " + std::to_string(batch) + " outside [1, max_batch=" + std::to_string(Lr->cfg.max_batch) + "]");
  if (batch < Lr->cfg.world_size) return fail(SPZ_EINVAL, "batch smaller than world_size");
  const int64_t F = Lr->ring->fill();
  if (F < batch) return fail(SPZ_ENODATA, "ring fill " + std::to_string(F) + " < batch " + std::to_string(batch));
  if (Lr->plan_B != batch || Lr->plan_track_gen != Lr->ring->track_gen) {
    SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
    spz_status s = Lr->bf16 ? build_plan<__nv_bfloat16>(Lr, batch) : build_plan<float>(Lr, batch);
    if (s != SPZ_OK) {
      Lr->plan_B = -1;
      return s;
    }
  }
  return SPZ_OK;
}


template <typename T>
static spz_status refresh_shadows_t(spz_learner* Lr) {
  launch_pdl(shadow_refresh_kernel<T>, dim3(dim3(64, (unsigned)Lr->n_shadow)), dim3(256), 0, Lr->stream, Lr->d_shadow, Lr->n_shadow, Lr->P,
                                                                                     static_cast<T*>(Lr->S));
  SPZ_CUDA_TRY(cudaGetLastError());
  return SPZ_OK;
}

spz_status refresh_shadows(spz_learner* Lr) {
  return Lr->bf16 ? refresh_shadows_t<__nv_bfloat16>(Lr) : refresh_shadows_t<float>(Lr);
}

static int variant_of(spz_learner* Lr, int64_t step) {
  if (!Lr->td3) return 0;
  const int delay = std::max(1, Lr->cfg.td3_policy_delay);
  return ((step + 1) % delay) == 0 ? 1 : 0;
}

static spz_status read_counters(spz_learner* Lr) {
  SPZ_CUDA_TRY(cudaMemcpyAsync(Lr->h_counters, Lr->counters, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, Lr->stream));
  SPZ_CUDA_TRY(cudaMemcpyAsync(Lr->h_flag, Lr->d_flag, sizeof(int), cudaMemcpyDeviceToHost, Lr->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  Lr->ctr_cached = true;
  return SPZ_OK;
}

}  // namespace spz

// ============================================================================= C API
extern "C" {

spz_status spz_config_default(spz_algo algo, int32_t obs_dim, int32_t act_dim, spz_config* out) {
  if (!out) return fail(SPZ_EINVAL, "spz_config_default: NULL out");
  if (obs_dim < 1 || act_dim < 1) return fail(SPZ_EINVAL, "spz_config_default: dims must be >= 1");
  std::memset(out, 0, sizeof(*out));
  out->algo = algo;
  out->precision = SPZ_BF16;
  out->obs_dim = obs_dim;
  out->act_dim = act_dim;
  out->hidden = 256;
  out->n_hidden = 2;
  out->max_batch = 8192;
  out->gamma = 0.99;
  out->tau = 0.005;
  out->lr_actor = out->lr_critic = out->lr_alpha = 3e-4;
  out->beta1 = 0.9;
  out->beta2 = 0.999;
  out->adam_eps = 1e-8;
  out->alpha_auto = algo == SPZ_SAC ? 1 : 0;  // SAC v1: fixed temperature (haarnoja2018soft)
  out->alpha_init = 0.2;
  out->target_entropy = -(double)act_dim;
  out->log_std_min = -20.0;
  out->log_std_max = 2.0;
  out->td3_noise = algo == SPZ_DDPG ? 0.0 : 0.2;
  out->td3_noise_clip = algo == SPZ_DDPG ? 0.0 : 0.5;
  out->td3_policy_delay = algo == SPZ_DDPG ? 1 : 2;
  out->seed = 6126;
  out->init_seed = 0;
  out->device = 0;
  out->world_size = 1;
  out->rank = 0;
  out->role = SPZ_ROLE_ALL;
  out->use_graph = 1;
  return SPZ_OK;
}

spz_status spz_plan_rank(const spz_config* cfg, int64_t batch, spz_plan* out) {
  if (!cfg || !out) return fail(SPZ_EINVAL, "spz_plan_rank: NULL argument");
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size)
    return fail(SPZ_EINVAL, "spz_plan_rank: bad rank/world_size");
  if (cfg->role != SPZ_ROLE_ALL && cfg->role != SPZ_ROLE_CRITIC && cfg->role != SPZ_ROLE_ACTOR)
    return fail(SPZ_EINVAL, "spz_plan_rank: unknown role");
  spz_plan p{};
  p.role = cfg->role;
  p.group_size = cfg->world_size;
  p.group_rank = cfg->rank;
  p.actor_root = p.critic_root = -1;
  if (cfg->role != SPZ_ROLE_ALL && cfg->world_size > 1) {
    // critic group = ranks [0, n_critic_ranks), actor group = the rest (P:239-247 generalised)
    const int nc = cfg->n_critic_ranks;
    if (nc < 1 || nc >= cfg->world_size) return fail(SPZ_EINVAL, "spz_plan_rank: split roles need 1 <= n_critic_ranks < world_size");
    if ((cfg->rank < nc) != (cfg->role == SPZ_ROLE_CRITIC))
      return fail(SPZ_EINVAL, "spz_plan_rank: ranks [0, n_critic_ranks) must be critic, the others actor");
    const bool critic = cfg->role == SPZ_ROLE_CRITIC;
    p.group_size = critic ? nc : cfg->world_size - nc;
    p.group_rank = critic ? cfg->rank : cfg->rank - nc;
    p.group_color = critic ? 0 : 1;
    p.critic_root = 0;
    p.actor_root = nc;
  }
  if (batch < p.group_size) return fail(SPZ_EINVAL, "spz_plan_rank: batch smaller than the group");
  const int64_t base = batch / p.group_size, rem = batch % p.group_size;
  p.rows = base + (p.group_rank < rem ? 1 : 0);
  p.row0 = p.group_rank * base + std::min<int64_t>(p.group_rank, rem);
  p.allreduce = p.group_size > 1 && cfg->comm_mode == 0;
  *out = p;
  return SPZ_OK;
}

spz_status spz_learner_create(const spz_config* cfg, spz_replay* ring, spz_learner** out) {
  if (!cfg || !ring || !out) return fail(SPZ_EINVAL, "spz_learner_create: NULL argument");
  *out = nullptr;
  if (cfg->obs_dim != ring->o || cfg->act_dim != ring->m)
    return fail(SPZ_EINVAL, "spz_learner_create: config dims do not match the ring");
  if (cfg->device != ring->device) return fail(SPZ_EINVAL, "spz_learner_create: ring lives on another device");
  if (cfg->hidden < 16 || cfg->hidden % 16 || cfg->n_hidden < 1 || cfg->n_hidden > 6)
    return fail(SPZ_EINVAL, "spz_learner_create: need hidden a positive multiple of 16 and 1 <= n_hidden <= 6");
  if (cfg->max_batch < 1) return fail(SPZ_EINVAL, "spz_learner_create: max_batch must be >= 1");
  if (cfg->act_dim > 32) return fail(SPZ_EINVAL, "spz_learner_create: act_dim must be <= 32");
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size) return fail(SPZ_EINVAL, "spz_learner_create: bad rank/world_size");
  if (cfg->world_size > 1 && cfg->comm_mode == 0 && !cfg->nccl_unique_id)
    return fail(SPZ_EINVAL, "spz_learner_create: world_size > 1 needs nccl_unique_id (or comm_mode = 1)");
  if (cfg->role != SPZ_ROLE_ALL && cfg->role != SPZ_ROLE_CRITIC && cfg->role != SPZ_ROLE_ACTOR)
    return fail(SPZ_EINVAL, "spz_learner_create: unknown role");
  spz_plan plan;  // validates the rank / role layout; the group shape below comes from it
  SPZ_TRY(spz_plan_rank(cfg, std::max<int64_t>(cfg->world_size, cfg->max_batch), &plan));
  if (cfg->algo != SPZ_SAC && cfg->algo != SPZ_TD3 && cfg->algo != SPZ_DDPG && cfg->algo != SPZ_SACV1)
    return fail(SPZ_EINVAL, "spz_learner_create: unknown algo");
  if (cfg->algo == SPZ_SACV1 && cfg->role != SPZ_ROLE_ALL)
    return fail(SPZ_EUNSUPPORTED, "spz_learner_create: SAC v1 runs with role ALL only");
  if (cfg->precision != SPZ_FP32 && cfg->precision != SPZ_BF16) return fail(SPZ_EINVAL, "spz_learner_create: unknown precision");
  spz_status st = check_device(cfg->device);
  if (st != SPZ_OK) return st;
  DeviceGuard dg(cfg->device);
  std::unique_ptr<spz_learner> Lr(new spz_learner());
  Lr->cfg = *cfg;
  Lr->ring = ring;
  Lr->device = cfg->device;
  Lr->td3 = cfg->algo == SPZ_TD3 || cfg->algo == SPZ_DDPG;
  Lr->ddpg = cfg->algo == SPZ_DDPG;
  Lr->v1 = cfg->algo == SPZ_SACV1;
  Lr->bf16 = cfg->precision == SPZ_BF16;
  Lr->esz = Lr->bf16 ? 2 : 4;
  Lr->o = cfg->obs_dim;
  Lr->m = cfg->act_dim;
  Lr->h = cfg->hidden;
  Lr->L = cfg->n_hidden;
  const int o = Lr->o, m = Lr->m, h = Lr->h, L = Lr->L;
  if (cudaStreamCreateWithFlags(&Lr->own_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SPZ_ECUDA, "spz_learner_create: stream creation failed");
  Lr->stream = Lr->own_stream;
  if (cudaEventCreateWithFlags(&Lr->ev_read, cudaEventDisableTiming) != cudaSuccess)
    return fail(SPZ_ECUDA, "spz_learner_create: event creation failed");
  {
    std::lock_guard<std::mutex> lk(ring->mu);
    ring->readers.push_back(Lr->ev_read);
  }
  Lr->split = cfg->role != SPZ_ROLE_ALL;
  Lr->gsize = plan.group_size;
  const int W = Lr->gsize;
  Lr->max_local = cfg->max_batch / W + (cfg->max_batch % W ? 1 : 0);
  // networks
  const int aout = Lr->td3 ? m : 2 * m;
  const int kpad = Lr->bf16 ? 64 : 8;
  Lr->net[NET_ACTOR] = make_layout(o, h, L, aout, kpad);
  Lr->net[NET_Q1] = Lr->net[NET_Q2] = Lr->net[NET_Q1T] = Lr->net[NET_Q2T] = make_layout(o + m, h, L, 1, kpad);
  Lr->net[NET_ACTORT] = Lr->net[NET_ACTOR];
  Lr->net[NET_V] = Lr->net[NET_VT] = make_layout(o, h, L, 1, kpad);
  int64_t p = 0, s = 0;
  for (int id = 0; id < N_NETS; ++id) {
    if (id == NET_ACTORT) Lr->has_net[id] = Lr->td3;
    else if (id == NET_Q1T || id == NET_Q2T) Lr->has_net[id] = !Lr->v1;
    else if (id == NET_V || id == NET_VT) Lr->has_net[id] = Lr->v1;
    else Lr->has_net[id] = true;
    if (!Lr->has_net[id]) continue;
    Lr->pbase[id] = p;
    p += round_up(Lr->net[id].np, 64);
    Lr->sbase[id] = s;
    s += Lr->net[id].ns;
  }
  Lr->p_log_alpha = p;
  p += 64;
  Lr->P_total = p;
  Lr->S_total = s;
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->P, p * sizeof(float)));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->Mo, p * sizeof(float)));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->Vo, p * sizeof(float)));
  SPZ_TRY(dalloc(Lr.get(), &Lr->S, s * Lr->esz));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->d_rb, sizeof(spz_learner::ReadBack)));
  Lr->counters = Lr->d_rb->ctr;
  Lr->d_flag = &Lr->d_rb->flag;
  Lr->d_stats = &Lr->d_rb->stats;
  if (cudaHostAlloc(&Lr->h_slots, 2 * sizeof(spz_learner::HostSlot), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&Lr->d_slots, Lr->h_slots, 0) != cudaSuccess ||
      cudaEventCreateWithFlags(&Lr->ev_slot[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&Lr->ev_slot[1], cudaEventDisableTiming) != cudaSuccess)
    return fail(SPZ_ENOMEM, "spz_learner_create: pinned read-back slots");
  if (cudaMallocHost(&Lr->h_stats, sizeof(StatsOut)) != cudaSuccess || cudaMallocHost(&Lr->h_flag, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&Lr->h_counters, 8 * sizeof(int64_t)) != cudaSuccess)
    return fail(SPZ_ENOMEM, "spz_learner_create: pinned host allocation failed");
  // activations
  const int64_t Bm = Lr->max_local;
  // input rows padded like the layer-0 weights (the padding columns stay zero)
  Lr->lda = (int)round_up(o, kpad);
  Lr->ldc = (int)round_up(o + m, kpad);
  Lr->ldh = (int)round_up(aout, 8);
  const size_t E = Lr->esz;
  SPZ_TRY(dalloc(Lr.get(), &Lr->Xa, 2 * Bm * Lr->lda * E));
  SPZ_TRY(dalloc(Lr.get(), &Lr->Xc, 3 * Bm * Lr->ldc * E));
  SPZ_TRY(dalloc(Lr.get(), &Lr->dH, Bm * Lr->ldh * E));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->H, 2 * Bm * Lr->ldh * sizeof(float)));
  Lr->mw = (int)cdiv(h, 32);
  Lr->qp = (int)cdiv(h, 256);
  for (int l = 0; l < L; ++l) {
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->mask_a[l], 2 * Bm * Lr->mw * 4));
    for (int i = 0; i < 2; ++i) SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->mask_c[i][l], 2 * Bm * Lr->mw * 4));
    SPZ_TRY(dalloc(Lr.get(), &Lr->Aact[l], 2 * Bm * h * E));
    SPZ_TRY(dalloc(Lr.get(), &Lr->dZa[l], Bm * h * E));
    for (int i = 0; i < 2; ++i) {
      SPZ_TRY(dalloc(Lr.get(), &Lr->Aon[i][l], 2 * Bm * h * E));
      SPZ_TRY(dalloc(Lr.get(), &Lr->Atg[i][l], Bm * h * E));
      SPZ_TRY(dalloc(Lr.get(), &Lr->dZc[i][l], 2 * Bm * h * E));
    }
  }
  for (int i = 0; i < 2; ++i) {
    // h > 256: the fused row dot leaves one partial per 256-column tile (QP of them)
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->q_on[i], 2 * Bm * Lr->qp * sizeof(float)));
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->q_tg[i], Bm * Lr->qp * sizeof(float)));
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->gq[i], 2 * Bm * sizeof(float)));
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->gq16[i], Bm * 8 * sizeof(__nv_bfloat16)));
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->dXc[i], Bm * Lr->ldc * sizeof(float)));
  }
  for (float** f : {&Lr->logp, &Lr->logp2, &Lr->r, &Lr->d, &Lr->y}) SPZ_TRY(dalloc(Lr.get(), (void**)f, Bm * sizeof(float)));
  if (Lr->v1) {
    for (int l = 0; l < L; ++l) {
      SPZ_TRY(dalloc(Lr.get(), &Lr->Av[l], Bm * h * E));
      SPZ_TRY(dalloc(Lr.get(), &Lr->AvT[l], Bm * h * E));
      SPZ_TRY(dalloc(Lr.get(), &Lr->dZv[l], Bm * h * E));
      SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->mask_v[l], Bm * Lr->mw * 4));
    }
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->v_on, Bm * Lr->qp * sizeof(float)));
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->v_tg, Bm * Lr->qp * sizeof(float)));
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->gv, Bm * sizeof(float)));
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->gv16, Bm * 8 * sizeof(__nv_bfloat16)));
  }
  for (float** f : {&Lr->cache.u, &Lr->cache.a, &Lr->cache.eps, &Lr->cache.sig, &Lr->cache.l})
    SPZ_TRY(dalloc(Lr.get(), (void**)f, Bm * m * sizeof(float)));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->idx, Bm * sizeof(int32_t)));
  Lr->max_stat_blocks = (int)cdiv(Bm, LOSS_MIN_ROWS);
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->stat_partials, (size_t)Lr->max_stat_blocks * NSTAT * sizeof(double)));
  {
    auto reg = [&](const std::string& n, void* p, size_t bytes, int es) { Lr->debug.push_back({n, p, bytes, es}); };
    reg("Xa", Lr->Xa, 2 * Bm * Lr->lda * E, (int)E);
    reg("Xc", Lr->Xc, 3 * Bm * Lr->ldc * E, (int)E);
    reg("H", Lr->H, 2 * Bm * Lr->ldh * 4, 4);
    reg("dH", Lr->dH, Bm * Lr->ldh * E, (int)E);
    for (int l = 0; l < L; ++l) {
      reg("Aact" + std::to_string(l), Lr->Aact[l], 2 * Bm * h * E, (int)E);
      reg("dZa" + std::to_string(l), Lr->dZa[l], Bm * h * E, (int)E);
      for (int i = 0; i < 2; ++i) {
        reg("Aon" + std::to_string(i) + "_" + std::to_string(l), Lr->Aon[i][l], 2 * Bm * h * E, (int)E);
        reg("Atg" + std::to_string(i) + "_" + std::to_string(l), Lr->Atg[i][l], Bm * h * E, (int)E);
        reg("dZc" + std::to_string(i) + "_" + std::to_string(l), Lr->dZc[i][l], 2 * Bm * h * E, (int)E);
      }
    }
    for (int l = 0; l < L; ++l) {  // packed ReLU masks (bf16 tensor-core path): [rows x mw] u32, bit c%32 of word c/32
      if (Lr->mask_a[l]) reg("mask_a" + std::to_string(l), Lr->mask_a[l], 2 * Bm * Lr->mw * 4, 4);
      for (int i = 0; i < 2; ++i)
        if (Lr->mask_c[i][l]) reg("mask_c" + std::to_string(i) + "_" + std::to_string(l), Lr->mask_c[i][l], 2 * Bm * Lr->mw * 4, 4);
    }
    for (int i = 0; i < 2; ++i) {
      // q partials: qp planes of 2 * max_local (online) / max_local (target) rows (h > 256: one per 256-column tile)
      reg("q_on" + std::to_string(i), Lr->q_on[i], 2 * Bm * Lr->qp * 4, 4);
      reg("q_tg" + std::to_string(i), Lr->q_tg[i], Bm * Lr->qp * 4, 4);
      reg("gq" + std::to_string(i), Lr->gq[i], 2 * Bm * 4, 4);
      reg("dXc" + std::to_string(i), Lr->dXc[i], Bm * Lr->ldc * 4, 4);
    }
    if (Lr->v1) {
      reg("v_on", Lr->v_on, Bm * 4, 4);
      reg("v_tg", Lr->v_tg, Bm * 4, 4);
      reg("gv", Lr->gv, Bm * 4, 4);
    }
    reg("logp", Lr->logp, Bm * 4, 4);
    reg("logp2", Lr->logp2, Bm * 4, 4);
    reg("r", Lr->r, Bm * 4, 4);
    reg("d", Lr->d, Bm * 4, 4);
    reg("y", Lr->y, Bm * 4, 4);
    reg("idx", Lr->idx, Bm * 4, 4);
    reg("P", Lr->P, Lr->P_total * 4, 4);
    reg("S", Lr->S, Lr->S_total * E, (int)E);
  }
  // gradients and optimizer tables
  std::vector<TensorSlot> slots = trained_tensors(Lr.get());
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->G, Lr->G_total * sizeof(float)));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->statsum, 8 * sizeof(double)));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->tickets, 256 * sizeof(unsigned)));  // [0] + per-group counters (critic_loss_kernel)
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->sched, 64 * sizeof(unsigned)));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->ctr_snap, 16 * sizeof(int64_t)));
  Lr->debug.push_back({"statsum", Lr->statsum, 8 * sizeof(double), 8});
  if (Lr->gsize > 1 || cfg->comm_mode == 2) {
    int64_t tot = 0;
    for (auto& t : slots) tot += round_up(t.numel, 16);  // >= the dense tensor sizes
    Lr->Gred_total = tot + 16;
    SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->Gred, Lr->Gred_total * sizeof(float)));
    Lr->debug.push_back({"Gred", Lr->Gred, (size_t)Lr->Gred_total * 4, 4});
  }
  if (cfg->comm_mode == 2) {
    // diagnostic: a single-rank NCCL group runs the sharded path (partials -> reduce -> allreduce -> Adam)
    if (cfg->world_size != 1 || Lr->split) return fail(SPZ_EINVAL, "spz_learner_create: comm_mode 2 needs world_size 1 and role ALL");
    uint8_t uid[128];
    SPZ_TRY(spz_nccl_unique_id(uid));
    SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
    SPZ_TRY(comm_init(&Lr->comm, uid, 1, 0));
    Lr->gcomm = Lr->comm;
  }
  if (cfg->world_size > 1 && cfg->comm_mode == 0) {
    SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
    spz_status cs = comm_init(&Lr->comm, cfg->nccl_unique_id, cfg->world_size, cfg->rank);
    if (cs != SPZ_OK) return cs;
    Lr->gcomm = Lr->comm;
    if (Lr->split) {  // the role's own group for the gradient allreduce
      cs = comm_split(Lr->comm, plan.group_color, plan.group_rank, &Lr->gcomm);
      if (cs != SPZ_OK) return cs;
    }
  }
  int64_t nseg = 0;
  for (auto& t : slots) nseg += cdiv(t.numel, ADAM_SEG);
  Lr->max_segs = (int)(4 * (nseg + 4));
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->d_segs, Lr->max_segs * sizeof(AdamSegment)));
  // shadow table: every W of every net
  std::vector<ShadowEntry> sh;
  for (int id = 0; id < N_NETS; ++id) {
    if (!Lr->has_net[id]) continue;
    const NetLayout& n = Lr->net[id];
    for (int l = 0; l < n.nl; ++l) sh.push_back({Lr->pbase[id] + n.w[l], n.out[l], n.in[l], n.ld[l], Lr->sbase[id] + n.sw[l]});
  }
  Lr->n_shadow = (int)sh.size();
  {
    // networks this role receives at the step boundary: the actor (and TD3 target actor) on the
    // critic side, the online critics on the actor side
    std::vector<ShadowEntry> rv;
    for (int id = 0; id < N_NETS; ++id) {
      if (!Lr->has_net[id]) continue;
      const bool recv = (cfg->role == SPZ_ROLE_CRITIC && (id == NET_ACTOR || id == NET_ACTORT)) ||
                        (cfg->role == SPZ_ROLE_ACTOR && (id == NET_Q1 || id == NET_Q2));
      if (!recv) continue;
      const NetLayout& n = Lr->net[id];
      for (int l = 0; l < n.nl; ++l) rv.push_back({Lr->pbase[id] + n.w[l], n.out[l], n.in[l], n.ld[l], Lr->sbase[id] + n.sw[l]});
    }
    Lr->n_shadow_recv = (int)rv.size();
    if (!rv.empty()) {
      SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->d_shadow_recv, rv.size() * sizeof(ShadowEntry)));
      SPZ_CUDA_TRY(cudaMemcpyAsync(Lr->d_shadow_recv, rv.data(), rv.size() * sizeof(ShadowEntry), cudaMemcpyHostToDevice, Lr->stream));
      SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
    }
  }
  SPZ_TRY(dalloc(Lr.get(), (void**)&Lr->d_shadow, sh.size() * sizeof(ShadowEntry)));
  SPZ_CUDA_TRY(cudaMemcpyAsync(Lr->d_shadow, sh.data(), sh.size() * sizeof(ShadowEntry), cudaMemcpyHostToDevice, Lr->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  // init: W, b ~ U(+-1/sqrt(fan_in)) (Philox stream S_INIT); targets copy online; log alpha = ln alpha_init
  for (int id : {NET_ACTOR, NET_Q1, NET_Q2, NET_V}) {
    if (!Lr->has_net[id]) continue;
    const NetLayout& n = Lr->net[id];
    for (int l = 0; l < n.nl; ++l) {
      const float bound = 1.0f / std::sqrt((float)n.in[l]);
      const int64_t cnt = (int64_t)n.out[l] * n.in[l] + n.out[l];
      launch_pdl(init_uniform_kernel, dim3((unsigned)std::min<int64_t>(cdiv(cnt, 256), 1024)), dim3(256), 0, Lr->stream, 
          Lr->P, Lr->pbase[id] + n.w[l], cnt, bound, cfg->init_seed, (uint32_t)id, n.w[l]);
    }
  }
  SPZ_CUDA_TRY(cudaGetLastError());
  auto copy_net = [&](int dst, int src) {
    return cudaMemcpyAsync(Lr->P + Lr->pbase[dst], Lr->P + Lr->pbase[src], Lr->net[src].np * sizeof(float),
                           cudaMemcpyDeviceToDevice, Lr->stream);
  };
  if (Lr->ddpg) SPZ_CUDA_TRY(copy_net(NET_Q2, NET_Q1));  // the tied twin
  if (Lr->has_net[NET_Q1T]) SPZ_CUDA_TRY(copy_net(NET_Q1T, NET_Q1));
  if (Lr->has_net[NET_Q2T]) SPZ_CUDA_TRY(copy_net(NET_Q2T, NET_Q2));
  if (Lr->v1) SPZ_CUDA_TRY(copy_net(NET_VT, NET_V));
  if (Lr->td3) SPZ_CUDA_TRY(copy_net(NET_ACTORT, NET_ACTOR));
  const float la = (float)std::log(cfg->alpha_init > 0 ? cfg->alpha_init : 1e-30);
  SPZ_CUDA_TRY(cudaMemcpyAsync(Lr->P + Lr->p_log_alpha, &la, sizeof(float), cudaMemcpyHostToDevice, Lr->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  spz_status rs = refresh_shadows(Lr.get());
  if (rs != SPZ_OK) return rs;
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  *out = Lr.release();
  return SPZ_OK;
}

spz_status spz_learner_set_stream(spz_learner* Lr, void* stream) {
  if (!Lr) return fail(SPZ_EINVAL, "spz_learner_set_stream: NULL learner");
  DeviceGuard dg(Lr->device);
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  Lr->stream = stream ? static_cast<cudaStream_t>(stream) : Lr->own_stream;
  return SPZ_OK;
}

namespace spz {
// completes the oldest update in flight: its statistics, the step counters and the non-finite flag
// (the counters mirror the device again once nothing is in flight)
static spz_status update_finish(spz_learner* Lr, spz_stats* last) {
  if (Lr->n_inflight == 0) {
    if (*Lr->h_flag)
      return fail(SPZ_ENONFINITE, "spz_update: learner halted by an earlier non-finite step " + std::to_string(Lr->h_counters[0]));
  } else {
    const int sl = Lr->inflight[0];
    Lr->inflight[0] = Lr->inflight[1];
    --Lr->n_inflight;
    SPZ_CUDA_TRY(cudaEventSynchronize(Lr->ev_slot[sl]));
    const spz_learner::ReadBack& rb = Lr->h_slots[sl].rb;
    for (int i = 0; i < 4; ++i) Lr->h_counters[i] = rb.ctr[i];
    *Lr->h_flag = rb.flag;
    *Lr->h_stats = rb.stats;
    Lr->ctr_cached = Lr->n_inflight == 0;
    if (rb.flag)
      return fail(SPZ_ENONFINITE, "spz_update: non-finite loss or gradient at step " + std::to_string(rb.ctr[0]) +
                                      (rb.flag == 2 ? " (gradient)" : " (loss)") + "; learner halted");
  }
  if (last) {
    const StatsOut& s = *Lr->h_stats;
    last->step = (int64_t)s.step;
    last->critic_loss = Lr->ddpg ? 0.5 * s.critic_loss : s.critic_loss;  // DDPG: one critic (tied twins)
    last->actor_loss = s.actor_loss;
    last->alpha = s.alpha;
    last->alpha_loss = s.alpha_loss;
    last->q1_mean = s.q1_mean;
    last->q2_mean = s.q2_mean;
    last->logp_mean = s.logp_mean;
    last->value_loss = Lr->v1 ? s.value_loss : 0.0;
  }
  return SPZ_OK;
}
// completes every update in flight (statistics dropped)
static spz_status update_drain(spz_learner* Lr) {
  spz_status st = SPZ_OK;
  while (Lr->n_inflight > 0) {
    const spz_status s = update_finish(Lr, nullptr);
    if (st == SPZ_OK) st = s;
  }
  return st;
}
}  // namespace spz

spz_status spz_update_async(spz_learner* Lr, int64_t batch, int64_t n_steps) {
  if (!Lr) return fail(SPZ_EINVAL, "spz_update_async: NULL learner");
  if (n_steps < 0) return fail(SPZ_EINVAL, "spz_update_async: n_steps < 0");
  DeviceGuard dg(Lr->device);
  if (Lr->n_inflight == 2) SPZ_TRY(update_finish(Lr, nullptr));  // at most two updates in flight
  if (Lr->plan_B != batch || Lr->plan_track_gen != Lr->ring->track_gen) SPZ_TRY(update_drain(Lr));
  SPZ_TRY(prepare(Lr, batch));
  int64_t step;
  if (Lr->n_inflight == 0) {
    if (!Lr->ctr_cached) SPZ_TRY(read_counters(Lr));
    if (*Lr->h_flag) return fail(SPZ_ENONFINITE, "spz_update: learner halted by an earlier non-finite step " + std::to_string(Lr->h_counters[0]));
    step = Lr->h_counters[0];
  } else {
    step = Lr->host_step;  // the device advances exactly n_steps per enqueued update (or halts: reported by wait)
  }
  Lr->ctr_cached = false;
  const int sl = Lr->next_slot;
  Lr->next_slot ^= 1;
  spz_learner::HostSlot& hs = Lr->h_slots[sl];
  // the last pinned push's deferred pack: on this learner's stream right before its steps when it is
  // the ring's only reader (stream order already follows its own earlier reads), else on the ring
  // stream after every reader; then the records (and the fill they leave on the device) are in place
  bool wait_pack = false;
  {
    std::lock_guard<std::mutex> lk(Lr->ring->mu);
    if (Lr->ring->pend.active) {
      if (Lr->ring->readers.size() == 1) SPZ_CUDA_TRY(ring_enqueue_pack(Lr->ring, Lr->stream));
      else SPZ_CUDA_TRY(ring_flush_pending(Lr->ring));
    }
    // a pack on the ring's stream that no push synchronised: wait for it (a pack on this stream is ordered
    // already, a synchronous push returned after its records landed); otherwise no cross-stream wait between
    // consecutive updates
    static const bool always = std::getenv("SPZ_PACK_WAIT_ALWAYS") != nullptr;  // A/B diagnostics
    wait_pack = always || Lr->ring->pack_gen != Lr->seen_pack_gen;
    Lr->seen_pack_gen = Lr->ring->pack_gen;
  }
  if (wait_pack) SPZ_CUDA_TRY(cudaStreamWaitEvent(Lr->stream, Lr->ring->ev_pack, 0));
  static const bool pub_sep = std::getenv("SPZ_PUBLISH_SEPARATE") != nullptr;  // A/B: the separate launch
  bool published = false;
  for (int64_t k = 0; k < n_steps; ++k, ++step) {
    const int v = variant_of(Lr, step);
    if (Lr->cfg.use_graph) {
      const int ps = k == n_steps - 1 && !pub_sep ? sl : -1;  // the call's last step publishes the read-back
      SPZ_TRY(ensure_graph(Lr, v, ps));
      SPZ_CUDA_TRY(cudaGraphLaunch(ps < 0 ? Lr->exec[v] : Lr->exec_pub[v][ps], Lr->stream));
      published = ps >= 0;
    } else {
      SPZ_TRY(run_ops(Lr, v, Lr->stream));
    }
  }
  // read-back of the statistics, counters and flag: a one-warp kernel writing host-mapped memory (a
  // device-to-host copy costs more stream time between consecutive updates) -- the last step graph's final node,
  // else (no graph, no steps) launched here
  if (!published) {
    SPZ_CUDA_TRY(enqueue_publish(Lr, sl, Lr->stream));
    SPZ_CUDA_TRY(cudaGetLastError());
  }
  (void)hs;
  SPZ_CUDA_TRY(cudaEventRecord(Lr->ev_read, Lr->stream));  // pushes overwrite records only after these reads
  SPZ_CUDA_TRY(cudaEventRecord(Lr->ev_slot[sl], Lr->stream));
  Lr->inflight[Lr->n_inflight++] = sl;
  Lr->host_step = step;
  return SPZ_OK;
}

spz_status spz_update_wait(spz_learner* Lr, spz_stats* last) {
  if (!Lr) return fail(SPZ_EINVAL, "spz_update_wait: NULL learner");
  DeviceGuard dg(Lr->device);
  return update_finish(Lr, last);  // the oldest in flight (nothing in flight: the last completed update)
}

spz_status spz_update(spz_learner* Lr, int64_t batch, int64_t n_steps, spz_stats* last) {
  SPZ_TRY(spz_update_async(Lr, batch, n_steps));
  DeviceGuard dg(Lr->device);
  while (Lr->n_inflight > 1) SPZ_TRY(update_finish(Lr, nullptr));
  return update_finish(Lr, last);
}

static spz_status tensor_region(spz_learner* Lr, spz_tensor t, spz_slot s, float** base, int64_t* n) {
  int id;
  switch (t) {
    case SPZ_T_ACTOR: id = NET_ACTOR; break;
    case SPZ_T_Q1: id = NET_Q1; break;
    case SPZ_T_Q2: id = NET_Q2; break;
    case SPZ_T_Q1_TARG: id = NET_Q1T; break;
    case SPZ_T_Q2_TARG: id = NET_Q2T; break;
    case SPZ_T_ACTOR_TARG: id = NET_ACTORT; break;
    case SPZ_T_LOG_ALPHA: id = -1; break;
    case SPZ_T_V: id = NET_V; break;
    case SPZ_T_V_TARG: id = NET_VT; break;
    default: return fail(SPZ_EINVAL, "unknown tensor id");
  }
  if (id >= 0 && !Lr->has_net[id]) return fail(SPZ_EINVAL, "tensor not present for this algorithm");
  const bool trained = id == NET_ACTOR || id == NET_Q1 || id == NET_Q2 || id == NET_V || id == -1;
  if (s != SPZ_S_PARAM && !trained) return fail(SPZ_EINVAL, "target networks have no Adam state");
  float* arr = s == SPZ_S_PARAM ? Lr->P : s == SPZ_S_ADAM_M ? Lr->Mo : s == SPZ_S_ADAM_V ? Lr->Vo : nullptr;
  if (!arr) return fail(SPZ_EINVAL, "unknown slot");
  *base = arr + (id >= 0 ? Lr->pbase[id] : Lr->p_log_alpha);
  *n = id >= 0 ? Lr->net[id].np : 1;
  return SPZ_OK;
}

spz_status spz_get_params(spz_learner* Lr, spz_tensor t, spz_slot s, float* host_out, int64_t n, int64_t* n_required) {
  if (!Lr) return fail(SPZ_EINVAL, "spz_get_params: NULL learner");
  DeviceGuard dg(Lr->device);
  float* base;
  int64_t cnt;
  SPZ_TRY(tensor_region(Lr, t, s, &base, &cnt));
  if (n_required) *n_required = cnt;
  if (n < cnt || !host_out) return fail(SPZ_EINVAL, "spz_get_params: output holds " + std::to_string(n) + " < " + std::to_string(cnt) + " floats");
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  SPZ_CUDA_TRY(cudaMemcpyAsync(host_out, base, cnt * sizeof(float), cudaMemcpyDeviceToHost, Lr->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  return SPZ_OK;
}

spz_status spz_set_params(spz_learner* Lr, spz_tensor t, spz_slot s, const float* host_in, int64_t n) {
  if (!Lr || !host_in) return fail(SPZ_EINVAL, "spz_set_params: NULL argument");
  DeviceGuard dg(Lr->device);
  float* base;
  int64_t cnt;
  SPZ_TRY(tensor_region(Lr, t, s, &base, &cnt));
  if (n != cnt) return fail(SPZ_EINVAL, "spz_set_params: expected " + std::to_string(cnt) + " floats, got " + std::to_string(n));
  if (Lr->ddpg && (t == SPZ_T_Q2 || t == SPZ_T_Q2_TARG))
    return fail(SPZ_EINVAL, "spz_set_params: DDPG's second critic is tied to the first (set Q1 / Q1_TARG)");
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  SPZ_CUDA_TRY(cudaMemcpyAsync(base, host_in, cnt * sizeof(float), cudaMemcpyHostToDevice, Lr->stream));
  if (Lr->ddpg && (t == SPZ_T_Q1 || t == SPZ_T_Q1_TARG)) {  // keep the twin tied (parameters and Adam state)
    float* twin;
    int64_t tc;
    SPZ_TRY(tensor_region(Lr, t == SPZ_T_Q1 ? SPZ_T_Q2 : SPZ_T_Q2_TARG, s, &twin, &tc));
    SPZ_CUDA_TRY(cudaMemcpyAsync(twin, host_in, cnt * sizeof(float), cudaMemcpyHostToDevice, Lr->stream));
  }
  SPZ_TRY(refresh_shadows(Lr));
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  return SPZ_OK;
}

spz_status spz_tune_batch(spz_learner* Lr, const int64_t* ladder, int32_t n, int64_t warmup, int64_t steps,
                          double min_update_hz, double tol, int32_t restore, spz_tune_point* out, int32_t* n_out,
                          int64_t* best) {
  if (!Lr || !ladder || !out || !n_out || !best) return fail(SPZ_EINVAL, "spz_tune_batch: NULL argument");
  if (n < 1 || steps < 1 || warmup < 0 || !(tol >= 0.0)) return fail(SPZ_EINVAL, "spz_tune_batch: bad n / steps / warmup / tol");
  for (int i = 1; i < n; ++i)
    if (ladder[i] <= ladder[i - 1]) return fail(SPZ_EINVAL, "spz_tune_batch: ladder must be strictly ascending");
  DeviceGuard dg(Lr->device);
  SPZ_TRY(update_drain(Lr));
  *n_out = 0;
  *best = ladder[0];
  // snapshot of everything the probe steps change (the bf16 operand shadow is refreshed from P)
  void* snap = nullptr;
  const size_t pbytes = (size_t)Lr->P_total * sizeof(float);
  if (restore) {
    SPZ_CUDA_TRY(cudaMalloc(&snap, 3 * pbytes + 8 * sizeof(int64_t) + sizeof(int)));
    uint8_t* s8 = static_cast<uint8_t*>(snap);
    SPZ_CUDA_TRY(cudaMemcpyAsync(s8, Lr->P, pbytes, cudaMemcpyDeviceToDevice, Lr->stream));
    SPZ_CUDA_TRY(cudaMemcpyAsync(s8 + pbytes, Lr->Mo, pbytes, cudaMemcpyDeviceToDevice, Lr->stream));
    SPZ_CUDA_TRY(cudaMemcpyAsync(s8 + 2 * pbytes, Lr->Vo, pbytes, cudaMemcpyDeviceToDevice, Lr->stream));
    SPZ_CUDA_TRY(cudaMemcpyAsync(s8 + 3 * pbytes, Lr->counters, 8 * sizeof(int64_t), cudaMemcpyDeviceToDevice, Lr->stream));
    SPZ_CUDA_TRY(cudaMemcpyAsync(s8 + 3 * pbytes + 8 * sizeof(int64_t), Lr->d_flag, sizeof(int), cudaMemcpyDeviceToDevice, Lr->stream));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  spz_status st = SPZ_OK;
  double best_fps = -1.0, peak_fps = 0.0;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) st = fail(SPZ_ECUDA, "spz_tune_batch: events");
  for (int i = 0; i < n && st == SPZ_OK; ++i) {
    const int64_t B = ladder[i];
    // at least one untimed step: the plan and CUDA graph of this B are built outside the timed region
    if ((st = spz_update(Lr, B, std::max<int64_t>(warmup, 1), nullptr)) != SPZ_OK) break;
    if ((st = prepare(Lr, B)) != SPZ_OK) break;  // plan + graph before the timed region
    if (cudaEventRecord(e0, Lr->stream) != cudaSuccess) { st = fail(SPZ_ECUDA, "spz_tune_batch: event record"); break; }
    if ((st = spz_update_async(Lr, B, steps)) != SPZ_OK) break;
    if (cudaEventRecord(e1, Lr->stream) != cudaSuccess) { st = fail(SPZ_ECUDA, "spz_tune_batch: event record"); break; }
    if ((st = update_finish(Lr, nullptr)) != SPZ_OK) break;
    float ms = 0.f;
    if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess || !(ms > 0.f)) {
      st = fail(SPZ_ECUDA, "spz_tune_batch: event timing failed");
      break;
    }
    spz_tune_point& pt = out[(*n_out)++];
    pt.batch = B;
    pt.ms_per_update = (double)ms / (double)steps;
    pt.updates_per_s = 1e3 / pt.ms_per_update;
    pt.frames_per_s = (double)B * pt.updates_per_s;
    const bool ok_hz = pt.updates_per_s >= min_update_hz;
    if (ok_hz && pt.frames_per_s > best_fps) {
      best_fps = pt.frames_per_s;
      *best = B;
    }
    peak_fps = std::max(peak_fps, pt.frames_per_s);
    if (!ok_hz || pt.frames_per_s < peak_fps * (1.0 - tol)) break;  // below the floor, or past the peak
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (restore) {
    cudaStreamSynchronize(Lr->stream);
    uint8_t* s8 = static_cast<uint8_t*>(snap);
    cudaMemcpyAsync(Lr->P, s8, pbytes, cudaMemcpyDeviceToDevice, Lr->stream);
    cudaMemcpyAsync(Lr->Mo, s8 + pbytes, pbytes, cudaMemcpyDeviceToDevice, Lr->stream);
    cudaMemcpyAsync(Lr->Vo, s8 + 2 * pbytes, pbytes, cudaMemcpyDeviceToDevice, Lr->stream);
    cudaMemcpyAsync(Lr->counters, s8 + 3 * pbytes, 8 * sizeof(int64_t), cudaMemcpyDeviceToDevice, Lr->stream);
    cudaMemcpyAsync(Lr->d_flag, s8 + 3 * pbytes + 8 * sizeof(int64_t), sizeof(int), cudaMemcpyDeviceToDevice, Lr->stream);
    spz_status rs = refresh_shadows(Lr);
    if (cudaStreamSynchronize(Lr->stream) != cudaSuccess && st == SPZ_OK) st = fail(SPZ_ECUDA, "spz_tune_batch: restore");
    cudaFree(snap);
    Lr->ctr_cached = false;
    if (st == SPZ_OK) st = rs;
  }
  return st;
}

spz_status spz_get_counters(spz_learner* Lr, int64_t* step, int64_t* t_critic, int64_t* t_actor, int64_t* t_alpha) {
  if (!Lr) return fail(SPZ_EINVAL, "spz_get_counters: NULL learner");
  DeviceGuard dg(Lr->device);
  SPZ_TRY(read_counters(Lr));
  if (step) *step = Lr->h_counters[0];
  if (t_critic) *t_critic = Lr->h_counters[1];
  if (t_actor) *t_actor = Lr->h_counters[2];
  if (t_alpha) *t_alpha = Lr->h_counters[3];
  return SPZ_OK;
}

spz_status spz_sync_actor(spz_learner* Lr, int32_t dst_device, void* dst, int64_t dst_bytes, uint64_t* version) {
  if (!Lr || !dst) return fail(SPZ_EINVAL, "spz_sync_actor: NULL argument");
  DeviceGuard dg(Lr->device);
  const int64_t nf = Lr->net[NET_ACTOR].np;
  if (dst_bytes < SPZ_SYNC_BYTES(nf))
    return fail(SPZ_EINVAL, "spz_sync_actor: destination smaller than SPZ_SYNC_BYTES(" + std::to_string(nf) + ") bytes");
  if (reinterpret_cast<uintptr_t>(dst) % 16) return fail(SPZ_EINVAL, "spz_sync_actor: destination not 16-byte aligned");
  if (dst_device != Lr->device) {
    int can = 0;
    SPZ_CUDA_TRY(cudaDeviceCanAccessPeer(&can, Lr->device, dst_device));
    if (can) {
      cudaError_t e = cudaDeviceEnablePeerAccess(dst_device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(SPZ_ECUDA, "cudaDeviceEnablePeerAccess failed");
      cudaGetLastError();
    }
  }
  if (!Lr->h_sync && cudaMallocHost(&Lr->h_sync, 8 * sizeof(uint64_t)) != cudaSuccess) {
    Lr->h_sync = nullptr;
    return fail(SPZ_ENOMEM, "spz_sync_actor: pinned header words");
  }
  // publication of version v into slot v & 1 (include/spz.h): seq odd, payload, seq even, header last --
  // each copy starts after the previous one completed (one stream), so the header never points at a slot
  // whose payload is incomplete, and a reader that overlaps the slot's rewrite sees its seq word change
  uint8_t* d8 = static_cast<uint8_t*>(dst);
  const uint64_t v = ++Lr->sync_version;
  const int slot = (int)(v & 1);
  uint64_t* w = Lr->h_sync;  // distinct host words: the copies read them when they execute
  w[0] = 2 * v - 1;
  w[1] = 2 * v;
  w[2] = v;
  w[3] = (uint64_t)nf;
  uint8_t* seq = d8 + 16 + 8 * slot;
  SPZ_CUDA_TRY(cudaMemcpyAsync(seq, &w[0], 8, cudaMemcpyHostToDevice, Lr->stream));
  SPZ_CUDA_TRY(cudaMemcpyPeerAsync(d8 + SPZ_SYNC_HEADER_BYTES + slot * SPZ_SYNC_SLOT_BYTES(nf), dst_device,
                                   Lr->P + Lr->pbase[NET_ACTOR], Lr->device, nf * sizeof(float), Lr->stream));
  SPZ_CUDA_TRY(cudaMemcpyAsync(seq, &w[1], 8, cudaMemcpyHostToDevice, Lr->stream));
  SPZ_CUDA_TRY(cudaMemcpyAsync(d8, &w[2], 16, cudaMemcpyHostToDevice, Lr->stream));
  SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  if (version) *version = v;
  return SPZ_OK;
}

spz_status spz_learner_profile(spz_learner* Lr, int64_t batch, int64_t n_steps, int32_t cap, const char** names, double* ms,
                               int32_t* count) {
  if (!Lr || n_steps < 1) return fail(SPZ_EINVAL, "spz_learner_profile: bad argument");
  DeviceGuard dg(Lr->device);
  SPZ_TRY(update_drain(Lr));
  SPZ_TRY(prepare(Lr, batch));
  SPZ_TRY(read_counters(Lr));
  int64_t step = Lr->h_counters[0];
  Lr->ctr_cached = false;
  {
    std::lock_guard<std::mutex> lk(Lr->ring->mu);
    SPZ_CUDA_TRY(ring_flush_pending(Lr->ring));
  }
  SPZ_CUDA_TRY(cudaStreamWaitEvent(Lr->stream, Lr->ring->ev_pack, 0));
  // No host gaps inside the timed ops: each step is enqueued behind a gate kernel that spins on a
  // host-mapped word, and the word is released only once the whole step (ops + events) is queued, so
  // every op starts right after the event that follows its predecessor (the events serialise the ops:
  // no PDL overlap, like ncu's per-launch times).
  if (!Lr->h_gate) {
    if (cudaHostAlloc((void**)&Lr->h_gate, sizeof(int), cudaHostAllocMapped) != cudaSuccess) {
      Lr->h_gate = nullptr;
      return fail(SPZ_ENOMEM, "spz_learner_profile: mapped gate word");
    }
    SPZ_CUDA_TRY(cudaHostGetDevicePointer((void**)&Lr->d_gate, Lr->h_gate, 0));
  }
  *const_cast<volatile int*>(Lr->h_gate) = 0;
  struct GateOpen {  // the gate always opens on exit (an error mid-enqueue must not leave the GPU spinning)
    volatile int* g;
    ~GateOpen() { *g = 1 << 30; }
  } gate_open{Lr->h_gate};
  std::vector<const char*> cls;
  std::vector<double> tot;
  std::vector<std::vector<cudaEvent_t>> ev(n_steps);
  std::vector<int> vars(n_steps);
  auto destroy = [&]() {
    for (auto& v : ev)
      for (auto e : v) cudaEventDestroy(e);
  };
  for (int64_t k = 0; k < n_steps; ++k) {
    const int v = variant_of(Lr, step + k);
    vars[k] = v;
    auto& ops = Lr->ops[v];
    ev[k].resize(ops.size() + 1);
    for (auto& e : ev[k])
      if (cudaEventCreate(&e) != cudaSuccess) {
        destroy();
        return fail(SPZ_ECUDA, "spz_learner_profile: event creation failed");
      }
    gate_kernel<<<1, 32, 0, Lr->stream>>>(Lr->d_gate, (int)(k + 1));
    SPZ_CUDA_TRY(cudaEventRecord(ev[k][0], Lr->stream));
    for (size_t i = 0; i < ops.size(); ++i) {
      cudaError_t e = ops[i].fn(Lr->stream);
      if (e != cudaSuccess) {
        destroy();
        return fail(SPZ_ECUDA, std::string("kernel ") + ops[i].cls + ": " + cudaGetErrorString(e));
      }
      SPZ_CUDA_TRY(cudaEventRecord(ev[k][i + 1], Lr->stream));
    }
    *const_cast<volatile int*>(Lr->h_gate) = (int)(k + 1);  // step k fully queued: release it
  }
  {
    cudaError_t e = cudaStreamSynchronize(Lr->stream);
    if (e != cudaSuccess) {
      destroy();
      return fail(SPZ_ECUDA, std::string("spz_learner_profile: ") + cudaGetErrorString(e));
    }
  }
  for (int64_t k = 0; k < n_steps; ++k) {
    auto& ops = Lr->ops[vars[k]];
    for (size_t i = 0; i < ops.size(); ++i) {
      float t = 0;
      SPZ_CUDA_TRY(cudaEventElapsedTime(&t, ev[k][i], ev[k][i + 1]));
      size_t c = 0;
      for (; c < cls.size(); ++c)
        if (std::strcmp(cls[c], ops[i].cls) == 0) break;
      if (c == cls.size()) {
        cls.push_back(ops[i].cls);
        tot.push_back(0.0);
      }
      tot[c] += t;
    }
  }
  SPZ_CUDA_TRY(cudaEventRecord(Lr->ev_read, Lr->stream));
  destroy();
  const int nc = (int)std::min<size_t>(cls.size(), (size_t)std::max(cap, 0));
  for (int i = 0; i < nc; ++i) {
    if (names) names[i] = cls[i];
    if (ms) ms[i] = tot[i] / (double)n_steps;
  }
  if (count) *count = (int)cls.size();
  SPZ_TRY(read_counters(Lr));
  return SPZ_OK;
}

spz_status spz_learner_launches_per_step(spz_learner* Lr, int64_t batch, int32_t* launches) {
  if (!Lr || !launches) return fail(SPZ_EINVAL, "spz_learner_launches_per_step: NULL argument");
  DeviceGuard dg(Lr->device);
  SPZ_TRY(prepare(Lr, batch));
  int n = 0;
  for (auto& op : Lr->ops[0]) n += op.launches;
  *launches = n;
  return SPZ_OK;
}

spz_status spz_split_exchange(spz_learner* critic_side, spz_learner* actor_side) {
  if (!critic_side || !actor_side) return fail(SPZ_EINVAL, "spz_split_exchange: NULL learner");
  if (critic_side->cfg.role != SPZ_ROLE_CRITIC || actor_side->cfg.role != SPZ_ROLE_ACTOR)
    return fail(SPZ_EINVAL, "spz_split_exchange: need a critic-role and an actor-role learner");
  if (critic_side->bf16 != actor_side->bf16 || critic_side->td3 != actor_side->td3 || critic_side->h != actor_side->h ||
      critic_side->L != actor_side->L || critic_side->o != actor_side->o || critic_side->m != actor_side->m)
    return fail(SPZ_EINVAL, "spz_split_exchange: learners of different configurations");
  spz_learner* C = critic_side;
  spz_learner* A = actor_side;
  {
    DeviceGuard g1(A->device);
    SPZ_CUDA_TRY(cudaStreamSynchronize(A->stream));
  }
  DeviceGuard dg(C->device);
  SPZ_CUDA_TRY(cudaStreamSynchronize(C->stream));
  auto cp = [&](spz_learner* dst, spz_learner* src, int64_t off, int64_t n) {
    return cudaMemcpyPeerAsync(dst->P + off, dst->device, src->P + off, src->device, n * sizeof(float), C->stream);
  };
  SPZ_CUDA_TRY(cp(C, A, A->pbase[NET_ACTOR], A->net[NET_ACTOR].np));
  SPZ_CUDA_TRY(cp(C, A, A->p_log_alpha, 1));
  if (A->td3) SPZ_CUDA_TRY(cp(C, A, A->pbase[NET_ACTORT], A->net[NET_ACTORT].np));
  SPZ_CUDA_TRY(cp(A, C, C->pbase[NET_Q1], C->pbase[NET_Q2] + C->net[NET_Q2].np - C->pbase[NET_Q1]));
  SPZ_CUDA_TRY(cudaStreamSynchronize(C->stream));
  for (spz_learner* Lr : {C, A}) {
    DeviceGuard g2(Lr->device);
    if (Lr->bf16)
      launch_pdl(shadow_refresh_kernel<__nv_bfloat16>, dim3(64, Lr->n_shadow_recv), dim3(256), 0, Lr->stream,
                 (const ShadowEntry*)Lr->d_shadow_recv, Lr->n_shadow_recv, (const float*)Lr->P, static_cast<__nv_bfloat16*>(Lr->S));
    else
      launch_pdl(shadow_refresh_kernel<float>, dim3(64, Lr->n_shadow_recv), dim3(256), 0, Lr->stream,
                 (const ShadowEntry*)Lr->d_shadow_recv, Lr->n_shadow_recv, (const float*)Lr->P, static_cast<float*>(Lr->S));
    SPZ_CUDA_TRY(cudaGetLastError());
    SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
  }
  return SPZ_OK;
}

spz_status spz_learner_debug_buffer(spz_learner* Lr, const char* name, void* host_out, int64_t bytes,
                                    int64_t* bytes_required, int32_t* elem_size) {
  if (!Lr || !name) return fail(SPZ_EINVAL, "spz_learner_debug_buffer: NULL argument");
  DeviceGuard dg(Lr->device);
  for (auto& b : Lr->debug) {
    if (b.name != name) continue;
    if (bytes_required) *bytes_required = (int64_t)b.bytes;
    if (elem_size) *elem_size = b.esz;
    if (!host_out) return SPZ_OK;
    if (bytes < (int64_t)b.bytes) return fail(SPZ_EINVAL, "spz_learner_debug_buffer: output too small");
    SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
    SPZ_CUDA_TRY(cudaMemcpyAsync(host_out, b.ptr, b.bytes, cudaMemcpyDeviceToHost, Lr->stream));
    SPZ_CUDA_TRY(cudaStreamSynchronize(Lr->stream));
    return SPZ_OK;
  }
  return fail(SPZ_EINVAL, std::string("spz_learner_debug_buffer: unknown buffer ") + name);
}

void spz_learner_destroy(spz_learner* Lr) { delete Lr; }

}  // extern "C"
