"""ctypes binding of libspz.so (include/spz.h) -- argument marshalling only.

Every function below forwards to the C entry point of the same name; no step of
the update runs in Python.  There is no CPU fallback: if libspz.so is missing or
cannot find an sm_100 device the calls fail loudly (``SpzError``).

Convenience classes ``Replay`` and ``Learner`` wrap the handles (RAII + numpy /
torch marshalling); they add no computation.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPZ_LIB_PATH") or os.path.join(_HERE, "libspz.so")  # override: A/B experiments only

SPZ_OK, SPZ_EINVAL, SPZ_ENODATA, SPZ_ENONFINITE, SPZ_ECUDA, SPZ_ENCCL, SPZ_ENOMEM, SPZ_ESTATE, SPZ_ETIMEOUT, SPZ_EUNSUPPORTED = (
    0, -1, -2, -3, -4, -5, -6, -7, -8, -9)
STATUS_NAMES = {0: "SPZ_OK", -1: "SPZ_EINVAL", -2: "SPZ_ENODATA", -3: "SPZ_ENONFINITE", -4: "SPZ_ECUDA",
                -5: "SPZ_ENCCL", -6: "SPZ_ENOMEM", -7: "SPZ_ESTATE", -8: "SPZ_ETIMEOUT", -9: "SPZ_EUNSUPPORTED"}
SPZ_SAC, SPZ_TD3, SPZ_DDPG, SPZ_SACV1 = 0, 1, 2, 3
ALGOS = {"sac": SPZ_SAC, "td3": SPZ_TD3, "ddpg": SPZ_DDPG, "sacv1": SPZ_SACV1}
SPZ_FP32, SPZ_BF16 = 0, 1
SPZ_ROLE_ALL, SPZ_ROLE_CRITIC, SPZ_ROLE_ACTOR = 0, 1, 2
SPZ_T_ACTOR, SPZ_T_Q1, SPZ_T_Q2, SPZ_T_Q1_TARG, SPZ_T_Q2_TARG, SPZ_T_ACTOR_TARG, SPZ_T_LOG_ALPHA, SPZ_T_V, SPZ_T_V_TARG = range(9)
SPZ_S_PARAM, SPZ_S_ADAM_M, SPZ_S_ADAM_V = 0, 1, 2

# Every symbol include/spz.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "spz_last_error", "spz_version", "spz_replay_create", "spz_replay_push", "spz_replay_push_async", "spz_replay_sync",
    "spz_replay_sample", "spz_replay_info",
    "spz_replay_records", "spz_replay_destroy", "spz_config_default", "spz_nccl_unique_id", "spz_learner_create",
    "spz_update", "spz_update_async", "spz_update_wait", "spz_learner_set_stream", "spz_get_params", "spz_set_params", "spz_get_counters", "spz_sync_actor",
    "spz_learner_profile", "spz_learner_launches_per_step", "spz_learner_debug_buffer", "spz_learner_destroy",
    "spz_diag_gemm_bf16", "spz_diag_gemm_f32", "spz_split_exchange", "spz_diag_tc_trace",
    "spz_policy_create", "spz_policy_load", "spz_policy_act", "spz_policy_get_params", "spz_policy_destroy", "spz_tune_batch",
    "spz_replay_track", "spz_replay_loss", "spz_plan_rank",
]


class SpzError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class spz_policy_desc(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int), ("precision", ctypes.c_int),
                ("obs_dim", ctypes.c_int32), ("act_dim", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("n_hidden", ctypes.c_int32), ("max_batch", ctypes.c_int64), ("device", ctypes.c_int32),
                ("log_std_min", ctypes.c_double), ("log_std_max", ctypes.c_double), ("expl_noise", ctypes.c_double)]


class spz_tune_point(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("updates_per_s", ctypes.c_double), ("frames_per_s", ctypes.c_double),
                ("ms_per_update", ctypes.c_double)]


class spz_replay_desc(ctypes.Structure):
    _fields_ = [("obs_dim", ctypes.c_int32), ("act_dim", ctypes.c_int32), ("capacity", ctypes.c_int64),
                ("device", ctypes.c_int32)]


class spz_config(ctypes.Structure):
    _fields_ = [
        ("algo", ctypes.c_int), ("precision", ctypes.c_int),
        ("obs_dim", ctypes.c_int32), ("act_dim", ctypes.c_int32),
        ("hidden", ctypes.c_int32), ("n_hidden", ctypes.c_int32),
        ("max_batch", ctypes.c_int64),
        ("gamma", ctypes.c_double), ("tau", ctypes.c_double),
        ("lr_actor", ctypes.c_double), ("lr_critic", ctypes.c_double), ("lr_alpha", ctypes.c_double),
        ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("adam_eps", ctypes.c_double),
        ("alpha_auto", ctypes.c_int32),
        ("alpha_init", ctypes.c_double), ("target_entropy", ctypes.c_double),
        ("log_std_min", ctypes.c_double), ("log_std_max", ctypes.c_double),
        ("td3_noise", ctypes.c_double), ("td3_noise_clip", ctypes.c_double), ("td3_policy_delay", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("init_seed", ctypes.c_uint64),
        ("device", ctypes.c_int32), ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
        ("n_critic_ranks", ctypes.c_int32), ("n_actor_ranks", ctypes.c_int32),
        ("role", ctypes.c_int),
        ("nccl_unique_id", ctypes.c_void_p),
        ("use_graph", ctypes.c_int32),
        ("comm_mode", ctypes.c_int32),
    ]


class spz_plan(ctypes.Structure):
    _fields_ = [("role", ctypes.c_int32), ("group_size", ctypes.c_int32), ("group_rank", ctypes.c_int32),
                ("group_color", ctypes.c_int32), ("row0", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("actor_root", ctypes.c_int32), ("critic_root", ctypes.c_int32), ("allreduce", ctypes.c_int32),
                ("pad_", ctypes.c_int32)]


class spz_stats(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int64), ("critic_loss", ctypes.c_double), ("actor_loss", ctypes.c_double),
                ("alpha", ctypes.c_double), ("alpha_loss", ctypes.c_double), ("q1_mean", ctypes.c_double),
                ("q2_mean", ctypes.c_double), ("logp_mean", ctypes.c_double),
                ("value_loss", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libspz.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SpzError(SPZ_ECUDA, f"{LIB_PATH} is missing: run `python -m paper_2312_06126_b200.build` "
                                      "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, U64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        sig = {
            "spz_last_error": (ctypes.c_char_p, []),
            "spz_version": (ctypes.c_char_p, []),
            "spz_replay_create": (ctypes.c_int, [ctypes.POINTER(spz_replay_desc), ctypes.POINTER(P)]),
            "spz_replay_push": (ctypes.c_int, [P, I64, P, P, P, P, P, I32, ctypes.POINTER(I64)]),
            "spz_replay_push_async": (ctypes.c_int, [P, I64, P, P, P, P, P, I32, ctypes.POINTER(I64)]),
            "spz_replay_sync": (ctypes.c_int, [P]),
            "spz_replay_sample": (ctypes.c_int, [P, I64, U64, U64, P, P, P, P, P, P]),
            "spz_replay_info": (ctypes.c_int, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
            "spz_replay_records": (ctypes.c_int, [P, ctypes.POINTER(P), ctypes.POINTER(I32)]),
            "spz_replay_destroy": (None, [P]),
            "spz_config_default": (ctypes.c_int, [ctypes.c_int, I32, I32, ctypes.POINTER(spz_config)]),
            "spz_nccl_unique_id": (ctypes.c_int, [P]),
            "spz_learner_create": (ctypes.c_int, [ctypes.POINTER(spz_config), P, ctypes.POINTER(P)]),
            "spz_update": (ctypes.c_int, [P, I64, I64, ctypes.POINTER(spz_stats)]),
            "spz_update_async": (ctypes.c_int, [P, I64, I64]),
            "spz_update_wait": (ctypes.c_int, [P, ctypes.POINTER(spz_stats)]),
            "spz_learner_set_stream": (ctypes.c_int, [P, P]),
            "spz_get_params": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, I64, ctypes.POINTER(I64)]),
            "spz_set_params": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, I64]),
            "spz_get_counters": (ctypes.c_int, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64),
                                                ctypes.POINTER(I64)]),
            "spz_sync_actor": (ctypes.c_int, [P, I32, P, I64, ctypes.POINTER(U64)]),
            "spz_learner_profile": (ctypes.c_int, [P, I64, I64, I32, ctypes.POINTER(ctypes.c_char_p),
                                                   ctypes.POINTER(D), ctypes.POINTER(I32)]),
            "spz_learner_launches_per_step": (ctypes.c_int, [P, I64, ctypes.POINTER(I32)]),
            "spz_learner_debug_buffer": (ctypes.c_int, [P, ctypes.c_char_p, P, I64, ctypes.POINTER(I64),
                                                        ctypes.POINTER(I32)]),
            "spz_learner_destroy": (None, [P]),
            "spz_split_exchange": (ctypes.c_int, [P, P]),
            "spz_diag_tc_trace": (ctypes.c_int, [I32, I32, P, I32]),
            "spz_diag_gemm_bf16": (ctypes.c_int, [I32, I32, I64, I64, I64, P, I64, I32, P, I64, I32, P, I64, I32, I64]),
            "spz_diag_gemm_f32": (ctypes.c_int, [I32, I32, I64, I64, I64, P, I64, I32, P, I64, I32, P, I64, I32, I64]),
            "spz_policy_create": (ctypes.c_int, [ctypes.POINTER(spz_policy_desc), ctypes.POINTER(P)]),
            "spz_policy_load": (ctypes.c_int, [P, P, I64, ctypes.POINTER(U64)]),
            "spz_policy_act": (ctypes.c_int, [P, I64, P, I32, U64, U64, P]),
            "spz_policy_get_params": (ctypes.c_int, [P, P, I64]),
            "spz_policy_destroy": (None, [P]),
            "spz_replay_track": (ctypes.c_int, [P, I32]),
            "spz_plan_rank": (ctypes.c_int, [ctypes.POINTER(spz_config), I64, ctypes.POINTER(spz_plan)]),
            "spz_replay_loss": (ctypes.c_int, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
            "spz_tune_batch": (ctypes.c_int, [P, ctypes.POINTER(I64), I32, I64, I64, D, D, I32,
                                              ctypes.POINTER(spz_tune_point), ctypes.POINTER(I32), ctypes.POINTER(I64)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status):
    if status != SPZ_OK:
        raise SpzError(status, lib().spz_last_error().decode())
    return status


# ----------------------------------------------------------------------------- same-name functions

def spz_version():
    return lib().spz_version().decode()


def spz_last_error():
    return lib().spz_last_error().decode()


def spz_replay_create(obs_dim, act_dim, capacity, device=0):
    h = ctypes.c_void_p()
    _check(lib().spz_replay_create(ctypes.byref(spz_replay_desc(obs_dim, act_dim, capacity, device)), ctypes.byref(h)))
    return h


def _ptr(x):
    """Host numpy array -> pointer (must be float32 C-contiguous); torch tensor -> data_ptr."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    assert x.flags["C_CONTIGUOUS"]
    return x.ctypes.data_as(ctypes.c_void_p)


def spz_replay_push(ring, obs, act, rew, next_obs, done, src_on_device=False, wait=True):
    """Host path: float32 numpy arrays; device path: torch CUDA float32 tensors.  wait=False:
    spz_replay_push_async (page-locked host arrays stay untouched until the next push or spz_replay_sync)."""
    n = len(rew)
    if not src_on_device:
        obs, act, rew, next_obs, done = [np.ascontiguousarray(a, dtype=np.float32) for a in (obs, act, rew, next_obs, done)]
    first = ctypes.c_int64()
    fn = lib().spz_replay_push if wait else lib().spz_replay_push_async
    _check(fn(ring, n, _ptr(obs), _ptr(act), _ptr(rew), _ptr(next_obs), _ptr(done), 1 if src_on_device else 0,
              ctypes.byref(first)))
    return first.value


def spz_replay_sample(ring, batch, seed, step, idx=None, obs=None, act=None, rew=None, next_obs=None, done=None):
    """Outputs are device tensors (torch) or None."""
    _check(lib().spz_replay_sample(ring, batch, seed, step, _ptr(idx), _ptr(obs), _ptr(act), _ptr(rew),
                                   _ptr(next_obs), _ptr(done)))


def spz_replay_info(ring):
    c, f, cap = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().spz_replay_info(ring, ctypes.byref(c), ctypes.byref(f), ctypes.byref(cap)))
    return c.value, f.value, cap.value


def spz_replay_destroy(ring):
    lib().spz_replay_destroy(ring)


def spz_nccl_unique_id():
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().spz_nccl_unique_id(buf))
    return bytes(buf)


def spz_plan_rank(batch, world_size, rank, role=SPZ_ROLE_ALL, n_critic_ranks=0, comm_mode=0, algo=SPZ_SAC, obs_dim=1,
                  act_dim=1):
    """The host-side multi-GPU plan of one rank (include/spz.h spz_plan_rank): a dict of its fields."""
    cfg = spz_config_default(algo, obs_dim, act_dim)
    cfg.world_size, cfg.rank, cfg.role, cfg.n_critic_ranks, cfg.comm_mode = world_size, rank, role, n_critic_ranks, comm_mode
    p = spz_plan()
    _check(lib().spz_plan_rank(ctypes.byref(cfg), batch, ctypes.byref(p)))
    return {f: getattr(p, f) for f, _ in spz_plan._fields_ if f != "pad_"}


def spz_config_default(algo, obs_dim, act_dim):
    c = spz_config()
    _check(lib().spz_config_default(algo, obs_dim, act_dim, ctypes.byref(c)))
    return c


def spz_learner_create(cfg, ring):
    h = ctypes.c_void_p()
    _check(lib().spz_learner_create(ctypes.byref(cfg), ring, ctypes.byref(h)))
    return h


def spz_update(learner, batch, n_steps):
    s = spz_stats()
    _check(lib().spz_update(learner, batch, n_steps, ctypes.byref(s)))
    return s.as_dict()


def spz_update_async(learner, batch, n_steps):
    _check(lib().spz_update_async(learner, batch, n_steps))


def spz_update_wait(learner):
    s = spz_stats()
    _check(lib().spz_update_wait(learner, ctypes.byref(s)))
    return s.as_dict()


def spz_learner_set_stream(learner, stream_handle):
    _check(lib().spz_learner_set_stream(learner, ctypes.c_void_p(stream_handle) if stream_handle else None))


def spz_get_params(learner, tensor, slot=SPZ_S_PARAM):
    need = ctypes.c_int64()
    lib().spz_get_params(learner, tensor, slot, None, 0, ctypes.byref(need))
    if need.value <= 0:
        _check(lib().spz_get_params(learner, tensor, slot, None, 0, ctypes.byref(need)))
    out = np.empty(need.value, np.float32)
    _check(lib().spz_get_params(learner, tensor, slot, _ptr(out), out.size, ctypes.byref(need)))
    return out


def spz_set_params(learner, tensor, values, slot=SPZ_S_PARAM):
    v = np.ascontiguousarray(values, dtype=np.float32)
    _check(lib().spz_set_params(learner, tensor, slot, _ptr(v), v.size))


def spz_get_counters(learner):
    a = [ctypes.c_int64() for _ in range(4)]
    _check(lib().spz_get_counters(learner, *[ctypes.byref(x) for x in a]))
    return dict(step=a[0].value, t_critic=a[1].value, t_actor=a[2].value, t_alpha=a[3].value)


SYNC_HEADER_BYTES = 64  # include/spz.h SPZ_SYNC_HEADER_BYTES


def sync_slot_bytes(n_floats):
    """include/spz.h SPZ_SYNC_SLOT_BYTES."""
    return (n_floats * 4 + 63) // 64 * 64


def sync_bytes(n_floats):
    """include/spz.h SPZ_SYNC_BYTES: size of an actor publication buffer (header + two slots)."""
    return SYNC_HEADER_BYTES + 2 * sync_slot_bytes(n_floats)


def spz_sync_actor(learner, dst_device, dst_ptr, dst_bytes):
    v = ctypes.c_uint64()
    _check(lib().spz_sync_actor(learner, dst_device, ctypes.c_void_p(dst_ptr), dst_bytes, ctypes.byref(v)))
    return v.value


def spz_learner_profile(learner, batch, n_steps, cap=64):
    names = (ctypes.c_char_p * cap)()
    ms = (ctypes.c_double * cap)()
    cnt = ctypes.c_int32()
    _check(lib().spz_learner_profile(learner, batch, n_steps, cap, names, ms, ctypes.byref(cnt)))
    return {names[i].decode(): ms[i] for i in range(min(cnt.value, cap))}


def spz_learner_launches_per_step(learner, batch):
    n = ctypes.c_int32()
    _check(lib().spz_learner_launches_per_step(learner, batch, ctypes.byref(n)))
    return n.value


def spz_learner_debug_buffer(learner, name):
    """Internal buffer as a numpy array (bf16 buffers widened to float32; "idx" as int32)."""
    need, es = ctypes.c_int64(), ctypes.c_int32()
    _check(lib().spz_learner_debug_buffer(learner, name.encode(), None, 0, ctypes.byref(need), ctypes.byref(es)))
    raw = np.empty(need.value, np.uint8)
    _check(lib().spz_learner_debug_buffer(learner, name.encode(), _ptr(raw), raw.size, ctypes.byref(need),
                                          ctypes.byref(es)))
    if name == "idx":
        return raw.view(np.int32)
    if name.startswith("mask"):
        return raw.view(np.uint32)
    if es.value == 2:
        return (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    if es.value == 8:
        return raw.view(np.float64)
    return raw.view(np.float32)


def spz_learner_destroy(learner):
    lib().spz_learner_destroy(learner)


def spz_diag_tc_trace(on, read=False, device=0):
    """Enable/disable GEMM tile timestamps; with read=True return them as uint64 [160, 8, 4]."""
    out = np.zeros(160 * 8 * 4, np.uint64) if read else None
    _check(lib().spz_diag_tc_trace(device, int(on), _ptr(out) if read else None, out.size if read else 0))
    return out.reshape(160, 8, 4) if read else None


def spz_diag_tc_trace_tiles(device=0):
    """Stamps [160, 8, 4], the linear tile index of each traced tile [160, 8] (-1: none) and per CTA [160, 2]
    (kernel entry, producer past the grid-dependency wait; 0: none) of the last traced GEMM launch."""
    n = 160 * 8 * 4
    out = np.zeros(n + 160 * 8 + 160 * 2, np.uint64)
    _check(lib().spz_diag_tc_trace(device, 0, _ptr(out), out.size))
    return (out[:n].reshape(160, 8, 4), out[n:n + 1280].view(np.int64).reshape(160, 8),
            out[n + 1280:].reshape(160, 2))


def spz_diag_mlp_trace(on, read=False, device=0):
    """Fused-MLP timestamps (spz_diag_tc_trace modes >= 100); with read=True: uint64 [160, 4, 3, 6]
    = (CTA, unit, layer, event: MMA start, MMA issued, epilogue sees accumulator, epilogue done,
    first / last weight slab present)."""
    out = np.zeros(160 * 4 * 3 * 6, np.uint64) if read else None
    _check(lib().spz_diag_tc_trace(device, 100 + int(on), _ptr(out) if read else None, out.size if read else 0))
    return out.reshape(160, 4, 3, 6) if read else None


def spz_split_exchange(critic_learner, actor_learner):
    _check(lib().spz_split_exchange(critic_learner, actor_learner))


def spz_diag_gemm_f32(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, ldc, tensor_cores=True, splits=1, k_per_split=0,
                      device=0):
    """A, B, C: fp32 torch CUDA tensors (see include/spz.h); tensor_cores=True runs the 3xTF32 kernel."""
    _check(lib().spz_diag_gemm_f32(device, 1 if tensor_cores else 0, M, N, K, _ptr(A), lda, a_mn, _ptr(B), ldb, b_mn,
                                   _ptr(C), ldc, splits, k_per_split))


def spz_diag_gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, ldc, tensor_cores=True, splits=1, k_per_split=0,
                       device=0):
    """A, B: bf16 torch CUDA tensors; C: fp32 torch CUDA tensor (see include/spz.h)."""
    _check(lib().spz_diag_gemm_bf16(device, 1 if tensor_cores else 0, M, N, K, _ptr(A), lda, a_mn, _ptr(B), ldb, b_mn,
                                    _ptr(C), ldc, splits, k_per_split))


# ----------------------------------------------------------------------------- RAII wrappers

class Replay:
    def __init__(self, obs_dim, act_dim, capacity, device=0):
        self.obs_dim, self.act_dim, self.capacity, self.device = obs_dim, act_dim, capacity, device
        self.h = spz_replay_create(obs_dim, act_dim, capacity, device)

    def push(self, obs, act, rew, next_obs, done, src_on_device=False, wait=True):
        return spz_replay_push(self.h, obs, act, rew, next_obs, done, src_on_device, wait)

    def sync(self):
        """Wait until the host buffers of the last push(..., wait=False) have been read."""
        _check(lib().spz_replay_sync(self.h))

    def info(self):
        return spz_replay_info(self.h)

    def track(self, on=True):
        """Start (or stop) experience-transmission-loss accounting (include/spz.h)."""
        _check(lib().spz_replay_track(self.h, 1 if on else 0))

    def loss(self):
        """(pushed, lost, resident_unsampled) since track(); lost / pushed is the transmission loss."""
        p, l, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().spz_replay_loss(self.h, ctypes.byref(p), ctypes.byref(l), ctypes.byref(r)))
        return p.value, l.value, r.value

    def close(self):
        if self.h:
            spz_replay_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PARAM_TENSORS = {"actor": SPZ_T_ACTOR, "q1": SPZ_T_Q1, "q2": SPZ_T_Q2, "q1_targ": SPZ_T_Q1_TARG,
                 "q2_targ": SPZ_T_Q2_TARG, "actor_targ": SPZ_T_ACTOR_TARG, "log_alpha": SPZ_T_LOG_ALPHA,
                 "v": SPZ_T_V, "v_targ": SPZ_T_V_TARG}


class Learner:
    def __init__(self, ring: Replay, algo="sac", precision="bf16", hidden=256, n_hidden=2, max_batch=8192,
                 device=0, use_graph=True, **overrides):
        cfg = spz_config_default(ALGOS[algo], ring.obs_dim, ring.act_dim)
        cfg.precision = SPZ_BF16 if precision == "bf16" else SPZ_FP32
        cfg.hidden, cfg.n_hidden, cfg.max_batch, cfg.device = hidden, n_hidden, max_batch, device
        cfg.use_graph = 1 if use_graph else 0
        self._uid = None
        if "nccl_unique_id" in overrides:
            uid = overrides.pop("nccl_unique_id")
            self._uid = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
            cfg.nccl_unique_id = ctypes.cast(self._uid, ctypes.c_void_p)
        for k, v in overrides.items():
            setattr(cfg, k, v)
        self.cfg = cfg
        self.ring = ring
        self.h = spz_learner_create(cfg, ring.h)

    def update(self, batch, n_steps=1):
        return spz_update(self.h, batch, n_steps)

    def update_async(self, batch, n_steps=1):
        spz_update_async(self.h, batch, n_steps)

    def wait(self):
        return spz_update_wait(self.h)

    def get(self, name, slot=SPZ_S_PARAM):
        return spz_get_params(self.h, PARAM_TENSORS[name], slot)

    def set(self, name, values, slot=SPZ_S_PARAM):
        spz_set_params(self.h, PARAM_TENSORS[name], values, slot)

    def counters(self):
        return spz_get_counters(self.h)

    def set_stream(self, handle):
        spz_learner_set_stream(self.h, handle)

    def profile(self, batch, n_steps):
        return spz_learner_profile(self.h, batch, n_steps)

    def debug(self, name):
        return spz_learner_debug_buffer(self.h, name)

    def launches_per_step(self, batch):
        return spz_learner_launches_per_step(self.h, batch)

    def tune_batch(self, ladder, warmup=3, steps=20, min_update_hz=0.0, tol=0.05, restore=True):
        return spz_tune_batch(self.h, ladder, warmup, steps, min_update_hz, tol, restore)

    def close(self):
        if self.h:
            spz_learner_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- sampler-side policy (f1)

def spz_policy_create(desc):
    h = ctypes.c_void_p()
    _check(lib().spz_policy_create(ctypes.byref(desc), ctypes.byref(h)))
    return h


def spz_policy_load(policy, payload_ptr, nbytes):
    v = ctypes.c_uint64()
    _check(lib().spz_policy_load(policy, ctypes.c_void_p(payload_ptr), nbytes, ctypes.byref(v)))
    return v.value


def spz_policy_act(policy, n, obs, deterministic, seed, step, act):
    """obs [n x o] / act [n x m]: float32 numpy arrays (host) or torch CUDA tensors."""
    _check(lib().spz_policy_act(policy, n, _ptr(obs), 1 if deterministic else 0, seed, step, _ptr(act)))


def spz_policy_get_params(policy, n):
    out = np.empty(n, dtype=np.float32)
    _check(lib().spz_policy_get_params(policy, out.ctypes.data_as(ctypes.c_void_p), n))
    return out


def spz_policy_destroy(policy):
    lib().spz_policy_destroy(policy)


class Policy:
    """Sampler-side actor inference (include/spz.h), fed by Learner.sync_actor payloads."""

    def __init__(self, obs_dim, act_dim, algo="sac", precision="bf16", hidden=256, n_hidden=2, max_batch=4096,
                 device=0, log_std_min=-20.0, log_std_max=2.0, expl_noise=0.1):
        d = spz_policy_desc(ALGOS[algo], SPZ_BF16 if precision == "bf16" else SPZ_FP32,
                            obs_dim, act_dim, hidden, n_hidden, max_batch, device, log_std_min, log_std_max,
                            expl_noise)
        self.obs_dim, self.act_dim = obs_dim, act_dim
        self.h = spz_policy_create(d)

    def load(self, payload_ptr, nbytes):
        return spz_policy_load(self.h, payload_ptr, nbytes)

    def params(self, n):
        return spz_policy_get_params(self.h, n)

    def act(self, obs, deterministic=False, seed=0, step=0, out=None):
        n = obs.shape[0]
        if out is None:
            out = np.empty((n, self.act_dim), dtype=np.float32)
        spz_policy_act(self.h, n, obs, deterministic, seed, step, out)
        return out

    def close(self):
        if self.h:
            spz_policy_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- batch-size adaptation (f3)

def spz_tune_batch(learner, ladder, warmup=3, steps=20, min_update_hz=0.0, tol=0.05, restore=True):
    """Returns (best_batch, [dict(batch, updates_per_s, frames_per_s, ms_per_update), ...])."""
    n = len(ladder)
    lad = (ctypes.c_int64 * n)(*ladder)
    pts = (spz_tune_point * n)()
    n_out, best = ctypes.c_int32(), ctypes.c_int64()
    _check(lib().spz_tune_batch(learner, lad, n, warmup, steps, min_update_hz, tol, 1 if restore else 0, pts,
                                ctypes.byref(n_out), ctypes.byref(best)))
    return best.value, [dict(batch=p.batch, updates_per_s=p.updates_per_s, frames_per_s=p.frames_per_s,
                             ms_per_update=p.ms_per_update) for p in pts[:n_out.value]]
