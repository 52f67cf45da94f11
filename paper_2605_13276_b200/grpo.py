"""Group-relative policy optimisation on B200: the learner's hot path.

Same public API as reference pkg/src/dvla/grpo.py (GrpoConfig :23-52,
GroupBatch :55-78, GrpoAbort :81-86, compute_advantages :89-99,
group_advantages :102-108, clipped_surrogate :111-119, AdamState :122-134,
adam_step :137-150, UpdateStats :153-174, grpo_loss :194-214, grpo_grad
:217-294, clip_grad_norm :297-301, grpo_update :304-320), with every
array-sized computation done by sm_100a kernels through the C-ABI.

Two policy heads share one learner epilogue (csrc/grpo_math.cuh):
  * the action-token head (the north-star path): `grpo_token_grad` /
    `TokenLoss` -- fused log-softmax gather + clipped surrogate + dlogits
    over logits [rows, V] in one pass (csrc/token_loss.cu);
  * the reference's Gaussian tanh-MLP chunk policy: `grpo_grad` on
    PolicyParams, bit-for-bit the reference's arithmetic contract
    (csrc/gauss.cu).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import ConfigError, UsageError

VALID_RATIO_GRANULARITY = ("chunk",)


@dataclass(frozen=True)
class GrpoConfig:
    group_size: int = 8
    clip_eps: float = 0.2
    adv_epsilon: float = 1e-8
    micro_batch: int = 8
    lr: float = 3e-3
    beta1: float = 0.9
    beta2: float = 0.999
    opt_eps: float = 1e-8
    max_grad_norm: float | None = None
    kl_coeff: float = 0.0
    ratio_granularity: str = "chunk"

    def validate(self):
        if self.group_size < 2:
            raise ConfigError(f"group_size must be >= 2, got {self.group_size}")
        if not (0.0 < self.clip_eps < 1.0):
            raise ConfigError(f"clip_eps must be in (0, 1), got {self.clip_eps}")
        if self.micro_batch < 1:
            raise ConfigError("micro_batch must be >= 1")
        if self.adv_epsilon <= 0:
            raise ConfigError("adv_epsilon must be > 0")
        if self.kl_coeff < 0:
            raise ConfigError("kl_coeff must be >= 0")
        if self.ratio_granularity not in VALID_RATIO_GRANULARITY:
            raise ConfigError(
                "ratio_granularity must be 'chunk'; per-sub-step ratios are "
                "unrepresentable (one behavior log-prob is stored per chunk)"
            )


@dataclass
class GroupBatch:
    """G trajectories sharing one initial condition and one behaviour version.

    obs: (G, C, obs_dim); actions: (G, C, chunk*act_dim);
    behavior_log_prob: (G, C); rewards: (G,).  Arrays may be numpy (host)
    or torch tensors (device).  For the action-token head `tokens`
    (G, C, T) int32 holds the target action-token ids.
    """

    group_id: int
    horizon: int
    chunk: int
    obs: object
    actions: object
    behavior_log_prob: object
    rewards: object
    behavior_version: int
    tokens: object = None

    @property
    def g(self) -> int:
        return self.obs.shape[0]

    @property
    def n_chunks(self) -> int:
        return self.obs.shape[1]


class GrpoAbort(RuntimeError):
    """Non-finite loss or gradient; carries the offending group id."""

    def __init__(self, group_id: int, detail: str):
        super().__init__(f"update aborted on group {group_id}: {detail}")
        self.group_id = group_id


ABORT_DETAILS = {
    1: "non-finite reward",
    2: "non-finite log-prob",
    3: "non-finite importance ratio",
    4: "non-finite loss or gradient",
}


def _torch():
    import torch
    return torch


def _dev(device=None):
    torch = _torch()
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("dvla_b200 kernels need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream_ptr(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def compute_advantages(rewards, delta: float):
    """A_i = (r_i - mean(r)) / (popstd(r) + delta); all-zero when var == 0.

    Computed on the GPU (csrc/grpo_math.cuh group_advantages), bit-identical
    to reference grpo.py:89-99 including numpy's pairwise mean order.
    Returns the input's kind: numpy in -> numpy f64 out, tensor -> tensor.
    """
    from . import _lib
    torch = _torch()
    is_t = isinstance(rewards, torch.Tensor)
    r = rewards if is_t else np.asarray(rewards, dtype=np.float64)
    if r.ndim != 1 or r.shape[0] < 2:
        raise ConfigError(f"a reward group needs >= 2 entries, got shape {tuple(r.shape)}")
    dev = rewards.device if (is_t and rewards.is_cuda) else _dev()
    rd = (r if is_t else torch.from_numpy(np.ascontiguousarray(r))).to(
        device=dev, dtype=torch.float64).contiguous()
    out = torch.empty_like(rd)
    with torch.cuda.device(dev):
        _lib.check(_lib.dvla_advantages(rd.data_ptr(), 1, rd.shape[0], float(delta),
                                        out.data_ptr(), _stream_ptr()), "dvla_advantages")
    if is_t:
        return out if rewards.is_cuda else out.cpu()
    return out.cpu().numpy()


def group_advantages(batch: GroupBatch, cfg: GrpoConfig):
    if batch.g != cfg.group_size:
        raise ConfigError(
            f"group {batch.group_id} has {batch.g} trajectories, "
            f"expected G={cfg.group_size}"
        )
    return compute_advantages(batch.rewards, cfg.adv_epsilon)


def clipped_surrogate(ratio: float, adv: float, clip_eps: float):
    """-min(ratio*A, clip(ratio)*A) and its d/d ratio; ties take the
    unclipped derivative (reference grpo.py:111-119).  Scalar helper only:
    the batched path evaluates the same expression on the device
    (grpo_math.cuh chunk_terms)."""
    clipped_ratio = min(max(ratio, 1.0 - clip_eps), 1.0 + clip_eps)
    unclipped = ratio * adv
    clipped = clipped_ratio * adv
    if unclipped <= clipped:
        return -unclipped, -adv
    return -clipped, 0.0


@dataclass
class UpdateStats:
    version: int
    loss: float
    mean_ratio: float
    clip_fraction: float
    grad_norm: float
    mean_reward: float
    n_traj: int
    n_groups: int
    n_chunks: int
    quarantined: int = 0
    group_ids: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {
            "version": self.version, "loss": self.loss,
            "mean_ratio": self.mean_ratio, "clip_fraction": self.clip_fraction,
            "grad_norm": self.grad_norm, "mean_reward": self.mean_reward,
            "n_traj": self.n_traj, "n_groups": self.n_groups,
            "n_chunks": self.n_chunks, "quarantined": self.quarantined,
        }


def canonical_order(group_ids) -> np.ndarray:
    """Stable sort by group_id (reference grpo.py:177-178 _ordered)."""
    ids = np.asarray(group_ids, dtype=np.int64)
    return np.argsort(ids, kind="stable").astype(np.int64)


def _mean_reward(rewards_2d: np.ndarray, order: np.ndarray) -> float:
    """float(np.mean([b.rewards.mean() for b in batches])) in canonical order
    (reference grpo.py:291); host f32 arithmetic, bit-identical."""
    # one row-wise reduction over the groups in canonical order: numpy's
    # per-row pairwise f32 sums, bit-identical to the per-group .mean()
    # (tests/test_oracle.py), without a Python loop over the groups
    per = np.asarray(rewards_2d, dtype=np.float32)[np.asarray(order)].mean(axis=1)
    return float(np.mean(per))


def stats_from_vector(sv: np.ndarray, group_ids: np.ndarray, order: np.ndarray,
                      n_traj: int, rewards_2d=None) -> dict:
    """Host view of the device stats vector + the abort contract."""
    from . import _lib
    code = int(sv[_lib.ST_ABORT])
    if int(sv[_lib.ST_KERNEL_ERR]) & 1:
        raise UsageError("target token id outside [0, V)")
    if int(sv[_lib.ST_KERNEL_ERR]) & 2:
        raise _lib.NativeError("fused loss kernel timed out waiting for a chunk")
    if code:
        raise GrpoAbort(int(sv[_lib.ST_ABORT_GROUP]), ABORT_DETAILS[code])
    n_chunks = int(sv[_lib.ST_CHUNK_COUNT])
    out = {
        "loss": float(sv[_lib.ST_LOSS]),
        "mean_ratio": float(sv[_lib.ST_RATIO_SUM]) / max(n_chunks, 1),
        "clip_fraction": float(sv[_lib.ST_CLIP_COUNT]) / max(n_chunks, 1),
        "n_traj": int(n_traj),
        "n_groups": int(len(group_ids)),
        "n_chunks": n_chunks,
        "group_ids": np.asarray(group_ids, dtype=np.int64)[np.asarray(order)].tolist(),
    }
    if rewards_2d is not None:
        out["mean_reward"] = _mean_reward(rewards_2d, order)
    return out


class TokenLoss:
    """Reusable launcher for the fused action-token GRPO loss.

    Holds the device workspace, stats vector and canonical group order for
    one batch shape so the trainer lane (and bench.py) can launch the fused
    kernel repeatedly without allocations:

        tl = TokenLoss(n_groups, G, C, T, V, cfg, dtype=torch.bfloat16)
        tl.set_groups(group_ids)                 # host ids -> canonical order
        tl.launch(logits, tokens, blp, rewards, dlogits)   # async
        stats = tl.stats(rewards)                # sync + GrpoAbort mapping

    Shapes (device tensors, input group order):
      logits  [n_groups*G*C*T, V] (bf16 or f32), tokens int32 [rows],
      blp f32 [n_groups*G*C], rewards f32 [n_groups*G],
      dlogits same shape/dtype as logits.
    """

    def __init__(self, n_groups: int, G: int, C: int, T: int, V: int, cfg: GrpoConfig,
                 dtype=None, device=None, fused: bool = True):
        from . import _lib
        torch = _torch()
        cfg.validate()
        if n_groups < 1:
            raise ConfigError("grpo update needs at least one group")
        if G != cfg.group_size:
            raise ConfigError(f"group has {G} trajectories, expected G={cfg.group_size}")
        self.cfg = cfg
        self.n_groups, self.G, self.C, self.T, self.V = n_groups, G, C, T, V
        self.dtype = dtype if dtype is not None else torch.bfloat16
        if self.dtype not in (torch.bfloat16, torch.float32):
            raise UsageError(f"logits dtype must be bf16 or f32, got {self.dtype}")
        self.code = _lib.BF16 if self.dtype == torch.bfloat16 else _lib.F32
        self.device = _dev(device)
        self.fused = fused
        self.rows = n_groups * G * C * T
        nbytes = _lib.dvla_token_loss_workspace_bytes(n_groups, G, C, T)
        self.workspace = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=self.device)
        self.lp_chunk = torch.empty(n_groups * G * C, dtype=torch.float64, device=self.device)
        self.stats_dev = torch.zeros(_lib.ST_LEN, dtype=torch.float64, device=self.device)
        offs = (_lib.C.c_size_t * 4)()
        _lib.check(_lib.dvla_token_loss_workspace_layout(n_groups, G, C, T, offs),
                   "dvla_token_loss_workspace_layout")
        ws64 = self.workspace.view(torch.float64)
        n_traj, nq = n_groups * G, n_groups * G * C
        # views of what the last launch left in the workspace (parity checks)
        self.adv = ws64[offs[0] // 8: offs[0] // 8 + n_traj]
        self.lp_tok = ws64[offs[1] // 8: offs[1] // 8 + self.rows]
        self.coeff = ws64[offs[3] // 8: offs[3] // 8 + nq]
        self.set_groups(np.arange(n_groups, dtype=np.int64))
        self._ids_ev.synchronize()   # usable from any stream from here on

    def set_groups(self, group_ids, stream=None):
        """Host group ids -> canonical order; the two small device vectors
        are refreshed by an asynchronous copy from a pinned staging buffer on
        `stream` (default: current) -- a pageable copy would block the host
        until the stream drained (no-op when the ids are unchanged)."""
        torch = _torch()
        ids = np.asarray(group_ids, dtype=np.int64)
        if ids.shape != (self.n_groups,):
            raise UsageError(f"expected {self.n_groups} group ids, got shape {ids.shape}")
        if getattr(self, "group_ids", None) is not None and np.array_equal(ids, self.group_ids):
            return
        self.group_ids = ids
        self.order = canonical_order(ids)
        if getattr(self, "_ids_host", None) is None:
            self._ids_host = torch.empty(2, self.n_groups, dtype=torch.int64, pin_memory=True)
            self._ids_dev = torch.empty(2, self.n_groups, dtype=torch.int64, device=self.device)
            self.order_dev, self.ids_dev = self._ids_dev[0], self._ids_dev[1]
            self._ids_ev = None
        if self._ids_ev is not None:
            self._ids_ev.synchronize()        # the previous copy has read the staging buffer
        self._ids_host[0].copy_(torch.from_numpy(self.order))
        self._ids_host[1].copy_(torch.from_numpy(ids))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            self._ids_dev.copy_(self._ids_host, non_blocking=True)
            self._ids_ev = torch.cuda.Event()
            self._ids_ev.record(st)

    def _check_tensor(self, t, shape, dtype, name):
        torch = _torch()
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise UsageError(f"{name} must be a CUDA tensor")
        if t.dtype != dtype:
            raise UsageError(f"{name} must be {dtype}, got {t.dtype}")
        if t.numel() != int(np.prod(shape)):
            raise UsageError(f"{name} has {t.numel()} elements, expected shape {shape}")
        if not t.is_contiguous():
            raise UsageError(f"{name} must be contiguous")

    def launch(self, logits, tokens, blp, rewards, dlogits=None, stream=None):
        """Enqueue the fused forward+backward on `stream` (default: current)."""
        from . import _lib
        torch = _torch()
        R, V = self.rows, self.V
        self._check_tensor(logits, (R, V), self.dtype, "logits")
        self._check_tensor(tokens, (R,), torch.int32, "tokens")
        self._check_tensor(blp, (self.n_groups * self.G * self.C,), torch.float32,
                           "behavior_log_prob")
        self._check_tensor(rewards, (self.n_groups * self.G,), torch.float32, "rewards")
        flags = 0 if self.fused else _lib.TL_UNFUSED
        dptr = None
        if dlogits is not None:
            self._check_tensor(dlogits, (R, V), self.dtype, "dlogits")
            flags |= _lib.TL_WRITE_DLOGITS
            dptr = dlogits.data_ptr()
        c = self.cfg
        with torch.cuda.device(self.device):
            st = _lib.dvla_token_loss_fwd_bwd(
                logits.data_ptr(), self.code, tokens.data_ptr(), blp.data_ptr(),
                rewards.data_ptr(), self.order_dev.data_ptr(), self.ids_dev.data_ptr(),
                self.n_groups, self.G, self.C, self.T, V, float(c.clip_eps),
                float(c.adv_epsilon), float(c.kl_coeff), flags, dptr,
                self.lp_chunk.data_ptr(), self.stats_dev.data_ptr(),
                self.workspace.data_ptr(), self.workspace.numel(), _stream_ptr(stream))
        _lib.check(st, "dvla_token_loss_fwd_bwd")

    def stats(self, rewards=None) -> dict:
        """Synchronise on the stats vector (64 B D2H) and apply the abort
        contract (GrpoAbort with the reference's group id and message)."""
        sv = self.stats_dev.cpu().numpy()
        r2d = None
        if rewards is not None:
            r = rewards.detach().cpu().numpy() if hasattr(rewards, "detach") else np.asarray(rewards)
            r2d = r.reshape(self.n_groups, self.G)
        return stats_from_vector(sv, self.group_ids, self.order, self.n_groups * self.G, r2d)


def grpo_token_grad(logits, tokens, behavior_log_prob, rewards, group_ids, cfg: GrpoConfig,
                    dlogits=None, write_dlogits: bool = True, fused: bool = True):
    """Token-head grpo_grad: (loss, dlogits, stats) for one learner batch.

    logits [n_groups, G, C, T, V] (or [rows, V]) bf16/f32 CUDA tensor in the
    same group order as `group_ids`; tokens int32 [n_groups, G, C, T];
    behavior_log_prob f32 [n_groups, G, C]; rewards f32 [n_groups, G].
    Canonical (sorted-by-group_id) order governs the loss accumulation and
    the abort group exactly as reference grpo.py:226-294.
    """
    torch = _torch()
    ids = np.asarray(group_ids, dtype=np.int64)
    n_groups = len(ids)
    if n_groups == 0:
        raise ConfigError("grpo update needs at least one group")
    tok = tokens
    if tok.dim() != 4:
        raise UsageError("tokens must be (n_groups, G, C, T)")
    _, G, C, T = tok.shape
    if G != cfg.group_size:
        k = 0
        raise ConfigError(f"group {int(ids[k])} has {G} trajectories, expected G={cfg.group_size}")
    V = logits.shape[-1]
    tl = TokenLoss(n_groups, G, C, T, V, cfg, dtype=logits.dtype, device=logits.device,
                   fused=fused)
    tl.set_groups(ids)
    lg = logits.reshape(-1, V)
    if write_dlogits and dlogits is None:
        dlogits = torch.empty_like(lg)
    tl.launch(lg, tok.reshape(-1).contiguous(), behavior_log_prob.reshape(-1).contiguous(),
              rewards.reshape(-1).contiguous(),
              dlogits.reshape(-1, V) if write_dlogits else None)
    st = tl.stats(rewards)
    st["lp_chunk"] = tl.lp_chunk.view(n_groups, G, C)
    st["coeff"] = tl.coeff.view(n_groups, G, C)
    st["lp_tok"] = tl.lp_tok.view(n_groups, G, C, T)
    return st["loss"], (dlogits if write_dlogits else None), st


def grpo_gauss_head_grad(means, log_std, actions, behavior_log_prob, rewards, group_ids,
                         cfg: GrpoConfig, dlog_std=None, stream=None):
    """Gaussian-head grpo_grad for an action expert whose chunk means come
    from the caller's model (BASELINE config 3, pi0-shaped): one
    `dvla_gauss_loss_fwd_bwd` call -> (loss, dmeans [.., D] f32,
    dlog_std [D] f64 (accumulated into `dlog_std` if given), stats).

    means/actions f32 [n_groups, G, C, D] CUDA tensors in `group_ids` order,
    log_std f32 [D], behavior_log_prob f32 [n_groups, G, C], rewards f32
    [n_groups, G]; the abort and canonical-order contract is grpo.py:226-294.
    """
    from . import _lib
    torch = _torch()
    cfg.validate()
    ids = np.asarray(group_ids, dtype=np.int64)
    n_groups = len(ids)
    if n_groups == 0:
        raise ConfigError("grpo update needs at least one group")
    if means.dim() != 4 or actions.shape != means.shape:
        raise UsageError("means/actions must be (n_groups, G, C, D) and equal in shape")
    _, G, C, D = means.shape
    if G != cfg.group_size:
        raise ConfigError(f"group {int(ids[0])} has {G} trajectories, expected G={cfg.group_size}")
    dev = means.device
    for name, t, dt in (("means", means, torch.float32), ("actions", actions, torch.float32),
                        ("log_std", log_std, torch.float32),
                        ("behavior_log_prob", behavior_log_prob, torch.float32),
                        ("rewards", rewards, torch.float32)):
        if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise UsageError(f"{name} must be a contiguous {dt} CUDA tensor")
    order = canonical_order(ids)
    order_d = torch.from_numpy(order).to(dev)
    ids_d = torch.from_numpy(ids).to(dev)
    B = n_groups * G * C
    lp = torch.empty(B, dtype=torch.float64, device=dev)
    stats = torch.zeros(_lib.ST_LEN, dtype=torch.float64, device=dev)
    dm = torch.empty((n_groups, G, C, D), dtype=torch.float32, device=dev)
    if dlog_std is None:
        dlog_std = torch.zeros(D, dtype=torch.float64, device=dev)
    ws = torch.empty(max(_lib.dvla_gauss_loss_workspace_bytes(n_groups, G, C), 8),
                     dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.dvla_gauss_loss_fwd_bwd(
            means.data_ptr(), log_std.data_ptr(), actions.data_ptr(), behavior_log_prob.data_ptr(),
            rewards.data_ptr(), order_d.data_ptr(), ids_d.data_ptr(), n_groups, G, C, D,
            float(cfg.clip_eps), float(cfg.adv_epsilon), float(cfg.kl_coeff), dm.data_ptr(),
            dlog_std.data_ptr(), lp.data_ptr(), stats.data_ptr(), ws.data_ptr(), ws.numel(),
            _stream_ptr(stream)), "dvla_gauss_loss_fwd_bwd")
    st = stats_from_vector(stats.cpu().numpy(), ids, order, n_groups * G,
                           rewards.reshape(n_groups, G).cpu().numpy())
    st["lp_chunk"] = lp.view(n_groups, G, C)
    return st["loss"], dm, dlog_std, st


# ------------------------------------------------------------------------
# Reference-shaped learner for the Gaussian tanh-MLP chunk policy
# ------------------------------------------------------------------------

@dataclass
class AdamState:
    """Adam moments (f64) and step count (reference grpo.py:122-134); m/v
    may be numpy arrays or device tensors (e.g. MODEL_COMPUTE pool views)."""

    m: object
    v: object
    step: int = 0

    @classmethod
    def zeros(cls, n: int, m_buf=None, v_buf=None) -> "AdamState":
        m = np.zeros(n, dtype=np.float64) if m_buf is None else m_buf
        v = np.zeros(n, dtype=np.float64) if v_buf is None else v_buf
        m[:] = 0.0
        v[:] = 0.0
        return cls(m=m, v=v)


def _is_t(x) -> bool:
    return type(x).__module__.startswith("torch")


def adam_step(flat_params, grad, state: AdamState, cfg: GrpoConfig):
    """One bias-corrected Adam step in place on flat_params (f32), on the
    GPU (csrc/optim.cu), element-wise identical to reference grpo.py:137-150."""
    from . import _lib
    from .policy import to_dev
    torch = _torch()
    p = flat_params if (_is_t(flat_params) and flat_params.is_cuda) else to_dev(flat_params)
    g = to_dev(grad, torch.float64)
    m = state.m if (_is_t(state.m) and state.m.is_cuda) else to_dev(state.m, torch.float64)
    v = state.v if (_is_t(state.v) and state.v.is_cuda) else to_dev(state.v, torch.float64)
    state.step += 1
    _lib.check(_lib.dvla_adam_step(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(),
                                   p.numel(), state.step, float(cfg.lr), float(cfg.beta1),
                                   float(cfg.beta2), float(cfg.opt_eps), _stream_ptr()),
               "dvla_adam_step")
    for host, dev in ((state.m, m), (state.v, v)):
        if not (_is_t(host) and host.is_cuda):
            host[:] = dev.cpu().numpy() if not _is_t(host) else dev.cpu()
    if not (_is_t(flat_params) and flat_params.is_cuda):
        flat_params[:] = p.cpu().numpy() if not _is_t(flat_params) else p.cpu()
    return flat_params


def clip_grad_norm(grad, max_norm: float | None) -> float:
    """L2 norm of grad; scales grad in place when norm > max_norm > 0
    (reference grpo.py:297-301)."""
    from . import _lib
    from .policy import to_dev
    torch = _torch()
    g = grad if (_is_t(grad) and grad.is_cuda) else to_dev(grad, torch.float64)
    n = g.numel()
    ws = torch.empty(_lib.dvla_grad_norm_workspace_bytes(n), dtype=torch.uint8, device=g.device)
    norm = torch.empty(1, dtype=torch.float64, device=g.device)
    flag = torch.zeros(1, dtype=torch.int32, device=g.device)
    mx = float(max_norm) if max_norm is not None else 0.0
    _lib.check(_lib.dvla_grad_norm(g.data_ptr(), n, mx, norm.data_ptr(), flag.data_ptr(),
                                   ws.data_ptr(), _stream_ptr()), "dvla_grad_norm")
    if not (_is_t(grad) and grad.is_cuda):
        grad[:] = g.cpu().numpy() if not _is_t(grad) else g.cpu()
    return float(norm.item())


def _ordered(batches) -> list:
    return sorted(batches, key=lambda b: b.group_id)


def _stack_batches(batches, cfg: GrpoConfig):
    """Device tensors of a list of GroupBatch in INPUT order + canonical order."""
    from .policy import to_dev
    torch = _torch()
    ordered = _ordered(batches)
    for b in ordered:  # group-size check in canonical order (grpo.py:235-236)
        if b.g != cfg.group_size:
            raise ConfigError(f"group {b.group_id} has {b.g} trajectories, "
                              f"expected G={cfg.group_size}")
    ids = np.array([b.group_id for b in batches], dtype=np.int64)
    order = canonical_order(ids)

    def stack(attr, dtype):
        xs = [getattr(b, attr) for b in batches]
        if all(_is_t(x) for x in xs):
            return torch.stack([x.to(dtype) for x in xs]).to(_dev()).contiguous()
        return to_dev(np.stack([np.asarray(x.cpu() if _is_t(x) else x) for x in xs]), dtype)

    obs = stack("obs", torch.float32)
    act = stack("actions", torch.float32)
    blp = stack("behavior_log_prob", torch.float32)
    rw = stack("rewards", torch.float32)
    return ids, order, obs, act, blp, rw


def grpo_grad(params, batches, cfg: GrpoConfig, out_grad=None):
    """Micro-batched GRPO loss + gradient for the Gaussian MLP policy
    (reference grpo.py:217-294) on the GPU: mlp_forward -> chunk_log_prob ->
    group advantages -> canonical-order epilogue -> policy_backward.

    Returns (loss, grad_sum f64 flat, stats) with the reference's stats keys
    and GrpoAbort / ConfigError contract.  grad is numpy when params are
    numpy, a device tensor when params are device tensors."""
    from . import _lib
    from .policy import _dims, _dparams, chunk_log_prob_dev, mlp_forward_dev, policy_backward_dev
    torch = _torch()
    cfg.validate()
    if not batches:
        raise ConfigError("grpo update needs at least one group")
    ids, order, obs, act, blp, rw = _stack_batches(batches, cfg)
    n_groups, G, C = blp.shape
    o, h, d = _dims(params)
    dev = obs.device
    n_traj = n_groups * G
    adv = torch.empty(n_traj, dtype=torch.float64, device=dev)
    bad = torch.empty(n_groups, dtype=torch.int32, device=dev)
    _lib.check(_lib.dvla_group_advantages(rw.data_ptr(), n_groups, G, float(cfg.adv_epsilon),
                                          adv.data_ptr(), bad.data_ptr(), _stream_ptr()),
               "dvla_group_advantages")
    dp = _dparams(params)
    means = mlp_forward_dev(dp, obs.reshape(-1, o), o, h, d)
    lp = chunk_log_prob_dev(means, dp[4], act.reshape(-1, d))
    coeff = torch.empty(n_traj * C, dtype=torch.float64, device=dev)
    stats = torch.zeros(_lib.ST_LEN, dtype=torch.float64, device=dev)
    order_d = torch.from_numpy(order).to(dev)
    ids_d = torch.from_numpy(ids).to(dev)
    _lib.check(_lib.dvla_grpo_epilogue(lp.data_ptr(), blp.data_ptr(), None, adv.data_ptr(),
                                       bad.data_ptr(), order_d.data_ptr(), ids_d.data_ptr(),
                                       n_groups, G, C, float(cfg.clip_eps), float(cfg.kl_coeff),
                                       coeff.data_ptr(), stats.data_ptr(), _stream_ptr()),
               "dvla_grpo_epilogue")
    st = stats_from_vector(stats.cpu().numpy(), ids, order, n_traj,
                           rw.reshape(n_groups, G).cpu().numpy())
    grad = torch.zeros(h * o + h + d * h + d + d, dtype=torch.float64, device=dev)
    policy_backward_dev(dp, obs.reshape(-1, o), act.reshape(-1, d), coeff, grad, o, h, d)
    if not np.isfinite(st["loss"]) or not bool(torch.isfinite(grad).all()):
        raise GrpoAbort(int(ids[order[0]]), "non-finite loss or gradient")
    if out_grad is not None:
        if _is_t(out_grad):
            out_grad.copy_(grad)
            grad = out_grad
        else:
            out_grad[:] = grad.cpu().numpy()
            grad = out_grad
    elif not _is_t(params.w1):
        grad = grad.cpu().numpy()
    return float(st["loss"]), grad, st


def grpo_loss(params, batches, cfg: GrpoConfig) -> float:
    """Scalar surrogate loss (reference grpo.py:194-214), from the same GPU
    forward + epilogue as grpo_grad (the independent f64 finite-difference
    path of the reference lives in the test oracle, oracle/grpo_oracle.py)."""
    loss, _, _ = grpo_grad(params, batches, cfg)
    return loss


def infer_policy_config(params):
    """The structural config a params object implies (reference
    grpo.py:323-330).  The reference fixes act_dim = 2 (its env) and sets
    chunk = out_dim // 2, which drops a unit for an odd out_dim; here the
    split keeps chunk * act_dim == out_dim (act_dim 2 when out_dim is even,
    else 1) -- unflatten only needs out_dim, so even-width heads behave
    exactly as in the reference."""
    from .policy import PolicyConfig
    hidden, obs_dim = tuple(params.w1.shape)
    out_dim = tuple(params.w2.shape)[0]
    act_dim = 2 if out_dim % 2 == 0 else 1
    return PolicyConfig(obs_dim=obs_dim, hidden=hidden, chunk=out_dim // act_dim,
                        act_dim=act_dim)


def grpo_update(params, batches, cfg: GrpoConfig, adam: AdamState, version: int):
    """grad, optional norm clip, Adam (reference grpo.py:304-320)."""
    from .policy import flatten, unflatten
    loss, grad, stats = grpo_grad(params, batches, cfg)
    norm = clip_grad_norm(grad, cfg.max_grad_norm)
    flat = flatten(params)
    adam_step(flat, grad, adam, cfg)
    new_params = unflatten(infer_policy_config(params), flat)
    ustats = UpdateStats(
        version=version + 1, loss=loss, mean_ratio=stats["mean_ratio"],
        clip_fraction=stats["clip_fraction"], grad_norm=norm,
        mean_reward=stats["mean_reward"], n_traj=stats["n_traj"],
        n_groups=stats["n_groups"], n_chunks=stats["n_chunks"],
        group_ids=stats["group_ids"],
    )
    return new_params, ustats
