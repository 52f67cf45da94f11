"""numpy restatement of the reference learner (TEST INFRASTRUCTURE ONLY).

Follows reference pkg/src/dvla/grpo.py and kernels/numpy_backend.py:
  compute_advantages      grpo.py:89-99
  clipped_surrogate       grpo.py:111-119
  adam_step               grpo.py:137-150
  clip_grad_norm          grpo.py:297-301
  grpo_grad (Gaussian)    grpo.py:217-294 with policy.log_prob_of
                          (policy.py:161-172), numpy_backend.mlp_forward
                          (:33-36), chunk_log_prob (:39-49),
                          policy_backward (:52-93)
  grpo_grad (token head)  the same epilogue with the action-token head
                          ("one Gaussian dim" -> "one
                          action token"; chunk lp = numpy pairwise sum over
                          the chunk's T token log-probs, f64)
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

LOG_2PI = float(np.log(2.0 * np.pi))


class OracleAbort(RuntimeError):
    def __init__(self, group_id: int, detail: str):
        super().__init__(f"update aborted on group {group_id}: {detail}")
        self.group_id = group_id
        self.detail = detail


# --------------------------------------------------------------- scalar math
def compute_advantages(rewards, delta: float) -> np.ndarray:
    r = np.asarray(rewards, dtype=np.float64)
    if r.ndim != 1 or r.shape[0] < 2:
        raise ValueError(f"a reward group needs >= 2 entries, got shape {r.shape}")
    mean = r.mean()
    centered = r - mean
    var = (centered * centered).mean()
    if var == 0.0:
        return np.zeros_like(r)
    return centered / (np.sqrt(var) + delta)


def clipped_surrogate(ratio: float, adv: float, clip_eps: float):
    clipped_ratio = min(max(ratio, 1.0 - clip_eps), 1.0 + clip_eps)
    unclipped = ratio * adv
    clipped = clipped_ratio * adv
    if unclipped <= clipped:
        return -unclipped, -adv
    return -clipped, 0.0


def adam_step(flat_params, grad, m, v, step, lr, beta1, beta2, opt_eps):
    """Returns (new f32 params, m, v, step) -- grpo.py:137-150."""
    g = np.asarray(grad, dtype=np.float64)
    step += 1
    m = m * beta1
    m = m + (1.0 - beta1) * g
    v = v * beta2
    v = v + (1.0 - beta2) * (g * g)
    m_hat = m / (1.0 - beta1 ** step)
    v_hat = v / (1.0 - beta2 ** step)
    update = flat_params.astype(np.float64) - lr * m_hat / (np.sqrt(v_hat) + opt_eps)
    return update.astype(np.float32), m, v, step


def clip_grad_norm(grad: np.ndarray, max_norm):
    norm = float(np.sqrt((grad * grad).sum()))
    if max_norm is not None and norm > max_norm > 0:
        grad = grad * (max_norm / norm)
    return norm, grad


# ----------------------------------------------------------- Gaussian head
def mlp_forward(w1, b1, w2, b2, obs):
    """f64 sequential accumulate (bias first, then k = 0..), f32 out
    (numba_backend.py:27-46 loop order; vectorised over rows only)."""
    x = obs.astype(np.float64)
    acc = np.broadcast_to(b1.astype(np.float64), (x.shape[0], w1.shape[0])).copy()
    for k in range(w1.shape[1]):
        acc = acc + w1[:, k].astype(np.float64)[None, :] * x[:, k][:, None]
    h = np.tanh(acc)
    out = np.broadcast_to(b2.astype(np.float64), (x.shape[0], w2.shape[0])).copy()
    for j in range(w2.shape[1]):
        out = out + w2[:, j].astype(np.float64)[None, :] * h[:, j][:, None]
    return out.astype(np.float32)


def chunk_log_prob(means, log_std, actions):
    mu = means.astype(np.float64)
    s = log_std.astype(np.float64)
    a = actions.astype(np.float64)
    eps = (a - mu) * np.exp(-s)
    d = means.shape[1]
    return (-0.5 * eps * eps - s).sum(axis=1) - 0.5 * LOG_2PI * d


def gauss_head_backward(means, log_std, actions, coeffs):
    """d(sum_b c_b lp_b)/d means (B,D) and /d log_std (D,), f64."""
    mu = means.astype(np.float64)
    s = log_std.astype(np.float64)
    inv = np.exp(-s)
    eps = (actions.astype(np.float64) - mu) * inv
    c = np.asarray(coeffs, dtype=np.float64)[:, None]
    return c * eps * inv, (c * (eps * eps - 1.0)).sum(axis=0)


def policy_backward(w1, b1, w2, b2, log_std, obs, actions, coeffs, out):
    x = obs.astype(np.float64)
    a = actions.astype(np.float64)
    fw1, fb1 = w1.astype(np.float64), b1.astype(np.float64)
    fw2, fb2 = w2.astype(np.float64), b2.astype(np.float64)
    s = log_std.astype(np.float64)
    c = np.asarray(coeffs, dtype=np.float64)
    h = np.tanh(x @ fw1.T + fb1)
    mu = h @ fw2.T + fb2
    inv_sig = np.exp(-s)
    eps = (a - mu) * inv_sig
    gmu = c[:, None] * (eps * inv_sig)
    g_w2 = gmu.T @ h
    g_b2 = gmu.sum(axis=0)
    gz = (gmu @ fw2) * (1.0 - h * h)
    g_w1 = gz.T @ x
    g_b1 = gz.sum(axis=0)
    g_s = (c[:, None] * (eps * eps - 1.0)).sum(axis=0)
    i = 0
    for part in (g_w1.ravel(), g_b1, g_w2.ravel(), g_b2, g_s):
        out[i:i + part.size] += part
        i += part.size


def _epilogue(lp_of_entry, entries, n_traj, clip_eps, kl_coeff):
    """grpo.py:242-276 per-entry loop; returns loss, stats, coeffs dict."""
    total_loss = 0.0
    ratio_sum = 0.0
    clip_count = 0
    chunk_count = 0
    coeffs = {}
    for key, gid, adv, n_chunks, blp in entries:
        weight = 1.0 / (n_traj * n_chunks)
        lp_now = lp_of_entry(key)
        blp64 = np.asarray(blp, dtype=np.float64)
        if not np.isfinite(lp_now).all():
            raise OracleAbort(gid, "non-finite log-prob")
        with np.errstate(over="ignore"):
            rhos = np.exp(lp_now - blp64)
        if not np.isfinite(rhos).all():
            raise OracleAbort(gid, "non-finite importance ratio")
        cs = np.empty(n_chunks)
        for c in range(n_chunks):
            rho = float(rhos[c])
            contrib, d_drho = clipped_surrogate(rho, adv, clip_eps)
            coeff = weight * d_drho * rho
            loss_term = weight * contrib
            if kl_coeff > 0.0:
                diff = float(lp_now[c] - blp64[c])
                loss_term += weight * 0.5 * kl_coeff * diff * diff
                coeff += weight * kl_coeff * diff
            total_loss += loss_term
            ratio_sum += rho
            chunk_count += 1
            if d_drho == 0.0:
                clip_count += 1
            cs[c] = coeff
        coeffs[key] = cs
    return total_loss, ratio_sum, clip_count, chunk_count, coeffs


def _entries(group_ids, rewards_2d, blp_3d, G, adv_eps):
    order = np.argsort(np.asarray(group_ids, dtype=np.int64), kind="stable")
    entries = []
    for k in order:
        r = np.asarray(rewards_2d[k])
        advs = compute_advantages(r, adv_eps)
        if not np.isfinite(r).all():
            raise OracleAbort(int(group_ids[k]), "non-finite reward")
        for i in range(G):
            entries.append(((int(k), i), int(group_ids[k]), float(advs[i]),
                            blp_3d.shape[2], blp_3d[k, i]))
    return order, entries


def grpo_grad_gauss(w1, b1, w2, b2, log_std, group_ids, obs, actions, blp, rewards,
                    clip_eps=0.2, adv_eps=1e-8, kl_coeff=0.0):
    """Reference grpo_grad for the Gaussian MLP policy.

    obs (n_groups, G, C, obs_dim), actions (n_groups, G, C, D), blp
    (n_groups, G, C) f32, rewards (n_groups, G) f32.  Returns
    (loss, grad f64 flat, stats)."""
    n_groups, G, _ = blp.shape
    if n_groups == 0:
        raise ValueError("grpo update needs at least one group")
    n_traj = n_groups * G
    order, entries = _entries(group_ids, rewards, blp, G, adv_eps)

    def lp_of(key):
        k, i = key
        means = mlp_forward(w1, b1, w2, b2, obs[k, i])
        return chunk_log_prob(means, log_std, actions[k, i])

    loss, ratio_sum, clip_count, chunk_count, coeffs = _epilogue(
        lp_of, entries, n_traj, clip_eps, kl_coeff)
    n_params = w1.size + b1.size + w2.size + b2.size + log_std.size
    grad = np.zeros(n_params)
    for (k, i), cs in coeffs.items():
        policy_backward(w1, b1, w2, b2, log_std, obs[k, i], actions[k, i], cs, grad)
    if not np.isfinite(loss) or not np.isfinite(grad).all():
        raise OracleAbort(int(group_ids[order[0]]), "non-finite loss or gradient")
    stats = {
        "loss": float(loss), "mean_ratio": ratio_sum / max(chunk_count, 1),
        "clip_fraction": clip_count / max(chunk_count, 1), "n_chunks": chunk_count,
        "group_ids": [int(group_ids[k]) for k in order],
    }
    return float(loss), grad, stats


# ------------------------------------------------------------- token head
def token_row_stats(x2d: np.ndarray, tokens: np.ndarray):
    """f64 log-softmax gather: (lse, lp_tok) per row."""
    x = x2d.astype(np.float64)
    m = x.max(axis=1)
    s = np.exp(x - m[:, None]).sum(axis=1)
    lse = m + np.log(s)
    lp_tok = x[np.arange(x.shape[0]), tokens.astype(np.int64)] - lse
    return lse, lp_tok


def _rows_parallel(fn, n_rows: int, threads: int, block: int = 64):
    spans = [(a, min(a + block, n_rows)) for a in range(0, n_rows, block)]
    if threads <= 1:
        return [fn(a, b) for a, b in spans]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda ab: fn(*ab), spans))


def grpo_token_grad(logits, tokens, blp, rewards, group_ids, clip_eps=0.2, adv_eps=1e-8,
                    kl_coeff=0.0, want_dlogits=True, threads: int | None = None):
    """Token-head grpo_grad restated in numpy f64.

    logits (n_groups, G, C, T, V) (f32 values; bf16 inputs are upcast
    exactly), tokens (n_groups, G, C, T) int, blp (n_groups, G, C) f32,
    rewards (n_groups, G) f32.  Returns (loss, dlogits f64 or None, stats)
    with stats["lp_chunk"] (n_groups, G, C) f64 and stats["coeff"].
    """
    n_groups, G, C, T, V = logits.shape
    if n_groups == 0:
        raise ValueError("grpo update needs at least one group")
    threads = threads or (os.cpu_count() or 1)
    x2d = logits.reshape(-1, V)
    tok = tokens.reshape(-1)
    R = x2d.shape[0]
    lse = np.empty(R)
    lp_tok = np.empty(R)

    def rows(a, b):
        lse[a:b], lp_tok[a:b] = token_row_stats(x2d[a:b], tok[a:b])

    _rows_parallel(rows, R, threads)
    # chunk-joint log-prob: numpy pairwise sum over the chunk's T tokens (the
    # order numpy_backend.chunk_log_prob's .sum(axis=1) uses over D dims)
    lp_chunk = lp_tok.reshape(-1, T).sum(axis=1).reshape(n_groups, G, C)
    n_traj = n_groups * G
    order, entries = _entries(group_ids, rewards, blp, G, adv_eps)
    loss, ratio_sum, clip_count, chunk_count, coeffs = _epilogue(
        lambda key: lp_chunk[key[0], key[1]], entries, n_traj, clip_eps, kl_coeff)
    if not np.isfinite(loss):
        raise OracleAbort(int(group_ids[order[0]]), "non-finite loss or gradient")
    coeff = np.zeros((n_groups, G, C))
    for (k, i), cs in coeffs.items():
        coeff[k, i] = cs
    dl = None
    if want_dlogits:
        dl = np.empty((R, V))
        crow = np.repeat(coeff.reshape(-1), T)

        def bwd(a, b):
            p = np.exp(x2d[a:b].astype(np.float64) - lse[a:b, None])
            oh = np.zeros_like(p)
            oh[np.arange(b - a), tok[a:b].astype(np.int64)] = 1.0
            dl[a:b] = crow[a:b, None] * (oh - p)

        _rows_parallel(bwd, R, threads)
        dl = dl.reshape(logits.shape)
    stats = {
        "loss": float(loss), "mean_ratio": ratio_sum / max(chunk_count, 1),
        "clip_fraction": clip_count / max(chunk_count, 1), "n_chunks": chunk_count,
        "group_ids": [int(group_ids[k]) for k in order],
        "lp_chunk": lp_chunk, "coeff": coeff, "lse": lse, "lp_tok": lp_tok,
    }
    return float(loss), dl, stats
