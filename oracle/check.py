"""Comparison criteria for d loss / d logits (TEST INFRASTRUCTURE ONLY).

Used by tests/, __graft_entry__.smoke() and bench.py's parity line; never by
the product package.

A max-scaled tolerance (err <= rtol*|want| + rtol*max|want|) cannot see a
systematic error in the off-target softmax entries of a long row: at
V = 32,064 they are ~1e-4 of the row maximum (the target column), so a 10 %
error on every one of them would pass.  The criterion here is per row:

  * row-wise relative L2:  ||got_r - want_r||_2 <= rtol * ||want_r||_2
  * element-wise relative: |got - want| <= rtol * |want| for every entry with
    |want| >= floor * max_r |want_r| (the entries that carry the row)
  * rows whose oracle gradient is exactly zero (coefficient 0: A = 0 or a
    clipped chunk) must be exactly zero.

Tolerances are the north star's: 1e-5 relative in fp32, 1e-2 in bf16.
"""

from __future__ import annotations

import numpy as np


def dlogits_rows(x_rows, tok_rows, lse_rows, coeff_rows):
    """Oracle d loss / d logits for a set of rows from f64 lse and the
    per-row coefficient: c * (1[v == tok] - exp(x - lse))."""
    x = np.asarray(x_rows, dtype=np.float64)
    p = np.exp(x - np.asarray(lse_rows, dtype=np.float64)[:, None])
    oh = np.zeros_like(p)
    oh[np.arange(x.shape[0]), np.asarray(tok_rows, dtype=np.int64)] = 1.0
    return np.asarray(coeff_rows, dtype=np.float64)[:, None] * (oh - p)


def dlogits_errors(got, want, floor: float = 1e-3, row_cond=None):
    """(max row-wise relative L2 error, max element-wise relative error over
    entries >= floor * row max, number of zero rows that are not zero).
    row_cond: optional per-row factor >= 1 (row_condition) dividing each
    row's errors."""
    g = np.asarray(got, dtype=np.float64).reshape(-1, np.shape(got)[-1])
    w = np.asarray(want, dtype=np.float64).reshape(g.shape)
    d = g - w
    rc = np.ones(g.shape[0]) if row_cond is None else \
        np.asarray(row_cond, dtype=np.float64).reshape(-1)
    wn = np.sqrt((w * w).sum(axis=1))
    dn = np.sqrt((d * d).sum(axis=1))
    zero = wn == 0.0
    bad_zero = int(np.count_nonzero(dn[zero] != 0.0))
    nz = ~zero
    row_l2 = float((dn[nz] / wn[nz] / rc[nz]).max()) if nz.any() else 0.0
    aw = np.abs(w[nz])
    big = aw >= floor * aw.max(axis=1, keepdims=True)
    rel = np.abs(d[nz]) / np.where(big, aw, 1.0) / rc[nz][:, None]
    elem = float(rel[big].max()) if big.any() else 0.0
    return row_l2, elem, bad_zero


def coeff_term_scale(lp_chunk, blp, rewards, clip_eps=0.2, adv_eps=1e-8, kl_coeff=0.0):
    """Per-chunk magnitude of the terms the coefficient is built from,
    w * (|A| rho + k (|lp - blp| + 1)), shape (n_groups, G, C).

    The coefficient w (-A rho + k (lp - blp)) cancels when the KL term
    offsets the surrogate term; its error is then set by these terms (and
    the lp error through d coeff / d lp = w (-A rho + k)), not by its own
    value.  Tolerances scale with max(|coeff|, this)."""
    from .grpo_oracle import compute_advantages
    lp = np.asarray(lp_chunk, dtype=np.float64)
    n_groups, G, C = lp.shape
    bl = np.asarray(blp, dtype=np.float32).astype(np.float64).reshape(lp.shape)
    rw = np.asarray(rewards, dtype=np.float32).reshape(n_groups, G)
    A = np.stack([compute_advantages(rw[k], adv_eps) for k in range(n_groups)])
    diff = lp - bl
    rho = np.exp(diff)
    w = 1.0 / (n_groups * G * C)
    return w * (np.abs(A)[:, :, None] * rho + kl_coeff * (np.abs(diff) + 1.0))


def row_condition(coeff, term_scale, T):
    """Per-row factor >= 1 by which a row's relative tolerance widens when
    its chunk coefficient cancels (term_scale / |coeff|), repeated over the
    chunk's T rows; rows of zero coefficients get 1 (they must be exact)."""
    c = np.abs(np.asarray(coeff, dtype=np.float64)).reshape(-1)
    s = np.asarray(term_scale, dtype=np.float64).reshape(-1)
    f = np.where(c > 0, np.maximum(1.0, s / np.where(c > 0, c, 1.0)), 1.0)
    return np.repeat(f, T)


def assert_dlogits_close(got, want, rtol: float, floor: float = 1e-3, row_cond=None) -> dict:
    row_l2, elem, bad_zero = dlogits_errors(got, want, floor, row_cond)
    assert bad_zero == 0, f"{bad_zero} rows with a zero oracle gradient are not exactly zero"
    assert row_l2 <= rtol, f"row-wise relative L2 error {row_l2:.3g} > {rtol:g}"
    assert elem <= rtol, f"element-wise relative error {elem:.3g} > {rtol:g} (|want| >= {floor:g} row max)"
    return {"row_l2": row_l2, "elem": elem}
