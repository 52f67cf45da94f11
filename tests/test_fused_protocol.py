"""Model check of the fused token-loss kernel's warp/mbarrier protocol
(csrc/token_loss.cu, tok_fused_bf16_kernel) on the CPU.

Every warp role is a generator that waits on simulated mbarriers with the
hardware's parity semantics; random interleavings must (a) finish, (b) never
let a barrier run two phases ahead of a waiter (parity aliasing), and (c)
never let a SMEM slot be overwritten before its consumer read it.  The op
sequence `op_of` mirrors the CUDA function of the same name.
"""

import random

import pytest

S = 3  # kFusedStages


def op_of(n, nloc, L):
    Le = min(nloc, L)
    if n < Le:
        return False, n
    m = n - Le
    pairs = nloc - Le
    if m < 2 * pairs:
        return (m & 1) == 1, (m >> 1) if (m & 1) else Le + (m >> 1)
    return True, pairs + (m - 2 * pairs)


class Bar:
    def __init__(self, cnt):
        self.cnt, self.pend, self.phase = cnt, cnt, 0

    def arrive(self):
        self.pend -= 1
        if self.pend == 0:
            self.phase += 1
            self.pend = self.cnt

    def done(self, idx):
        assert idx <= self.phase + 1 and self.phase <= idx + 1, "parity aliasing"
        return (self.phase & 1) != (idx & 1)


def coef_order(nops, nloc, L):
    """The coefficient warp handles B(k) before the A(k+L) that precedes it
    in the op sequence (its coefficient never depends on that A), so the
    compute warps never wait for the tail of the row they just finished."""
    order = []
    n = 0
    Le = min(nloc, L)
    pair_end = Le + 2 * (nloc - Le)
    while n < nops:
        isb, _ = op_of(n, nloc, L)
        nxt = op_of(n + 1, nloc, L)[0] if n + 1 < nops else None
        if not isb and nxt and Le >= 2 and n + 1 < pair_end:
            order += [n + 1, n]
            n += 2
        else:
            order.append(n)
            n += 1
    return order


def simulate(nloc, L, seed, write_dl=True):
    """Roles as generators (v8 protocol): the loader streams every op's row
    into a 3-stage SMEM ring; compute warps free a stage as soon as they have
    read it (dlogits leave through 16-byte stores from registers); A-row
    partials go through an 8-slot ring guarded by afree; B coefficients
    through a 3-slot ring guarded by adoneB."""
    AS = 8
    rnd = random.Random(seed)
    nops = 2 * nloc if write_dl else nloc
    Lx = L if write_dl else 1 << 30
    full = [Bar(1) for _ in range(S)]
    empty = [Bar(16) for _ in range(S)]
    ad_a = [Bar(16) for _ in range(AS)]
    a_free = [Bar(1) for _ in range(AS)]
    ad_b = [Bar(16) for _ in range(S)]
    cf_b = [Bar(1) for _ in range(S)]
    slot_p, slot_c, rows_b = [None] * AS, [None] * S, []
    stage_owner = [None] * S

    def wait(b, idx):
        while not b.done(idx):
            yield 1

    def loader():
        for n in range(nops):
            if n >= S:
                yield from wait(empty[n % S], n // S - 1)
            assert stage_owner[n % S] is None, "stage reloaded while in use"
            stage_owner[n % S] = n
            full[n % S].arrive()

    tails = set()
    readers = {}

    def coef():
        a = b = 0
        for n in coef_order(nops, nloc, Lx):
            isb, k = op_of(n, nloc, Lx)
            if isb:
                # the chunk of row k spans rounds k and k+1: both tails of this
                # CTA must already be published (else: cross-CTA deadlock)
                assert k in tails and (k + 1 >= nloc or k + 1 in tails), (k, sorted(tails))
                if b >= S:
                    yield from wait(ad_b[(b - S) % S], (b - S) // S)
                slot_c[b % S] = b
                cf_b[b % S].arrive()
                b += 1
            else:
                yield from wait(ad_a[a % AS], a // AS)
                assert slot_p[a % AS] == a
                a_free[a % AS].arrive()
                tails.add(k)
                a += 1

    def compute(w):
        a = b = 0
        for n in range(nops):
            isb, k = op_of(n, nloc, Lx)
            yield from wait(full[n % S], n // S)
            assert stage_owner[n % S] == n
            readers[n] = readers.get(n, 0) + 1
            if readers[n] == 16:
                stage_owner[n % S] = None  # last reader done (arrives below)
            if not isb:
                empty[n % S].arrive()
                if a >= AS:
                    yield from wait(a_free[a % AS], (a - AS) // AS)
                if w == 0:
                    slot_p[a % AS] = a
                ad_a[a % AS].arrive()
                a += 1
            else:
                yield from wait(cf_b[b % S], b // S)
                assert slot_c[b % S] == b
                if w == 0:
                    rows_b.append(k)
                empty[n % S].arrive()
                ad_b[b % S].arrive()
                b += 1

    gens = [loader(), coef()] + [compute(w) for w in range(16)]
    live = list(gens)
    for _ in range(400000):
        if not live:
            break
        g = rnd.choice(live)
        try:
            next(g)
        except StopIteration:
            live.remove(g)
    assert not live, "protocol deadlocked"
    if write_dl:
        assert sorted(rows_b) == list(range(nloc))


@pytest.mark.parametrize("nloc", [1, 2, 3, 4, 7, 13, 20])
@pytest.mark.parametrize("L", [1, 2, 3, 4])
def test_protocol_completes_without_aliasing(nloc, L):
    for seed in range(3):
        simulate(nloc, L, seed)


def test_forward_only_protocol():
    for nloc in (1, 5, 13):
        simulate(nloc, 3, 0, write_dl=False)


def test_coef_order_is_a_permutation():
    for nloc in range(1, 20):
        for L in (1, 2, 3):
            assert sorted(coef_order(2 * nloc, nloc, L)) == list(range(2 * nloc))


def test_op_sequence_is_a_permutation():
    for nloc in range(1, 30):
        for L in (1, 2, 3, 5):
            ops = [op_of(n, nloc, L) for n in range(2 * nloc)]
            assert sorted(k for b, k in ops if not b) == list(range(nloc))
            assert sorted(k for b, k in ops if b) == list(range(nloc))
            # A(k) always precedes B(k), and A(k + L) precedes B(k)
            pos = {op: i for i, op in enumerate(ops)}
            for k in range(nloc):
                assert pos[(False, k)] < pos[(True, k)]
                if k + L < nloc:
                    assert pos[(False, k + L)] < pos[(True, k)]
