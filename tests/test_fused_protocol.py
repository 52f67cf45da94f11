"""Model check of the fused token-loss kernel's warp/mbarrier protocol
(csrc/token_loss.cu, tok_fused_kernel<TE, P>) on the CPU.

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


def simulate(nloc, L, seed, write_dl=True, W=4, P=1):
    """Roles as generators (v10 protocol): the loader streams every op's row
    into a 3-stage SMEM ring; compute warps free an A stage as soon as they
    have read it, write B rows in place and hand them to the store warp
    (bdone), which frees the stage once its bulk copy has read it (one
    arrival worth W on empty).  A-row partials go to the tail warp through an
    8-slot ring guarded by afree; the tail warp leaves (lse, target) in an
    8-row ring for the prep warp (tdone); B coefficients go through a 3-slot
    ring guarded by adoneB.  The prep warp's wait for the chunk to complete
    on all CTAs is modelled by waiting for this CTA's own tails of rows k and
    k + 1 (a chunk spans at most two consecutive rounds when T <= grid).
    With P pieces per row, ops walk virtual rows u = k P + p (lag L P); the
    tail consumes the P partial slots of a row, the prep hands the row's
    coefficient to each of its P B ops."""
    AS, RING = 8, 8
    rnd = random.Random(seed)
    nvr = nloc * P
    nops = 2 * nvr if write_dl else nvr
    Lx = L if write_dl else 1 << 30  # lag in pieces (>= 2P - 1, <= 8P - 1)
    full = [Bar(1) for _ in range(S)]
    empty = [Bar(W) for _ in range(S)]
    ad_a = [Bar(W) for _ in range(AS)]
    a_free = [Bar(1) for _ in range(AS)]
    tdone = [Bar(1) for _ in range(RING)]
    ad_b = [Bar(W) for _ in range(S)]
    cf_b = [Bar(1) for _ in range(S)]
    bdone = [Bar(W) for _ in range(S)]
    slot_p, slot_c, ring = [None] * AS, [None] * S, [None] * RING
    ring_read = set()
    stage_op = [None] * S
    done_ops = set()  # ops whose stage use is over (read for A, stored for B)
    readers, writers = {}, {}
    rows_b, tails = [], set()

    def wait(b, idx):
        while not b.done(idx):
            yield 1

    def loader():
        for n in range(nops):
            if n >= S:
                yield from wait(empty[n % S], n // S - 1)
                assert n - S in done_ops, "stage reloaded while in use"
            stage_op[n % S] = n
            full[n % S].arrive()

    def tail():
        for k in range(nloc):
            for pc in range(P):
                u = k * P + pc
                yield from wait(ad_a[u % AS], u // AS)
                assert slot_p[u % AS] == u
                a_free[u % AS].arrive()
            if write_dl:
                assert k < RING or (k - RING) in ring_read, "(lse, target) ring overrun"
                ring[k % RING] = k
                tdone[k % RING].arrive()
            tails.add(k)

    def prep():
        if not write_dl:
            return
        for k in range(nloc):
            while not (k in tails and (k + 1 >= nloc or k + 1 in tails)):
                yield 1  # chunk incomplete on "other CTAs"
            yield from wait(tdone[k % RING], k // RING)
            assert ring[k % RING] == k
            ring_read.add(k)
            for pc in range(P):
                u = k * P + pc
                if u >= S:
                    yield from wait(ad_b[u % S], (u - S) // S)
                slot_c[u % S] = u
                cf_b[u % S].arrive()

    def store():
        if not write_dl:
            return
        nb = 0
        for n in range(nops):
            isb, k = op_of(n, nvr, Lx)
            if not isb:
                continue
            yield from wait(bdone[nb % S], nb // S)
            assert stage_op[n % S] == n and writers.get(n) == W
            nb += 1
            done_ops.add(n)
            for _ in range(W):  # one arrival worth W
                empty[n % S].arrive()

    def compute(w):
        a = b = 0
        for n in range(nops):
            isb, k = op_of(n, nvr, Lx)
            yield from wait(full[n % S], n // S)
            assert stage_op[n % S] == n
            if not isb:
                readers[n] = readers.get(n, 0) + 1
                if readers[n] == W:
                    done_ops.add(n)
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
                writers[n] = writers.get(n, 0) + 1
                bdone[b % S].arrive()
                ad_b[b % S].arrive()
                b += 1

    gens = [loader(), tail(), prep(), store()] + [compute(w) for w in range(W)]
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
        assert sorted(rows_b) == list(range(nvr))


@pytest.mark.parametrize("nloc", [1, 2, 3, 4, 7, 13, 20])
@pytest.mark.parametrize("L", [2, 3, 4, 7])
def test_protocol_completes_without_aliasing(nloc, L):
    for seed in range(3):
        simulate(nloc, L, seed)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("nloc", [1, 2, 5, 11])
@pytest.mark.parametrize("lag", ["min", "mid", "max"])
def test_protocol_with_row_pieces(P, nloc, lag):
    L = {"min": 2 * P - 1, "mid": 4 * P, "max": 8 * P - 1}[lag]
    for seed in range(2):
        simulate(nloc, L, seed, P=P)


def test_forward_only_protocol():
    for nloc in (1, 5, 13):
        simulate(nloc, 3, 0, write_dl=False)


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
