"""f1: the paper's schedulers with real OS processes as ranks (gloo
point-to-point messages, Alg. 1), checked by trace-only verifiers, plus mutation
tests showing each verifier catches its fault."""
import copy

import numpy as np
import pytest

from paper_2309_07270_b200 import ranks as R


def test_token_order_unit():
    ring = R.Ring([0, 1, 2], [2, 2, 1], 1)          # the counts that deadlock Alg. 1 read literally
    seq, u, b, it = [], 0, 1, 1
    while u >= 0:
        seq.append((ring.members[u], b))
        nx = ring.next(u, b, it)
        if nx < 0:
            break
        nb = b + (1 if nx <= u else 0)
        assert ring.prev(nx, nb, 1) == u              # prev inverts next
        u, b = nx, nb
    assert seq == [(0, 1), (1, 1), (2, 1), (0, 2), (1, 2)]
    assert R.subbatches(0, 25000, 10000, 4)[2][0].size == 1250
    assert [len(s) for s in R.subbatches(0, 10001, 10000, 3)[1]] == [1, 0, 0]   # empty kept (Q22)


@pytest.mark.parametrize("policy", R.POLICIES)
@pytest.mark.parametrize("n_ranks,m,c,n", [(3, 1, 2, 41), (4, 2, 3, 57)])
def test_multiprocess_schedule_verifies(policy, n_ranks, m, c, n):
    seq = np.frombuffer(b"ACGT" * 8, np.uint8)
    off = np.array([0, 32], np.int64)
    pairs = np.zeros((n, 4), np.int32)
    _, _, turns, met, bad = R.spawn(n_ranks, policy, m, seq, off, pairs, batch_size=4, c=c, use_gpu=False,
                                    sleep_ns_per_pair=2e5, timeout=120)
    assert bad == [], bad
    assert met["turns"] > 0
    if policy == "one2all":
        assert met["exchange_msgs"] == n_ranks * (n_ranks - 1)


def _fake_trace(policy="one2one", n_ranks=3, m=1, c=2, n=24, bs=4):
    turns, t = [], 0.0
    rings = {}
    for r in range(n_ranks):
        lo, hi = R.rank_chunk(n, n_ranks, r)
        rings.setdefault(0 if policy == "one2all" else r % m, []).append((r, R.subbatches(lo, hi, bs, c)))
    for rid, mem in rings.items():
        nb = max(len(w) for _, w in mem)
        for b in range(1, nb + 1):
            for it in range(1, c + 1):
                for r, w in mem:
                    if len(w) >= b:
                        idx = w[b - 1][it - 1]
                        turns.append(R.Turn(r, r % m, b, it, int(idx.size), t, t + 1.0))
                        t += 1.0
    return turns


def test_verifiers_pass_and_catch_mutations():
    base = _fake_trace()
    assert R.verify(base, 24, 3, 1, "one2one", 4, 2) == []
    overlap = copy.deepcopy(base); overlap[3].t0 -= 0.5                      # mutual exclusion
    assert any("overlap" in v for v in R.verify(overlap, 24, 3, 1, "one2one", 4, 2))
    dup = copy.deepcopy(base) + [copy.deepcopy(base[2])]                      # duplicate
    dup[-1].t0 += 100; dup[-1].t1 += 100
    assert any("duplicate" in v for v in R.verify(dup, 24, 3, 1, "one2one", 4, 2))
    miss = copy.deepcopy(base); del miss[4]                                   # omission
    assert any("missing" in v for v in R.verify(miss, 24, 3, 1, "one2one", 4, 2))
    swap = copy.deepcopy(base)                                                # order swap
    swap[0].t0, swap[1].t0 = swap[1].t0, swap[0].t0
    swap[0].t1, swap[1].t1 = swap[0].t0 + 1, swap[1].t0 + 1
    assert any("order" in v for v in R.verify(swap, 24, 3, 1, "one2one", 4, 2))
    aff = copy.deepcopy(_fake_trace(m=2)); aff[0].gpu = 1 - aff[0].gpu        # pipeline affinity
    assert any("affinity" in v for v in R.verify(aff, 24, 3, 2, "one2one", 4, 2))
