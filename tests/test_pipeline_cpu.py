"""Host logic of xd.Pipeline on CPU (no GPU): results come back in submission order, every context
is reused, at most n_inflight calls run at once, and an error in one call reaches its future."""
import threading
import time

import pytest


def test_pipeline_order_concurrency_and_errors(monkeypatch):
    import paper_2309_07270_b200 as xd

    state = {"active": 0, "peak": 0, "made": 0}
    lock = threading.Lock()

    class FakeAligner:
        def __init__(self, **kw):
            with lock:
                state["made"] += 1
            self.closed = False

        def align(self, seqA, offA, pairs, k, X, **kw):
            with lock:
                state["active"] += 1
                state["peak"] = max(state["peak"], state["active"])
            time.sleep(0.01 * (pairs % 3))
            with lock:
                state["active"] -= 1
            if pairs == 7:
                raise ValueError("bad batch")
            return ("res", pairs), ("cells", pairs)

        def close(self):
            self.closed = True

    monkeypatch.setattr(xd, "Aligner", FakeAligner)
    with xd.Pipeline(n_inflight=3) as pl:
        jobs = [dict(seqA=None, offA=None, pairs=i, k=17, X=15) for i in range(12) if i != 7]
        outs = pl.map(jobs)
        assert [o[0][1] for o in outs] == [j["pairs"] for j in jobs]
        fut = pl.submit(None, None, 7, k=17, X=15)
        with pytest.raises(ValueError):
            fut.result()
        assert pl.submit(None, None, 5, k=17, X=15).result()[1] == ("cells", 5)   # contexts still usable
    assert state["made"] == 3 and 1 <= state["peak"] <= 3
