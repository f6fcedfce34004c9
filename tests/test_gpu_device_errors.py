"""Device-API validation (xdrop_align_batch_device, include/xdrop.h): invalid pairs must return
XDROP_ESEED with the smallest offending pair index, WITHOUT any band kernel touching the bad pair
(the queue is emptied on the device by scan_kernel before the band kernels start), and the context
must stay usable.  Each case runs in a child process against libxdrop.so and against the
bounds-checked build (which traps on any out-of-pool read, so a kernel that dereferenced the bad id
or position would turn the expected ESEED into ECUDA).  Run parameters the ABI validates:
PAPER.md:221-224 (§IV-A: k, --ga X, scoring)."""
import os
import subprocess
import sys
import textwrap

import pytest

from test_gpu_checked import ROOT, child_env

pytestmark = pytest.mark.gpu

CHILD = textwrap.dedent("""
    import numpy as np
    import torch
    import oracle
    import paper_2309_07270_b200 as xd
    from synth import workload as W
    dev = torch.device("cuda:0")
    w = W.random_pairs_workload(seed=41, n_pairs=300, len_lo=200, len_hi=3000, k=17, X=15)
    seq = torch.from_numpy(w.seq).to(dev)
    off = torch.from_numpy(w.offsets).to(dev)
    n = w.n_pairs
    L = np.diff(w.offsets)
    ref, rcells = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, w.M, w.mu, w.g, w.X)
    F = ("score", "a_begin", "a_end", "b_begin", "b_end")

    def call(al, pairs_np, off_t=off, lenA=None):
        pairs = torch.from_numpy(np.ascontiguousarray(pairs_np, dtype=np.int32)).to(dev)
        out = torch.zeros((n, 5), dtype=torch.int32, device=dev)
        cells = torch.zeros(n, dtype=torch.int64, device=dev)
        al.align_device(seq, off_t, pairs, out, cells, k=w.k, X=w.X, lenA=lenA)
        return out.cpu().numpy(), cells.cpu().numpy()

    def good(al):
        o, c = call(al, w.pairs)
        for i, f in enumerate(F):
            assert np.array_equal(o[:, i], ref[f]), f
        assert np.array_equal(c, rcells)

    cases = []
    p = w.pairs.copy(); p[137, 0] = 1 << 30; p[200, 0] = -3; cases.append(("a_id huge", p, 137))
    p = w.pairs.copy(); p[55, 1] = len(L); cases.append(("b_id out of range", p, 55))
    p = w.pairs.copy(); p[9, 1] = (len(L) + 5) | -(1 << 31); cases.append(("RC b_id out of range", p, 9))
    p = w.pairs.copy(); p[77, 2] = -1; cases.append(("negative a_pos", p, 77))
    p = w.pairs.copy(); r = p[250, 1] & 0x7fffffff; p[250, 3] = L[r] - w.k + 1; cases.append(("seed past B end", p, 250))
    p = w.pairs.copy(); r = p[3, 0]; p[3, 2] = L[r] - w.k + 1; p[4, 2] = 1 << 29; cases.append(("seed past A end", p, 3))
    with xd.Aligner(devices=[0]) as al:
        good(al)
        for name, pairs, want in cases:
            try:
                call(al, pairs)
                raise SystemExit(f"{name}: no error")
            except xd.XdropError as e:
                assert e.status == -5, (name, e.status)
                assert al_index(al) == want, (name, al_index(al), want)
            good(al)                      # the context is still usable
            print("case ok", name, flush=True)
        # offsets beyond the pool: the last read ends past lenA
        last = len(L) - 1
        p = w.pairs.copy(); p[11, 0] = last; p[11, 2] = 0
        try:
            call(al, p, lenA=int(w.offsets[-1]) - 1)
            raise SystemExit("offsets past lenA: no error")
        except xd.XdropError as e:
            assert e.status == -5 and al_index(al) == 11, (e.status, al_index(al))
        good(al)
        print("case ok offsets", flush=True)
        # marshalling guards (ValueError before the C call)
        for bad in (torch.from_numpy(w.pairs.astype(np.int64)).to(dev),
                    torch.from_numpy(w.pairs).to(dev).t().contiguous().t()):
            try:
                al.align_device(seq, off, bad, torch.zeros((n, 5), dtype=torch.int32, device=dev), None,
                                k=w.k, X=w.X)
                raise SystemExit("guard missed")
            except ValueError:
                pass
    print("device errors ok")
""").replace("al_index(al)", "xd._native.lib.xdrop_last_error_index(al._h)")


@pytest.mark.parametrize("lib", ["libxdrop.so", "libxdrop_checked.so"])
def test_device_api_invalid_pairs(lib):
    path = os.path.join(ROOT, "paper_2309_07270_b200", lib)
    if lib == "libxdrop_checked.so":
        sys.path.insert(0, os.path.join(ROOT, "paper_2309_07270_b200"))
        try:
            import build as B
            B.build_checked()
        finally:
            sys.path.pop(0)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=child_env(path))
    assert r.returncode == 0 and "device errors ok" in r.stdout, (r.stdout[-3000:], r.stderr[-3000:])
