"""The paper's experiment shape on one box: N OS-process ranks share the
GPU(s) under each policy; reports the alignment span (Table I "Alignment Time" analog),
message counts and the verifier verdict.  usage: python tools/ranks_demo.py [ranks] [m]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_07270_b200 import ranks as R  # noqa: E402
from synth import workload as W  # noqa: E402

def main():
    n_ranks = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    w = W.config("ecoli")
    print(f"| policy | ranks | GPUs | c | span ms | handoffs | exchange msgs | turns | verifier |")
    print("|---|---|---|---|---|---|---|---|---|")
    for policy, c in [("one2all", 1), ("one2one", 1), ("opt_one2one", 1), ("one2one", 4), ("opt_one2one", 4)]:
        t = time.time()
        out, cells, turns, met, bad = R.spawn(n_ranks, policy, m, w.seq, w.offsets, w.pairs, batch_size=10000, c=c,
                                              params=dict(k=w.k, X=w.X), use_gpu=True, timeout=1800)
        print(f"| {policy} | {n_ranks} | {m} | {c} | {met['span_ms']:.1f} | {met['handoffs']} | {met['exchange_msgs']} | "
              f"{met['turns']} | {'pass' if not bad else bad[:2]} |", flush=True)


if __name__ == "__main__":
    main()
