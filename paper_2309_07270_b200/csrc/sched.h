// sched.h -- L3 multi-GPU scheduler (host-only C++, no CUDA dependency).
//
// Policies (include/xdrop.h xdrop_policy):
//  CELLS        pairs sorted by estimated cost, LPT-assigned to the m GPUs, one
//               host thread per GPU (the default; no paper counterpart).
//  ONE2ALL      PAPER.md §III-B + Alg. 1: n logical ranks own equal chunks of
//               pairs, split into batches of batch_size and c
//               sub-batches; a token ring (Alg. 1 l.18-30)
//               serialises the ranks; the holder spreads its sub-batch over
//               all m GPUs.
//  ONE2ONE      PAPER.md §III-C: rank r drives GPU r mod m; one ring per
//               pipeline, token per sub-batch (l.186 "n mod m").
//  OPT_ONE2ONE  PAPER.md §III-D: as ONE2ONE, token held for a whole batch.
// Logical ranks are host threads; MPI_Send/MPI_Recv become a mailbox of
// per-(src,dst) message counters (buffered send, blocking source-matched
// receive -- the semantics Alg. 1 relies on).
#pragma once
#include <cstdint>
#include <functional>
#include <vector>

#include "../../include/xdrop.h"

struct xdrop_sched_cfg {
  int m;            // GPUs
  int policy;       // xdrop_policy
  int n_ranks;      // logical ranks (ONE2ALL / ONE2ONE / OPT)
  int batch_size;   // pairs per batch
  int subbatches;   // c
};

// Runs pairs idx[0..n) on GPU `gpu`; returns 0 or an xdrop_status.
using xdrop_runner = std::function<int(int gpu, const int64_t* idx, int64_t n)>;

// w: estimated cost per pair (> 0).  Fills st (may be null).
int xdrop_sched_run(const xdrop_sched_cfg& cfg, const int64_t* w, int64_t n, const xdrop_runner& run,
                    xdrop_sched_stats* st, std::vector<xdrop_trace_event>* trace);

// ---- pure helpers (Alg. 1 ring search; SPEC.md:221-249 test vectors) -------
// Literal Alg. 1 l.18-30: walk down (up) from rank-1 (rank+1) with wrap over
// ranks 0..n-1; return the first r with batch <= counts[r], or -1 if the walk
// returns to `rank`.
int xdrop_left_predecessor(int rank, int batch, const int* counts, int n);
int xdrop_right_successor(int rank, int batch, const int* counts, int n);
