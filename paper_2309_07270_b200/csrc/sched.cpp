// sched.cpp -- L3 scheduler: CELLS sharding and the paper's token-ring
// policies (§III-B/C/D, Alg. 1).  Host-only C++; see sched.h.
//
// Token protocol.  Alg. 1 passes a token along a ring of the ranks that still
// have work at the current batch level (l.18-30, "traversing in a ring-array
// fashion", l.167).  Read literally (source-matched MPI_Recv) it deadlocks when
// the last ring member of batch b has no batch b+1: e.g. batch counts [2,2,1]
// -- rank 2 sends its batch-1 token to rank 0, while rank 0 waits at batch 2
// for rank 1, which waits for rank 0.  DESIGN.md reading Q21: the token visits
// turns in the order (batch, iteration, rank) over the ranks with work at that
// batch, i.e. Alg. 1's ring within a batch (xdrop_ring_left/right) and, at the
// wrap-around that ends a batch level, the first member of the next level's
// ring.  Every batch has exactly c iterations (empty sub-batches are no-op
// turns), so every member of a level takes the same number of turns.
#include "sched.h"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <map>
#include <mutex>
#include <queue>
#include <thread>
#include <utility>
#include <vector>

namespace {

using clk = std::chrono::steady_clock;

struct Mailbox {   // MPI_Send (buffered) / MPI_Recv (blocking, source-matched)
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::queue<int64_t>> q;
  int64_t sent = 0;
  void send(int src, int dst, int64_t payload) {
    {
      std::lock_guard<std::mutex> lk(mu);
      q[{src, dst}].push(payload);
      ++sent;
    }
    cv.notify_all();
  }
  int64_t recv(int src, int dst) {
    std::unique_lock<std::mutex> lk(mu);
    auto key = std::make_pair(src, dst);
    cv.wait(lk, [&] { auto it = q.find(key); return it != q.end() && !it->second.empty(); });
    int64_t v = q[key].front();
    q[key].pop();
    return v;
  }
};

struct Tracer {
  std::mutex mu;
  clk::time_point t0 = clk::now();
  std::vector<xdrop_trace_event> ev;
  int running = 0, max_running = 0;
  double now_ms() const { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }
  double begin() {
    std::lock_guard<std::mutex> lk(mu);
    ++running;
    max_running = std::max(max_running, running);
    return now_ms();
  }
  void end(int rank, int gpu, int batch, int sub, int64_t n, double t_begin) {
    std::lock_guard<std::mutex> lk(mu);
    --running;
    xdrop_trace_event e;
    e.rank = rank; e.gpu = gpu; e.batch = batch; e.sub = sub; e.n_pairs = n; e.t0_ms = t_begin; e.t1_ms = now_ms();
    ev.push_back(e);
  }
};

// LPT: assign items (by descending w) to the least-loaded of m bins.
std::vector<std::vector<int64_t>> lpt(const int64_t* idx, int64_t n, const int64_t* w, int m) {
  std::vector<int64_t> order(idx, idx + n);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return w[a] > w[b]; });
  std::vector<std::vector<int64_t>> bins((size_t)m);
  using E = std::pair<int64_t, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
  for (int g = 0; g < m; ++g) heap.push({0, g});
  for (int64_t t : order) {
    E e = heap.top(); heap.pop();
    bins[(size_t)e.second].push_back(t);
    heap.push({e.first + w[t], e.second});
  }
  return bins;
}

// Equal chunks per rank (remainder to the lowest ranks), then
// batches of batch_size, each split into c near-equal sub-batches, larger
// first.  Empty sub-batches are kept (no-op turns, reading Q21).
struct RankWork {
  std::vector<std::vector<std::vector<int64_t>>> batches;   // [batch][sub] -> pair indices
};

std::vector<RankWork> partition(int64_t n, int n_ranks, int batch_size, int c) {
  std::vector<RankWork> R((size_t)n_ranks);
  int64_t pos = 0;
  for (int r = 0; r < n_ranks; ++r) {
    const int64_t cnt = n / n_ranks + (r < n % n_ranks ? 1 : 0);
    for (int64_t b0 = 0; b0 < cnt; b0 += batch_size) {
      const int64_t bs = std::min<int64_t>(batch_size, cnt - b0);
      std::vector<std::vector<int64_t>> subs((size_t)c);
      int64_t q = pos + b0;
      for (int s = 0; s < c; ++s) {
        const int64_t ss = bs / c + (s < bs % c ? 1 : 0);
        for (int64_t u = 0; u < ss; ++u) subs[(size_t)s].push_back(q + u);
        q += ss;
      }
      R[(size_t)r].batches.push_back(std::move(subs));
    }
    pos += cnt;
  }
  return R;
}

// Turn order within one ring (members sorted), reading Q21.
struct Ring {
  std::vector<int> members;        // rank ids
  std::vector<int> counts;         // batches per member (same order)
  int turns_per_batch;             // c (one2all/one2one) or 1 (opt)
  // position of rank in members
  int pos(int rank) const {
    return (int)(std::lower_bound(members.begin(), members.end(), rank) - members.begin());
  }
  // next turn after (batch b, iteration it) of member index u; returns member index or -1
  int next(int u, int b, int it, int& nb, int& nit) const {
    const int n = (int)members.size();
    for (int v = u + 1; v < n; ++v) if (counts[(size_t)v] >= b) { nb = b; nit = it; return v; }
    // wrap: next iteration of the same batch, else next batch level
    int bb = b, ii = it + 1;
    if (ii > turns_per_batch) { bb = b + 1; ii = 1; }
    for (int v = 0; v < n; ++v) if (counts[(size_t)v] >= bb) { nb = bb; nit = ii; return v; }
    return -1;
  }
  int prev(int u, int b, int it) const {
    for (int v = u - 1; v >= 0; --v) if (counts[(size_t)v] >= b) return v;
    int bb = b, ii = it - 1;
    if (ii < 1) { bb = b - 1; ii = turns_per_batch; }
    if (bb < 1) return -1;
    const int n = (int)members.size();
    for (int v = n - 1; v >= 0; --v) if (counts[(size_t)v] >= bb) return v;
    return -1;
  }
};

}  // namespace

// ------------------------------------------------- Alg. 1 helpers (literal)
int xdrop_left_predecessor(int rank, int batch, const int* counts, int n) {
  int left = (rank - 1 + n) % n;
  while (batch > counts[left] && left != rank) left = (left - 1 + n) % n;
  return left == rank ? -1 : left;
}
int xdrop_right_successor(int rank, int batch, const int* counts, int n) {
  int right = (rank + 1) % n;
  while (batch > counts[right] && right != rank) right = (right + 1) % n;
  return right == rank ? -1 : right;
}

static int run_cells(const xdrop_sched_cfg& cfg, const int64_t* w, int64_t n, const xdrop_runner& run,
                     Tracer& tr) {
  std::vector<int64_t> all((size_t)n);
  for (int64_t t = 0; t < n; ++t) all[(size_t)t] = t;
  auto bins = lpt(all.data(), n, w, cfg.m);
  std::vector<int> rcs((size_t)cfg.m, 0);
  std::vector<std::thread> th;
  for (int g = 0; g < cfg.m; ++g) {
    th.emplace_back([&, g] {
      const auto& b = bins[(size_t)g];
      const double t0 = tr.begin();
      rcs[(size_t)g] = run(g, b.data(), (int64_t)b.size());
      tr.end(0, g, 0, 0, (int64_t)b.size(), t0);
    });
  }
  for (auto& t : th) t.join();
  for (int r : rcs) if (r) return r;
  return 0;
}

static int run_rings(const xdrop_sched_cfg& cfg, const int64_t* w, int64_t n, const xdrop_runner& run,
                     Tracer& tr, xdrop_sched_stats* st) {
  const int N = cfg.n_ranks, m = cfg.m, c = cfg.subbatches;
  const bool one2all = cfg.policy == XDROP_POLICY_ONE2ALL;
  const bool opt = cfg.policy == XDROP_POLICY_OPT_ONE2ONE;
  std::vector<RankWork> work = partition(n, N, cfg.batch_size, c);
  // rings: one global ring (one2all) or one per pipeline g = r mod m
  const int n_rings = one2all ? 1 : std::min(m, N);
  std::vector<Ring> rings((size_t)n_rings);
  for (int r = 0; r < N; ++r) {
    Ring& R = rings[(size_t)(one2all ? 0 : r % m)];
    R.members.push_back(r);
    R.counts.push_back((int)work[(size_t)r].batches.size());
    R.turns_per_batch = opt ? 1 : c;
  }
  Mailbox mb, ex;
  std::mutex err_mu;
  int first_rc = 0;
  auto note = [&](int rc) { if (rc) { std::lock_guard<std::mutex> lk(err_mu); if (!first_rc) first_rc = rc; } };

  auto turn_gpu = [&](int rank, int b, int s, const std::vector<int64_t>& idx) {
    if (idx.empty()) return;
    if (one2all) {         // the holder spreads its sub-batch over all GPUs
      auto bins = lpt(idx.data(), (int64_t)idx.size(), w, m);
      std::vector<std::thread> th;
      for (int g = 0; g < m; ++g) {
        if (bins[(size_t)g].empty()) continue;
        th.emplace_back([&, g] {
          const double t0 = tr.begin();
          note(run(g, bins[(size_t)g].data(), (int64_t)bins[(size_t)g].size()));
          tr.end(rank, g, b, s, (int64_t)bins[(size_t)g].size(), t0);
        });
      }
      for (auto& t : th) t.join();
    } else {
      const int g = rank % m;
      const double t0 = tr.begin();
      note(run(g, idx.data(), (int64_t)idx.size()));
      tr.end(rank, g, b, s, (int64_t)idx.size(), t0);
    }
  };

  std::vector<std::thread> th;
  for (int r = 0; r < N; ++r) {
    th.emplace_back([&, r] {
      const Ring& R = rings[(size_t)(one2all ? 0 : r % m)];
      const int u = R.pos(r);
      const int nr = (int)R.members.size();
      // Alg. 1 l.5-11: all-to-all exchange of batch counts within the ring
      const int mine = R.counts[(size_t)u];
      for (int v = 0; v < nr; ++v)
        if (v != u) ex.send(r, R.members[(size_t)v], mine);
      for (int v = 0; v < nr; ++v)
        if (v != u) (void)ex.recv(R.members[(size_t)v], r);
      const int B = mine;
      for (int b = 1; b <= B; ++b) {
        const int iters = opt ? 1 : c;
        for (int it = 1; it <= iters; ++it) {
          const int pv = R.prev(u, b, it);
          if (pv >= 0 && pv != u) (void)mb.recv(R.members[(size_t)pv], r);   // l.18-24 implicit barrier
          const auto& subs = work[(size_t)r].batches[(size_t)(b - 1)];
          if (opt) for (int s = 0; s < c; ++s) turn_gpu(r, b, s + 1, subs[(size_t)s]);
          else turn_gpu(r, b, it, subs[(size_t)(it - 1)]);
          int nb, nit;
          const int nx = R.next(u, b, it, nb, nit);
          if (nx >= 0 && nx != u) mb.send(r, R.members[(size_t)nx], 1);       // l.26-30
        }
      }
    });
  }
  for (auto& t : th) t.join();
  if (st) { st->handoffs = mb.sent; st->exchange_msgs = ex.sent; }
  return first_rc;
}

int xdrop_sched_run(const xdrop_sched_cfg& cfg, const int64_t* w, int64_t n, const xdrop_runner& run,
                    xdrop_sched_stats* st, std::vector<xdrop_trace_event>* trace) {
  Tracer tr;
  xdrop_sched_stats local{};
  int rc;
  if (cfg.policy == XDROP_POLICY_CELLS || cfg.n_ranks < 1) rc = run_cells(cfg, w, n, run, tr);
  else rc = run_rings(cfg, w, n, run, tr, &local);
  double lo = 1e300, hi = 0;
  for (const auto& e : tr.ev) {
    lo = std::min(lo, e.t0_ms); hi = std::max(hi, e.t1_ms);
    if (e.gpu >= 0 && e.gpu < 16) local.busy_ms[e.gpu] += e.t1_ms - e.t0_ms;
  }
  local.turns = (int64_t)tr.ev.size();
  local.span_ms = tr.ev.empty() ? 0.0 : hi - lo;
  local.max_concurrent = tr.max_running;
  local.n_events = (int32_t)tr.ev.size();
  if (st) *st = local;
  if (trace) *trace = std::move(tr.ev);
  return rc;
}

extern "C" int xdrop_ring_left(int rank, int batch, const int* counts, int n) {
  if (!counts || n < 1 || rank < 0 || rank >= n) return -1;
  return xdrop_left_predecessor(rank, batch, counts, n);
}
extern "C" int xdrop_ring_right(int rank, int batch, const int* counts, int n) {
  if (!counts || n < 1 || rank < 0 || rank >= n) return -1;
  return xdrop_right_successor(rank, batch, counts, n);
}

// Reading Q21's token order over one ring (members 0..n-1 with counts[v] batches each, turns_per_batch
// turns per batch): the member owning the turn after / before (batch b, iteration it) of member u.
// Exported so that the multi-process rank mode (ranks.py) uses this one implementation.
extern "C" int xdrop_ring_turn_next(int u, int b, int it, const int* counts, int n, int turns_per_batch,
                                    int* next_b, int* next_it) {
  if (!counts || n < 1 || u < 0 || u >= n || turns_per_batch < 1) return -1;
  Ring r;
  r.members.resize((size_t)n);
  for (int v = 0; v < n; ++v) r.members[(size_t)v] = v;
  r.counts.assign(counts, counts + n);
  r.turns_per_batch = turns_per_batch;
  int nb = 0, nit = 0;
  const int v = r.next(u, b, it, nb, nit);
  if (next_b) *next_b = nb;
  if (next_it) *next_it = nit;
  return v;
}
extern "C" int xdrop_ring_turn_prev(int u, int b, int it, const int* counts, int n, int turns_per_batch) {
  if (!counts || n < 1 || u < 0 || u >= n || turns_per_batch < 1) return -1;
  Ring r;
  r.members.resize((size_t)n);
  for (int v = 0; v < n; ++v) r.members[(size_t)v] = v;
  r.counts.assign(counts, counts + n);
  r.turns_per_batch = turns_per_batch;
  return r.prev(u, b, it);
}

extern "C" int64_t xdrop_sched_simulate(int m, int policy, int n_ranks, int batch_size, int subbatches,
                                        const int64_t* w, int64_t n, double ns_per_unit, xdrop_sched_stats* st,
                                        xdrop_trace_event* trace, int64_t cap, int32_t* gpu_of_pair) {
  if (m < 1 || m > 16 || policy < 0 || policy > 3 || n < 0 || (n > 0 && !w)) return XDROP_EINVAL;
  xdrop_sched_cfg cfg{m, policy, std::max(1, n_ranks), batch_size > 0 ? batch_size : 10000,
                      subbatches > 0 ? subbatches : 1};
  std::vector<int> busy((size_t)m, 0);
  std::mutex mu;
  bool overlap = false;
  auto runner = [&](int gpu, const int64_t* idx, int64_t k) -> int {
    {
      std::lock_guard<std::mutex> lk(mu);
      if (busy[(size_t)gpu]++) overlap = true;   // two turns on one GPU at once
    }
    double units = 0;
    for (int64_t t = 0; t < k; ++t) {
      units += (double)w[idx[t]];
      if (gpu_of_pair) gpu_of_pair[idx[t]] = gpu;
    }
    if (ns_per_unit > 0) std::this_thread::sleep_for(std::chrono::nanoseconds((int64_t)(units * ns_per_unit)));
    {
      std::lock_guard<std::mutex> lk(mu);
      --busy[(size_t)gpu];
    }
    return 0;
  };
  std::vector<xdrop_trace_event> tv;
  int rc = xdrop_sched_run(cfg, w, n, runner, st, &tv);
  if (rc) return rc;
  if (overlap) return XDROP_ESTATE;
  for (int64_t t = 0; t < (int64_t)tv.size() && t < cap; ++t) trace[t] = tv[(size_t)t];
  return (int64_t)tv.size();
}
