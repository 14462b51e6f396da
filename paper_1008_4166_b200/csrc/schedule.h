// Ring schedule of the 2F driver: a host-side restatement of the reference's
// strategy steppers (pkg/src/hjacobi/strategies.py:58-136).  Data-independent,
// so the whole sequence of block pairs can be generated before the solve.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace hjb {

struct StepPlan {
  int32_t snd_rnk, snd_blk, rcv_rnk, rcv_blk;
};

class RingSchedule {
 public:
  // strategy: 0 = modulus, 1 = round robin (include/hjb200.h)
  RingSchedule(int strategy, int p);
  int p() const { return p_; }
  int nbl() const { return nbl_; }
  int steps_per_sweep() const { return strategy_ == 0 ? 2 * p_ : 2 * p_ - 1; }
  // (i_blk, j_blk) held by worker q (1-based block indices)
  int i_blk(int q) const { return st_[q].i_blk; }
  int j_blk(int q) const { return st_[q].j_blk; }
  // one step for every worker (strategies.py:75-136); nsweep selects the
  // neighbour direction (strategies.py:69-72).  Throws on an inconsistent
  // exchange (strategies.py:164-175).
  std::vector<StepPlan> advance(int nsweep);

 private:
  struct State { int ip, jp, i_blk, j_blk; };
  void step_modulus(State &s, int &snd, int &rcv) const;
  void step_round_robin(State &s, int &snd, int &rcv) const;
  int strategy_, p_, nbl_;
  std::vector<State> st_;
};

// ---- several GPUs: ring ranks are split into contiguous ranges per GPU ----
// GPU g hosts workers [workers_lo(g), workers_lo(g+1)).
inline int workers_lo(int p, int world, int g) { return int((int64_t(g) * p) / world); }
int gpu_of_worker(int p, int world, int q);

// One block column that crosses a GPU boundary after a step (0-based block).
struct Xfer {
  int blk, peer;
  bool send;
};
// The transfers of GPU `rank` implied by one step's plans: worker q on this
// GPU sends snd_blk to snd_rnk and receives rcv_blk from rcv_rnk
// (parallel.py:212-221); only partners on another GPU need a transfer.
void step_transfers(const std::vector<StepPlan> &plans, int p, int world, int rank, std::vector<Xfer> &out);

// GPU holding each block (0-based) after `sweeps` whole sweeps of the ring
// (the layout the reference reassembles from, parallel.py:299-301).  The
// layout has period 2 sweeps, so odd and even sweep counts differ.
std::vector<int> final_block_owners(int strategy, int p, int world, int sweeps);

}  // namespace hjb
