// Host restatement of strategies.py:58-136 (see schedule.h).
#include "schedule.h"

#include <string>

namespace hjb {

RingSchedule::RingSchedule(int strategy, int p) : strategy_(strategy), p_(p), nbl_(2 * p) {
  if (p < 1) throw std::invalid_argument("p must be >= 1");
  if (strategy != 0 && strategy != 1) throw std::invalid_argument("unknown strategy");
  st_.resize(p);
  for (int q = 0; q < p; ++q) {  // antidiagonal start, strategies.py:58-66
    st_[q] = State{q + 1, nbl_ - q, q + 1, nbl_ - q};
  }
}

// strategies.py:75-92
void RingSchedule::step_modulus(State &s, int &snd, int &rcv) const {
  if (s.ip + s.jp > nbl_) {
    snd = s.i_blk;
    s.ip += 1;
    if (s.ip == s.jp) {
      s.ip -= nbl_ / 2;
      s.jp = s.ip;
    }
    s.i_blk = s.ip;
    rcv = s.i_blk;
  } else {
    snd = s.j_blk;
    s.jp += 1;
    s.j_blk = s.jp;
    rcv = s.j_blk;
  }
}

// strategies.py:95-136 (the reference's reconstruction of the modified
// round-robin stepper, including the swflag renumbering branch)
void RingSchedule::step_round_robin(State &s, int &snd, int &rcv) const {
  if (s.ip + s.jp > nbl_) {
    if (s.jp < nbl_) {
      snd = s.i_blk;
      s.ip += 1;
      if (s.ip < s.jp) {
        s.i_blk = s.ip;
        rcv = s.i_blk;
      } else {
        s.ip = s.jp;
        s.i_blk = s.j_blk;
        s.jp = nbl_;
        s.j_blk = nbl_;
        rcv = s.j_blk;
      }
    } else if (s.ip > nbl_ / 2) {
      snd = s.i_blk;
      s.ip = s.ip - nbl_ / 2 + 1;
      s.i_blk = s.ip;
      rcv = s.i_blk;
    } else {
      snd = s.j_blk;
      s.jp = s.ip + 1;
      s.j_blk = s.jp;
      rcv = s.j_blk;
    }
  } else {
    snd = s.j_blk;
    s.jp += 1;
    s.j_blk = s.jp;
    rcv = s.j_blk;
  }
}

std::vector<StepPlan> RingSchedule::advance(int nsweep) {
  std::vector<StepPlan> plans(p_);
  for (int q = 0; q < p_; ++q) {
    int snd = 0, rcv = 0;
    if (strategy_ == 0)
      step_modulus(st_[q], snd, rcv);
    else
      step_round_robin(st_[q], snd, rcv);
    // strategies.py:69-72: odd sweeps send to q-1 and receive from q+1
    int down = (p_ + q - 1) % p_, up = (p_ + q + 1) % p_;
    if (nsweep % 2)
      plans[q] = StepPlan{down, snd, up, rcv};
    else
      plans[q] = StepPlan{up, snd, down, rcv};
  }
  for (int q = 0; q < p_; ++q) {
    const StepPlan &pl = plans[q];
    const StepPlan &sender = plans[pl.rcv_rnk];
    if (sender.snd_blk != pl.rcv_blk || sender.snd_rnk != q)
      throw std::runtime_error("inconsistent exchange at rank " + std::to_string(q));
  }
  return plans;
}

int gpu_of_worker(int p, int world, int q) {
  int g = int((int64_t(q) * world) / p);
  while (g + 1 < world && workers_lo(p, world, g + 1) <= q) ++g;
  while (g > 0 && workers_lo(p, world, g) > q) --g;
  return g;
}

void step_transfers(const std::vector<StepPlan> &plans, int p, int world, int rank, std::vector<Xfer> &out) {
  const int lo = workers_lo(p, world, rank), hi = workers_lo(p, world, rank + 1);
  for (int q = lo; q < hi; ++q) {
    const int gs = gpu_of_worker(p, world, plans[q].snd_rnk);
    const int gr = gpu_of_worker(p, world, plans[q].rcv_rnk);
    if (gs != rank) out.push_back(Xfer{plans[q].snd_blk - 1, gs, true});
    if (gr != rank) out.push_back(Xfer{plans[q].rcv_blk - 1, gr, false});
  }
}

std::vector<int> final_block_owners(int strategy, int p, int world, int sweeps) {
  RingSchedule rs(strategy, p);
  for (int sw = 1; sw <= sweeps; ++sw)
    for (int s = 0; s < rs.steps_per_sweep(); ++s) rs.advance(sw);
  std::vector<int> owner(2 * p, -1);
  for (int q = 0; q < p; ++q) {
    owner[rs.i_blk(q) - 1] = gpu_of_worker(p, world, q);
    owner[rs.j_blk(q) - 1] = gpu_of_worker(p, world, q);
  }
  return owner;
}

}  // namespace hjb
