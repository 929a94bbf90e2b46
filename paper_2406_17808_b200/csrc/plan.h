// plan.h -- host control plane: the deterministic mirror of Alg. 2's counters and the
// per-chunk schedule (library-private).
//
// Alg. 2 is simulated for the m tokens of a chunk *without payloads*: every
// slot holds a symbolic reference to its occupant -- the pre-chunk occupant of a flat
// slot, a chunk row, or the winner of a selection of this chunk -- so the schedule is
// the same for every (b, g) and needs no device->host read.  Only the selection
// outcomes are data dependent; the device resolves them (k_maint.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/cascade.h"

namespace cascade {

struct Plan {
  // select k: {slot, cand_ref, inc_ref}; refs as in internal.h (PlanDev)
  std::vector<int32_t> sel;
  std::vector<int32_t> sel_depth;
  std::vector<int32_t> sel_order;          // select indices sorted by depth
  std::vector<int32_t> depth_begin;        // offsets into sel_order per depth (+ end)
  std::vector<int32_t> mov;                // {dst, ref} grouped by phase
  std::vector<int32_t> phase_begin;        // N + 2 entries: C_N, ..., C_1, sinks, end
  int64_t drops = 0;
};

class Planner {
 public:
  // selection = false: the ablation without token selection (reading Q3: the resident stays,
  // the carried token is dropped)
  void configure(int32_t alpha, int32_t N, int32_t c, bool selection = true);
  // Advances `mr` by m insertions starting at stream index mr.t; fills plan if non-null.
  void advance(cascade_mirror& mr, int32_t m, Plan* plan);

 private:
  int32_t alpha_ = 0, N_ = 0, c_ = 0, S_tot_ = 0;
  bool selection_ = true;
  std::vector<int32_t> occ_;
  std::vector<uint32_t> stamp_;
  std::vector<int32_t> touched_;
  uint32_t cur_ = 0;
  int32_t get(int32_t x) const { return stamp_[x] == cur_ ? occ_[x] : x; }
  void set(int32_t x, int32_t v) {
    if (stamp_[x] != cur_) { stamp_[x] = cur_; touched_.push_back(x); }
    occ_[x] = v;
  }
};

// gamma^m by right-to-left binary exponentiation in double (documented in cascade.h).
double gamma_pow(double gamma, int64_t m);

// pe of every flat slot for a mirror (-1 empty), host side.
void mirror_positions(const cascade_mirror& mr, int32_t alpha, int32_t N, int32_t c, int32_t* pe);

}  // namespace cascade
