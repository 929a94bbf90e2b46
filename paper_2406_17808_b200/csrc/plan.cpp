// plan.cpp -- see plan.h.  Restates Alg. 2 over symbolic occupants.
#include "plan.h"

#include <algorithm>

namespace cascade {

void Planner::configure(int32_t alpha, int32_t N, int32_t c, bool selection) {
  alpha_ = alpha; N_ = N; c_ = c; S_tot_ = alpha + N * c;
  selection_ = selection;
  occ_.assign(S_tot_, 0);
  stamp_.assign(S_tot_, 0);
  cur_ = 0;
}

void Planner::advance(cascade_mirror& mr, int32_t m, Plan* plan) {
  ++cur_;
  if (cur_ == 0) { std::fill(stamp_.begin(), stamp_.end(), 0u); cur_ = 1; }
  touched_.clear();
  if (plan) {
    plan->sel.clear(); plan->sel_depth.clear(); plan->sel_order.clear();
    plan->depth_begin.clear(); plan->mov.clear(); plan->phase_begin.clear(); plan->drops = 0;
  }
  int64_t drops = 0;
  for (int32_t r = 0; r < m; ++r) {
    const int64_t t = mr.t + r;                       // 0-based stream index (Q1)
    int32_t item = S_tot_ + r;                        // chunk row r
    if (mr.sink_count < alpha_) {
      set(mr.sink_count, item);
      ++mr.sink_count;
      continue;
    }
    bool placed = false;
    for (int32_t i = 0; i < N_ && !placed; ++i) {     // sub-cache i+1
      const bool acc = (t & ((int64_t(1) << i) - 1)) == 0;   // t mod 2^i == 0
      const bool full = mr.counts[i] == c_;
      const int32_t base = alpha_ + i * c_;
      if (!full) {                                    // accepting fill or eager add
        set(base + mr.counts[i], item);
        ++mr.counts[i];
        mr.xi[i] = mr.counts[i] % c_;
        placed = true;
      } else if (acc) {                               // overwrite oldest, carry evictee
        const int32_t x = base + mr.xi[i];
        const int32_t ev = get(x);
        set(x, item);
        mr.xi[i] = (mr.xi[i] + 1) % c_;
        item = ev;
      } else if (!selection_) {                       // ablation (Q3): resident stays, carried dropped
        ++drops;
        placed = true;
      } else {                                        // token selection vs newest
        const int32_t ns = base + (mr.xi[i] - 1 + c_) % c_;
        const int32_t inc = get(ns);
        if (plan) {
          const int32_t k = (int32_t)plan->sel_depth.size();
          int32_t dep = 0;
          if (item < 0) dep = std::max(dep, plan->sel_depth[-item - 1] + 1);
          if (inc < 0) dep = std::max(dep, plan->sel_depth[-inc - 1] + 1);
          plan->sel.push_back(ns); plan->sel.push_back(item); plan->sel.push_back(inc);
          plan->sel_depth.push_back(dep);
          set(ns, -(k + 1));
        }
        ++drops;                                      // exactly one of the two is dropped
        placed = true;
      }
    }
    if (!placed) ++drops;                             // carried past C_N
  }
  mr.t += m;
  if (!plan) return;
  plan->drops = drops;
  // selections by dependency depth
  const int32_t nsel = (int32_t)plan->sel_depth.size();
  int32_t maxd = -1;
  for (int32_t d : plan->sel_depth) maxd = std::max(maxd, d);
  plan->depth_begin.push_back(0);
  for (int32_t d = 0; d <= maxd; ++d) {
    for (int32_t k = 0; k < nsel; ++k)
      if (plan->sel_depth[k] == d) plan->sel_order.push_back(k);
    plan->depth_begin.push_back((int32_t)plan->sel_order.size());
  }
  // final writes grouped by phase: C_N ... C_1, then sinks
  std::sort(touched_.begin(), touched_.end());
  auto emit_range = [&](int32_t lo, int32_t hi) {
    auto a = std::lower_bound(touched_.begin(), touched_.end(), lo);
    auto b = std::lower_bound(touched_.begin(), touched_.end(), hi);
    for (auto it = a; it != b; ++it) {
      const int32_t ref = occ_[*it];
      if (ref == *it) continue;
      plan->mov.push_back(*it);
      plan->mov.push_back(ref);
    }
  };
  for (int32_t i = N_ - 1; i >= 0; --i) {
    plan->phase_begin.push_back((int32_t)(plan->mov.size() / 2));
    emit_range(alpha_ + i * c_, alpha_ + (i + 1) * c_);
  }
  plan->phase_begin.push_back((int32_t)(plan->mov.size() / 2));
  emit_range(0, alpha_);
  plan->phase_begin.push_back((int32_t)(plan->mov.size() / 2));
}

double gamma_pow(double gamma, int64_t m) {
  double result = 1.0, base = gamma;
  int64_t e = m;
  while (e > 0) {
    if (e & 1) result = result * base;
    base = base * base;
    e >>= 1;
  }
  return result;
}

void mirror_positions(const cascade_mirror& mr, int32_t alpha, int32_t N, int32_t c, int32_t* pe) {
  for (int32_t x = 0; x < alpha; ++x) pe[x] = x < mr.sink_count ? x : -1;
  int32_t base = mr.sink_count;
  for (int32_t i = N - 1; i >= 0; --i) {
    const int32_t cnt = mr.counts[i];
    for (int32_t s = 0; s < c; ++s) {
      int32_t x = alpha + i * c + s;
      if (s >= cnt) { pe[x] = -1; continue; }
      pe[x] = base + (cnt == c ? (s - mr.xi[i] + c) % c : s);
    }
    base += cnt;
  }
}

}  // namespace cascade
