// Discrete-event schedule model of one worker/server pipeline — the C++ port of the
// reference simulator (sim.py:241-365). Four resources: the compute
// chain (forward/backward per layer), a serial uplink, an update stage (per-key concurrent
// or serial) and a serial downlink; integer ticks. With `device_queue` the uplink's
// pending set IS the device slice queue (p3_queue_*): layers are published into it at their
// backward-done tick and every uplink dispatch pops from it — the scripted tick replay that
// checks the GPU scheduler against the reference's transmission sequences.
#include <algorithm>
#include <cstring>
#include <queue>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "p3_internal.h"

namespace {

enum Kind { BOOT = 0, FWD_DONE = 1, BWD_DONE = 2, UP_DONE = 3, UPDATE_DONE = 4, DOWN_DONE = 5 };
using Ev = std::tuple<int64_t, int, int64_t, int64_t, int64_t>;  // (tick, kind, iteration, layer, slice)

struct Link {
  bool busy = false;
  // (arrival, iteration, layer, slice)
  std::vector<std::tuple<int64_t, int64_t, int64_t, int64_t>> pending;
  int64_t arrivals = 0;
  void enqueue(int64_t k, int64_t l, int64_t s) { pending.emplace_back(arrivals++, k, l, s); }
  // priority key (priority = layer, layer, slice, iteration, arrival) — plan.py:70-72 +
  // sim.py:231-238; FIFO key: arrival
  std::tuple<int64_t, int64_t, int64_t> pick(bool priority) {
    size_t best = 0;
    for (size_t i = 1; i < pending.size(); ++i) {
      const auto& a = pending[i];
      const auto& b = pending[best];
      const bool less = priority ? std::make_tuple(std::get<2>(a), std::get<3>(a), std::get<1>(a), std::get<0>(a)) <
                                       std::make_tuple(std::get<2>(b), std::get<3>(b), std::get<1>(b), std::get<0>(b))
                                 : std::get<0>(a) < std::get<0>(b);
      if (less) best = i;
    }
    auto e = pending[best];
    pending.erase(pending.begin() + best);
    return {std::get<1>(e), std::get<2>(e), std::get<3>(e)};
  }
};

}  // namespace

extern "C" int p3_simulate(const p3_sim_scenario_t* sc, p3_sim_entry_t* out, uint64_t cap, uint64_t* n_out) {
  using p3::set_thread_error;
  if (!sc || !sc->fwd || !sc->bwd || !sc->stages || sc->n_layers == 0) {
    set_thread_error("scenario needs at least one layer");
    return P3_EUSAGE;
  }
  const int64_t L = sc->n_layers, n_iter = sc->iterations, T = sc->slice_ticks, ovh = sc->per_slice_overhead;
  if (T < 1 || n_iter < 1 || ovh < 0 || sc->policy > P3_SIM_PRIORITY_SLICED) {
    set_thread_error("slice_ticks/num_iterations/per_slice_overhead/policy out of range");
    return P3_EUSAGE;
  }
  const bool coarse = sc->policy == P3_SIM_AGGRESSIVE_COARSE, prio = sc->policy == P3_SIM_PRIORITY_SLICED;
  std::vector<int64_t> ns(L), cu(L), cupd(L), cd(L);
  for (int64_t l = 0; l < L; ++l) {
    const p3_sim_stage_t& st = sc->stages[l];
    if (sc->fwd[l] < 0 || sc->bwd[l] < 0 || st.up < 0 || st.update < 0 || st.down < 0) {
      set_thread_error("layer " + std::to_string(l) + ": negative time or stage cost");
      return P3_EUSAGE;
    }
    if (coarse || st.up == 0) {
      ns[l] = 1;
    } else {
      if (st.up % T) {
        set_thread_error("layer " + std::to_string(l) + ": up cost not divisible by slice_ticks");
        return P3_EUSAGE;
      }
      ns[l] = st.up / T;
    }
    if (st.up % ns[l] || st.update % ns[l] || st.down % ns[l]) {
      set_thread_error("layer " + std::to_string(l) + ": stage costs not divisible into slices");
      return P3_EUSAGE;
    }
    cu[l] = st.up / ns[l];
    cupd[l] = st.update / ns[l];
    cd[l] = st.down / ns[l];
  }
  auto up_cost = [&](int64_t l) { return cu[l] > 0 ? cu[l] + ovh : 0; };
  auto down_cost = [&](int64_t l) { return cd[l] > 0 ? cd[l] + ovh : 0; };

  p3_queue_t* dq = nullptr;
  if (sc->device_queue) {
    std::vector<uint32_t> nsl(L);
    for (int64_t l = 0; l < L; ++l) nsl[l] = (uint32_t)ns[l];
    int rc = p3_queue_create(nsl.data(), (uint32_t)L, prio ? P3_SCHED_PRIORITY : P3_SCHED_FIFO, &dq);
    if (rc) return rc;
  }
  std::vector<p3_sim_entry_t> entries;
  auto record = [&](uint32_t res, uint32_t op, int64_t k, int64_t l, int64_t s, int64_t a, int64_t b) {
    p3_sim_entry_t e;
    e.resource = res;
    e.op = op;
    e.iteration = k;
    e.layer = l;
    e.slice = s;
    e.start = a;
    e.end = b;
    entries.push_back(e);
  };

  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> ev;
  ev.emplace(0, BOOT, 0, 0, 0);
  Link uplink, downlink, updlink;
  bool dq_busy = false, dq_pending = false;  // device-queue uplink: busy flag + "something queued"
  int64_t dq_iter = 0;
  std::set<std::pair<int64_t, int64_t>> bwd_ready, chain_ok, params_ok, started;
  std::vector<int64_t> remaining((size_t)(n_iter * L));
  for (int64_t k = 0; k < n_iter; ++k)
    for (int64_t l = 0; l < L; ++l) remaining[(size_t)(k * L + l)] = ns[l];
  int rc = P3_OK;

  auto start_ready_computes = [&](int64_t t) {
    while (!bwd_ready.empty()) {
      auto kl = *bwd_ready.begin();
      bwd_ready.erase(bwd_ready.begin());
      record(P3_SIM_COMPUTE, P3_SIM_BWD, kl.first, kl.second, 0, t, t + sc->bwd[kl.second]);
      ev.emplace(t + sc->bwd[kl.second], BWD_DONE, kl.first, kl.second, 0);
      if (sc->bwd[kl.second] > 0) break;  // the chain resumes when this backward completes
    }
    for (int64_t k = 1; k <= n_iter; ++k)
      for (int64_t l = 0; l < L; ++l) {
        const auto kl = std::make_pair(k, l);
        if (started.count(kl) || !chain_ok.count(kl) || !params_ok.count(kl)) continue;
        started.insert(kl);
        record(P3_SIM_COMPUTE, P3_SIM_FWD, k, l, 0, t, t + sc->fwd[l]);
        ev.emplace(t + sc->fwd[l], FWD_DONE, k, l, 0);
      }
  };
  auto into_update = [&](int64_t t, int64_t k, int64_t l, int64_t s) {
    const int64_t c = cupd[l];
    if (c == 0) {
      ev.emplace(t, UPDATE_DONE, k, l, s);
    } else if (sc->serial_update) {
      updlink.enqueue(k, l, s);
    } else {
      record(P3_SIM_UPDATE, P3_SIM_UPD, k, l, s, t, t + c);
      ev.emplace(t + c, UPDATE_DONE, k, l, s);
    }
  };
  auto handle = [&](const Ev& e) {
    const int64_t t = std::get<0>(e), k = std::get<2>(e), l = std::get<3>(e), s = std::get<4>(e);
    switch (std::get<1>(e)) {
      case BOOT:
        bwd_ready.insert({0, L - 1});
        break;
      case BWD_DONE:
        if (up_cost(l) == 0) {
          for (int64_t sl = 0; sl < ns[l]; ++sl) ev.emplace(t, UP_DONE, k, l, sl);
        } else if (dq) {
          if (p3_queue_put_layer(dq, (uint32_t)l, (uint32_t)k) != P3_OK) rc = P3_ECUDA;
          dq_pending = true;
          dq_iter = k;
        } else {
          for (int64_t sl = 0; sl < ns[l]; ++sl) uplink.enqueue(k, l, sl);
        }
        if (l > 0) bwd_ready.insert({k, l - 1});
        else chain_ok.insert({k + 1, 0});
        break;
      case FWD_DONE:
        if (l < L - 1) chain_ok.insert({k, l + 1});
        else if (k < n_iter) bwd_ready.insert({k, L - 1});
        break;
      case UP_DONE:
        if (up_cost(l) > 0) (dq ? dq_busy : uplink.busy) = false;
        into_update(t, k, l, s);
        break;
      case UPDATE_DONE:
        if (sc->serial_update && cupd[l] > 0) updlink.busy = false;
        if (down_cost(l) == 0) ev.emplace(t, DOWN_DONE, k, l, s);
        else downlink.enqueue(k, l, s);
        break;
      case DOWN_DONE:
        if (down_cost(l) > 0) downlink.busy = false;
        if (--remaining[(size_t)(k * L + l)] == 0) params_ok.insert({k + 1, l});
        break;
    }
  };
  auto dispatch = [&](int64_t t) {
    if (dq) {
      if (!dq_busy && dq_pending) {
        uint32_t l = 0, s = 0;
        const int r = p3_queue_poll(dq, &l, &s);
        if (r == P3_OK) {
          dq_busy = true;
          record(P3_SIM_UPLINK, P3_SIM_UP, dq_iter, l, s, t, t + up_cost(l));
          ev.emplace(t + up_cost(l), UP_DONE, dq_iter, (int64_t)l, (int64_t)s);
        } else if (r == P3_ETIMEOUT) {
          dq_pending = false;  // drained
        } else {
          rc = r;
        }
      }
    } else if (!uplink.busy && !uplink.pending.empty()) {
      auto [k, l, s] = uplink.pick(prio);
      uplink.busy = true;
      record(P3_SIM_UPLINK, P3_SIM_UP, k, l, s, t, t + up_cost(l));
      ev.emplace(t + up_cost(l), UP_DONE, k, l, s);
    }
    if (sc->serial_update && !updlink.busy && !updlink.pending.empty()) {
      auto [k, l, s] = updlink.pick(prio);
      updlink.busy = true;
      record(P3_SIM_UPDATE, P3_SIM_UPD, k, l, s, t, t + cupd[l]);
      ev.emplace(t + cupd[l], UPDATE_DONE, k, l, s);
    }
    if (!downlink.busy && !downlink.pending.empty()) {
      auto [k, l, s] = downlink.pick(prio);
      downlink.busy = true;
      record(P3_SIM_DOWNLINK, P3_SIM_DOWN, k, l, s, t, t + down_cost(l));
      ev.emplace(t + down_cost(l), DOWN_DONE, k, l, s);
    }
  };

  while (!ev.empty() && rc == P3_OK) {
    const int64_t t = std::get<0>(ev.top());
    while (!ev.empty() && std::get<0>(ev.top()) == t) {
      std::vector<Ev> batch;
      while (!ev.empty() && std::get<0>(ev.top()) == t) {
        batch.push_back(ev.top());
        ev.pop();
      }
      for (const Ev& e : batch) handle(e);
      start_ready_computes(t);
    }
    dispatch(t);
  }
  if (dq) p3_queue_destroy(dq);
  if (rc != P3_OK) {
    set_thread_error("device queue failed during the replay");
    return rc;
  }
  if (n_out) *n_out = entries.size();
  if (out) {
    if (cap < entries.size()) {
      set_thread_error("output capacity too small");
      return P3_EUSAGE;
    }
    std::memcpy(out, entries.data(), entries.size() * sizeof(p3_sim_entry_t));
  }
  return P3_OK;
}
