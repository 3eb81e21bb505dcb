// Host-side planning and hashing of the P3 sync path (no device code).
//
//   p3_plan_p3        <- make_p3_plan        plan.py:94-119 (+ _chunk_layer plan.py:82-91)
//   p3_plan_baseline  <- make_baseline_plan  plan.py:122-164
//   p3_splitmix64_*   <- hashing.py:24-35
//   p3_fnv1a64        <- hashing.py:79-83
//   p3_fq_*           <- FrameQueue ordering (queues.py:16-62) for host-resident frames
#include "p3_internal.h"

#include <cstring>
#include <queue>

namespace p3 {

uint64_t splitmix64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Slice count of one layer under greedy max_slice chunking (full chunks first, one
// shorter remainder chunk last).
static inline uint64_t chunks_of(uint64_t count, uint64_t max_slice) {
  return count / max_slice + (count % max_slice ? 1 : 0);
}

int build_p3_plan(const uint64_t* counts, uint32_t n_layers, uint32_t servers, uint64_t max_slice,
                  std::vector<p3_slice_t>* out, std::string* err) {
  if (servers < 1) { *err = "num_servers must be >= 1"; return P3_EUSAGE; }
  if (max_slice < 1) { *err = "max_slice must be >= 1"; return P3_EUSAGE; }
  out->clear();
  uint64_t total = 0;
  for (uint32_t l = 0; l < n_layers; ++l) {
    if (counts[l] < 1) { *err = "layer " + std::to_string(l) + ": param_count must be >= 1"; return P3_EUSAGE; }
    total += chunks_of(counts[l], max_slice);
  }
  out->reserve(total);
  uint64_t rr = 0;  // round-robin owner counter runs across layer boundaries
  for (uint32_t l = 0; l < n_layers; ++l) {
    const uint64_t n = chunks_of(counts[l], max_slice);
    for (uint64_t s = 0; s < n; ++s, ++rr) {
      p3_slice_t row;
      row.layer = l;
      row.slice = (uint32_t)s;
      row.offset = s * max_slice;
      row.length = (s + 1 < n || counts[l] % max_slice == 0) ? max_slice : counts[l] % max_slice;
      row.priority = l;
      row.server = (uint32_t)(rr % servers);
      out->push_back(row);
    }
  }
  return P3_OK;
}

int build_baseline_plan(const uint64_t* counts, uint32_t n_layers, uint32_t servers,
                        uint64_t big_threshold, uint64_t rng_seed, std::vector<p3_slice_t>* out,
                        std::string* err) {
  if (servers < 1) { *err = "num_servers must be >= 1"; return P3_EUSAGE; }
  out->clear();
  for (uint32_t l = 0; l < n_layers; ++l) {
    const uint64_t c = counts[l];
    if (c < big_threshold) {
      // whole layer on a pseudo-random server (KVStore default placement)
      p3_slice_t row{l, 0, 0, c, l, (uint32_t)(p3_splitmix64_stream(rng_seed, l) % servers)};
      out->push_back(row);
      continue;
    }
    const uint64_t part = c / servers;
    for (uint32_t s = 0; s < servers; ++s) {
      const uint64_t off = (uint64_t)s * part;
      const uint64_t len = (s + 1 == servers) ? c - off : part;
      p3_slice_t row{l, s, off, len, l, s};
      out->push_back(row);
    }
  }
  return P3_OK;
}

}  // namespace p3

extern "C" {

uint64_t p3_splitmix64_stream(uint64_t seed, uint64_t index) {
  return p3::splitmix64_mix(seed + (index + 1) * 0x9E3779B97F4A7C15ull);
}

uint64_t p3_fnv1a64(const void* data, uint64_t nbytes, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (uint64_t i = 0; i < nbytes; ++i) h = (h ^ p[i]) * 0x100000001B3ull;
  return h;
}

static int emit(const std::vector<p3_slice_t>& rows, p3_slice_t* out, uint64_t cap, uint64_t* n_out,
                std::string* err) {
  if (n_out) *n_out = rows.size();
  if (!out) return P3_OK;
  if (cap < rows.size()) { *err = "output capacity too small"; return P3_EUSAGE; }
  std::memcpy(out, rows.data(), rows.size() * sizeof(p3_slice_t));
  return P3_OK;
}

int p3_plan_p3(const uint64_t* counts, uint32_t n_layers, uint32_t num_servers, uint64_t max_slice,
               p3_slice_t* out, uint64_t cap, uint64_t* n_out) {
  std::vector<p3_slice_t> rows;
  std::string err;
  int rc = p3::build_p3_plan(counts, n_layers, num_servers, max_slice, &rows, &err);
  if (rc == P3_OK) rc = emit(rows, out, cap, n_out, &err);
  if (rc != P3_OK) p3::set_thread_error(err);
  return rc;
}

int p3_plan_baseline(const uint64_t* counts, uint32_t n_layers, uint32_t num_servers,
                     uint64_t big_threshold, uint64_t rng_seed, p3_slice_t* out, uint64_t cap,
                     uint64_t* n_out) {
  std::vector<p3_slice_t> rows;
  std::string err;
  int rc = p3::build_baseline_plan(counts, n_layers, num_servers, big_threshold, rng_seed, &rows, &err);
  if (rc == P3_OK) rc = emit(rows, out, cap, n_out, &err);
  if (rc != P3_OK) p3::set_thread_error(err);
  return rc;
}

// ------------------------------------------------------------ host frame queue

// FrameQueue order for frames that live on the host (the wire path beyond one NVSwitch
// domain, tests): a min-heap of (priority, layer, slice, arrival) in priority mode, of
// arrival alone in FIFO mode (queues.py:16-17, 34-38). Frames themselves stay with the
// caller; the heap orders opaque handles. Not thread-safe: the caller serialises (the
// Python FrameQueue holds its condition lock around every call, which also makes a batch
// atomic, queues.py:44-50). The GPU path never uses it: there the comm kernel pops the
// device slice queue.
struct p3_fq {
  struct Ent {
    uint64_t p, l, s, seq, h;
    bool operator>(const Ent& o) const {
      if (p != o.p) return p > o.p;
      if (l != o.l) return l > o.l;
      if (s != o.s) return s > o.s;
      return seq > o.seq;
    }
  };
  bool priority = true;
  uint64_t seq = 0;
  std::priority_queue<Ent, std::vector<Ent>, std::greater<Ent>> heap;
};

int p3_fq_create(uint32_t priority_mode, p3_fq_t** out) {
  if (!out) return P3_EUSAGE;
  p3_fq* q = new p3_fq();
  q->priority = priority_mode != 0;
  *out = q;
  return P3_OK;
}

int p3_fq_put_batch(p3_fq_t* q, const uint64_t* keys3, const uint64_t* handles, uint64_t n) {
  if (!q || (n && (!keys3 || !handles))) return P3_EUSAGE;
  for (uint64_t i = 0; i < n; ++i) {
    p3_fq::Ent e{0, 0, 0, q->seq++, handles[i]};
    if (q->priority) {
      e.p = keys3[3 * i];
      e.l = keys3[3 * i + 1];
      e.s = keys3[3 * i + 2];
    }
    q->heap.push(e);
  }
  return P3_OK;
}

int p3_fq_poll(p3_fq_t* q, uint64_t* handle) {
  if (!q || !handle) return P3_EUSAGE;
  if (q->heap.empty()) return P3_ETIMEOUT;
  *handle = q->heap.top().h;
  q->heap.pop();
  return P3_OK;
}

uint64_t p3_fq_size(p3_fq_t* q) { return q ? (uint64_t)q->heap.size() : 0; }

int p3_fq_snapshot(p3_fq_t* q, uint64_t* handles, uint64_t cap, uint64_t* n_out) {
  if (!q || !n_out) return P3_EUSAGE;
  *n_out = q->heap.size();
  if (!handles) return P3_OK;
  if (cap < q->heap.size()) return P3_EUSAGE;
  auto copy = q->heap;  // queued frames in dequeue order (queues.py:69-71)
  for (uint64_t i = 0; !copy.empty(); ++i, copy.pop()) handles[i] = copy.top().h;
  return P3_OK;
}

int p3_fq_destroy(p3_fq_t* q) {
  delete q;
  return P3_OK;
}

}  // extern "C"
