// Internal declarations shared by the host planner, the kernels and the context.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/p3.h"

// P3_EXP=1 compiles the comm-kernel experiment switches in (P3_PUSH_CAP, P3_LAZY_PICK,
// P3_SRV_PIECE, P3_BCAST_PULL; measured slower or neutral, profiles/r02_summary.md §7);
// the default build leaves them out so they cost the scheduler nothing.
// Signaler warps of the N > 1 comm kernel (1, or one per job slot).
#ifndef P3_NSIG
#define P3_NSIG 2
#endif
#ifndef P3_EXP
#define P3_EXP 0
#endif
#ifndef P3_COMM_MAX_THREADS
#define P3_COMM_MAX_THREADS 512  // comm CTA size bound (launch bounds: 126 registers at 512)
#endif
#define P3_MAX_LOCAL 8      // ranks one process hosts (1 per GPU; up to 8 when emulating)
#define P3_SIDE_STREAMS 4   // comm streams DRAIN launches rotate over
#define P3_DBG_CTAS 512
#define P3_COMM_DRAIN 0   // exit as soon as nothing is poppable or reducible
#define P3_COMM_FINISH 1  // exit when the iteration's local work is complete

namespace p3 {

uint64_t splitmix64_mix(uint64_t z);
int build_p3_plan(const uint64_t* counts, uint32_t n_layers, uint32_t servers, uint64_t max_slice,
                  std::vector<p3_slice_t>* out, std::string* err);
int build_baseline_plan(const uint64_t* counts, uint32_t n_layers, uint32_t servers,
                        uint64_t big_threshold, uint64_t rng_seed, std::vector<p3_slice_t>* out,
                        std::string* err);
void set_thread_error(const std::string& msg);

// ---------------------------------------------------------------- device-side views

// Read-only plan tables (one copy per GPU). Global slice id g enumerates the plan in
// (layer, slice) order, i.e. in priority order.
struct PlanDev {
  uint32_t n_layers;
  uint32_t total_slices;
  uint32_t world;
  uint32_t rr_owner;  // owner(g) == g % world for every slice (make_p3_plan)
  const uint32_t* layer_nslices;  // [L]
  const uint32_t* layer_first;    // [L] first global slice id of the layer
  const uint64_t* layer_woff;     // [L] element offset of the layer in W / G arenas
  const uint64_t* slice_off;      // [S] element offset inside the layer
  const uint32_t* slice_len;      // [S]
  const uint32_t* slice_layer;    // [S]
  const uint32_t* slice_owner;    // [S]
  const uint64_t* slice_slot;     // [S] element offset in the owner's per-pusher R block
  const uint32_t* own_list;       // [S] slice ids grouped by owner, plan order inside
  const uint32_t* slice_opos;     // [S] position of the slice in own_list (indexes arrivals, claim)
  const uint32_t* own_lfirst;     // [world*L] index into own_list of (owner, layer)
  const uint32_t* own_lcount;     // [world*L] owned slices of (owner, layer)
  const uint32_t* own_total;      // [world] owned slices per owner
  const uint64_t* own_stride;     // [world] R block stride (padded owned elements)
  const uint32_t* layer_group;    // [L] forward-gate group of the layer
  const uint32_t* own_base;       // [world] first own_list position of each owner
  const uint64_t* layer_flat;     // [L+1] start of each layer in the single-rank streaming order
                                  // (layers in priority order, each padded to 8 elements)
};

// Peer-visible state of every rank (pointers valid in this process: local or IPC-mapped).
struct PeersDev {
  float* W[P3_MAX_RANKS];          // parameter replica
  float* R[P3_MAX_RANKS];          // receive slots [world][own_stride]
  uint32_t* arrivals[P3_MAX_RANKS];  // [S] pushes received per owned slice, by own_list position (monotone)
  uint32_t* hint[P3_MAX_RANKS];      // [L] owned slices completed per layer (monotone)
  uint32_t* tally[P3_MAX_RANKS];     // [2] pushes arrived, owned slices completed (monotone)
  uint32_t* done[P3_MAX_RANKS];      // [L] slices of a layer broadcast into W (monotone)
  uint32_t* gdone[P3_MAX_RANKS];     // [G] slices of a gate group broadcast into W (monotone)
  // notify mode: NOTIFY ring of each rank (entries ((k+1) << 32) | slice, appended by owners)
  // and PULL ring of each owner (entries ((k+1) << 40) | (requester << 32) | slice)
  uint32_t* ntf_tail[P3_MAX_RANKS];
  unsigned long long* ntf_ring[P3_MAX_RANKS];
  uint32_t* pull_tail[P3_MAX_RANKS];
  unsigned long long* pull_ring[P3_MAX_RANKS];
};

// Per-iteration scratch of one local rank; zeroed before each comm launch.
struct IterState {
  uint32_t pushed;   // worker slices claimed
  uint32_t reduced;  // owned slices claimed
  uint32_t exited;   // CTAs of the FINISH launch that left (diagnostics)
  uint32_t jobs;     // jobs executed (diagnostics)
  // time (ns, summed over CTAs) spent by the scheduler picking, the scheduler waiting for a
  // free slot, the movers moving data, the signaler publishing completions (diagnostics)
  unsigned long long t_pick, t_slot_wait, t_move, t_signal;
  uint32_t push_live;  // remote pushes popped and not yet signalled (the push_cap gate)
  uint32_t pad_;
};

// Local-only state of one rank hosted in this process.
// One publication (enqueue_layer) in the host-written ring: written by the host when the
// layer's backward is issued, consumed by the device once a stream-ordered write of the
// ring tail says the producing kernels have run.
struct PubEntry {
  uint32_t layer;
  uint32_t key;             // FIFO publish sequence
  unsigned long long word;  // publication word: iteration tag << 48 | gradient pointer
};

struct LocalDev {
  uint32_t rank;
  uint32_t trace_cap;
  uint64_t* pub;        // [L] publication word: iteration tag + 256-B aligned gradient pointer
  uint32_t* fifo_key;   // [L] publish sequence (FIFO discipline)
  uint32_t* claim;      // [S] server claim tag by own_list position (monotone: k -> k+1)
  uint32_t* cursor;     // [L] worker claim cursor (per iteration)
  uint32_t* srv_lo;     // [L] server scan watermark (per iteration)
  uint32_t* srv_taken;  // [L] owned slices claimed (per iteration)
  IterState* it;        // per iteration
  float* V;             // momentum of owned elements [own_stride] (may be null)
  float* M;             // param_bf16: fp32 master of owned elements [own_stride] (else null)
  unsigned long long* bytes;  // [2] in, out
  unsigned long long* trace_n;
  p3_trace_rec_t* trace;
  uint32_t* cta_phase;  // [P3_DBG_CTAS] last phase of each comm CTA (diagnostics)
  unsigned long long* vclock;  // K7 token bucket: time (ns) at which granted bytes drain
  const PubEntry* ring;        // host-mapped publication ring
  uint32_t ring_cap;
  uint32_t* pubseq;            // ring entries published (stream memory write, monotone)
  uint32_t* ingested;          // ring entries turned into publication words (monotone)
  uint32_t* ingested_host;     // host-mapped mirror of `ingested` (host back-pressure)
  uint32_t* ntf_head;          // notify mode: NOTIFY entries consumed (monotone)
  uint32_t* pull_head;         // notify mode: PULL requests answered or claimed (monotone)
  uint32_t* pcount;            // [2] notify mode, per iteration: PULLs sent, PULLs answered
  uint32_t* slice_elems;       // [S] single-rank stream: elements of each slice updated (per iteration)
  unsigned long long* stream_next;  // single-rank stream: next warp tile to claim (per iteration)
  uint32_t* piece_next;  // [S] by own-list position: server pieces claimed (srv_piece; per iteration)
  uint32_t* piece_done;  // [S] by own-list position: server pieces signalled (per iteration)
};

struct CommArgs {
  PlanDev plan;
  PeersDev peers;
  LocalDev loc[P3_MAX_LOCAL];
  uint32_t n_local;
  uint32_t mode;    // P3_COMM_DRAIN or P3_COMM_FINISH
  uint32_t remote;  // some peer lives on another GPU: system-scope fences
  uint32_t k;  // iteration
  uint32_t sched;
  float lr;
  float momentum;
  unsigned long long linger_ns;  // DRAIN: wait this long for peers' pushes of partial slices
  uint32_t pop_run;   // single rank: consecutive slices claimed per pop
  uint32_t pop_relax; // a pop may take any of this many most urgent layers (1: strict)
  uint32_t pop_multi; // candidate layers claimed per round of pop atomics
  uint32_t push_bf16; // pushes travel as bf16
  uint32_t notify;    // notify mode (P3 config notify_pull, N > 1)
  uint32_t pb16;      // param_bf16: bf16 replicas / gradients, fp32 masters
  uint32_t ntf_cap, pull_cap;  // ring entries
  uint32_t push_split; // every push_split-th CTA prefers pushes over server work (0: none)
  uint32_t srv_filter; // server picks: only srv_filter x (ready slices) consumers look (0: all)
  uint32_t srv_reserve; // N > 1: every srv_reserve-th CTA does server work only (0: none)
  uint32_t tma_store;  // fp32 push tiles leave shared memory as TMA bulk stores
  uint32_t tma_store_red; // reduce results leave shared memory as TMA bulk stores (1: all, 2: remote)
  uint32_t push_cap;
  uint32_t srv_piece;  // >0: a completed owned slice is reduced in pieces of this many elements
                       // (multiple of 8), each claimed by whichever CTA is free
  uint32_t lazy_pick;
  uint32_t push_ctas;
  float* mcw;  // nvls: multicast address of the replica region (every rank's W); null = unicast  // FINISH, N > 1: CTAs [0, push_ctas) only push, the others only reduce  // FINISH, N > 1: once every local slice is claimed, pick the next job only
                       // when the CTA's movers are idle (no job bound to a busy CTA)  // >0: at most this many remote pushes of a rank in flight (pops wait)
  uint32_t push_max;  // FINISH: 1 = a CTA keeps at most one push in flight (the other slot for reduces)
  uint32_t use_tma;   // movers stage sources through shared memory with TMA (else direct loads)
  uint32_t trace_cta; // diagnostics (P3_TRACE_CTA=1): trace records carry the CTA index as `rank`
  float ns_per_byte;  // K7 link emulation (0: unthrottled)
  unsigned long long burst_ns;
  unsigned long long timeout_ns;
  uint32_t* err;  // device error word (P3_* code)
};

// Launchers (p3_kernels.cu)
int preload_kernels();
int launch_comm(const CommArgs& a, uint32_t ctas, uint32_t threads, void* stream);
int launch_update_stream(const CommArgs& a, uint32_t ctas, void* stream);
int launch_gradgen(uint64_t seed, uint64_t iteration, uint64_t layer, uint64_t start, uint64_t count,
                   float* out, void* stream);
int launch_mark(const LocalDev& L, uint32_t k, uint32_t ev, void* stream);
int launch_bump(uint32_t* done, uint32_t* gdone, uint32_t v, void* stream);
int launch_master_init(const CommArgs& a, void* stream);
int launch_queue_pop(const uint32_t* nslices, const uint32_t* first, const uint64_t* pub,
                     const uint32_t* fifo_key, uint32_t* cursor, uint32_t n_layers, uint32_t sched,
                     uint32_t tag, uint32_t* result, void* stream);

}  // namespace p3
