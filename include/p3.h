/*
 * p3.h — C ABI of the B200-native P3 (Priority-based Parameter Propagation) sync path.
 *
 * This is the drop-in boundary. Every entry point replaces one call site of the
 * reference's Python API (`/root/reference/pkg/src/p3sync`); the citation above each
 * declaration names the reference interface (file:line) it stands in for.
 *
 * Conventions
 *   - Return codes mirror the reference CLI exit codes (cli.py:49-52):
 *       P3_OK 0, P3_EUSAGE 1 (ValueError / PlanError / ProfileError),
 *       P3_EPROTOCOL 2 (ProtocolError), P3_ETIMEOUT 3 (DeadlockError), P3_ECUDA 4.
 *   - Plain pointers and sizes only. `stream` arguments are CUstream / cudaStream_t
 *     handles passed as void* (NULL = legacy default stream).
 *   - Host arrays are owned by the caller. Device pointers are borrowed. A p3_ctx_t owns
 *     its device arenas (parameters, receive slots, flags, trace) and frees them in
 *     p3_ctx_destroy.
 *   - Hot calls (p3_layer_ready, p3_wait_layer, p3_iteration_begin/end, p3_gradgen_layer)
 *     are asynchronous and stream-ordered; none of them synchronises the host.
 *   - The library has no CPU fallback: every compute entry point runs sm_100a code and
 *     returns P3_ECUDA when no device is available.
 */
#ifndef P3_H_
#define P3_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P3_OK 0
#define P3_EUSAGE 1
#define P3_EPROTOCOL 2
#define P3_ETIMEOUT 3
#define P3_ECUDA 4

/* Plan modes: plan.py:53-54 (P3_MODE / BASELINE_MODE). */
#define P3_PLAN_P3 0
#define P3_PLAN_BASELINE 1

/* Queue disciplines: FrameQueue(priority_mode=True/False), queues.py:28-39. */
#define P3_SCHED_PRIORITY 0
#define P3_SCHED_FIFO 1

/* Maximum ranks (workers == servers) in one NVSwitch domain handled by one context. */
#define P3_MAX_RANKS 16

/* Trace events. PUSH / BCAST are the Frame msg types that cross the link (proto.py:26-32);
 * PUBLISH, COMPLETE and PICK record the queue operations around them, so a live run can be
 * replayed through FrameQueue (queues.py:44-62): PUBLISH = put_batch of a layer (worker.py:
 * 173-182), PUSH = the sender's poll (worker.py:184-190), COMPLETE = the last on_push of a
 * slice (server.py:36-53), PICK = the server consumer's poll of a complete slice
 * (server.py:208-226). */
#define P3_EV_PUSH 0     /* worker popped a slice (claim) and stored it into the owner's slot;
                            t0_ns = start of the pop's queue snapshot, t_ns = after the claim */
#define P3_EV_BCAST 1    /* owner reduced + updated a slice and broadcast it */
#define P3_EV_PUBLISH 2  /* a layer's publication word became visible to the pops (ingest);
                            slice = the publish sequence number (FIFO key) */
#define P3_EV_COMPLETE 3 /* the last push of an owned slice arrived; rank = owner */
#define P3_EV_PICK 4     /* owner claimed a complete slice for reduce + broadcast; t0_ns = start
                            of the pick's scan, t_ns = after the claim */
#define P3_EV_ITER_START 5 /* p3_trace_mark: a rank's forward pass of `iteration` starts
                              (IterationRecord.start, worker.py:312-313) */
#define P3_EV_SYNCED 6     /* p3_trace_mark: every layer of `iteration` synced on that rank
                              (sync_end_times, worker.py:265-268) */
#define P3_EV_NOTIFY 7     /* notify mode: owner told rank `rank` that slice (layer, slice) is
                              updated (server.py:227-239) */
#define P3_EV_PULL 8       /* notify mode: this rank asked owner `rank` for the slice
                              (worker.py:226-239); the answer is a BCAST record at the owner
                              with rank = the requester */

/* One row of a SlicePlan (plan.py:30-45: SliceKey + Slice). */
typedef struct p3_slice {
  uint32_t layer;    /* SliceKey.layer_index */
  uint32_t slice;    /* SliceKey.slice_index */
  uint64_t offset;   /* Slice.offset (elements into the layer) */
  uint64_t length;   /* Slice.length (elements) */
  uint32_t priority; /* Slice.priority (== layer index) */
  uint32_t server;   /* Slice.server (owner rank) */
} p3_slice_t;

/* One device trace record; the wire header fields of proto.py:20-21 minus the codec. */
typedef struct p3_trace_rec {
  uint64_t t_ns;      /* %globaltimer at the event */
  uint64_t t0_ns;     /* PUSH / PICK: %globaltimer before the queue snapshot the claim came
                         from (0 for other events) */
  uint32_t iteration; /* Frame.iteration */
  uint32_t layer;     /* Frame.layer_index (== priority) */
  uint32_t slice;     /* Frame.slice_index */
  uint16_t rank;      /* Frame.worker_rank (pusher for PUSH, owner for BCAST) */
  uint16_t event;     /* P3_EV_* */
} p3_trace_rec_t;

/* ---------------------------------------------------------------- planning (host) */

/* make_p3_plan, plan.py:94-119 (greedy max_slice chunks, remainder last, server =
 * running counter % num_servers, priority = layer index). Rows are written in
 * (layer, slice) order. With out == NULL only *n_out is computed. */
int p3_plan_p3(const uint64_t* param_counts, uint32_t n_layers, uint32_t num_servers,
               uint64_t max_slice, p3_slice_t* out, uint64_t cap, uint64_t* n_out);

/* make_baseline_plan, plan.py:122-164 (small layer -> splitmix64_stream(seed, L) % N,
 * layer >= big_threshold -> N equal parts, remainder on the last part). */
int p3_plan_baseline(const uint64_t* param_counts, uint32_t n_layers, uint32_t num_servers,
                     uint64_t big_threshold, uint64_t rng_seed, p3_slice_t* out,
                     uint64_t cap, uint64_t* n_out);

/* splitmix64_stream, hashing.py:32-35. */
uint64_t p3_splitmix64_stream(uint64_t seed, uint64_t index);

/* fnv1a64 over `nbytes` bytes with chaining seed `h`, hashing.py:79-83. */
uint64_t p3_fnv1a64(const void* data, uint64_t nbytes, uint64_t h);

/* ------------------------------------------------------- standalone device kernels */

/* gradient_block, hashing.py:55-63: out_dev[i] = gradient_value(seed, it, layer,
 * start + i) for i < count, bit-exact, written by the K1 gradgen kernel. */
int p3_gradient_block(uint64_t seed, uint64_t iteration, uint64_t layer, uint64_t start,
                      uint64_t count, float* out_dev, void* stream);

/* ShardState.aggregate_and_update, server.py:55-68, for one slice:
 *   acc = 0; for r in 0..num_workers-1 (ascending): acc += grads[r]; g = acc / N;
 *   params -= lr * g            (IEEE fp32, no contraction; bit-exact)
 * grads_dev is a HOST array of num_workers device pointers (rank order).
 * momentum_dev may be NULL (plain SGD, the reference); otherwise
 *   v = momentum * v + g; params -= lr * v   (extension, not in the reference). */
int p3_shard_update(float* params_dev, const float* const* grads_dev, uint32_t num_workers,
                    uint64_t n, float lr, float momentum, float* momentum_dev, void* stream);

/* Device-side sleep for `duration_us` (TrainingWorker._emulate, worker.py:299-310). */
int p3_emulate_compute(uint64_t duration_us, void* stream);

/* ---------------------------------------------------- scripted device priority queue */

/* The device slice queue driven one operation at a time (FrameQueue, queues.py:20-75).
 * Used for tick-replay parity against the reference simulator; the same __device__ pop
 * routine runs inside the comm kernel. */
typedef struct p3_queue p3_queue_t;
int p3_queue_create(const uint32_t* layer_nslices, uint32_t n_layers, uint32_t sched,
                    p3_queue_t** out);
/* FrameQueue.put_batch of all slices of `layer` (queues.py:44-50): atomic. */
int p3_queue_put_layer(p3_queue_t* q, uint32_t layer, uint32_t iteration);
/* FrameQueue.poll (queues.py:52-62) without blocking: returns P3_OK and the popped
 * (layer, slice), or P3_ETIMEOUT when nothing is queued. */
int p3_queue_poll(p3_queue_t* q, uint32_t* layer, uint32_t* slice);
int p3_queue_destroy(p3_queue_t* q);

/* ------------------------------------------------------------- host frame queue */

/* FrameQueue ordering (queues.py:16-62) for frames that stay on the host (wire path beyond
 * the NVSwitch domain): a heap of opaque handles keyed (priority, layer, slice, arrival) in
 * priority mode, arrival in FIFO mode. Callers serialise access. put_batch takes n keys as
 * 3 u64 each (priority, layer, slice; ignored in FIFO mode). poll returns P3_ETIMEOUT when
 * empty; snapshot lists the handles in dequeue order. */
typedef struct p3_fq p3_fq_t;
int p3_fq_create(uint32_t priority_mode, p3_fq_t** out);
int p3_fq_put_batch(p3_fq_t* q, const uint64_t* keys3, const uint64_t* handles, uint64_t n);
int p3_fq_poll(p3_fq_t* q, uint64_t* handle);
uint64_t p3_fq_size(p3_fq_t* q);
int p3_fq_snapshot(p3_fq_t* q, uint64_t* handles, uint64_t cap, uint64_t* n_out);
int p3_fq_destroy(p3_fq_t* q);

/* ------------------------------------------------------------- schedule model (host) */

/* sim.py:26-34: policies and resources of the discrete-event model. */
#define P3_SIM_AGGRESSIVE_COARSE 0
#define P3_SIM_AGGRESSIVE_SLICED 1
#define P3_SIM_PRIORITY_SLICED 2
#define P3_SIM_COMPUTE 0
#define P3_SIM_UPLINK 1
#define P3_SIM_UPDATE 2
#define P3_SIM_DOWNLINK 3
#define P3_SIM_FWD 0
#define P3_SIM_BWD 1
#define P3_SIM_UP 2
#define P3_SIM_UPD 3
#define P3_SIM_DOWN 4

typedef struct p3_sim_stage { int64_t up, update, down; } p3_sim_stage_t;  /* StageCost, sim.py:41-45 */

typedef struct p3_sim_scenario {      /* Scenario, sim.py:48-57 */
  uint32_t n_layers;
  const int64_t* fwd;                 /* LayerSpec.fwd_time per layer (ticks) */
  const int64_t* bwd;                 /* LayerSpec.bwd_time per layer (ticks) */
  const p3_sim_stage_t* stages;
  uint32_t policy;                    /* P3_SIM_* */
  int64_t slice_ticks;
  int64_t iterations;
  int64_t per_slice_overhead;
  uint32_t serial_update;
  uint32_t device_queue;              /* 1: the uplink pops from the device slice queue */
} p3_sim_scenario_t;

typedef struct p3_sim_entry {         /* TimelineEntry, sim.py:135-140 (item = op:k:Ll[:ss]) */
  uint32_t resource, op;
  int64_t iteration, layer, slice, start, end;
} p3_sim_entry_t;

/* simulate (sim.py:241-365): the timeline entries in creation order. With device_queue the
 * uplink transmission order comes from the device priority/FIFO queue (the same warp_pop
 * the comm kernel runs), which must reproduce the reference's sequences exactly. */
int p3_simulate(const p3_sim_scenario_t* scenario, p3_sim_entry_t* out, uint64_t cap, uint64_t* n_out);

/* --------------------------------------------------------------- sync context (K3) */

typedef struct p3_ctx p3_ctx_t;

typedef struct p3_config {
  uint32_t world;                      /* N workers == N servers (cli.py:81-82) */
  uint32_t n_local;                    /* ranks hosted by this process (1, or N when
                                          emulating all ranks on one GPU) */
  uint32_t local_ranks[P3_MAX_RANKS];  /* which ranks */
  uint32_t n_layers;
  const uint64_t* layer_counts;        /* LayerSpec.param_count per layer */
  uint64_t max_slice;                  /* make_p3_plan max_slice (plan.py:22) */
  uint32_t plan_mode;                  /* P3_PLAN_P3 or P3_PLAN_BASELINE (KVStore layer-wise
                                          placement, plan.py:122-164) */
  uint32_t sched;                      /* P3_SCHED_PRIORITY (p3) or P3_SCHED_FIFO */
  float lr;                            /* RunConfig.lr (cli.py:69) */
  float momentum;                      /* 0 == the reference's plain SGD */
  uint32_t comm_ctas;                  /* CTAs of each DRAIN launch of the comm kernel */
  uint32_t comm_threads;               /* threads per comm CTA (multiple of 32 in [128, 512],
                                          [160, 512] when world > 1: scheduler, signaler(s),
                                          TMA producer, consumers) */
  double timeout_s;                    /* device spin deadline (deadlock_timeout) */
  uint32_t trace_cap;                  /* trace records per local rank (0 = off) */
  uint32_t emulate_grads;              /* allocate a gradient arena for gradgen mode */
  uint64_t drain_bytes;                /* launch a DRAIN comm kernel once this many gradient
                                          bytes were published since the last one (0: on
                                          every publication) */
  uint64_t big_threshold;              /* baseline plan: layers >= this are split N ways */
  uint64_t rng_seed;                   /* baseline plan: placement seed of small layers */
  double throttle_bps;                 /* K7 link emulation: per-rank egress rate in bit/s
                                          (TokenBucket, transport.py:22-55); 0 = full NVLink */
  uint64_t throttle_burst;             /* bucket depth in bytes (transport.py:18: 50 KiB) */
  uint64_t pub_batch_bytes;            /* publish (one stream memory write of the ring tail)
                                          once this many gradient bytes were enqueued
                                          (0: every layer at once — finest preemption) */
  uint32_t drain_linger_us;            /* a DRAIN launch with nothing to do keeps waiting this
                                          long while peers' pushes of partially arrived owned
                                          slices are outstanding (never for local compute) */
  uint32_t finish_ctas;                /* CTAs of the FINISH launch (0: comm_ctas) */
  uint32_t pop_relax;                  /* bounded relaxation: a pop takes one of this many most
                                          urgent published slices (0: the launch's CTA count;
                                          1: strict order); capped at the CTA count */
  uint32_t pop_run;                    /* single rank: consecutive slices per job (0: auto) */
  uint32_t pop_multi;                  /* layers claimed per round of pop atomics, 1..4 (0: 1) */
  uint32_t push_bf16;                  /* declared lossy transport: pushes carry bf16 (RNE)
                                          contributions, summed in fp32 in rank order;
                                          parameters, update and broadcasts stay fp32 */
  const uint32_t* gate_groups;         /* optional per-layer forward-gate group id (layers of
                                          one module gated together); NULL = one group per
                                          layer. Ids must be 0..G-1 */
  uint32_t drain_streams;              /* side streams DRAIN launches rotate over (0: 4). With 1,
                                          comm_ctas = finish_ctas = 1 and pop_relax = 1 there is
                                          one consumer at a time: the strict FrameQueue order
                                          (queues.py:52-62), checked by trace replay */
  uint32_t notify_pull;                /* N > 1, the baseline's protocol (server.py:227-247,
                                          worker.py:226-239): the owner updates only its own
                                          replica and NOTIFYs the other ranks; each replica
                                          queues a PULL behind its pushes and the owner answers
                                          it with the slice (one more round trip than P3's
                                          broadcast) */
  uint32_t param_bf16;                 /* declared bf16 replicas: the model's parameters and
                                          gradients are bf16 (W holds bf16); each owner keeps an
                                          fp32 master of its slices. Pushes carry the bf16
                                          gradients, the owner sums them in fp32 in rank order,
                                          updates the fp32 master (same arithmetic as the fp32
                                          path) and broadcasts bf16(master), round to nearest
                                          even. Call p3_master_init once the replica holds the
                                          initial parameters. */
  uint32_t nvls;                       /* N > 1, one local rank per process, fp32 replicas, not
                                          notify_pull: broadcasts go through an NVLS multicast
                                          object spanning every rank's replica W (one
                                          multimem.st per element; the NVSwitch delivers it to
                                          all N replicas). The arena is then a VMM allocation
                                          shared by file descriptor: bootstrap with
                                          p3_ctx_export_fd / p3_ctx_open_peers_fd and
                                          p3_nvls_create / _attach / _bind instead of IPC. */
} p3_config_t;

/* Builds the plan, allocates per-local-rank arenas (parameters W zero-initialised like
 * worker.py:72 / server.py:112-115, receive slots R, flags) and uploads plan tables. */
int p3_ctx_create(const p3_config_t* cfg, p3_ctx_t** out);
int p3_ctx_destroy(p3_ctx_t* ctx);

/* Multi-process bootstrap: the IPC handle of a local rank's arena (P3_IPC_BYTES bytes),
 * and opening every rank's handle (world * P3_IPC_BYTES bytes, rank order; entries of
 * local ranks are ignored). Replaces the TCP connect/HELLO of worker.py:136-148. */
#define P3_IPC_BYTES 64
int p3_ctx_ipc_handle(p3_ctx_t* ctx, uint32_t local_idx, void* out);
int p3_ctx_open_peers(p3_ctx_t* ctx, const void* handles);

/* NVLS bootstrap (cfg.nvls; replaces p3_ctx_ipc_handle / p3_ctx_open_peers; the descriptors
 * travel between processes over a Unix socket, SCM_RIGHTS):
 *   p3_ctx_export_fd     a POSIX file descriptor of the local rank's arena (caller closes it);
 *   p3_ctx_open_peers_fd map every other rank's arena (fds[r]; the local entry is ignored);
 *   p3_nvls_create       one rank: create the multicast object for the replica region, fd out;
 *   p3_nvls_attach       every rank: import it (fd >= 0; the creator passes -1) and add its GPU;
 *   p3_nvls_bind         every rank, once all have attached: bind its replica and map the
 *                        multicast address. */
int p3_ctx_export_fd(p3_ctx_t* ctx, uint32_t local_idx, int* fd);
int p3_ctx_open_peers_fd(p3_ctx_t* ctx, const int* fds);
int p3_nvls_create(p3_ctx_t* ctx, int* fd);
int p3_nvls_attach(p3_ctx_t* ctx, int fd);
int p3_nvls_bind(p3_ctx_t* ctx);

/* Device pointer of local rank's parameter replica and each layer's element offset in
 * it (layers are 16-byte aligned). TrainingWorker.params, worker.py:72. */
int p3_ctx_params(p3_ctx_t* ctx, uint32_t local_idx, float** params_dev);
int p3_ctx_layer_offset(p3_ctx_t* ctx, uint32_t layer, uint64_t* elem_offset);
/* param_bf16: initialise the fp32 master of the local rank's owned slices from its (bf16)
 * replica W — once, after the initial parameters were written into W (stream-ordered). */
int p3_master_init(p3_ctx_t* ctx, uint32_t local_idx, void* stream);

/* Device pointer of the local rank's gradient arena (emulate_grads only). */
int p3_ctx_grads(p3_ctx_t* ctx, uint32_t local_idx, float** grads_dev);

/* Open iteration k on `comm_stream`: reset the per-iteration queue state (stream-ordered
 * after the previous iteration's comm work). The comm kernel (K3: worker pop/push +
 * server reduce/update/broadcast for all local ranks) replaces the _priority_sender /
 * _fifo_sender threads (worker.py:184-198) and ServerEngine._consumer (server.py:208-249);
 * it is launched by p3_layer_ready and p3_iteration_end below. */
int p3_iteration_begin(p3_ctx_t* ctx, uint64_t iteration, void* comm_stream);

/* TrainingWorker.enqueue_layer (worker.py:173-182): publish all slices of `layer` for
 * `iteration` atomically (one word: iteration tag + gradient pointer). `grad_dev` is the
 * layer's fp32 gradient (param_count elements); NULL = the context's gradient arena.
 * When an iteration is open the entry goes to a pinned, device-mapped ring; once
 * `pub_batch_bytes` are pending one stream memory write on `stream` advances the ring tail
 * (so the entries become visible only after the kernels that produced them), and any
 * running comm kernel picks them up at its next pick (slice-granular preemption). Once
 * `drain_bytes` are pending a DRAIN launch is queued on the comm stream behind this point
 * of `stream`: it pops the most urgent published slices, reduces owned slices whose pushes
 * are complete and exits once nothing is poppable — it never spins on compute that has not
 * been published. Outside an open iteration the word is written at once. */
int p3_layer_ready(p3_ctx_t* ctx, uint32_t local_idx, uint32_t layer, uint64_t iteration,
                   const float* grad_dev, void* stream);

/* End of iteration k's backward for every local rank: launch the comm kernel in FINISH
 * mode on the comm stream; it exits when every local slice is pushed and every owned
 * slice reduced and broadcast (waiting only for pushes of peers), or at the deadline. */
int p3_iteration_end(p3_ctx_t* ctx, uint64_t iteration);

/* K1 emulate mode: fill the gradient arena for `layer` with GradGen(seed) values
 * (TrainingWorker._materialize, worker.py:166-171). The reference pushes the same seed
 * from every rank (worker.py:71); callers wanting rank-distinct gradients pass a
 * per-rank seed. */
int p3_gradgen_layer(p3_ctx_t* ctx, uint32_t local_idx, uint64_t seed, uint64_t iteration,
                     uint32_t layer, void* stream);

/* TrainingWorker._wait_layer (worker.py:277-285): make `stream` wait until `layer` holds
 * the parameters for forward pass `iteration` (flags[layer] >= iteration). A stream
 * memory wait: no SM is occupied. */
int p3_wait_layer(p3_ctx_t* ctx, uint32_t local_idx, uint32_t layer, uint64_t iteration,
                  void* stream);

/* _wait_layer for a gate group: wait until every layer of `group` holds the parameters
 * for forward pass `iteration` — one stream memory wait for a whole module. */
int p3_wait_group(p3_ctx_t* ctx, uint32_t local_idx, uint32_t group, uint64_t iteration,
                  void* stream);

/* TrainingWorker.on_bcast (worker.py:241-269) for a BCAST frame that arrived on the host
 * (the wire path beyond the NVSwitch domain): copy `n` fp32 values of slice (layer, slice)
 * into the local replica W at the slice's offset and count the slice towards the layer's
 * forward gate (done[layer], its gate group) — stream-ordered on `stream`. `n` must equal the
 * slice length (P3_EPROTOCOL otherwise). Iteration / duplicate checks are the caller's. */
int p3_apply_slice(p3_ctx_t* ctx, uint32_t local_idx, uint32_t layer, uint32_t slice, const float* values_host,
                   uint64_t n, void* stream);

/* flags[layer] of the reference worker (worker.py:74-75): the forward pass whose parameters
 * layer `layer` of a local rank holds = done[layer] / slices of the layer (device read). */
int p3_layer_flag(p3_ctx_t* ctx, uint32_t local_idx, uint32_t layer, uint64_t* iteration);

/* TrainingWorker._wait_all (worker.py:287-289) + error check: block the host until the
 * comm kernels finished and every local layer reached `iteration`, or timeout. */
int p3_sync_all(p3_ctx_t* ctx, uint64_t iteration, double timeout_s);

/* Transmission sequence (trace) of a local rank, in device append order. */
int p3_trace_read(p3_ctx_t* ctx, uint32_t local_idx, p3_trace_rec_t* out, uint64_t cap,
                  uint64_t* n_out);
int p3_trace_clear(p3_ctx_t* ctx);

/* Append a stream-ordered record (P3_EV_ITER_START / P3_EV_SYNCED) with the device clock to
 * a local rank's trace: the iteration timeline of the reference worker (worker.py:312-368)
 * on the same %globaltimer clock as the queue records. One 1-thread kernel on `stream`. */
int p3_trace_mark(p3_ctx_t* ctx, uint32_t local_idx, uint64_t iteration, uint32_t event, void* stream);

/* Comm kernel launches issued by this context so far (DRAIN + FINISH). */
int p3_comm_launches(p3_ctx_t* ctx, uint64_t* n);

/* NetCounters.totals (metrics.py:31-45): NVLink/HBM payload bytes in / out. */
int p3_counters(p3_ctx_t* ctx, uint32_t local_idx, uint64_t* bytes_in, uint64_t* bytes_out);

/* Diagnostics snapshot of a local rank (deadlock dumps, worker.py:291-297): 5 arrays of
 * n_layers u32 — ready tag, claim cursor, server claims, completed-hint, done counter —
 * then the per-iteration counters (pushed, reduced, exited CTAs, jobs; then 4 u64 ns totals:
 * scheduler pick, scheduler slot wait, consumers, signaler), the last phase word of the
 * first 512 comm CTAs, and per slice the arrival counter and server claim tag. Copied on a private stream (never blocks on the
 * compute or comm streams). */
int p3_debug_snapshot(p3_ctx_t* ctx, uint32_t local_idx, uint32_t* out, uint64_t cap,
                      uint64_t* n_out);

/* Diagnostics of the last failing call on this context (thread-local when ctx == NULL). */
const char* p3_last_error(p3_ctx_t* ctx);

/* Device attributes the runtime depends on (stream memory ops, SM count). */
int p3_device_info(int* sm_count, int* stream_memops, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------------ wire frames (multi-node)
 * The framed wire protocol of proto.py:18-141 for traffic that leaves the NVSwitch domain
 * (SURVEY §8(f) item 4): a 39-byte little-endian header "<4sBIQHIIQI" — magic "P3W1",
 * msg_type u8, priority u32, iteration u64, worker_rank u16, layer u32, slice u32,
 * offset u64, payload_len u32 — followed by the float32 payload of PUSH / BCAST frames.
 * Inside one box the comm kernel never serialises (stores go straight over NVLink). */
#define P3_FRAME_HEADER_BYTES 39
#define P3_FRAME_DEFAULT_MAX_PAYLOAD (16u * 1024u * 1024u)
#define P3_MSG_PUSH 0
#define P3_MSG_BCAST 1
#define P3_MSG_PULL 2
#define P3_MSG_NOTIFY 3
#define P3_MSG_HELLO 4
#define P3_MSG_FIN 5
#define P3_EMORE 5 /* p3_frame_decode: incomplete frame, *n_out = bytes still needed */

typedef struct {
  uint32_t msg_type;    /* P3_MSG_* */
  uint32_t priority;
  uint64_t iteration;
  uint32_t worker_rank; /* u16 on the wire */
  uint32_t layer;
  uint32_t slice;
  uint64_t offset;
  uint32_t payload_len; /* bytes */
  uint32_t reserved;
} p3_frame_t;

/* encode_frame (proto.py:61-79): header + payload into out (cap bytes); *n_out = frame
 * bytes. P3_EPROTOCOL for a PUSH/BCAST payload that is not a float32 array or a payload on
 * a control frame; P3_EUSAGE for out-of-range fields or a short buffer. */
int p3_frame_encode(const p3_frame_t* f, const void* payload, uint8_t* out, uint64_t cap, uint64_t* n_out);
/* try_decode (proto.py:82-120) of the frame at the head of buf: P3_OK with *n_out = frame
 * bytes (the payload is buf + P3_FRAME_HEADER_BYTES), P3_EMORE with *n_out = bytes still
 * needed, or P3_EPROTOCOL (bad magic, unknown msg_type, payload over max_payload, payload on
 * a control frame; p3_last_error says which). */
int p3_frame_decode(const uint8_t* buf, uint64_t n, uint64_t max_payload, p3_frame_t* f, uint64_t* n_out);
/* Device: build n frames in out_dev — frame i at byte out_off_dev[i], its payload copied
 * from src_dev[i] (payload_len bytes; may be NULL for control frames). All arrays are
 * device memory; the headers are validated on the host side by the caller (see above). */
int p3_frames_pack(const p3_frame_t* frames_dev, const float* const* src_dev, const uint64_t* out_off_dev,
                   uint32_t n, uint8_t* out_dev, void* stream);
/* Device: decode n frames of in_dev (frame i at byte in_off_dev[i]) into frames_out_dev and
 * copy each payload to dst_dev[i] (NULL: header only). err_dev[0..2] receive the first
 * failure: P3_EPROTOCOL, the frame index, the reason (1 magic, 2 msg_type, 3 payload over
 * max_payload, 4 payload on a control frame); err_dev must be zeroed by the caller. */
int p3_frames_unpack(const uint8_t* in_dev, const uint64_t* in_off_dev, uint32_t n, uint64_t max_payload,
                     float* const* dst_dev, p3_frame_t* frames_out_dev, uint32_t* err_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* P3_H_ */
