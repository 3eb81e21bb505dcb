// Sync context: plan tables on the device, per-rank arenas, IPC bootstrap, stream memory
// operations for layer publication (enqueue_layer) and forward gating (_wait_layer), and
// the per-iteration launch of the comm kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "p3_internal.h"

namespace p3 {

static thread_local std::string g_thread_error;
void set_thread_error(const std::string& msg) { g_thread_error = msg; }

// ------------------------------------------------------------ driver entry points

// Virtual memory management and multicast (NVLS) entry points, resolved on first use.
struct Vmm {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) alloc_gran = nullptr;
  decltype(&cuMemExportToShareableHandle) export_h = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_h = nullptr;
  decltype(&cuMulticastCreate) mc_create = nullptr;
  decltype(&cuMulticastAddDevice) mc_add = nullptr;
  decltype(&cuMulticastBindMem) mc_bind = nullptr;
  decltype(&cuMulticastUnbind) mc_unbind = nullptr;
  decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
  bool ok = false;
};

static Vmm& vmm() {
  static Vmm v;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    auto get = [&](const char* name, void** fp) {
      cudaDriverEntryPointQueryResult q;
      ok &= cudaGetDriverEntryPointByVersion(name, fp, 12080, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess;
    };
    get("cuMemCreate", (void**)&v.create);
    get("cuMemRelease", (void**)&v.release);
    get("cuMemAddressReserve", (void**)&v.reserve);
    get("cuMemAddressFree", (void**)&v.addr_free);
    get("cuMemMap", (void**)&v.map);
    get("cuMemUnmap", (void**)&v.unmap);
    get("cuMemSetAccess", (void**)&v.set_access);
    get("cuMemGetAllocationGranularity", (void**)&v.alloc_gran);
    get("cuMemExportToShareableHandle", (void**)&v.export_h);
    get("cuMemImportFromShareableHandle", (void**)&v.import_h);
    get("cuMulticastCreate", (void**)&v.mc_create);
    get("cuMulticastAddDevice", (void**)&v.mc_add);
    get("cuMulticastBindMem", (void**)&v.mc_bind);
    get("cuMulticastUnbind", (void**)&v.mc_unbind);
    get("cuMulticastGetGranularity", (void**)&v.mc_gran);
    v.ok = ok;
  });
  return v;
}

typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_attr)(int*, CUdevice_attribute, CUdevice);

struct Driver {
  PFN_wait32 wait32 = nullptr;
  PFN_write32 write32 = nullptr;
  PFN_write64 write64 = nullptr;
  PFN_attr attr = nullptr;
  bool ok = false;
  bool has64 = false;
};

static Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    // the v2 stream memory operations (CUDA >= 11.7 semantics, incl. NO_MEMORY_BARRIER on
    // writes) straight from the driver library the runtime already loaded
    if (void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD)) {
      d.wait32 = (PFN_wait32)dlsym(h, "cuStreamWaitValue32_v2");
      d.write32 = (PFN_write32)dlsym(h, "cuStreamWriteValue32_v2");
      d.write64 = (PFN_write64)dlsym(h, "cuStreamWriteValue64_v2");
      d.attr = (PFN_attr)dlsym(h, "cuDeviceGetAttribute");
      if (d.wait32 && d.write32 && d.write64 && d.attr) {
        d.ok = true;
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (d.attr(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, dev) == CUDA_SUCCESS) d.has64 = v != 0;
        return;
      }
    }
    cudaDriverEntryPointQueryResult q;
    void* fp = nullptr;
    bool ok = true;
    ok &= cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &fp, 12000, cudaEnableDefault, &q) ==
              cudaSuccess && q == cudaDriverEntryPointSuccess;
    d.wait32 = (PFN_wait32)fp;
    ok &= cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &fp, 12000, cudaEnableDefault, &q) ==
              cudaSuccess && q == cudaDriverEntryPointSuccess;
    d.write32 = (PFN_write32)fp;
    ok &= cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", &fp, 12000, cudaEnableDefault, &q) ==
              cudaSuccess && q == cudaDriverEntryPointSuccess;
    d.write64 = (PFN_write64)fp;
    ok &= cudaGetDriverEntryPointByVersion("cuDeviceGetAttribute", &fp, 12000, cudaEnableDefault, &q) ==
              cudaSuccess && q == cudaDriverEntryPointSuccess;
    d.attr = (PFN_attr)fp;
    d.ok = ok;
    if (ok) {
      int dev = 0, v = 0;
      cudaGetDevice(&dev);
      if (d.attr(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, dev) == CUDA_SUCCESS) d.has64 = v != 0;
    }
  });
  return d;
}

static inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

}  // namespace p3

using namespace p3;

// Peer-visible arena of one rank: W | R | arrivals | hint | done (256-byte aligned parts).
struct PeerLayout {
  uint64_t w, r, arrivals, hint, tally, done, gdone, ntf_tail, ntf_ring, pull_tail, pull_ring, bytes;
};

// Local arena of one rank. The per-iteration part (cursor | srv_lo | srv_taken | it) is
// contiguous so one memset resets it before each launch.
struct LocalLayout {
  uint64_t pub, fifo_key, claim, iter_begin, cursor, srv_lo, srv_taken, it, pcount, slice_elems, stream_next, piece, iter_end, V,
      M, bytes, trace_n, trace, cta_phase, vclock, pubseq, ingested, heads, total;
};

struct p3_ctx {
  p3_config_t cfg;
  std::vector<uint64_t> counts;
  std::vector<p3_slice_t> plan;
  uint32_t L = 0, S = 0, N = 0, G = 0;
  std::vector<uint32_t> layer_group, group_slices;
  std::vector<uint64_t> layer_woff;
  std::vector<uint32_t> layer_nslices, layer_first;
  std::vector<uint32_t> slice_opos;  // position of each slice in the owner-grouped list
  // experiment / diagnostics switches, read once from the environment at creation:
  // P3_TMA=0 (direct loads instead of the TMA stage ring), P3_PUSH_SPLIT=n, P3_SRV_FILTER=n,
  // P3_TRACE_CTA=1 (trace records carry CTA indices; CTA start / exit records)
  struct {
    uint32_t use_tma = 1, push_split = 0xffffffffu, srv_filter = 0, trace_cta = 0, srv_reserve = 0, tma_store = 1, tma_store_red = 0, pop_relax = 0,
             push_max = 2, stream = 1, push_cap = 0, bcast_pull = 0, lazy_pick = 0, srv_piece = 0, push_ctas = 0;
  } knobs;
  std::vector<uint32_t> own_total;
  std::vector<uint64_t> own_stride;
  std::vector<uint64_t> bcast_in_bytes;  // per rank: broadcast payload received per iteration
  uint64_t w_elems = 0;
  int device = 0;
  // NVLS (cfg.nvls): VMM arenas shared by fd, and the multicast object over the replicas
  size_t alloc_gran = 0, mc_gran = 0, w_pad = 0;
  CUmemGenericAllocationHandle arena_h = 0;
  size_t arena_sz = 0;
  CUmemGenericAllocationHandle peer_h[P3_MAX_RANKS]{};
  size_t peer_sz[P3_MAX_RANKS]{};
  CUmemGenericAllocationHandle mc_h = 0;
  bool mc_added = false, mc_bound = false;
  float* mcw = nullptr;

  void* d_plan = nullptr;
  PlanDev plan_dev{};
  PeersDev peers{};
  LocalDev loc[P3_MAX_LOCAL]{};
  PeerLayout peer_layout[P3_MAX_RANKS]{};
  LocalLayout local_layout{};
  void* peer_arena[P3_MAX_LOCAL]{};
  void* local_arena[P3_MAX_LOCAL]{};
  float* grads[P3_MAX_LOCAL]{};
  void* opened[P3_MAX_RANKS]{};
  uint32_t* d_err = nullptr;
  uint32_t fifo_seq[P3_MAX_LOCAL]{};
  cudaEvent_t comm_done = nullptr;
  cudaEvent_t ready_ev[P3_MAX_LOCAL]{};
  cudaStream_t poll_stream = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaStream_t side[P3_SIDE_STREAMS]{};
  cudaEvent_t side_ev[P3_SIDE_STREAMS]{};
  cudaEvent_t iter_ev = nullptr;
  uint32_t side_next = 0;
  uint32_t side_used = 0;  // side streams that carry a DRAIN launch of the open iteration
  uint64_t open_iter = 0;
  bool iter_open = false;
  uint64_t launches = 0;
  uint64_t published[P3_MAX_LOCAL]{};  // gradient bytes published since the last DRAIN launch
  // publication ring (pinned, device-mapped) of each local rank
  PubEntry* ring_host[P3_MAX_LOCAL]{};
  uint32_t* ring_ingested_host[P3_MAX_LOCAL]{};
  uint32_t ring_tail[P3_MAX_LOCAL]{}, ring_flushed[P3_MAX_LOCAL]{};
  uint64_t pub_pending[P3_MAX_LOCAL]{};
  cudaStream_t pend_stream[P3_MAX_LOCAL]{};  // may be the legacy default stream (NULL)
  bool pend_valid[P3_MAX_LOCAL]{};           // pend_stream holds a publishing stream
  // every stream that published in the open iteration (the FINISH launch comes after all)
  std::vector<cudaStream_t> pub_streams[P3_MAX_LOCAL];
  cudaEvent_t switch_ev[P3_MAX_LOCAL]{};     // orders a new publishing stream after the previous one
  uint32_t n_side = P3_SIDE_STREAMS;         // side streams DRAIN launches rotate over
  bool comm_pending = false;
  uint64_t synced_iterations = 0;
  std::string err;
};

namespace {

int fail(p3_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  set_thread_error(msg);
  return code;
}

int cuda_fail(p3_ctx* c, cudaError_t e, const char* what) {
  return fail(c, P3_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                           \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #call); \
  } while (0)

#define CU_OK(call, what)                                                                          \
  do {                                                                                             \
    CUresult r_ = (call);                                                                          \
    if (r_ != CUDA_SUCCESS) return fail(c, P3_ECUDA, std::string(what) + " failed (CUresult " + std::to_string((int)r_) + ")"); \
  } while (0)

CUmemAllocationProp vmm_prop(const p3_ctx* c) {
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return ap;
}

CUmemAccessDesc vmm_access(const p3_ctx* c) {
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = c->device;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return ad;
}

// Map `h` (size bytes) at a fresh address aligned to the multicast granule, readable and
// writable from this context's GPU.
int vmm_map(p3_ctx* c, CUmemGenericAllocationHandle h, size_t size, void** out) {
  Vmm& v = vmm();
  CUdeviceptr va = 0;
  CU_OK(v.reserve(&va, size, c->mc_gran, 0, 0), "cuMemAddressReserve");
  CUresult r = v.map(va, size, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    v.addr_free(va, size);
    return fail(c, P3_ECUDA, "cuMemMap failed (CUresult " + std::to_string((int)r) + ")");
  }
  const CUmemAccessDesc ad = vmm_access(c);
  r = v.set_access(va, size, &ad, 1);
  if (r != CUDA_SUCCESS) {
    v.unmap(va, size);
    v.addr_free(va, size);
    return fail(c, P3_ECUDA, "cuMemSetAccess failed (CUresult " + std::to_string((int)r) + ")");
  }
  *out = reinterpret_cast<void*>(va);
  return P3_OK;
}

void vmm_unmap(void* va, size_t size) {
  vmm().unmap(reinterpret_cast<CUdeviceptr>(va), size);
  vmm().addr_free(reinterpret_cast<CUdeviceptr>(va), size);
}

PeerLayout peer_layout_of(const p3_ctx* c, uint32_t rank) {
  PeerLayout p;
  uint64_t o = 0;
  p.w = o;
  // (nvls: the replica region is bound to the multicast object in whole granules)
  o = align_up(o + c->w_elems * (c->cfg.param_bf16 ? 2 : 4), c->cfg.nvls ? c->mc_gran : 256);
  p.r = o;
  o = align_up(o + (uint64_t)c->N * c->own_stride[rank] * 4, 256);
  p.arrivals = o;
  o = align_up(o + (uint64_t)c->S * 4, 256);
  p.hint = o;
  o = align_up(o + (uint64_t)c->L * 4, 256);
  p.tally = o;
  o = align_up(o + 8, 256);
  p.done = o;
  o = align_up(o + (uint64_t)c->L * 4, 256);
  p.gdone = o;
  o = align_up(o + (uint64_t)c->G * 4, 256);
  const bool ring = (c->cfg.notify_pull || c->knobs.bcast_pull) && c->N > 1;
  p.ntf_tail = o;
  o = align_up(o + 4, 256);
  p.ntf_ring = o;
  o = align_up(o + (ring ? (uint64_t)c->S * 8 : 8), 256);
  p.pull_tail = o;
  o = align_up(o + 4, 256);
  p.pull_ring = o;
  o = align_up(o + (ring ? (uint64_t)c->S * (c->N - 1) * 8 : 8), 256);
  p.bytes = o;
  return p;
}

LocalLayout local_layout_of(const p3_ctx* c, uint64_t v_elems, uint64_t m_elems) {
  LocalLayout q;
  uint64_t o = 0;
  auto take = [&](uint64_t& field, uint64_t bytes) {
    field = o;
    o = align_up(o + bytes, 256);
  };
  take(q.pub, c->L * 8ull);
  take(q.fifo_key, c->L * 4ull);
  take(q.claim, c->S * 4ull);
  q.iter_begin = o;
  take(q.cursor, c->L * 4ull);
  take(q.srv_lo, c->L * 4ull);
  take(q.srv_taken, c->L * 4ull);
  take(q.it, sizeof(IterState));
  take(q.pcount, 8);
  take(q.slice_elems, c->N == 1 ? c->S * 4ull : 4ull);
  take(q.stream_next, 8);
  take(q.piece, c->N > 1 ? c->S * 8ull : 8ull);
  q.iter_end = o;
  take(q.V, v_elems * 4);
  take(q.M, m_elems * 4);
  take(q.bytes, 16);
  take(q.trace_n, 8);
  take(q.trace, (uint64_t)c->cfg.trace_cap * sizeof(p3_trace_rec_t));
  take(q.cta_phase, P3_DBG_CTAS * 4ull);
  take(q.vclock, 8);
  take(q.pubseq, 4);
  take(q.ingested, 4);
  take(q.heads, 8);
  q.total = o;
  return q;
}

void set_peer_pointers(p3_ctx* c, uint32_t rank, char* base) {
  const PeerLayout& p = c->peer_layout[rank];
  c->peers.W[rank] = reinterpret_cast<float*>(base + p.w);
  c->peers.R[rank] = reinterpret_cast<float*>(base + p.r);
  c->peers.arrivals[rank] = reinterpret_cast<uint32_t*>(base + p.arrivals);
  c->peers.hint[rank] = reinterpret_cast<uint32_t*>(base + p.hint);
  c->peers.tally[rank] = reinterpret_cast<uint32_t*>(base + p.tally);
  c->peers.done[rank] = reinterpret_cast<uint32_t*>(base + p.done);
  c->peers.gdone[rank] = reinterpret_cast<uint32_t*>(base + p.gdone);
  c->peers.ntf_tail[rank] = reinterpret_cast<uint32_t*>(base + p.ntf_tail);
  c->peers.ntf_ring[rank] = reinterpret_cast<unsigned long long*>(base + p.ntf_ring);
  c->peers.pull_tail[rank] = reinterpret_cast<uint32_t*>(base + p.pull_tail);
  c->peers.pull_ring[rank] = reinterpret_cast<unsigned long long*>(base + p.pull_ring);
}

int check_local(p3_ctx* c, uint32_t li) {
  if (!c) return fail(nullptr, P3_EUSAGE, "null context");
  if (li >= c->cfg.n_local) return fail(c, P3_EUSAGE, "local rank index out of range");
  return P3_OK;
}

}  // namespace

extern "C" {

const char* p3_last_error(p3_ctx_t* ctx) { return ctx ? ctx->err.c_str() : g_thread_error.c_str(); }

int p3_device_info(int* sm_count, int* stream_memops, int* cc_major, int* cc_minor) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_thread_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
    return P3_ECUDA;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (sm_count) cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  Driver& d = driver();
  if (stream_memops) *stream_memops = d.ok ? (d.has64 ? 2 : 1) : 0;
  return P3_OK;
}

int p3_ctx_create(const p3_config_t* cfg, p3_ctx_t** out) {
  p3_ctx* c = nullptr;
  if (!cfg || !out) return fail(nullptr, P3_EUSAGE, "null argument");
  if (cfg->world < 1 || cfg->world > P3_MAX_RANKS) return fail(nullptr, P3_EUSAGE, "world must be in [1, 16]");
  if (cfg->n_local < 1 || cfg->n_local > cfg->world || cfg->n_local > P3_MAX_LOCAL)
    return fail(nullptr, P3_EUSAGE, "bad n_local (1..min(world, 8))");
  if (cfg->n_layers < 1 || !cfg->layer_counts) return fail(nullptr, P3_EUSAGE, "profile needs at least one layer");
  if (cfg->plan_mode != P3_PLAN_P3 && cfg->plan_mode != P3_PLAN_BASELINE) return fail(nullptr, P3_EUSAGE, "bad plan_mode");
  if (cfg->throttle_bps < 0) return fail(nullptr, P3_EUSAGE, "throttle rate must be >= 0 (0 disables shaping)");
  // scheduler + signaler(s) + producer + at least one consumer warp (N > 1: P3_NSIG signalers)
  const uint32_t min_thr = 32u * (3u + (cfg->world > 1 ? (uint32_t)P3_NSIG : 1u));
  if (cfg->comm_threads < min_thr || cfg->comm_threads > P3_COMM_MAX_THREADS || cfg->comm_threads % 32)
    return fail(nullptr, P3_EUSAGE,
                "comm_threads must be a multiple of 32 in [" + std::to_string(min_thr) + ", " +
                    std::to_string(P3_COMM_MAX_THREADS) + "] (scheduler + signalers + producer + consumer warps)");
  if (cfg->comm_ctas < 1) return fail(nullptr, P3_EUSAGE, "comm_ctas must be >= 1");
  if (cfg->param_bf16 && (cfg->push_bf16 || cfg->emulate_grads))
    return fail(nullptr, P3_EUSAGE, "param_bf16 takes bf16 gradients from the model (no push_bf16, no emulate_grads)");
  if (cfg->drain_streams > P3_SIDE_STREAMS)
    return fail(nullptr, P3_EUSAGE, "drain_streams must be in [0, " + std::to_string(P3_SIDE_STREAMS) + "]");
  for (uint32_t i = 0; i < cfg->n_local; ++i)
    if (cfg->local_ranks[i] >= cfg->world) return fail(nullptr, P3_EUSAGE, "local rank out of range");
  if (!driver().ok) return fail(nullptr, P3_ECUDA, "CUDA driver stream memory operations unavailable");
  if (cfg->nvls) {
    if (cfg->world < 2 || cfg->n_local != 1)
      return fail(nullptr, P3_EUSAGE, "nvls needs world > 1 and one local rank per process");
    if (cfg->notify_pull || cfg->param_bf16)
      return fail(nullptr, P3_EUSAGE, "nvls broadcasts fp32 replicas in the P3 protocol (no notify_pull, no param_bf16)");
    if (!vmm().ok) return fail(nullptr, P3_ECUDA, "CUDA VMM / multicast driver entry points unavailable");
  }
  if (preload_kernels() != P3_OK) return fail(nullptr, P3_ECUDA, "loading the sm_100a kernels failed");

  c = new p3_ctx();
  c->cfg = *cfg;
  c->counts.assign(cfg->layer_counts, cfg->layer_counts + cfg->n_layers);
  c->cfg.layer_counts = c->counts.data();
  c->cfg.gate_groups = nullptr;  // consumed below, not retained
  c->L = cfg->n_layers;
  c->N = cfg->world;
  c->n_side = cfg->drain_streams ? cfg->drain_streams : P3_SIDE_STREAMS;
  {
    auto env_u32 = [](const char* name, uint32_t dflt) {
      const char* e = getenv(name);
      return e ? (uint32_t)atoi(e) : dflt;
    };
    c->knobs.use_tma = env_u32("P3_TMA", 1);
    // (unset: auto, see comm_args)
    c->knobs.push_split = env_u32("P3_PUSH_SPLIT", 0xffffffffu);
    c->knobs.srv_filter = env_u32("P3_SRV_FILTER", 0);
    c->knobs.trace_cta = getenv("P3_TRACE_CTA") != nullptr;
    c->knobs.srv_reserve = env_u32("P3_SRV_RESERVE", 0);
    c->knobs.tma_store = env_u32("P3_TMA_STORE", 1);
    c->knobs.pop_relax = env_u32("P3_POP_RELAX", 0);  // 0: the config's
    c->knobs.tma_store_red = env_u32("P3_TMA_STORE_RED", 0);
    c->knobs.push_max = env_u32("P3_PUSH_MAX", 2);
    if (P3_EXP) {  // experiment switches (a -DP3_EXP=1 build)
      c->knobs.push_cap = env_u32("P3_PUSH_CAP", 0);
      c->knobs.bcast_pull = env_u32("P3_BCAST_PULL", 0);
      c->knobs.lazy_pick = env_u32("P3_LAZY_PICK", 0);
      c->knobs.srv_piece = env_u32("P3_SRV_PIECE", 0) & ~7u;
      c->knobs.push_ctas = env_u32("P3_PUSH_CTAS", 0);
    } else {
      for (const char* k : {"P3_PUSH_CAP", "P3_BCAST_PULL", "P3_LAZY_PICK", "P3_SRV_PIECE", "P3_PUSH_CTAS"})
        if (getenv(k)) fprintf(stderr, "p3: %s ignored (experiment switch; build with -DP3_EXP=1)\n", k);
    }
    c->knobs.stream = env_u32("P3_STREAM", 1);  // single rank: streaming FINISH (0: slice pops)
  }
  std::string perr;
  int rc = cfg->plan_mode == P3_PLAN_P3
               ? build_p3_plan(c->counts.data(), c->L, c->N, cfg->max_slice, &c->plan, &perr)
               : build_baseline_plan(c->counts.data(), c->L, c->N, cfg->big_threshold, cfg->rng_seed, &c->plan, &perr);
  if (rc != P3_OK) {
    delete c;
    return fail(nullptr, rc, perr);
  }
  if (c->plan.size() >= 0x7fffffffull) {
    delete c;
    return fail(nullptr, P3_EUSAGE, "too many slices");
  }
  c->S = (uint32_t)c->plan.size();
  cudaGetDevice(&c->device);
  if (cfg->nvls) {  // allocation and multicast granules (the replica region is bound in whole granules)
    int mc = 0;
    driver().attr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, c->device);
    if (!mc) {
      int r2 = fail(c, P3_EUSAGE, "nvls: this GPU does not support multicast objects (no NVSwitch / fabric manager)");
      delete c;
      return r2;
    }
    const CUmemAllocationProp ap = vmm_prop(c);
    CUmulticastObjectProp mp = {};
    mp.numDevices = c->N;
    mp.size = 2ull << 20;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    if (vmm().alloc_gran(&c->alloc_gran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS ||
        vmm().mc_gran(&c->mc_gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) {
      int r2 = fail(c, P3_ECUDA, "nvls: granularity query failed");
      delete c;
      return r2;
    }
    c->mc_gran = std::max(c->mc_gran, c->alloc_gran);
  }

  // ---- host-side plan tables
  const uint32_t L = c->L, S = c->S, N = c->N;
  c->layer_woff.resize(L);
  c->layer_nslices.assign(L, 0);
  c->layer_first.assign(L, 0);
  uint64_t w = 0;
  for (uint32_t l = 0; l < L; ++l) {
    c->layer_woff[l] = w;
    w = align_up(w + c->counts[l], 64);  // 256-byte aligned layer starts
  }
  c->w_elems = w;
  std::vector<uint64_t> slice_off(S), slice_slot(S);
  std::vector<uint32_t> slice_len(S), slice_layer(S), slice_owner(S);
  std::vector<uint32_t> own_list;
  std::vector<uint32_t> own_lfirst((size_t)N * L, 0), own_lcount((size_t)N * L, 0);
  c->own_total.assign(N, 0);
  c->own_stride.assign(N, 0);
  c->bcast_in_bytes.assign(N, 0);
  for (uint32_t g = 0; g < S; ++g) {
    const p3_slice_t& r = c->plan[g];
    if (r.slice == 0) c->layer_first[r.layer] = g;
    c->layer_nslices[r.layer]++;
    slice_off[g] = r.offset;
    slice_len[g] = (uint32_t)r.length;
    slice_layer[g] = r.layer;
    slice_owner[g] = r.server;
    if (r.length >= 0xffffffffull) {
      delete c;
      return fail(nullptr, P3_EUSAGE, "max_slice too large");
    }
  }
  own_list.reserve(S);
  c->slice_opos.assign(S, 0);
  for (uint32_t o = 0; o < N; ++o) {
    uint64_t slot = 0;
    for (uint32_t l = 0; l < L; ++l) {
      own_lfirst[(size_t)o * L + l] = (uint32_t)own_list.size();
      for (uint32_t s = 0; s < c->layer_nslices[l]; ++s) {
        const uint32_t g = c->layer_first[l] + s;
        if (slice_owner[g] != o) continue;
        c->slice_opos[g] = (uint32_t)own_list.size();
        own_list.push_back(g);
        own_lcount[(size_t)o * L + l]++;
        slice_slot[g] = slot;
        slot = align_up(slot + slice_len[g], 64);
      }
    }
    c->own_stride[o] = std::max<uint64_t>(slot, 64);
  }
  {
    std::vector<uint32_t> tot(N, 0);
    for (uint32_t g = 0; g < S; ++g) tot[slice_owner[g]]++;
    c->own_total = tot;
    for (uint32_t r = 0; r < N; ++r)
      for (uint32_t g = 0; g < S; ++g)
        if (slice_owner[g] != r) c->bcast_in_bytes[r] += 4ull * slice_len[g];
  }

  // ---- forward-gate groups
  c->layer_group.resize(L);
  for (uint32_t l = 0; l < L; ++l) c->layer_group[l] = cfg->gate_groups ? cfg->gate_groups[l] : l;
  for (uint32_t l = 0; l < L; ++l) c->G = std::max(c->G, c->layer_group[l] + 1);
  if (c->G > L) {
    delete c;
    return fail(nullptr, P3_EUSAGE, "gate group ids must be < n_layers");
  }
  c->group_slices.assign(c->G, 0);
  for (uint32_t l = 0; l < L; ++l) c->group_slices[c->layer_group[l]] += c->layer_nslices[l];

  // ---- device plan tables: one allocation
  std::vector<char> blob;
  auto put = [&](const void* src, size_t bytes) -> size_t {
    size_t off = align_up(blob.size(), 256);
    blob.resize(off + std::max<size_t>(bytes, 4));
    if (bytes) std::memcpy(blob.data() + off, src, bytes);
    return off;
  };
  const size_t o_lns = put(c->layer_nslices.data(), L * 4ull);
  const size_t o_lf = put(c->layer_first.data(), L * 4ull);
  const size_t o_lw = put(c->layer_woff.data(), L * 8ull);
  const size_t o_so = put(slice_off.data(), S * 8ull);
  const size_t o_sl = put(slice_len.data(), S * 4ull);
  const size_t o_sly = put(slice_layer.data(), S * 4ull);
  const size_t o_sow = put(slice_owner.data(), S * 4ull);
  const size_t o_ss = put(slice_slot.data(), S * 8ull);
  const size_t o_ol = put(own_list.data(), own_list.size() * 4ull);
  const size_t o_sop = put(c->slice_opos.data(), S * 4ull);
  const size_t o_olf = put(own_lfirst.data(), own_lfirst.size() * 4ull);
  const size_t o_olc = put(own_lcount.data(), own_lcount.size() * 4ull);
  const size_t o_ot = put(c->own_total.data(), N * 4ull);
  const size_t o_ost = put(c->own_stride.data(), N * 8ull);
  const size_t o_lg = put(c->layer_group.data(), L * 4ull);
  std::vector<uint32_t> own_base(N, 0);
  for (uint32_t o = 1; o < N; ++o) own_base[o] = own_base[o - 1] + c->own_total[o - 1];
  const size_t o_ob = put(own_base.data(), N * 4ull);
  std::vector<uint64_t> flat(L + 1, 0);
  for (uint32_t l = 0; l < L; ++l) flat[l + 1] = flat[l] + align_up(c->counts[l], 8);
  const size_t o_fl = put(flat.data(), (L + 1) * 8ull);
  bool rr = true;
  for (uint32_t g = 0; g < S && rr; ++g) rr = slice_owner[g] == g % N;
  cudaError_t e = cudaMalloc(&c->d_plan, blob.size());
  if (e == cudaSuccess) e = cudaMemcpy(c->d_plan, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_err, 256);
  if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, 256);
  if (e != cudaSuccess) {
    int r2 = cuda_fail(c, e, "plan upload");
    p3_ctx_destroy(c);
    return r2;
  }
  char* pb = static_cast<char*>(c->d_plan);
  PlanDev& P = c->plan_dev;
  P.n_layers = L;
  P.total_slices = S;
  P.world = N;
  P.layer_nslices = reinterpret_cast<const uint32_t*>(pb + o_lns);
  P.layer_first = reinterpret_cast<const uint32_t*>(pb + o_lf);
  P.layer_woff = reinterpret_cast<const uint64_t*>(pb + o_lw);
  P.slice_off = reinterpret_cast<const uint64_t*>(pb + o_so);
  P.slice_len = reinterpret_cast<const uint32_t*>(pb + o_sl);
  P.slice_layer = reinterpret_cast<const uint32_t*>(pb + o_sly);
  P.slice_owner = reinterpret_cast<const uint32_t*>(pb + o_sow);
  P.slice_slot = reinterpret_cast<const uint64_t*>(pb + o_ss);
  P.own_list = reinterpret_cast<const uint32_t*>(pb + o_ol);
  P.slice_opos = reinterpret_cast<const uint32_t*>(pb + o_sop);
  P.own_lfirst = reinterpret_cast<const uint32_t*>(pb + o_olf);
  P.own_lcount = reinterpret_cast<const uint32_t*>(pb + o_olc);
  P.own_total = reinterpret_cast<const uint32_t*>(pb + o_ot);
  P.own_stride = reinterpret_cast<const uint64_t*>(pb + o_ost);
  P.layer_group = reinterpret_cast<const uint32_t*>(pb + o_lg);
  P.own_base = reinterpret_cast<const uint32_t*>(pb + o_ob);
  P.layer_flat = reinterpret_cast<const uint64_t*>(pb + o_fl);
  P.rr_owner = rr ? 1u : 0u;

  // ---- per-rank arenas
  for (uint32_t r = 0; r < N; ++r) c->peer_layout[r] = peer_layout_of(c, r);
  for (uint32_t i = 0; i < cfg->n_local; ++i) {
    const uint32_t rank = cfg->local_ranks[i];
    const PeerLayout& pl = c->peer_layout[rank];
    if (cfg->nvls) {  // VMM allocation, shareable by file descriptor (p3_ctx_export_fd)
      const CUmemAllocationProp ap = vmm_prop(c);
      c->arena_sz = align_up(pl.bytes, c->mc_gran);
      e = cudaErrorMemoryAllocation;
      if (vmm().create(&c->arena_h, c->arena_sz, &ap, 0) == CUDA_SUCCESS &&
          vmm_map(c, c->arena_h, c->arena_sz, &c->peer_arena[i]) == P3_OK)
        e = cudaMemset(c->peer_arena[i], 0, c->arena_sz);
      c->w_pad = pl.r;  // the replica region, whole multicast granules
    } else {
      e = cudaMalloc(&c->peer_arena[i], pl.bytes);
      if (e == cudaSuccess) e = cudaMemset(c->peer_arena[i], 0, pl.bytes);
    }
    const uint64_t v_elems = cfg->momentum != 0.f ? c->own_stride[rank] : 0;
    const uint64_t m_elems = cfg->param_bf16 ? c->own_stride[rank] : 0;
    LocalLayout ll = local_layout_of(c, v_elems, m_elems);
    c->local_layout = ll;
    if (e == cudaSuccess) e = cudaMalloc(&c->local_arena[i], ll.total);
    if (e == cudaSuccess) e = cudaMemset(c->local_arena[i], 0, ll.total);
    if (e == cudaSuccess && cfg->emulate_grads) {
      e = cudaMalloc(&c->grads[i], std::max<uint64_t>(c->w_elems, 4) * 4);
      if (e == cudaSuccess) e = cudaMemset(c->grads[i], 0, std::max<uint64_t>(c->w_elems, 4) * 4);
    }
    if (e != cudaSuccess) {
      int r2 = cuda_fail(c, e, "arena allocation");
      p3_ctx_destroy(c);
      return r2;
    }
    set_peer_pointers(c, rank, static_cast<char*>(c->peer_arena[i]));
    char* lb = static_cast<char*>(c->local_arena[i]);
    LocalDev& D = c->loc[i];
    D.rank = rank;
    D.trace_cap = cfg->trace_cap;
    D.pub = reinterpret_cast<uint64_t*>(lb + ll.pub);
    D.fifo_key = reinterpret_cast<uint32_t*>(lb + ll.fifo_key);
    D.claim = reinterpret_cast<uint32_t*>(lb + ll.claim);
    D.cursor = reinterpret_cast<uint32_t*>(lb + ll.cursor);
    D.srv_lo = reinterpret_cast<uint32_t*>(lb + ll.srv_lo);
    D.srv_taken = reinterpret_cast<uint32_t*>(lb + ll.srv_taken);
    D.it = reinterpret_cast<IterState*>(lb + ll.it);
    D.V = v_elems ? reinterpret_cast<float*>(lb + ll.V) : nullptr;
    D.M = m_elems ? reinterpret_cast<float*>(lb + ll.M) : nullptr;
    D.bytes = reinterpret_cast<unsigned long long*>(lb + ll.bytes);
    D.trace_n = reinterpret_cast<unsigned long long*>(lb + ll.trace_n);
    D.trace = reinterpret_cast<p3_trace_rec_t*>(lb + ll.trace);
    D.cta_phase = reinterpret_cast<uint32_t*>(lb + ll.cta_phase);
    D.vclock = reinterpret_cast<unsigned long long*>(lb + ll.vclock);
    D.pubseq = reinterpret_cast<uint32_t*>(lb + ll.pubseq);
    D.ingested = reinterpret_cast<uint32_t*>(lb + ll.ingested);
    D.pcount = reinterpret_cast<uint32_t*>(lb + ll.pcount);
    D.slice_elems = reinterpret_cast<uint32_t*>(lb + ll.slice_elems);
    D.stream_next = reinterpret_cast<unsigned long long*>(lb + ll.stream_next);
    D.piece_next = reinterpret_cast<uint32_t*>(lb + ll.piece);
    D.piece_done = D.piece_next + (c->N > 1 ? c->S : 1u);
    D.ntf_head = reinterpret_cast<uint32_t*>(lb + ll.heads);
    D.pull_head = D.ntf_head + 1;
    D.ring_cap = 4 * L + 64;
    if (e == cudaSuccess)
      e = cudaHostAlloc((void**)&c->ring_host[i], D.ring_cap * sizeof(PubEntry) + 256, cudaHostAllocMapped);
    if (e == cudaSuccess) {
      std::memset(c->ring_host[i], 0, D.ring_cap * sizeof(PubEntry) + 256);
      c->ring_ingested_host[i] = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c->ring_host[i]) +
                                                             D.ring_cap * sizeof(PubEntry));
      void* dp = nullptr;
      e = cudaHostGetDevicePointer(&dp, c->ring_host[i], 0);
      D.ring = static_cast<const PubEntry*>(dp);
      D.ingested_host = reinterpret_cast<uint32_t*>(static_cast<char*>(dp) + D.ring_cap * sizeof(PubEntry));
    }
    if (e != cudaSuccess) {
      int r2 = cuda_fail(c, e, "publication ring");
      p3_ctx_destroy(c);
      return r2;
    }
  }
  e = cudaEventCreateWithFlags(&c->comm_done, cudaEventDisableTiming);
  for (uint32_t i = 0; i < cfg->n_local && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&c->ready_ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->switch_ev[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->iter_ev, cudaEventDisableTiming);
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (int j = 0; j < P3_SIDE_STREAMS && e == cudaSuccess; ++j) {
      e = cudaStreamCreateWithPriority(&c->side[j], cudaStreamNonBlocking, hi);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->side_ev[j], cudaEventDisableTiming);
    }
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->poll_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    int r2 = cuda_fail(c, e, "context init");
    p3_ctx_destroy(c);
    return r2;
  }
  *out = c;
  return P3_OK;
}

int p3_ctx_destroy(p3_ctx_t* c) {
  if (!c) return P3_OK;
  cudaDeviceSynchronize();
  if (c->cfg.nvls) {  // multicast mapping and binding, peers' and the own VMM arena
    Vmm& v = vmm();
    if (c->mcw) vmm_unmap(c->mcw, c->w_pad);
    if (c->mc_bound) v.mc_unbind(c->mc_h, (CUdevice)c->device, 0, c->w_pad);
    if (c->mc_h) v.release(c->mc_h);
    for (uint32_t r = 0; r < P3_MAX_RANKS; ++r)
      if (c->peer_h[r]) {
        if (c->opened[r]) vmm_unmap(c->opened[r], c->peer_sz[r]);
        v.release(c->peer_h[r]);
        c->opened[r] = nullptr;
      }
    if (c->arena_h) {
      if (c->peer_arena[0]) vmm_unmap(c->peer_arena[0], c->arena_sz);
      v.release(c->arena_h);
      c->peer_arena[0] = nullptr;
    }
  }
  for (uint32_t r = 0; r < P3_MAX_RANKS; ++r)
    if (c->opened[r]) cudaIpcCloseMemHandle(c->opened[r]);
  for (uint32_t i = 0; i < P3_MAX_LOCAL; ++i) {
    if (c->peer_arena[i]) cudaFree(c->peer_arena[i]);
    if (c->local_arena[i]) cudaFree(c->local_arena[i]);
    if (c->grads[i]) cudaFree(c->grads[i]);
    if (c->ring_host[i]) cudaFreeHost(c->ring_host[i]);
  }
  if (c->d_plan) cudaFree(c->d_plan);
  if (c->d_err) cudaFree(c->d_err);
  if (c->comm_done) cudaEventDestroy(c->comm_done);
  if (c->iter_ev) cudaEventDestroy(c->iter_ev);
  for (int j = 0; j < P3_SIDE_STREAMS; ++j) {
    if (c->side[j]) cudaStreamDestroy(c->side[j]);
    if (c->side_ev[j]) cudaEventDestroy(c->side_ev[j]);
  }
  for (uint32_t i = 0; i < P3_MAX_LOCAL; ++i) {
    if (c->ready_ev[i]) cudaEventDestroy(c->ready_ev[i]);
    if (c->switch_ev[i]) cudaEventDestroy(c->switch_ev[i]);
  }
  if (c->poll_stream) cudaStreamDestroy(c->poll_stream);
  delete c;
  return P3_OK;
}

int p3_ctx_ipc_handle(p3_ctx_t* c, uint32_t li, void* out) {
  int rc = check_local(c, li);
  if (rc) return rc;
  static_assert(sizeof(cudaIpcMemHandle_t) <= P3_IPC_BYTES, "ipc handle size");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->peer_arena[li]));
  std::memset(out, 0, P3_IPC_BYTES);
  std::memcpy(out, &h, sizeof(h));
  return P3_OK;
}

int p3_ctx_open_peers(p3_ctx_t* c, const void* handles) {
  if (!c || !handles) return fail(c, P3_EUSAGE, "null argument");
  const char* hb = static_cast<const char*>(handles);
  for (uint32_t r = 0; r < c->N; ++r) {
    bool local = false;
    for (uint32_t i = 0; i < c->cfg.n_local; ++i) local |= c->cfg.local_ranks[i] == r;
    if (local || c->opened[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + (size_t)r * P3_IPC_BYTES, sizeof(h));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->opened[r] = p;
    set_peer_pointers(c, r, static_cast<char*>(p));
  }
  return P3_OK;
}

int p3_ctx_export_fd(p3_ctx_t* c, uint32_t li, int* fd) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (!c->cfg.nvls || !fd) return fail(c, P3_EUSAGE, "p3_ctx_export_fd needs an nvls context and an output");
  int f = -1;
  CU_OK(vmm().export_h(&f, c->arena_h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle");
  *fd = f;
  return P3_OK;
}

int p3_ctx_open_peers_fd(p3_ctx_t* c, const int* fds) {
  if (!c || !fds) return fail(c, P3_EUSAGE, "null argument");
  if (!c->cfg.nvls) return fail(c, P3_EUSAGE, "p3_ctx_open_peers_fd needs an nvls context (else p3_ctx_open_peers)");
  const uint32_t me = c->cfg.local_ranks[0];
  for (uint32_t r = 0; r < c->N; ++r) {
    if (r == me || c->opened[r]) continue;
    CUmemGenericAllocationHandle h = 0;
    CU_OK(vmm().import_h(&h, reinterpret_cast<void*>((intptr_t)fds[r]), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
          "cuMemImportFromShareableHandle");
    const size_t sz = align_up(c->peer_layout[r].bytes, c->mc_gran);
    void* va = nullptr;
    int rc = vmm_map(c, h, sz, &va);
    if (rc) {
      vmm().release(h);
      return rc;
    }
    c->peer_h[r] = h;
    c->peer_sz[r] = sz;
    c->opened[r] = va;
    set_peer_pointers(c, r, static_cast<char*>(va));
  }
  return P3_OK;
}

int p3_nvls_create(p3_ctx_t* c, int* fd) {
  if (!c || !fd) return fail(c, P3_EUSAGE, "null argument");
  if (!c->cfg.nvls || c->mc_h) return fail(c, P3_EUSAGE, "p3_nvls_create: not an nvls context, or it already has a multicast object");
  CUmulticastObjectProp mp = {};
  mp.numDevices = c->N;
  mp.size = c->w_pad;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CU_OK(vmm().mc_create(&c->mc_h, &mp), "cuMulticastCreate");
  int f = -1;
  CU_OK(vmm().export_h(&f, c->mc_h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle (multicast)");
  *fd = f;
  return P3_OK;
}

int p3_nvls_attach(p3_ctx_t* c, int fd) {
  if (!c || !c->cfg.nvls) return fail(c, P3_EUSAGE, "p3_nvls_attach needs an nvls context");
  if (fd >= 0) {
    if (c->mc_h) return fail(c, P3_EUSAGE, "p3_nvls_attach: the creator passes -1");
    CU_OK(vmm().import_h(&c->mc_h, reinterpret_cast<void*>((intptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
          "cuMemImportFromShareableHandle (multicast)");
  }
  if (!c->mc_h) return fail(c, P3_EUSAGE, "p3_nvls_attach: no multicast object (p3_nvls_create on one rank, its fd on the others)");
  if (!c->mc_added) CU_OK(vmm().mc_add(c->mc_h, (CUdevice)c->device), "cuMulticastAddDevice");
  c->mc_added = true;
  return P3_OK;
}

int p3_nvls_bind(p3_ctx_t* c) {
  if (!c || !c->cfg.nvls || !c->mc_added) return fail(c, P3_EUSAGE, "p3_nvls_bind: attach first (every rank)");
  if (c->mcw) return P3_OK;
  CU_OK(vmm().mc_bind(c->mc_h, 0, c->arena_h, 0, c->w_pad, 0), "cuMulticastBindMem");
  c->mc_bound = true;
  void* va = nullptr;
  int rc = vmm_map(c, c->mc_h, c->w_pad, &va);
  if (rc) return rc;
  c->mcw = static_cast<float*>(va);
  return P3_OK;
}

int p3_ctx_params(p3_ctx_t* c, uint32_t li, float** params) {
  int rc = check_local(c, li);
  if (rc) return rc;
  *params = c->peers.W[c->cfg.local_ranks[li]];
  return P3_OK;
}

static CommArgs comm_args(p3_ctx* c, uint32_t mode, uint32_t ctas);

int p3_master_init(p3_ctx_t* c, uint32_t li, void* stream) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (!c->cfg.param_bf16) return fail(c, P3_EUSAGE, "p3_master_init needs param_bf16");
  CommArgs a = comm_args(c, P3_COMM_FINISH, 1);
  a.loc[0] = c->loc[li];
  a.n_local = 1;
  if (launch_master_init(a, stream) != P3_OK) return cuda_fail(c, cudaGetLastError(), "master init launch");
  return P3_OK;
}

int p3_ctx_grads(p3_ctx_t* c, uint32_t li, float** grads) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (!c->grads[li]) return fail(c, P3_EUSAGE, "context has no gradient arena (emulate_grads = 0)");
  *grads = c->grads[li];
  return P3_OK;
}

int p3_ctx_layer_offset(p3_ctx_t* c, uint32_t layer, uint64_t* off) {
  if (!c || layer >= c->L) return fail(c, P3_EUSAGE, "layer out of range");
  *off = c->layer_woff[layer];
  return P3_OK;
}

static CommArgs comm_args(p3_ctx* c, uint32_t mode, uint32_t ctas) {
  CommArgs a;
  std::memset(&a, 0, sizeof(a));
  a.plan = c->plan_dev;
  a.peers = c->peers;
  for (uint32_t i = 0; i < c->cfg.n_local; ++i) a.loc[i] = c->loc[i];
  a.n_local = c->cfg.n_local;
  a.mode = mode;
  for (uint32_t r = 0; r < c->N; ++r) a.remote |= c->opened[r] != nullptr;
  a.k = (uint32_t)c->open_iter;
  a.sched = c->cfg.sched;
  a.lr = c->cfg.lr;
  a.momentum = c->cfg.momentum;
  a.timeout_ns = (unsigned long long)(c->cfg.timeout_s * 1e9);
  a.err = c->d_err;
  a.linger_ns = (unsigned long long)c->cfg.drain_linger_us * 1000ull;
  // single rank: about two jobs per CTA, at most 8 slices per job
  // (measured, tools/sync_sweep.py: about four jobs per CTA balances per-job overhead and the
  // tail; a stash of extra claims loses more to imbalance than it saves in pick time)
  a.pop_run = c->cfg.pop_run ? c->cfg.pop_run
                             : std::max<uint32_t>(1, std::min<uint32_t>(8, c->S / std::max<uint32_t>(1, 4 * ctas)));
  a.pop_multi = std::max<uint32_t>(1, std::min<uint32_t>(4, c->cfg.pop_multi ? c->cfg.pop_multi : 1));
  a.push_bf16 = c->cfg.push_bf16 ? 1u : 0u;
  a.pb16 = c->cfg.param_bf16 ? 1u : 0u;
  a.notify = c->N < 2 ? 0u : c->cfg.notify_pull ? 1u : c->knobs.bcast_pull ? 2u : 0u;
  a.ntf_cap = c->S;
  a.pull_cap = c->S * (c->N > 1 ? c->N - 1 : 1);
  a.trace_cta = c->knobs.trace_cta;
  // auto: every 2nd CTA of an unthrottled FINISH launch looks for pushes before server work
  // (N=2 sync-only with one signaler per slot: ResNet-50 -3%, seq2seq -2%, VGG-19 -1%); not in
  // DRAIN launches or under the K7 throttle, where it cost throttled P3 training 17% at N=2
  // (profiles/r02_summary.md §7)
  a.push_split = c->knobs.push_split != 0xffffffffu ? c->knobs.push_split
                 : (mode == P3_COMM_FINISH && c->cfg.throttle_bps <= 0) ? 2u : 0u;
  a.srv_filter = c->knobs.srv_filter;
  a.use_tma = c->knobs.use_tma;
  a.srv_reserve = c->knobs.srv_reserve;
  a.tma_store = c->knobs.tma_store;
  a.tma_store_red = c->mcw ? 0u : c->knobs.tma_store_red;  // (nvls: replicas by multimem.st)
  a.push_max = c->knobs.push_max;
  a.push_cap = c->knobs.push_cap;
  a.lazy_pick = c->knobs.lazy_pick;
  a.srv_piece = c->knobs.srv_piece;
  a.push_ctas = c->knobs.push_ctas;
  a.mcw = c->mcw;
  // bounded relaxation of the pop order: a pop takes one of the C most urgent slices, C =
  // the launch's concurrent consumers (its CTAs) unless configured lower
  // (measured, tools/sync_sweep.py, ResNet-50 N=1 sync-only: C=8 2.2 TB/s, C=148 3.4 TB/s —
  // 148 schedulers racing for the same few one-slice layers lose an atomic round trip per try)
  const uint32_t relax_cfg = c->knobs.pop_relax ? c->knobs.pop_relax : c->cfg.pop_relax;
  a.pop_relax = std::min<uint32_t>(ctas, relax_cfg ? relax_cfg : ctas);
  if (c->cfg.throttle_bps > 0) {
    a.ns_per_byte = (float)(8e9 / c->cfg.throttle_bps);
    a.burst_ns = (unsigned long long)((double)c->cfg.throttle_burst * 8e9 / c->cfg.throttle_bps);
  }
  return a;
}

// Publish local rank li's ring entries up to its tail: one stream memory write of the tail,
// ordered after the kernels that produced those gradients on their stream.
static int flush_publications(p3_ctx* c, uint32_t li) {
  if (c->ring_flushed[li] == c->ring_tail[li]) return P3_OK;
  CUresult r = driver().write32((CUstream)c->pend_stream[li], (CUdeviceptr)c->loc[li].pubseq, c->ring_tail[li], 0);
  if (r != CUDA_SUCCESS) return fail(c, P3_ECUDA, "cuStreamWriteValue32 failed (code " + std::to_string(r) + ")");
  c->ring_flushed[li] = c->ring_tail[li];
  c->pub_pending[li] = 0;
  return P3_OK;
}

// DRAIN launches rotate over side streams so a long-running launch (link-bound, or down to
// its last CTAs while it keeps ingesting newly published layers) never holds back the next
// one: concurrent launches share the device queue. Each side stream starts the iteration
// after the per-iteration reset on the main comm stream; the FINISH launch on the main comm
// stream comes after all of them.
static int launch_drain(p3_ctx* c, int li) {
  const uint32_t j = c->side_next++ % c->n_side;
  cudaStream_t s = c->side[j];
  if (!(c->side_used & (1u << j))) {  // first launch of the iteration here: after the reset
    CK(cudaStreamWaitEvent(s, c->iter_ev, 0));
    c->side_used |= 1u << j;
  }
  CK(cudaEventRecord(c->ready_ev[li], c->pend_stream[li]));
  CK(cudaStreamWaitEvent(s, c->ready_ev[li], 0));
  c->published[li] = 0;
  if (launch_comm(comm_args(c, P3_COMM_DRAIN, c->cfg.comm_ctas), c->cfg.comm_ctas, c->cfg.comm_threads, s) != P3_OK)
    return cuda_fail(c, cudaGetLastError(), "comm kernel launch");
  c->launches++;
  return P3_OK;
}

int p3_iteration_begin(p3_ctx_t* c, uint64_t k, void* stream) {
  if (!c) return fail(nullptr, P3_EUSAGE, "null context");
  if (k >= 0x3fffffffull) return fail(c, P3_EUSAGE, "iteration out of range");
  if (c->iter_open) return fail(c, P3_EUSAGE, "previous iteration not ended (p3_iteration_end)");
  for (uint32_t r = 0; r < c->N; ++r)
    if (!c->peers.W[r]) return fail(c, P3_EUSAGE, "peer arenas not opened (call p3_ctx_open_peers)");
  if (c->cfg.nvls && !c->mcw) return fail(c, P3_EUSAGE, "nvls multicast not bound (p3_nvls_attach + p3_nvls_bind)");
  cudaStream_t s = (cudaStream_t)stream;
  const LocalLayout& ll = c->local_layout;
  for (uint32_t i = 0; i < c->cfg.n_local; ++i) {
    CK(cudaMemsetAsync(static_cast<char*>(c->local_arena[i]) + ll.iter_begin, 0, ll.iter_end - ll.iter_begin, s));
    c->pend_valid[i] = false;  // (everything of the previous iteration was flushed at its end)
    c->pub_streams[i].clear();
  }
  CK(cudaEventRecord(c->iter_ev, s));  // side streams wait for it when they get a DRAIN launch
  c->side_used = 0;
  c->comm_stream = s;
  c->open_iter = k;
  c->iter_open = true;
  return P3_OK;
}

int p3_iteration_end(p3_ctx_t* c, uint64_t k) {
  if (!c) return fail(nullptr, P3_EUSAGE, "null context");
  if (!c->iter_open || c->open_iter != k) return fail(c, P3_EUSAGE, "iteration not open");
  // publish what is still pending and order the FINISH launch after every producing stream
  for (uint32_t i = 0; i < c->cfg.n_local; ++i) {
    if (!c->pend_valid[i]) continue;
    int rc = flush_publications(c, i);
    if (rc) return rc;
    for (cudaStream_t ps : c->pub_streams[i]) {
      CK(cudaEventRecord(c->ready_ev[i], ps));
      CK(cudaStreamWaitEvent(c->comm_stream, c->ready_ev[i], 0));
    }
    c->published[i] = 0;
  }
  for (int j = 0; j < P3_SIDE_STREAMS; ++j) {  // only the side streams used this iteration
    if (!(c->side_used & (1u << j))) continue;
    CK(cudaEventRecord(c->side_ev[j], c->side[j]));
    CK(cudaStreamWaitEvent(c->comm_stream, c->side_ev[j], 0));
  }
  const uint32_t ctas = c->cfg.finish_ctas ? c->cfg.finish_ctas : c->cfg.comm_ctas;
  // Single rank, no DRAIN launch this iteration, relaxed order allowed: nothing to exchange and
  // every layer published — the FINISH work is one priority-ordered streaming update of the
  // whole parameter space (k_update_stream); otherwise the comm kernel.
  const bool stream = c->N == 1 && c->side_used == 0 && c->cfg.pop_relax != 1 && !c->cfg.param_bf16 &&
                      c->knobs.stream;
  if (stream) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    if (launch_update_stream(comm_args(c, P3_COMM_FINISH, ctas), (uint32_t)sms, c->comm_stream) != P3_OK)
      return cuda_fail(c, cudaGetLastError(), "update kernel launch");
  } else if (launch_comm(comm_args(c, P3_COMM_FINISH, ctas), ctas, c->cfg.comm_threads, c->comm_stream) != P3_OK) {
    return cuda_fail(c, cudaGetLastError(), "comm kernel launch");
  }
  c->launches++;
  CK(cudaEventRecord(c->comm_done, c->comm_stream));
  c->comm_pending = true;
  c->iter_open = false;
  return P3_OK;
}

int p3_layer_ready(p3_ctx_t* c, uint32_t li, uint32_t layer, uint64_t k, const float* grad, void* stream) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (layer >= c->L) return fail(c, P3_EUSAGE, "layer out of range");
  if (!grad) {
    if (!c->grads[li]) return fail(c, P3_EUSAGE, "no gradient pointer and no gradient arena");
    grad = c->grads[li] + c->layer_woff[layer];
  }
  const uint64_t gp = (uint64_t)(uintptr_t)grad;
  if (gp >> 48) return fail(c, P3_EUSAGE, "gradient pointer does not fit the 48-bit publication word");
  // FrameQueue.put_batch is atomic (queues.py:44-50): one word makes every slice of the layer
  // poppable — the iteration tag and the gradient pointer together
  const uint64_t word = (((k + 1) & 0xffffull) << 48) | gp;
  if (c->iter_open && c->open_iter == k) {
    // Batched publication: the layer becomes poppable when the comm launch that carries it
    // starts — stream-ordered after this point of `stream` by an event — so no stream memory
    // write is needed (each costs ~3 us of stream time, tools/exp_memop_cost.py).
    const LocalDev& D = c->loc[li];
    // back-pressure: never overwrite an entry the device has not ingested yet
    const auto t0 = std::chrono::steady_clock::now();
    while (c->ring_tail[li] - *(volatile uint32_t*)c->ring_ingested_host[li] >= D.ring_cap) {
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > c->cfg.timeout_s)
        return fail(c, P3_ETIMEOUT, "publication ring full: the comm kernels stopped ingesting");
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    if (c->pend_valid[li] && c->pend_stream[li] != (cudaStream_t)stream) {
      // A new publishing stream: the ring tail it advances also exposes the entries queued
      // from the previous stream, so it must be ordered after that stream's producing work.
      CK(cudaEventRecord(c->switch_ev[li], c->pend_stream[li]));
      CK(cudaStreamWaitEvent((cudaStream_t)stream, c->switch_ev[li], 0));
    }
    PubEntry& e = c->ring_host[li][c->ring_tail[li] % D.ring_cap];
    e.layer = layer;
    e.key = c->fifo_seq[li]++;
    e.word = word;
    c->ring_tail[li]++;
    c->pend_stream[li] = (cudaStream_t)stream;
    c->pend_valid[li] = true;
    if (std::find(c->pub_streams[li].begin(), c->pub_streams[li].end(), (cudaStream_t)stream) == c->pub_streams[li].end())
      c->pub_streams[li].push_back((cudaStream_t)stream);
    c->published[li] += 4ull * c->counts[layer];
    c->pub_pending[li] += 4ull * c->counts[layer];
    if (c->pub_pending[li] >= c->cfg.pub_batch_bytes) {
      rc = flush_publications(c, li);
      if (rc) return rc;
    }
    if (c->published[li] >= c->cfg.drain_bytes) {
      rc = flush_publications(c, li);  // a DRAIN launch must see what it was queued for
      if (rc) return rc;
      return launch_drain(c, (int)li);
    }
    return P3_OK;
  }
  // no iteration open: publish right away with stream memory writes on `stream`
  Driver& d = driver();
  const LocalDev& D = c->loc[li];
  CUstream s = (CUstream)stream;
  CUresult r = CUDA_SUCCESS;
  if (c->cfg.sched == P3_SCHED_FIFO) r = d.write32(s, (CUdeviceptr)(D.fifo_key + layer), c->fifo_seq[li]++, 0);
  if (r == CUDA_SUCCESS) {
    if (d.has64) {
      r = d.write64(s, (CUdeviceptr)(D.pub + layer), word, 0);
    } else {  // low half (pointer) first, then the half holding the tag
      r = d.write32(s, (CUdeviceptr)(D.pub + layer), (cuuint32_t)(word & 0xffffffffu), 0);
      if (r == CUDA_SUCCESS) r = d.write32(s, (CUdeviceptr)(D.pub + layer) + 4, (cuuint32_t)(word >> 32), 0);
    }
  }
  if (r != CUDA_SUCCESS) return fail(c, P3_ECUDA, "cuStreamWriteValue failed (code " + std::to_string(r) + ")");
  return P3_OK;
}

int p3_gradgen_layer(p3_ctx_t* c, uint32_t li, uint64_t seed, uint64_t k, uint32_t layer, void* stream) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (layer >= c->L) return fail(c, P3_EUSAGE, "layer out of range");
  if (!c->grads[li]) return fail(c, P3_EUSAGE, "context has no gradient arena (emulate_grads = 0)");
  if (launch_gradgen(seed, k, layer, 0, c->counts[layer], c->grads[li] + c->layer_woff[layer], stream) != P3_OK)
    return cuda_fail(c, cudaGetLastError(), "gradgen launch");
  return P3_OK;
}

int p3_wait_layer(p3_ctx_t* c, uint32_t li, uint32_t layer, uint64_t k, void* stream) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (layer >= c->L) return fail(c, P3_EUSAGE, "layer out of range");
  if (k == 0) return P3_OK;  // forward pass 0 reads the initial parameters
  const uint32_t target = (uint32_t)(k * c->layer_nslices[layer]);
  uint32_t* flag = c->peers.done[c->cfg.local_ranks[li]] + layer;
  CUresult r = driver().wait32((CUstream)stream, (CUdeviceptr)flag, target, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(c, P3_ECUDA, "cuStreamWaitValue32 failed (code " + std::to_string(r) + ")");
  return P3_OK;
}

int p3_wait_group(p3_ctx_t* c, uint32_t li, uint32_t group, uint64_t k, void* stream) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (group >= c->G) return fail(c, P3_EUSAGE, "gate group out of range");
  if (k == 0) return P3_OK;
  const uint32_t target = (uint32_t)(k * c->group_slices[group]);
  uint32_t* flag = c->peers.gdone[c->cfg.local_ranks[li]] + group;
  CUresult r = driver().wait32((CUstream)stream, (CUdeviceptr)flag, target, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(c, P3_ECUDA, "cuStreamWaitValue32 failed (code " + std::to_string(r) + ")");
  return P3_OK;
}

int p3_apply_slice(p3_ctx_t* c, uint32_t li, uint32_t layer, uint32_t slice, const float* values, uint64_t n,
                   void* stream) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (layer >= c->L || slice >= c->layer_nslices[layer]) return fail(c, P3_EPROTOCOL, "BCAST for unknown slice");
  const p3_slice_t& r = c->plan[c->layer_first[layer] + slice];
  if (n != r.length)
    return fail(c, P3_EPROTOCOL, "slice payload holds " + std::to_string(n) + " values, expected " +
                                     std::to_string(r.length));
  if (!values) return fail(c, P3_EUSAGE, "null payload");
  const uint32_t rank = c->cfg.local_ranks[li];
  const uint64_t e = c->layer_woff[layer] + r.offset;
  if (c->cfg.param_bf16) {  // the replica holds bf16: round to nearest even on the host
    std::vector<uint16_t> h(n);
    for (uint64_t i = 0; i < n; ++i) {
      uint32_t x;
      std::memcpy(&x, values + i, 4);
      h[i] = (x & 0x7fffffffu) > 0x7f800000u ? (uint16_t)((x >> 16) | 0x40u)
                                             : (uint16_t)((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
    }
    CK(cudaMemcpyAsync(reinterpret_cast<uint16_t*>(c->peers.W[rank]) + e, h.data(), n * 2, cudaMemcpyHostToDevice,
                       (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));  // (h is released on return)
  } else {
    CK(cudaMemcpyAsync(c->peers.W[rank] + e, values, n * 4, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  }
  if (launch_bump(c->peers.done[rank] + layer, c->peers.gdone[rank] + c->layer_group[layer], 1, stream) != P3_OK)
    return cuda_fail(c, cudaGetLastError(), "gate counter update");
  return P3_OK;
}

int p3_layer_flag(p3_ctx_t* c, uint32_t li, uint32_t layer, uint64_t* iteration) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (layer >= c->L || !iteration) return fail(c, P3_EUSAGE, "layer out of range");
  uint32_t d = 0;
  CK(cudaMemcpyAsync(&d, c->peers.done[c->cfg.local_ranks[li]] + layer, 4, cudaMemcpyDeviceToHost, c->poll_stream));
  CK(cudaStreamSynchronize(c->poll_stream));
  *iteration = d / c->layer_nslices[layer];
  return P3_OK;
}

int p3_sync_all(p3_ctx_t* c, uint64_t k, double timeout_s) {
  if (!c) return fail(nullptr, P3_EUSAGE, "null context");
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  if (c->comm_pending) {
    for (;;) {
      cudaError_t q = cudaEventQuery(c->comm_done);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) return cuda_fail(c, q, "comm kernel");
      if (elapsed() > timeout_s) return fail(c, P3_ETIMEOUT, "comm kernel did not finish before the timeout");
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    c->comm_pending = false;
  }
  uint32_t ew[64] = {0};
  CK(cudaMemcpyAsync(ew, c->d_err, sizeof(ew), cudaMemcpyDeviceToHost, c->poll_stream));
  CK(cudaStreamSynchronize(c->poll_stream));
  if (ew[0]) {
    std::string m = "comm kernel of iteration " + std::to_string(ew[1]) +
                    " stalled (timeout waiting for peers or gradients);";
    for (uint32_t i = 0; i < c->cfg.n_local; ++i) {
      std::vector<uint64_t> pub(c->L);
      cudaMemcpyAsync(pub.data(), c->loc[i].pub, c->L * 8ull, cudaMemcpyDeviceToHost, c->poll_stream);
      cudaStreamSynchronize(c->poll_stream);
      uint32_t nready = 0;
      for (uint32_t l = 0; l < c->L; ++l) nready += (uint32_t)(pub[l] >> 48) == ((ew[1] + 1) & 0xffffu);
      m += " rank " + std::to_string(c->cfg.local_ranks[i]) + ": pushed " + std::to_string(ew[2 + 2 * i]) + "/" +
           std::to_string(c->S) + " reduced " + std::to_string(ew[3 + 2 * i]) + "/" +
           std::to_string(c->own_total[c->cfg.local_ranks[i]]) + " ready layers " + std::to_string(nready) + "/" +
           std::to_string(c->L) + ";";
    }
    return fail(c, (int)ew[0], m);
  }
  std::vector<uint32_t> done(c->L);
  for (uint32_t i = 0; i < c->cfg.n_local; ++i) {
    const uint32_t rank = c->cfg.local_ranks[i];
    for (;;) {
      CK(cudaMemcpyAsync(done.data(), c->peers.done[rank], c->L * 4ull, cudaMemcpyDeviceToHost, c->poll_stream));
      CK(cudaStreamSynchronize(c->poll_stream));
      std::vector<uint32_t> unmet;
      for (uint32_t l = 0; l < c->L; ++l)
        if ((int32_t)(done[l] - (uint32_t)(k * c->layer_nslices[l])) < 0) unmet.push_back(l);
      if (unmet.empty()) break;
      if (elapsed() > timeout_s) {
        std::string m = "rank " + std::to_string(rank) + " stalled waiting for iteration-" + std::to_string(k) +
                        " parameters; unmet layers [";
        for (size_t j = 0; j < unmet.size() && j < 16; ++j) m += (j ? "," : "") + std::to_string(unmet[j]);
        return fail(c, P3_ETIMEOUT, m + (unmet.size() > 16 ? ",...]" : "]"));
      }
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }
  if (k > c->synced_iterations) c->synced_iterations = k;
  return P3_OK;
}

int p3_trace_read(p3_ctx_t* c, uint32_t li, p3_trace_rec_t* out, uint64_t cap, uint64_t* n_out) {
  int rc = check_local(c, li);
  if (rc) return rc;
  unsigned long long n = 0;
  CK(cudaMemcpyAsync(&n, c->loc[li].trace_n, 8, cudaMemcpyDeviceToHost, c->poll_stream));
  CK(cudaStreamSynchronize(c->poll_stream));
  n = std::min<unsigned long long>(n, c->cfg.trace_cap);
  if (n_out) *n_out = n;
  if (out && n) {
    if (cap < n) return fail(c, P3_EUSAGE, "trace buffer too small");
    CK(cudaMemcpyAsync(out, c->loc[li].trace, n * sizeof(p3_trace_rec_t), cudaMemcpyDeviceToHost, c->poll_stream));
    CK(cudaStreamSynchronize(c->poll_stream));
  }
  return P3_OK;
}

int p3_trace_clear(p3_ctx_t* c) {
  if (!c) return fail(nullptr, P3_EUSAGE, "null context");
  for (uint32_t i = 0; i < c->cfg.n_local; ++i) CK(cudaMemsetAsync(c->loc[i].trace_n, 0, 8, c->poll_stream));
  CK(cudaStreamSynchronize(c->poll_stream));
  return P3_OK;
}

int p3_trace_mark(p3_ctx_t* c, uint32_t li, uint64_t k, uint32_t ev, void* stream) {
  int rc = check_local(c, li);
  if (rc) return rc;
  if (ev != P3_EV_ITER_START && ev != P3_EV_SYNCED) return fail(c, P3_EUSAGE, "mark event must be ITER_START or SYNCED");
  if (launch_mark(c->loc[li], (uint32_t)k, ev, stream) != P3_OK) return cuda_fail(c, cudaGetLastError(), "mark launch");
  return P3_OK;
}

int p3_comm_launches(p3_ctx_t* c, uint64_t* n) {
  if (!c || !n) return fail(c, P3_EUSAGE, "null argument");
  *n = c->launches;
  return P3_OK;
}

int p3_counters(p3_ctx_t* c, uint32_t li, uint64_t* bytes_in, uint64_t* bytes_out) {
  int rc = check_local(c, li);
  if (rc) return rc;
  unsigned long long b[2] = {0, 0};
  CK(cudaMemcpyAsync(b, c->loc[li].bytes, 16, cudaMemcpyDeviceToHost, c->poll_stream));
  CK(cudaStreamSynchronize(c->poll_stream));
  // broadcasts land by remote stores; their byte count follows from the plan per synced iteration
  if (bytes_in) *bytes_in = b[0] + c->bcast_in_bytes[c->cfg.local_ranks[li]] * c->synced_iterations;
  if (bytes_out) *bytes_out = b[1];
  return P3_OK;
}

int p3_debug_snapshot(p3_ctx_t* c, uint32_t li, uint32_t* out, uint64_t cap, uint64_t* n_out) {
  int rc = check_local(c, li);
  if (rc) return rc;
  const uint64_t n = 5ull * c->L + 12 + P3_DBG_CTAS + 2ull * c->S;
  if (n_out) *n_out = n;
  if (!out) return P3_OK;
  if (cap < n) return fail(c, P3_EUSAGE, "snapshot buffer too small");
  const LocalDev& D = c->loc[li];
  const uint32_t rank = c->cfg.local_ranks[li];
  const uint32_t* src[5] = {nullptr, D.cursor, D.srv_taken, c->peers.hint[rank], c->peers.done[rank]};
  for (int a = 1; a < 5; ++a)
    CK(cudaMemcpyAsync(out + (uint64_t)a * c->L, src[a], c->L * 4ull, cudaMemcpyDeviceToHost, c->poll_stream));
  std::vector<uint64_t> pub(c->L);
  CK(cudaMemcpyAsync(pub.data(), D.pub, c->L * 8ull, cudaMemcpyDeviceToHost, c->poll_stream));
  static_assert(sizeof(IterState) == 56, "IterState layout");
  CK(cudaMemcpyAsync(out + 5ull * c->L, D.it, 48, cudaMemcpyDeviceToHost, c->poll_stream));  // (up to t_signal)
  CK(cudaMemcpyAsync(out + 5ull * c->L + 12, D.cta_phase, P3_DBG_CTAS * 4ull, cudaMemcpyDeviceToHost, c->poll_stream));
  uint32_t* tail = out + 5ull * c->L + 12 + P3_DBG_CTAS;
  CK(cudaMemcpyAsync(tail, c->peers.arrivals[rank], c->S * 4ull, cudaMemcpyDeviceToHost, c->poll_stream));
  CK(cudaMemcpyAsync(tail + c->S, D.claim, c->S * 4ull, cudaMemcpyDeviceToHost, c->poll_stream));
  CK(cudaStreamSynchronize(c->poll_stream));
  for (uint32_t l = 0; l < c->L; ++l) out[l] = (uint32_t)(pub[l] >> 48);  // iteration tag
  {  // arrivals and claims are stored by owner-list position: report them per slice id
    std::vector<uint32_t> byp(tail, tail + 2ull * c->S);
    for (uint32_t g = 0; g < c->S; ++g) {
      tail[g] = byp[c->slice_opos[g]];
      tail[c->S + g] = byp[c->S + c->slice_opos[g]];
    }
  }
  return P3_OK;
}

// ------------------------------------------------------------ scripted device queue

struct p3_queue {
  uint32_t L = 0, sched = 0, tag = 0, seq = 0;
  std::vector<uint32_t> nslices;
  char* d = nullptr;  // nslices | first | pub | fifo_key | cursor | result
  uint32_t *d_nslices, *d_first, *d_fifo, *d_cursor, *d_result;
  uint64_t* d_pub;
  cudaStream_t s = nullptr;
};

int p3_queue_create(const uint32_t* layer_nslices, uint32_t n_layers, uint32_t sched, p3_queue_t** out) {
  p3_ctx* c = nullptr;
  if (!layer_nslices || !out || n_layers == 0) return fail(nullptr, P3_EUSAGE, "bad queue arguments");
  if (sched > P3_SCHED_FIFO) return fail(nullptr, P3_EUSAGE, "bad queue discipline");
  if (preload_kernels() != P3_OK) return fail(nullptr, P3_ECUDA, "loading the sm_100a kernels failed");
  p3_queue* q = new p3_queue();
  q->L = n_layers;
  q->sched = sched;
  q->nslices.assign(layer_nslices, layer_nslices + n_layers);
  std::vector<uint32_t> first(n_layers);
  uint64_t f = 0;
  for (uint32_t l = 0; l < n_layers; ++l) {
    first[l] = (uint32_t)f;
    f += layer_nslices[l];
  }
  const size_t stride = align_up(n_layers * 8ull, 256);
  cudaError_t e = cudaMalloc(&q->d, stride * 6);
  if (e == cudaSuccess) e = cudaMemset(q->d, 0, stride * 6);
  q->d_nslices = reinterpret_cast<uint32_t*>(q->d);
  q->d_first = reinterpret_cast<uint32_t*>(q->d + stride);
  q->d_pub = reinterpret_cast<uint64_t*>(q->d + 2 * stride);
  q->d_fifo = reinterpret_cast<uint32_t*>(q->d + 3 * stride);
  q->d_cursor = reinterpret_cast<uint32_t*>(q->d + 4 * stride);
  q->d_result = reinterpret_cast<uint32_t*>(q->d + 5 * stride);
  if (e == cudaSuccess) e = cudaMemcpy(q->d_nslices, layer_nslices, n_layers * 4ull, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(q->d_first, first.data(), n_layers * 4ull, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q->s, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    p3_queue_destroy(q);
    return cuda_fail(c, e, "queue init");
  }
  *out = q;
  return P3_OK;
}

int p3_queue_put_layer(p3_queue_t* q, uint32_t layer, uint32_t iteration) {
  p3_ctx* c = nullptr;
  if (!q || layer >= q->L) return fail(nullptr, P3_EUSAGE, "layer out of range");
  const uint32_t tag = iteration + 1, zero = 0, key = q->seq++;
  const uint64_t word = ((uint64_t)(tag & 0xffffu)) << 48;
  CK(cudaMemcpyAsync(q->d_cursor + layer, &zero, 4, cudaMemcpyHostToDevice, q->s));
  CK(cudaMemcpyAsync(q->d_fifo + layer, &key, 4, cudaMemcpyHostToDevice, q->s));
  CK(cudaMemcpyAsync(q->d_pub + layer, &word, 8, cudaMemcpyHostToDevice, q->s));
  CK(cudaStreamSynchronize(q->s));
  q->tag = std::max(q->tag, tag);
  return P3_OK;
}

int p3_queue_poll(p3_queue_t* q, uint32_t* layer, uint32_t* slice) {
  p3_ctx* c = nullptr;
  if (!q) return fail(nullptr, P3_EUSAGE, "null queue");
  if (q->tag == 0) return P3_ETIMEOUT;
  if (launch_queue_pop(q->d_nslices, q->d_first, q->d_pub, q->d_fifo, q->d_cursor, q->L, q->sched, q->tag,
                       q->d_result, q->s) != P3_OK)
    return cuda_fail(c, cudaGetLastError(), "queue pop launch");
  uint32_t g = 0;
  CK(cudaMemcpyAsync(&g, q->d_result, 4, cudaMemcpyDeviceToHost, q->s));
  CK(cudaStreamSynchronize(q->s));
  if (g == 0xffffffffu) return P3_ETIMEOUT;
  // global slice id -> (layer, slice)
  uint32_t l = 0;
  uint64_t f = 0;
  while (l < q->L && f + q->nslices[l] <= g) f += q->nslices[l++];
  *layer = l;
  *slice = (uint32_t)(g - f);
  return P3_OK;
}

int p3_queue_destroy(p3_queue_t* q) {
  if (!q) return P3_OK;
  if (q->s) cudaStreamSynchronize(q->s);
  if (q->d) cudaFree(q->d);
  if (q->s) cudaStreamDestroy(q->s);
  delete q;
  return P3_OK;
}

}  // extern "C"
