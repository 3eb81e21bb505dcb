// sm_100a kernels of the P3 sync path.
//
//   K1 k_gradgen       gradient_block / _materialize          hashing.py:55-63, worker.py:166-171
//   K4 k_shard_update  ShardState.aggregate_and_update        server.py:55-68
//   K3 k_comm          the comm kernel (DRAIN launches during the backward pass, one FINISH
//                      launch per iteration), warp-specialised, TMA-staged:
//        worker role   FrameQueue.poll + _priority_sender     queues.py:52-62, worker.py:184-190
//        server role   ShardState.on_push/aggregate/bcast     server.py:36-88, 208-226
//        apply role    on_bcast -> flags[layer]               worker.py:241-269 (remote stores +
//                                                             per-layer counters)
//   k_queue_pop        one FrameQueue.poll on the device queue (scripted tick replay)
//   k_sleep            TrainingWorker._emulate                worker.py:299-310
//
// All traffic is bandwidth-bound streaming (TMA bulk copies through shared memory, 16-byte
// vector stores), no tensor cores.
// Floating point follows the reference's numpy fp32 semantics exactly: the sum is taken in
// ascending rank order starting from +0.0, then divided by N, then p - lr*g with the multiply
// and the subtract rounded separately (explicit _rn intrinsics: no FMA contraction).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "p3_internal.h"

namespace p3 {

#define FULL_MASK 0xffffffffu
#define P3_NONE 0xffffffffu

// Protocol invariants, compiled in for the checked build (libp3_checked.so, -DP3_CHECKS):
// a violated one prints where and traps, so the host sees a launch failure instead of wrong
// values (compute-sanitizer is not available on the GPU pool).
#ifdef P3_CHECKS
#define P3_CHECK(cond)                                                                                  \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("P3_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x);                                                                             \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define P3_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_add_release_sys(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.release.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_relaxed_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_add_relaxed_sys(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_add_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// mbarrier / TMA bulk copy (cp.async.bulk, 1-D) helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_1d(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// TMA bulk store shared -> global (any global address: a peer's memory over NVLink too)
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// bulk store without its own commit (a stage's stores form one bulk group)
__device__ __forceinline__ void tma_store_1d_nc(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// every bulk group but the most recent one has finished reading shared memory
__device__ __forceinline__ void tma_store_wait_read_all_but_one() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// P3_COLD: functions off the N=1 hot loop (N>1 server role, notify mode, K7, the trace) may be
// compiled out of line so the scheduler's inlined code stays small (experiment switch).
#ifndef P3_COLD
#define P3_COLD
#endif
// P3_TRACE=0 compiles the device trace out (experiment switch; the tests need it on).
#ifndef P3_TRACE
#define P3_TRACE 1
#endif

// Diagnostics clock of the per-job time totals (t_pick / t_slot_wait / t_move / t_signal in
// the debug snapshot): %globaltimer reads are not free, so they compile out with P3_STATS=0.
#ifndef P3_STATS
#define P3_STATS 1
#endif
__device__ __forceinline__ uint64_t stat_clock() { return P3_STATS ? globaltimer() : 0ull; }

// Bounded mbarrier wait: every wait of the stage pipeline ends within the iteration timeout
// (the scheduler posts EXIT by then), so one that outlives it is a protocol bug — trap (the
// host sees a launch failure) rather than hang the GPU.
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* b, uint32_t parity, const CommArgs& a) {
  if (mbar_try_wait(b, parity)) return;
  const uint64_t t0 = globaltimer();
  while (!mbar_try_wait(b, parity))
    if (globaltimer() - t0 > a.timeout_ns + 2000000000ull) __trap();
}

// ------------------------------------------------------------------ K1: gradient source

// gradient_value (hashing.py:45-52): x = seed ^ it*Gi ^ L*Gl ^ e*Ge; top24 = mix(x) >> 40;
// value = top24 * 2^-23 - 1. (top24 - 2^23) is a 24-bit integer, so the fp32 result is exact.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float grad_value(uint64_t base, uint64_t e) {
  const uint32_t top24 = (uint32_t)(mix64(base ^ (e * 0x165667B19E3779F9ull)) >> 40);
  return (float)((int32_t)top24 - 8388608) * 1.1920928955078125e-7f;
}

__global__ void __launch_bounds__(256) k_gradgen(uint64_t base, uint64_t start, uint64_t count,
                                                 float* __restrict__ out) {
  // head elements until `out` is 16-byte aligned, then float4 body, then tail
  const uint64_t head = min((unsigned long long)count, (unsigned long long)(((16 - ((uintptr_t)out & 15)) & 15) / 4));
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  if (tid < head) out[tid] = grad_value(base, start + tid);
  const uint64_t nvec = (count - head) / 4;
  float4* o4 = reinterpret_cast<float4*>(out + head);
  for (uint64_t v = tid; v < nvec; v += nthr) {
    const uint64_t e = start + head + 4 * v;
    float4 r;
    r.x = grad_value(base, e);
    r.y = grad_value(base, e + 1);
    r.z = grad_value(base, e + 2);
    r.w = grad_value(base, e + 3);
    __stcs(o4 + v, r);
  }
  const uint64_t tail0 = head + 4 * nvec;
  if (tid < count - tail0) out[tail0 + tid] = grad_value(base, start + tail0 + tid);
}

int launch_gradgen(uint64_t seed, uint64_t iteration, uint64_t layer, uint64_t start, uint64_t count,
                   float* out, void* stream) {
  if (count == 0) return P3_OK;
  const uint64_t base =
      seed ^ (iteration * 0x9E3779B97F4A7C15ull) ^ (layer * 0xC2B2AE3D27D4EB4Full);
  uint64_t blocks = (count / 4 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_gradgen<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(base, start, count, out);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

// ------------------------------------------------------------------ K4: reduce + update

struct UpdCoef {
  float nw;       // N as fp32 (the reference divides by np.float32(num_workers))
  float inv_nw;   // exact 1/N when N is a power of two (then x*inv == x/N bit-for-bit)
  int pow2;
  float lr;
  float mu;
};

__device__ __forceinline__ float sgd_step(float p, float gsum, const UpdCoef& c, float* v) {
  const float g = c.pow2 ? __fmul_rn(gsum, c.inv_nw) : __fdiv_rn(gsum, c.nw);
  float step = g;
  if (v) {
    step = __fadd_rn(__fmul_rn(c.mu, *v), g);
    *v = step;
  }
  return __fsub_rn(p, __fmul_rn(c.lr, step));
}

// fp32 sum of one float4 lane-set in ascending rank order, starting from +0.0 exactly like
// np.zeros(...) followed by `acc += g_rank` (server.py:60-63).
template <int NW>
__device__ __forceinline__ float4 sum_in_rank_order(const float4 (&v)[NW]) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    acc.x = __fadd_rn(acc.x, v[q].x);
    acc.y = __fadd_rn(acc.y, v[q].y);
    acc.z = __fadd_rn(acc.z, v[q].z);
    acc.w = __fadd_rn(acc.w, v[q].w);
  }
  return acc;
}

__device__ __forceinline__ float sum_sources_scalar(const float* const* src, int nw, uint64_t i) {
  float acc = 0.f;
  for (int q = 0; q < nw; ++q) acc = __fadd_rn(acc, __ldcg(src[q] + i));
  return acc;
}

__device__ __forceinline__ float4 sgd4(float4 p, const float4& acc, const UpdCoef& c, float4* v) {
  if (v) {
    p.x = sgd_step(p.x, acc.x, c, &v->x);
    p.y = sgd_step(p.y, acc.y, c, &v->y);
    p.z = sgd_step(p.z, acc.z, c, &v->z);
    p.w = sgd_step(p.w, acc.w, c, &v->w);
  } else {
    p.x = sgd_step(p.x, acc.x, c, nullptr);
    p.y = sgd_step(p.y, acc.y, c, nullptr);
    p.z = sgd_step(p.z, acc.z, c, nullptr);
    p.w = sgd_step(p.w, acc.w, c, nullptr);
  }
  return p;
}

// CTA-wide reduce + update over n4 float4s: dst[0..ndst) all receive the result (dst[0]
// is also the master copy read as p), src[0..NW) are the gradient sources in rank order,
// v the optional momentum. U float4 columns per thread are loaded before any arithmetic
// so each thread keeps (NW + 1) * U independent 16-byte loads in flight.
template <int NW, int U, bool MOM>
__device__ void cta_update_vec(const float* p_src, float* const* dst, int ndst, const float* const* src,
                               float* v, uint64_t n4, const UpdCoef& c, uint32_t tid, uint32_t nthr) {
  // Every round issues all of its (predicated) loads before any use, including the last,
  // partial round: a remainder walked one float4 at a time would cost one memory round trip
  // per element per thread (measured: ~4 us of a 50K-element job).
  const uint32_t stride = nthr, m4 = (uint32_t)n4;  // a job is < 2^32 elements
  for (uint32_t j = tid; j < m4; j += U * stride) {
    float4 g[U][NW], p[U], vv[MOM ? U : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // out-of-range columns reload column j (in range) instead of branching: the loads stay
      // unconditional, only the stores are predicated
      const uint32_t i = 4 * (j + u * stride < m4 ? j + u * stride : j);
#pragma unroll
      for (int q = 0; q < NW; ++q) g[u][q] = __ldcg(reinterpret_cast<const float4*>(src[q] + i));
      p[u] = __ldcg(reinterpret_cast<const float4*>(p_src + i));
      if (MOM) vv[MOM ? u : 0] = __ldcg(reinterpret_cast<const float4*>(v + i));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = 4 * (j + u * stride);
      if (j + u * stride < m4) {
        const float4 r = sgd4(p[u], sum_in_rank_order<NW>(g[u]), c, MOM ? &vv[MOM ? u : 0] : nullptr);
        if (MOM) *reinterpret_cast<float4*>(v + i) = vv[MOM ? u : 0];
        for (int d = 0; d < ndst; ++d) *reinterpret_cast<float4*>(dst[d] + i) = r;
      }
    }
  }
}

__device__ void cta_update_generic(const float* p_src, float* const* dst, int ndst, const float* const* src,
                                   int nw, float* v, uint64_t n, bool aligned, const UpdCoef& c, uint32_t tid,
                                   uint32_t nthr) {
  // (callers pass pointers already offset to the range; see move_range for sub-ranges)
  uint64_t done = 0;
  if (aligned) {
    const uint64_t n4 = n / 4;
    switch (nw) {
#define P3_CASE(K)                                                                                      \
  case K:                                                                                               \
    if (v)                                                                                              \
      cta_update_vec<K, (K <= 1 ? 4 : K <= 2 ? 2 : 1), true>(p_src, dst, ndst, src, v, n4, c, tid, nthr);  \
    else                                                                                                \
      cta_update_vec<K, (K <= 1 ? 8 : K <= 2 ? 4 : K <= 4 ? 2 : 1), false>(p_src, dst, ndst, src, v, n4, c, tid, nthr); \
    break;
      P3_CASE(1) P3_CASE(2) P3_CASE(3) P3_CASE(4) P3_CASE(5) P3_CASE(6) P3_CASE(7) P3_CASE(8)
#undef P3_CASE
      default: aligned = false; break;
    }
    if (aligned) done = 4 * n4;
  }
  for (uint64_t i = done + tid; i < n; i += nthr) {
    const float acc = sum_sources_scalar(src, nw, i);
    float p = __ldcg(p_src + i);
    p = sgd_step(p, acc, c, v ? v + i : nullptr);
    for (int d = 0; d < ndst; ++d) dst[d][i] = p;
  }
}

__device__ __forceinline__ UpdCoef make_coef(uint32_t nw, float lr, float mu) {
  UpdCoef c;
  c.nw = (float)nw;
  c.pow2 = (nw & (nw - 1)) == 0;
  c.inv_nw = 1.0f / (float)nw;  // exact for powers of two
  c.lr = lr;
  c.mu = mu;
  return c;
}

struct GradPtrs {
  const float* p[P3_MAX_RANKS];
};

__global__ void __launch_bounds__(256) k_shard_update(float* params, GradPtrs g, uint32_t nw, uint64_t n,
                                                      float lr, float mu, float* V) {
  // one CTA per 64K-element chunk: the same CTA-wide routine the comm kernel runs per slice
  const uint64_t chunk = 65536;
  const uint64_t lo = blockIdx.x * chunk;
  if (lo >= n) return;
  const uint64_t len = min(chunk, n - lo);
  __shared__ const float* src[P3_MAX_RANKS];
  __shared__ float* dst[1];
  if (threadIdx.x < nw) src[threadIdx.x] = g.p[threadIdx.x] + lo;
  if (threadIdx.x == 0) dst[0] = params + lo;
  __syncthreads();
  uintptr_t al = (uintptr_t)(params + lo) | (V ? (uintptr_t)(V + lo) : 0);
  for (uint32_t q = 0; q < nw; ++q) al |= (uintptr_t)(g.p[q] + lo);
  cta_update_generic(params + lo, dst, 1, src, (int)nw, V ? V + lo : nullptr, len, (al & 15) == 0,
                     make_coef(nw, lr, mu), threadIdx.x, blockDim.x);
}

}  // namespace p3

extern "C" int p3_shard_update(float* params_dev, const float* const* grads_dev, uint32_t num_workers,
                               uint64_t n, float lr, float momentum, float* momentum_dev, void* stream) {
  using namespace p3;
  if (num_workers < 1 || num_workers > P3_MAX_RANKS) {
    set_thread_error("num_workers must be in [1, 16]");
    return P3_EUSAGE;
  }
  if (n == 0) return P3_OK;
  GradPtrs g{};
  for (uint32_t q = 0; q < num_workers; ++q) g.p[q] = grads_dev[q];
  const uint64_t blocks = (n + 65535) / 65536;
  k_shard_update<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(params_dev, g, num_workers, n, lr,
                                                                     momentum, momentum_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_thread_error(cudaGetErrorString(e));
    return P3_ECUDA;
  }
  return P3_OK;
}

extern "C" int p3_gradient_block(uint64_t seed, uint64_t iteration, uint64_t layer, uint64_t start,
                                 uint64_t count, float* out_dev, void* stream) {
  int rc = p3::launch_gradgen(seed, iteration, layer, start, count, out_dev, stream);
  if (rc != P3_OK) p3::set_thread_error(cudaGetErrorString(cudaGetLastError()));
  return rc;
}

namespace p3 {

// ------------------------------------------------------------------ emulated compute

__global__ void k_sleep(uint64_t ns) {
  const uint64_t t0 = globaltimer();
  while (globaltimer() - t0 < ns) __nanosleep(1000);
}

// ------------------------------------------------------------------ trace ring

__device__ __forceinline__ void trace_append(const LocalDev& L, uint32_t k, uint32_t layer, uint32_t slice,
                                             uint32_t rank, uint32_t ev, uint64_t t0 = 0) {
  if (!P3_TRACE || !L.trace_cap) return;
  const unsigned long long idx = atomicAdd(L.trace_n, 1ull);
  if (idx < L.trace_cap) {
    p3_trace_rec_t r;
    r.t_ns = globaltimer();
    r.t0_ns = t0;
    r.iteration = k;
    r.layer = layer;
    r.slice = slice;
    r.rank = (uint16_t)rank;
    r.event = (uint16_t)ev;
    L.trace[idx] = r;
  }
}

// ------------------------------------------------------------------ device slice queue

// The outbox of one worker: per layer a publication word (iteration tag in the top 16 bits,
// gradient pointer below, written by one stream memory write), a publish sequence
// (fifo_key) and a claim cursor. The minimum under the FrameQueue order is the lowest ready
// layer with unclaimed slices (priority == layer index, plan.py:112, ties by slice index
// through the ascending cursor), or the earliest-published such layer in FIFO mode.
struct QueueView {
  uint32_t n_layers;
  uint32_t sched;
  uint32_t relax;  // pops may take any of the `relax` most urgent layers (1: strict)
  uint32_t multi;  // candidate layers claimed per round of atomics (<= P3_MULTI)
  const uint32_t* nslices;
  const uint32_t* first;
  const uint64_t* pub;
  const uint32_t* fifo_key;
  uint32_t* cursor;
  const LocalDev* ring;  // publication ring to ingest from (nullptr: scripted queue)
};

#ifndef P3_INGEST_U
#define P3_INGEST_U 8  // publication-ring entries per lane loaded before use (ingest)
#endif
__device__ __noinline__ void ingest(const LocalDev& L, uint32_t sched);
__device__ __forceinline__ uint64_t globaltimer_lane0() {
  uint64_t t = (threadIdx.x & 31) == 0 ? globaltimer() : 0ull;
  return __shfl_sync(0xffffffffu, (unsigned long long)t, 0);
}

// Publication word: iteration tag (16 bits) above the 48-bit gradient pointer, written by one
// 64-bit stream memory write, so the tag and the pointer become visible together.
__device__ __forceinline__ bool pub_ready(uint64_t w, uint32_t tag) { return (uint32_t)(w >> 48) == (tag & 0xffffu); }
__device__ __forceinline__ const float* pub_ptr(uint64_t w) {
  return reinterpret_cast<const float*>(w & 0x0000ffffffffffffull);
}

// Executed by one full warp; returns the popped global slice id or P3_NONE.
// Priority discipline: layers are examined in ascending order 32 at a time (lane i owns
// layer base+i); each lane first loads the availability of all its layers (independent
// loads, one memory round trip), then the warp walks the availability ballots in layer
// order and claims the first slice it wins. A lost race moves on to the next candidate
// without rescanning. FIFO discipline: arg-min of the publish sequence, then claim.
// `want` > 1 claims up to that many consecutive slices of the chosen layer at once (they
// would be the next pops anyway); `*run` receives how many were claimed.
// Priority discipline with a stash: up to P3_MULTI candidate layers are claimed with one
// round of atomics (one per lane); the most urgent win is returned, the other wins are
// appended to the caller's stash (processed next by the same CTA). Against many concurrent
// consumers this turns a walk of lost races into one memory round trip.
#define P3_MULTI 4
struct Stash {
  uint32_t n;
  uint32_t g[P3_MULTI];
  uint32_t run[P3_MULTI];
  uint32_t layer[P3_MULTI];
  uint64_t word[P3_MULTI];
  uint64_t t0[P3_MULTI];
};

// What a pop hands to the caller besides the slice id: the slice's layer and the layer's
// publication word (already loaded by the pop), so preparing the job needs no dependent
// round trip through slice_layer[] / pub[].
struct Popped {
  uint32_t run;
  uint32_t piece;  // server pick with srv_piece: the piece of the slice claimed
  uint32_t layer;
  uint64_t word;
  uint64_t t0;  // %globaltimer before the queue snapshot the claim came from (trace)
};

__device__ uint32_t warp_pop(const QueueView& q, uint32_t tag, uint32_t* dbg = nullptr, uint32_t want = 1,
                             Popped* out = nullptr, Stash* stash = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
  if (q.sched == P3_SCHED_PRIORITY) {
    constexpr uint32_t CH = 8;  // chunks of 32 layers examined per memory round trip
    for (uint32_t group = 0, attempt = 0; group < q.n_layers; ++attempt) {
      // all loads of the group issued before any is used: one round trip, not 2*CH
      // (trace only: the time before this snapshot's loads; %globaltimer is not free)
      const uint64_t t_snap = P3_TRACE && q.ring && q.ring->trace_cap ? globaltimer_lane0() : 0ull;
      uint64_t w[CH];
      uint32_t cur[CH], ns[CH];
      // the ring check rides on the same round trip as the first group's loads
      const bool ring_check = q.ring && group == 0 && lane == 0;
      const uint32_t r_lo = ring_check ? ld_relaxed_gpu(q.ring->ingested) : 0u;
      const uint32_t r_hi = ring_check ? ld_relaxed_gpu(q.ring->pubseq) : 0u;
#pragma unroll
      for (uint32_t c = 0; c < CH; ++c) {
        const uint32_t l = group + 32 * c + lane;
        const bool in = l < q.n_layers;
        w[c] = in ? ld_relaxed_gpu64(q.pub + l) : 0ull;
        cur[c] = in ? ld_relaxed_gpu(q.cursor + l) : 0u;
        ns[c] = in ? q.nslices[l] : 0u;
      }
      if (q.ring && group == 0 && __shfl_sync(FULL_MASK, (uint32_t)(r_lo != r_hi), 0)) {
        ingest(*q.ring, q.sched);  // new publications: turn them into words, then look again
        continue;
      }
      uint32_t bits = 0;  // bit c: layer group + 32*c + lane is poppable
#pragma unroll
      for (uint32_t c = 0; c < CH; ++c) bits |= (uint32_t)(pub_ready(w[c], tag) && cur[c] < ns[c]) << c;
      const uint32_t nchunk = min(CH, (q.n_layers - group + 31) / 32);
      bool first = true;
      if (q.relax > 1 && !(stash && q.multi > 1) && attempt < 4) {
        // Bounded relaxation, ranked by slice: with `relax` consumers popping at once, this
        // CTA aims at the job of rank (blockIdx % relax) among the most urgent available
        // slices of the group — one claim that rarely collides, where racing for the same few
        // most urgent layers (one-slice layers: most of ResNet-50) costs a lost atomic round
        // trip per try. A lost claim reloads the group and aims again (the snapshot is stale).
        uint32_t tot[CH], total = 0;
#pragma unroll
        for (uint32_t c = 0; c < CH; ++c) {
          tot[c] = __reduce_add_sync(FULL_MASK, ((bits >> c) & 1u) ? ns[c] - cur[c] : 0u);
          total += tot[c];
        }
        if (!total) {  // nothing available in this group
          group += 32 * CH;
          attempt = 0;
          continue;
        }
        {
          uint32_t t = ((blockIdx.x % q.relax) * want) % total, tc = 0;
#pragma unroll
          for (uint32_t c = 0; c < CH; ++c) {  // chunk holding rank t (uniform)
            if (c == tc && t >= tot[c] && c + 1 < CH) {
              t -= tot[c];
              tc = c + 1;
            }
          }
          uint32_t r = 0, my_ns = 0;
          uint64_t my_w = 0;
#pragma unroll
          for (uint32_t c = 0; c < CH; ++c) {
            if (c == tc) {
              r = ((bits >> c) & 1u) ? ns[c] - cur[c] : 0u;
              my_ns = ns[c];
              my_w = w[c];
            }
          }
          uint32_t incl = r;  // inclusive scan over the lanes (layer order)
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL_MASK, incl, off);
            if (lane >= (uint32_t)off) incl += y;
          }
          const bool hit = r && incl - r <= t && t < incl;
          uint32_t s = 0;
          bool won = false;
          if (hit) {
            s = atomicAdd(q.cursor + group + 32 * tc + lane, want);
            won = s < my_ns;
          }
          const uint32_t wm = __ballot_sync(FULL_MASK, won);
          if (wm) {
            const uint32_t j0 = __ffs(wm) - 1;
            const uint32_t l = group + 32 * tc + j0;
            const uint32_t g0 = __shfl_sync(FULL_MASK, won ? q.first[l] + s : 0u, j0);
            if (out) {
              out->run = __shfl_sync(FULL_MASK, won ? min(want, my_ns - s) : 0u, j0);
              out->layer = l;
              out->word = __shfl_sync(FULL_MASK, (unsigned long long)my_w, j0);
              out->t0 = t_snap;
            }
            return g0;
          }
        }
        continue;  // lost the claim: reload the group and aim again
      }
      for (uint32_t c = 0; c < nchunk; ++c) {
        uint32_t m = __ballot_sync(FULL_MASK, (bits >> c) & 1u);
        uint32_t my_ns = 0;
        uint64_t my_w = 0;
#pragma unroll
        for (uint32_t cc = 0; cc < CH; ++cc) {
          my_ns = cc == c ? ns[cc] : my_ns;
          my_w = cc == c ? w[cc] : my_w;
        }
        while (m) {
          // candidates: the most urgent available layers of the chunk — starting, on the
          // first round, at a CTA-dependent one of the `relax` most urgent (a pop is then
          // among the `relax` smallest, as with `relax` consumers popping at once)
          uint32_t mm = m;
          if (first && q.relax > 1) {
            const uint32_t skip = blockIdx.x % min((uint32_t)__popc(m), q.relax);
            for (uint32_t t = 0; t < skip; ++t) mm &= mm - 1;
          }
          first = false;
          uint32_t cand = 0;
          const uint32_t k = stash ? q.multi : 1u;
          for (uint32_t t = 0; t < k && mm; ++t) {
            cand |= mm & (~mm + 1);  // lowest remaining set bit
            mm &= mm - 1;
          }
          uint32_t s = 0;
          bool won = false;
          if ((cand >> lane) & 1u) {
            s = atomicAdd(q.cursor + group + 32 * c + lane, want);
            won = s < my_ns;
          }
          const uint32_t wm = __ballot_sync(FULL_MASK, won);
          if (wm) {
            const uint32_t l = group + 32 * c + lane;
            const uint32_t my_g = won ? q.first[l] + s : 0u, my_run = won ? min(want, my_ns - s) : 0u;
            const uint32_t j0 = __ffs(wm) - 1;
            if (won && lane != j0) {  // the other wins: next jobs of this CTA, in layer order
              const uint32_t idx = stash->n + __popc(wm & ((1u << lane) - 1u)) - 1u;
              stash->g[idx] = my_g;
              stash->run[idx] = my_run;
              stash->layer[idx] = l;
              stash->word[idx] = my_w;
              stash->t0[idx] = t_snap;
            }
            __syncwarp();
            if (lane == 0 && stash) stash->n += __popc(wm) - 1u;
            __syncwarp();
            if (out) {
              out->run = __shfl_sync(FULL_MASK, my_run, j0);
              out->layer = group + 32 * c + j0;
              out->word = __shfl_sync(FULL_MASK, (unsigned long long)my_w, j0);
              out->t0 = t_snap;
            }
            return __shfl_sync(FULL_MASK, my_g, j0);
          }
          m &= ~cand;  // every candidate lost the race for its layer's last slices
        }
      }
      group += 32 * CH;
      attempt = 0;
    }
    return P3_NONE;
  }
  if (q.ring) ingest(*q.ring, q.sched);
  for (uint32_t retry = 0;; ++retry) {
    if (dbg && lane == 0) *(volatile uint32_t*)dbg = (6u << 20) | (retry & 0xfffff);
    const uint64_t t_snap = q.ring && q.ring->trace_cap ? globaltimer_lane0() : 0ull;
    uint32_t best_key = P3_NONE, best_l = P3_NONE;
    uint64_t best_w = 0;
    for (uint32_t l = lane; l < q.n_layers; l += 32) {
      // acquire: the layer's publish sequence (fifo_key) was stored before its word (ingest)
      const uint64_t w = ld_acquire_gpu64(q.pub + l);
      if (!pub_ready(w, tag)) continue;
      if (ld_relaxed_gpu(q.cursor + l) >= q.nslices[l]) continue;
      const uint32_t key = ld_relaxed_gpu(q.fifo_key + l);
      if (key < best_key || (key == best_key && l < best_l)) {
        best_key = key;
        best_l = l;
        best_w = w;
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const uint32_t ok = __shfl_xor_sync(FULL_MASK, best_key, off);
      const uint32_t ol = __shfl_xor_sync(FULL_MASK, best_l, off);
      const uint64_t ow = __shfl_xor_sync(FULL_MASK, (unsigned long long)best_w, off);
      if (ok < best_key || (ok == best_key && ol < best_l)) {
        best_key = ok;
        best_l = ol;
        best_w = ow;
      }
    }
    if (best_l == P3_NONE) return P3_NONE;
    uint32_t s = 0;
    if (lane == 0) s = atomicAdd(q.cursor + best_l, want);
    s = __shfl_sync(FULL_MASK, s, 0);
    if (s < q.nslices[best_l]) {
      if (out) {
        out->run = min(want, q.nslices[best_l] - s);
        out->layer = best_l;
        out->word = best_w;
        out->t0 = t_snap;
      }
      return q.first[best_l] + s;
    }
    // lost the race for the last slice of that layer: rescan
  }
}

__global__ void k_queue_pop(QueueView q, uint32_t tag, uint32_t* result) {
  const uint32_t g = warp_pop(q, tag);
  if (threadIdx.x == 0) *result = g;
}

int launch_queue_pop(const uint32_t* nslices, const uint32_t* first, const uint64_t* pub,
                     const uint32_t* fifo_key, uint32_t* cursor, uint32_t n_layers, uint32_t sched,
                     uint32_t tag, uint32_t* result, void* stream) {
  QueueView q{n_layers, sched, 1u, 1u, nslices, first, pub, fifo_key, cursor, nullptr};
  k_queue_pop<<<1, 32, 0, (cudaStream_t)stream>>>(q, tag, result);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

// ------------------------------------------------------------------ K3: comm kernel

// Server role pick (one warp): the lowest layer with a completed, unclaimed owned slice,
// then the first such slice of that layer (ascending slice index). The inbox of
// ServerEngine is priority ordered (server.py:118), so the same order is used here.
// Round trips: one to see whether any owned slice completed unclaimed (the common "no"
// ends here), one to scan 256 layers, one for a window of 32 owned slices (arrivals and
// claims are indexed by the slice's position in the owner's list, so no indirection), one
// claim.
__device__ P3_COLD uint32_t warp_server_pick(const CommArgs& a, const LocalDev& L, uint32_t* layer_out,
                                     uint32_t* dbg = nullptr, uint32_t* piece_out = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
  const PlanDev& P = a.plan;
  const uint32_t o = L.rank, nl = P.n_layers, k = a.k;
  const uint32_t* hint = a.peers.hint[o];
  const uint32_t* arrivals = a.peers.arrivals[o];
  const uint32_t* lcount = P.own_lcount + (uint64_t)o * nl;
  const uint32_t* lfirst = P.own_lfirst + (uint64_t)o * nl;
  const uint32_t need = (k + 1) * P.world;
  {
    // completed but unclaimed owned slices (with `srv_filter` > 0, only srv_filter x as many
    // of the launch's consumers as there are such slices look; the rest go to their pushes)
    int32_t avail = 0;
    if (lane == 0) {
      const uint32_t claimed = ld_relaxed_gpu(&L.it->reduced);
      const uint32_t completed = ld_relaxed_sys(a.peers.tally[o] + 1) - k * P.own_total[o];
      avail = (int32_t)(completed - claimed);
    }
    avail = __shfl_sync(FULL_MASK, avail, 0);
    if (avail <= 0 || (a.srv_filter && (blockIdx.x % a.pop_relax) >= a.srv_filter * (uint32_t)avail)) return P3_NONE;
  }
  constexpr uint32_t CH = 8;
  // A scan is a snapshot: with many consumers the candidates it shows are claimed within
  // microseconds, and walking a stale list costs a window round trip per dead candidate
  // (measured: 50 dead candidates, ~50 us per pick, at N=2 for ResNet-50). So each attempt
  // takes one candidate — the (blockIdx + attempt)-th of the most urgent ones, spreading the
  // consumers like the pops do — and a miss rescans.
  for (uint32_t attempt = 0; attempt < 4; ++attempt) {
    const uint64_t t_snap = L.trace_cap ? globaltimer_lane0() : 0ull;  // (trace: before this scan's loads)
    uint32_t ncand = 0, tl = P3_NONE, t_start = 0, t_cnt = 0;
    for (uint32_t group = 0; group < nl && tl == P3_NONE; group += 32 * CH) {
      uint32_t oc[CH], hv[CH], tk[CH], lo[CH];
#pragma unroll
      for (uint32_t c = 0; c < CH; ++c) {
        const uint32_t l = group + 32 * c + lane;
        const bool in = l < nl;
        oc[c] = in ? lcount[l] : 0u;
        hv[c] = in ? ld_relaxed_sys(hint + l) : 0u;
        tk[c] = in ? ld_relaxed_gpu(L.srv_taken + l) : 0u;
        lo[c] = in ? ld_relaxed_gpu(L.srv_lo + l) : 0u;
      }
      uint32_t cnt_c[CH], total = 0;
#pragma unroll
      for (uint32_t c = 0; c < CH; ++c) {
        const bool cand = oc[c] && (int32_t)((hv[c] - k * oc[c]) - tk[c]) > 0 && lo[c] < oc[c];
        cnt_c[c] = __popc(__ballot_sync(FULL_MASK, cand));
        total += cnt_c[c];
        oc[c] = cand ? oc[c] : 0u;  // (reused below as the candidate flag)
      }
      if (!total) continue;
      const uint32_t spread = a.pop_relax > 1 ? min(total, a.pop_relax) : 1u;
      uint32_t t = (blockIdx.x + attempt) % spread;
#pragma unroll
      for (uint32_t c = 0; c < CH; ++c) {
        const uint32_t m = __ballot_sync(FULL_MASK, oc[c] != 0);
        if (tl == P3_NONE && t < cnt_c[c]) {
          uint32_t mm = m;
          for (uint32_t x = 0; x < t; ++x) mm &= mm - 1;
          const uint32_t j = __ffs(mm) - 1;
          tl = group + 32 * c + j;
          t_cnt = __shfl_sync(FULL_MASK, oc[c], j);
          t_start = __shfl_sync(FULL_MASK, lo[c], j);
        } else if (tl == P3_NONE) {
          t -= cnt_c[c];
        }
      }
      ncand += total;
    }
    if (tl == P3_NONE) return P3_NONE;  // nothing completed and unclaimed in the snapshot
    const uint32_t l = tl, cnt = t_cnt;
    const uint32_t lf = lfirst[l];
    for (uint32_t i0 = t_start; i0 < cnt; i0 += 32) {
      if (dbg && lane == 0) *(volatile uint32_t*)dbg = (8u << 20) | ((l & 0x3ff) << 10) | (i0 & 0x3ff);
      const uint32_t i = i0 + lane, pos = lf + i;
      uint32_t g = P3_NONE;
      bool ok = false, claimed = true;
      if (i < cnt) {
        g = P.own_list[pos];
        claimed = ld_relaxed_gpu(L.claim + pos) != k;
        ok = !claimed && (int32_t)(ld_relaxed_sys(arrivals + pos) - need) >= 0;
      }
      // advance the watermark only contiguously: a window below this one may still
      // hold an unclaimed slice even if this window is fully claimed
      if (__all_sync(FULL_MASK, claimed) && lane == 0) atomicCAS(L.srv_lo + l, i0, i0 + 32);
      uint32_t m = __ballot_sync(FULL_MASK, ok);
      // first try a CTA-dependent one of the window's ready slices (consumers spread over
      // them instead of racing for the lowest), then the rest in ascending order
      int pref = -1;
      if (m && a.pop_relax > 1) {
        uint32_t mm = m;
        for (uint32_t skip = blockIdx.x % __popc(m); skip; --skip) mm &= mm - 1;
        pref = __ffs(mm) - 1;
      }
      for (uint32_t tries = 0; m; ++tries) {
        const int jj = (tries == 0 && pref >= 0) ? pref : __ffs(m) - 1;
        m &= ~(1u << jj);
        const uint32_t gj = __shfl_sync(FULL_MASK, g, jj);
        const uint32_t pj = lf + i0 + jj;
        uint32_t won = 0, piece = 0;
        if (lane == 0) {
          if (P3_EXP && a.srv_piece) {
            // pieces: claim the next piece; the claim of the last one claims the slice
            const uint32_t np = (P.slice_len[gj] + a.srv_piece - 1) / a.srv_piece;
            piece = atomicAdd(L.piece_next + pj, 1u);
            won = piece < np;
            if (won && piece + 1 < np) {
              if (L.trace_cap && piece == 0) trace_append(L, k, l, gj - P.layer_first[l], o, P3_EV_PICK, t_snap);
              won = 2;  // a piece; the slice stays open for the other pieces
            } else if (won) {
              atomicExch(L.claim + pj, k + 1);
            }
          } else {
            won = atomicCAS(L.claim + pj, k, k + 1) == k;
          }
          if (won == 1) {
            atomicAdd(L.srv_taken + l, 1u);
            atomicAdd(&L.it->reduced, 1u);
            if (L.trace_cap && (!(P3_EXP && a.srv_piece) || piece == 0))
              trace_append(L, k, l, gj - P.layer_first[l], o, P3_EV_PICK, t_snap);
          }
        }
        won = __shfl_sync(FULL_MASK, won, 0);
        if (won) {
          *layer_out = l;
          if (piece_out) *piece_out = __shfl_sync(FULL_MASK, piece, 0);
          return gj;
        }
      }
    }
  }
  return P3_NONE;
}

__device__ void cta_copy(float* dst, const float* src, uint32_t n, uint32_t tid, uint32_t nthr) {
  constexpr int U = 8;  // 8 independent 16-byte loads in flight per thread
  uint32_t done = 0;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const uint32_t n4 = n / 4;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (uint32_t j = tid; j < n4; j += U * nthr) {  // the partial last round predicated, not serial
      float4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = __ldcg(s4 + (j + u * nthr < n4 ? j + u * nthr : j));
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j + u * nthr < n4) d4[j + u * nthr] = r[u];
    }
    done = 4 * n4;
  }
  for (uint32_t i = done + tid; i < n; i += nthr) dst[i] = __ldcg(src + i);
}

__device__ __forceinline__ QueueView queue_of(const CommArgs& a, const LocalDev& L) {
  QueueView q;
  q.n_layers = a.plan.n_layers;
  q.sched = a.sched;
  q.relax = a.pop_relax;
  q.multi = a.pop_multi;
  q.nslices = a.plan.layer_nslices;
  q.first = a.plan.layer_first;
  q.pub = L.pub;
  q.fifo_key = L.fifo_key;
  q.cursor = L.cursor;
  q.ring = &L;
  return q;
}

// One job handed from the scheduler warp to the producer / consumer warps of a CTA.
#define JOB_NONE 0
#define JOB_REDUCE 1
#define JOB_PUSH 2
#define JOB_EXIT 3
#define JOB_ANSWER 4  // scheduler only: becomes a PUSH-shaped slot with `answer` set
#define JOB_FETCH 5   // scheduler only (broadcast pull): a PUSH-shaped slot with `answer` = 2
struct Job {
  uint32_t kind, li, g, layer, opos, rank, len, n, aligned, run;  // opos: position in the owner's list
  uint32_t ndst;    // REDUCE: replicas written (dst[0..ndst)): N, or 1 when peers pull (notify mode)
  uint32_t pb16;    // REDUCE, param_bf16: bf16 contributions, fp32 master m, bf16 replicas
  float* m;         // REDUCE, param_bf16: the owner's fp32 master of the slice
  uint32_t answer;  // PUSH-shaped copy of an updated slice to a peer that pulled it (notify mode)
  uint32_t pieces;  // REDUCE: pieces the slice is reduced in (srv_piece; 1 = whole)
  uint32_t mc;      // REDUCE, nvls: dst[0] is the multicast address of every replica (multimem.st),
                    // m the owner's own replica (the master p read back)
  uint32_t bf16;  // pushes travel as bf16 (declared lossy mode); own = index of the fp32 source
  const float* src[P3_MAX_RANKS];  // PUSH: src[0]; REDUCE: contributions in rank order
  float* dst[P3_MAX_RANKS];        // PUSH: dst[0]; REDUCE: replicas, dst[0] = owner's master
  float* v;
};

// Named barriers (0 is __syncthreads), per job slot b:
//   FULL(b)  scheduler arrives, producer + signaler sync    (slot b holds a job)
//   DONE(b)  consumers arrive, signaler syncs               (the job's data has moved)
//   EMPTY(b) signaler arrives, scheduler syncs              (slot b may be refilled)
#ifndef P3_SLOTS
#define P3_SLOTS 2  // job slots: the scheduler prepares up to P3_SLOTS - 1 jobs ahead of the movers
                    // (measured: 4 slots hold more claims per CTA and lose the tail balance)
#endif
#define BAR_FULL(b) (1 + (b))
#define BAR_DONE(b) (1 + P3_SLOTS + (b))
#define BAR_EMPTY(b) (1 + 2 * P3_SLOTS + (b))
#define BAR_RANGE (1 + 3 * P3_SLOTS)  // consumers among themselves (direct-path scratch)
static_assert(BAR_RANGE <= 15, "16 named barriers per CTA");
__device__ __forceinline__ void bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// K7 link emulation (TokenBucket.consume, transport.py:42-55) on %globaltimer, one bucket
// per rank's egress: take `bytes` tokens at the bucket rate with `burst` of capacity, and
// wait until they are all taken — the reference's consume() returns at that point. As a
// virtual clock V (the time the bucket has paid for): a grant moves it to
// max(V, now - burst) + bytes/rate and may proceed once now >= V'.
__device__ P3_COLD void pace(const CommArgs& a, const LocalDev& L, uint64_t bytes) {
  if (a.ns_per_byte == 0.f || bytes == 0) return;
  const unsigned long long cost = (unsigned long long)((double)bytes * a.ns_per_byte);
  const unsigned long long now = globaltimer();
  unsigned long long v = *(volatile unsigned long long*)L.vclock, d;
  for (;;) {
    const unsigned long long start = max(v, now - a.burst_ns);
    d = start + cost;
    const unsigned long long old = atomicCAS(L.vclock, v, d);
    if (old == v) break;
    v = old;
  }
  while (globaltimer() < d) __nanosleep(2000);
}

// Turn newly published ring entries into publication words (one warp). The ring tail is
// advanced by a stream memory write ordered after the kernels that produced the gradients,
// so entries below it are safe to expose; the first warp to move `ingested` forward copies
// them, the others see the layers on a later pick.
// The single-rank streaming kernel keeps the one-entry-per-lane ingest inline: the batched,
// out-of-line one changed its register allocation (111 -> 128) and cost ~0.8% there.
__device__ __forceinline__ void ingest_lanes(const LocalDev& L) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = 0, won = 0;
  if (lane == 0) {
    lo = ld_relaxed_gpu(L.ingested);
    hi = ld_acquire_gpu(L.pubseq);
    if ((int32_t)(hi - lo) > 0) won = atomicCAS(L.ingested, lo, hi) == lo;
  }
  won = __shfl_sync(FULL_MASK, won, 0);
  if (!won) return;
  lo = __shfl_sync(FULL_MASK, lo, 0);
  hi = __shfl_sync(FULL_MASK, hi, 0);
  __syncwarp();
  fence_acq_rel_gpu();
  for (uint32_t i = lo + lane; (int32_t)(hi - i) > 0; i += 32) {
    const volatile PubEntry* e = L.ring + (i % L.ring_cap);
    const uint32_t layer = e->layer;
    const unsigned long long word = e->word;
    *(volatile unsigned long long*)(L.pub + layer) = word;
    if (L.trace_cap) {
      __threadfence();
      trace_append(L, (uint32_t)(word >> 48) - 1u, layer, e->key, L.rank, P3_EV_PUBLISH);
    }
  }
  __syncwarp();
  if (lane == 0) *(volatile uint32_t*)L.ingested_host = hi;
}

__device__ __noinline__ void ingest(const LocalDev& L, uint32_t sched) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = 0, won = 0;
  if (lane == 0) {
    lo = ld_relaxed_gpu(L.ingested);  // issued first: both loads share one round trip
    hi = ld_acquire_gpu(L.pubseq);
    if ((int32_t)(hi - lo) > 0) won = atomicCAS(L.ingested, lo, hi) == lo;
  }
  won = __shfl_sync(FULL_MASK, won, 0);
  if (!won) return;
  lo = __shfl_sync(FULL_MASK, lo, 0);
  hi = __shfl_sync(FULL_MASK, hi, 0);
  // release: a consumer that reads a publication word relaxed and then fences (acquire
  // pattern) sees the gradients the memory write of pubseq was ordered after
  __syncwarp();
  fence_acq_rel_gpu();
  // The ring is in pinned host memory: every read is a PCIe round trip, so each lane issues
  // the 16-byte loads of up to P3_INGEST_U entries before using any (a whole iteration's
  // publications — 161 for ResNet-50 — in one or two round trips instead of one per 32).
  constexpr uint32_t U = P3_INGEST_U;
  for (uint32_t base = lo; (int32_t)(hi - base) > 0; base += 32 * U) {
    uint4 ent[U];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const uint32_t i = base + 32 * u + lane;
      if ((int32_t)(hi - i) > 0) {
        const PubEntry* e = L.ring + (i % L.ring_cap);
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(ent[u].x), "=r"(ent[u].y), "=r"(ent[u].z), "=r"(ent[u].w)
                     : "l"(e));
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const uint32_t i = base + 32 * u + lane;
      if ((int32_t)(hi - i) <= 0) continue;
      const uint32_t layer = ent[u].x;
      const uint32_t key = ent[u].y;
      const unsigned long long word = (unsigned long long)ent[u].z | ((unsigned long long)ent[u].w << 32);
      if (sched == P3_SCHED_FIFO) {
        // the publish sequence is visible before the word (FIFO pops load the word with acquire)
        *(volatile uint32_t*)(L.fifo_key + layer) = key;
        __threadfence();
      }
      *(volatile unsigned long long*)(L.pub + layer) = word;
      if (L.trace_cap) {  // PUBLISH (put_batch) once the word is visible to every pop
        __threadfence();
        trace_append(L, (uint32_t)(word >> 48) - 1u, layer, key, L.rank, P3_EV_PUBLISH);
      }
    }
  }
  __syncwarp();
  if (lane == 0) *(volatile uint32_t*)L.ingested_host = hi;  // host may reuse the entries
}

// Scheduler side of a push. With job == nullptr, classify the popped slice: a remote
// owner needs a push job (PUSH_REMOTE); for a local owner the contribution stays in place
// and only the arrival is counted here — and when that arrival completes the slice the
// scheduler claims its reduction at once (PUSH_REDUCE) instead of leaving it to a later
// server pick. With a slot: fill it for the producer / consumers, who store the slice into the owner's
// receive slot over NVLink.
#define PUSH_DONE 0
#define PUSH_REMOTE 1
#define PUSH_REDUCE 2
__device__ uint32_t prepare_push(const CommArgs& a, uint32_t li, uint32_t g, uint32_t l, uint64_t w, Job* job,
                                 uint64_t t0 = 0) {
  const PlanDev& P = a.plan;
  const LocalDev& L = a.loc[li];
  const uint32_t r = L.rank;
  // round-robin plans (make_p3_plan: owner = slice counter % N) need no table load here:
  // the owner is g % N and its own-list position own_base[o] + g / N
  const uint32_t o = P.rr_owner ? g % P.world : P.slice_owner[g];
  const uint32_t opos = P.rr_owner ? P.own_base[o] + g / P.world : P.slice_opos[g];
  const uint32_t lane = threadIdx.x & 31;
  if (!job) {
    uint32_t verdict = o == r ? PUSH_DONE : PUSH_REMOTE;
    if (lane == 0) {
      // the pop read the publication word relaxed: this fence makes it an acquire, so the
      // gradient is visible from here on (ingest released it)
      fence_acq_rel_gpu();
      if (L.trace_cap) trace_append(L, a.k, l, g - P.layer_first[l], a.trace_cta ? blockIdx.x : r, P3_EV_PUSH, t0);
      if (o == r) {
        // the contribution stays in place (published to this rank by the acquire above)
        const uint32_t old = atom_add_relaxed_gpu(a.peers.arrivals[o] + opos, 1u);
        P3_CHECK(old >= a.k * P.world && old < (a.k + 1) * P.world);
        red_add_relaxed_sys(a.peers.tally[o], 1u);
        if (old + 1 == (a.k + 1) * P.world) {  // the last arrival: the slice is complete
          red_add_relaxed_sys(a.peers.hint[o] + l, 1u);
          const uint32_t done_before = atom_add_relaxed_sys(a.peers.tally[o] + 1, 1u);
          if (L.trace_cap) {  // COMPLETE once the completion is visible to every server pick
            __threadfence();
            trace_append(L, a.k, l, g - P.layer_first[l], o, P3_EV_COMPLETE);
          }
          // Claim the reduction right here only when no other completed owned slice waits
          // (else the server picks take them in priority order, this one included). The pick
          // time is taken before the backlog is read.
          const uint64_t tc = L.trace_cap ? globaltimer() : 0ull;
          const uint32_t backlog = done_before + 1u - a.k * P.own_total[o] - ld_relaxed_gpu(&L.it->reduced);
          if (!(P3_EXP && a.srv_piece) && (int32_t)backlog <= 1 && atomicCAS(L.claim + opos, a.k, a.k + 1) == a.k) {
            atomicAdd(L.srv_taken + l, 1u);
            atomicAdd(&L.it->reduced, 1u);
            if (L.trace_cap) trace_append(L, a.k, l, g - P.layer_first[l], o, P3_EV_PICK, tc);
            verdict = PUSH_REDUCE;
          }
        }
      }
    }
    return __shfl_sync(FULL_MASK, verdict, 0);
  }
  if (lane == 0) {
    job->kind = JOB_PUSH;
    job->ndst = 1;
    job->answer = 0;
    job->pb16 = 0;
    job->run = 1;
    job->n = 1;  // one source (the slot keeps no stale rank count from a previous reduce)
    job->li = li;
    job->g = g;
    job->layer = l;
    job->opos = opos;
    job->rank = o;
    job->len = P.slice_len[g];
    const uint64_t ri = (uint64_t)r * P.own_stride[o] + P.slice_slot[g];
    if (a.pb16) {  // bf16 gradient copied as is into a bf16 receive slot (2-byte elements)
      job->src[0] = reinterpret_cast<const float*>(reinterpret_cast<const __nv_bfloat16*>(pub_ptr(w)) + P.slice_off[g]);
      job->bf16 = 2;
      job->dst[0] = reinterpret_cast<float*>(reinterpret_cast<__nv_bfloat16*>(a.peers.R[o]) + ri);
    } else {
      job->src[0] = pub_ptr(w) + P.slice_off[g];
      job->bf16 = a.push_bf16;
      job->dst[0] = a.push_bf16 ? reinterpret_cast<float*>(reinterpret_cast<__nv_bfloat16*>(a.peers.R[o]) + ri)
                                : a.peers.R[o] + ri;
    }
  }
  return PUSH_REMOTE;
}

// Scheduler side of a reduce: contributions of every rank (the owner's own straight from
// its gradient) and every replica to write, master first.
// `w` is the layer's publication word when the caller already holds it (0: load it).
__device__ void prepare_reduce(const CommArgs& a, uint32_t li, uint32_t g, uint32_t l, uint64_t w, Job* job,
                               uint32_t run = 1, uint32_t piece = 0) {
  const PlanDev& P = a.plan;
  const LocalDev& L = a.loc[li];
  // srv_piece: elements [piece * srv_piece, +srv_piece) of the slice
  const uint32_t o = L.rank, N = P.world;
  const bool pieces = P3_EXP && a.srv_piece && N > 1;
  const uint32_t pe0 = pieces ? piece * a.srv_piece : 0u;
  const uint32_t q = threadIdx.x & 31;
  // independent loads first (one round trip), then the acquire that orders the data reads
  const uint64_t soff = P.slice_off[g] + pe0;
  const uint64_t woff = P.layer_woff[l] + soff;
  const uint64_t slot = P.slice_slot[g] + pe0;
  const uint32_t opos = N > 1 ? P.slice_opos[g] : 0u;
  const uint64_t stride = P.own_stride[o];
  uint32_t len = q < run ? P.slice_len[g + q] : 0u;  // consecutive slices: contiguous
  if (!w) w = ld_relaxed_gpu64(L.pub + l);
  if (N > 1) {
    if (q == 0) (void)ld_acquire_sys(a.peers.arrivals[o] + opos);  // all N pushes are visible
  } else if (q == 0) {
    fence_acq_rel_gpu();  // acquire of the publication word (single rank: nothing arrives)
  }
  __syncwarp();
  uintptr_t al = 0;
  if (q < N) {
    const uint64_t ri = (uint64_t)q * stride + slot;
    const bool b16 = a.push_bf16 || a.pb16;  // receive slots hold bf16
    const float* rsrc = b16 ? reinterpret_cast<const float*>(reinterpret_cast<__nv_bfloat16*>(a.peers.R[o]) + ri)
                            : a.peers.R[o] + ri;
    const float* own = a.pb16 ? reinterpret_cast<const float*>(reinterpret_cast<const __nv_bfloat16*>(pub_ptr(w)) + soff)
                              : pub_ptr(w) + soff;
    const float* src = q == o ? own : rsrc;
    float* dst = a.pb16 ? reinterpret_cast<float*>(reinterpret_cast<__nv_bfloat16*>(a.peers.W[q]) + woff)
                        : a.peers.W[q] + woff;
    job->src[q] = src;
    job->dst[q == o ? 0 : (q < o ? q + 1 : q)] = dst;
    al = (uintptr_t)src | (uintptr_t)dst;
  }
  float* v = L.V ? L.V + slot : nullptr;
  float* m = L.M ? L.M + slot : nullptr;
#pragma unroll
  for (int off = 16; off; off >>= 1) al |= __shfl_xor_sync(FULL_MASK, (unsigned long long)al, off);
#pragma unroll
  for (int off = 16; off; off >>= 1) len += __shfl_xor_sync(FULL_MASK, len, off);
  const uint32_t np = pieces ? (len + a.srv_piece - 1) / a.srv_piece : 1u;
  if (pieces) len = min(a.srv_piece, len - pe0);
  if (q == 0) {
    job->kind = JOB_REDUCE;
    job->pieces = np;
    job->opos = opos;
    job->ndst = a.notify ? 1u : N;  // notify mode: peers pull the update (server.py:227-247)
    job->answer = 0;
    job->li = li;
    job->g = g;
    job->layer = l;
    job->rank = o;
    job->run = run;
    job->len = len;
    job->n = N;
    job->v = v;
    job->m = m;
    job->pb16 = a.pb16;
    job->bf16 = a.push_bf16 ? 1u + o : 0u;  // 1 + index of the owner's own (fp32) contribution
    job->aligned = ((al | (uintptr_t)v | (uintptr_t)m) & 15) == 0;
  }
  __syncwarp();
  if (q == 0) {
    // nvls: one multicast store per element reaches every replica (the NVSwitch fans it out);
    // the master p is read from the owner's own replica
    job->mc = a.mcw && N > 1 ? 1u : 0u;
    if (job->mc) {
      job->ndst = 1;
      job->m = a.peers.W[o] + woff;
      job->dst[0] = a.mcw + woff;
    }
  }
}

// bf16 transport (declared lossy mode): each rank's contribution is rounded to bf16 (round
// to nearest even) — the owner's own one too, so every rank counts alike — then summed in
// fp32 in ascending rank order; the update and the broadcast parameters stay fp32.
__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ uint2 to_bf16x4(const float4& v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  uint2 w;
  w.x = *reinterpret_cast<uint32_t*>(&lo);
  w.y = *reinterpret_cast<uint32_t*>(&hi);
  return w;
}
__device__ __forceinline__ float4 from_bf16x4(const uint2& w) {
  const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&w.x);
  const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&w.y);
  const float2 a = __bfloat1622float2(lo), b = __bfloat1622float2(hi);
  return make_float4(a.x, a.y, b.x, b.y);
}

__device__ void cta_copy_to_bf16(__nv_bfloat16* dst, const float* src, uint32_t n, uint32_t tid, uint32_t nthr) {
  uint32_t done = 0;
  if ((((uintptr_t)src & 15) | ((uintptr_t)dst & 7)) == 0) {
    constexpr int U = 8;
    const uint32_t n4 = n / 4;
    for (uint32_t j = tid; j < n4; j += U * nthr) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcg(reinterpret_cast<const float4*>(src) + (j + u * nthr < n4 ? j + u * nthr : j));
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j + u * nthr < n4) *reinterpret_cast<uint2*>(dst + 4 * (j + u * nthr)) = to_bf16x4(v[u]);
    }
    done = 4 * n4;
  }
  for (uint32_t i = done + tid; i < n; i += nthr) dst[i] = __float2bfloat16_rn(__ldcg(src + i));
}

__device__ void cta_update_bf16(float* const* dst, int ndst, const float* const* src, int nw, int own, float* v,
                                uint64_t n, const UpdCoef& c, uint32_t tid, uint32_t nthr) {
  uintptr_t al8 = 0, al16 = (uintptr_t)v;
  for (int q = 0; q < nw; ++q) {
    if (q == own) al16 |= (uintptr_t)src[q];
    else al8 |= (uintptr_t)src[q];
  }
  for (int d = 0; d < ndst; ++d) al16 |= (uintptr_t)dst[d];
  uint64_t done = 0;
  if ((al8 & 7) == 0 && (al16 & 15) == 0) {
    // 4 elements per vector: the other ranks' bf16 contributions as 8-byte loads, the own
    // fp32 one rounded here; per rank U loads in flight, summed in ascending rank order
    constexpr int U = 4;
    const uint32_t m4 = (uint32_t)(n / 4);
    for (uint32_t j = tid; j < m4; j += U * nthr) {
      float4 acc[U], p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        p[u] = __ldcg(reinterpret_cast<const float4*>(dst[0]) + (j + u * nthr < m4 ? j + u * nthr : j));
      }
      for (int q = 0; q < nw; ++q) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t e = j + u * nthr < m4 ? j + u * nthr : j;
          if (q == own) {
            const float4 f = __ldcg(reinterpret_cast<const float4*>(src[q]) + e);
            x[u] = make_float4(bf16_round(f.x), bf16_round(f.y), bf16_round(f.z), bf16_round(f.w));
          } else {
            x[u] = from_bf16x4(__ldcg(reinterpret_cast<const uint2*>(src[q]) + e));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          acc[u].x = __fadd_rn(acc[u].x, x[u].x);
          acc[u].y = __fadd_rn(acc[u].y, x[u].y);
          acc[u].z = __fadd_rn(acc[u].z, x[u].z);
          acc[u].w = __fadd_rn(acc[u].w, x[u].w);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t e = j + u * nthr;
        if (e >= m4) continue;
        float4 vv = v ? __ldcg(reinterpret_cast<const float4*>(v) + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 r = sgd4(p[u], acc[u], c, v ? &vv : nullptr);
        if (v) reinterpret_cast<float4*>(v)[e] = vv;
        for (int d = 0; d < ndst; ++d) reinterpret_cast<float4*>(dst[d])[e] = r;
      }
    }
    done = 4 * (uint64_t)m4;
  }
  for (uint64_t i = done + tid; i < n; i += nthr) {
    float acc = 0.f;
    for (int q = 0; q < nw; ++q) {
      const float x = q == own ? bf16_round(__ldcg(src[q] + i))
                               : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src[q])[i]);
      acc = __fadd_rn(acc, x);
    }
    const float p = sgd_step(__ldcg(dst[0] + i), acc, c, v ? v + i : nullptr);
    for (int d = 0; d < ndst; ++d) dst[d][i] = p;
  }
}

// Consumers, direct path: elements [e0, e0 + n) of the job straight from global memory
// (jobs the TMA path cannot take — unaligned sources — and the < 8-element residue of the
// others). `ptrs` is consumer-shared scratch for the offset pointer arrays.
struct RangePtrs {
  const float* src[P3_MAX_RANKS];
  float* dst[P3_MAX_RANKS];
};
__device__ __noinline__ void move_range_pb16(const CommArgs& a, const Job& j, uint32_t e0, uint32_t n, uint32_t tid,
                                             uint32_t nthr);
__device__ void move_range(const CommArgs& a, const Job& j, uint32_t e0, uint32_t n, RangePtrs* ptrs, uint32_t tid,
                           uint32_t nthr) {
  const bool bf = j.bf16 != 0;
  if (j.pb16 || (j.kind == JOB_PUSH && j.bf16 == 2)) {
    move_range_pb16(a, j, e0, n, tid, nthr);
    return;
  }
  if (j.kind == JOB_PUSH) {
    if (bf)
      cta_copy_to_bf16(reinterpret_cast<__nv_bfloat16*>(j.dst[0]) + e0, j.src[0] + e0, n, tid, nthr);
    else
      cta_copy(j.dst[0] + e0, j.src[0] + e0, n, tid, nthr);
    return;
  }
  const int own = bf ? (int)j.bf16 - 1 : -1;
  if (tid < j.n) {  // bf16 receive slots are offset in bf16 elements
    ptrs->src[tid] = (bf && (int)tid != own)
                         ? reinterpret_cast<const float*>(reinterpret_cast<const __nv_bfloat16*>(j.src[tid]) + e0)
                         : j.src[tid] + e0;
    ptrs->dst[tid] = j.dst[tid] + e0;
  }
  if (j.mc && tid == 0) ptrs->dst[0] = j.m + e0;  // nvls: update the own replica, multicast below
  bar_sync(BAR_RANGE, nthr);
  float* v = j.v ? j.v + e0 : nullptr;
  if (j.mc) {
    if (bf)
      cta_update_bf16(ptrs->dst, 1, ptrs->src, (int)j.n, own, v, n, make_coef(j.n, a.lr, a.momentum), tid, nthr);
    else
      cta_update_generic(ptrs->dst[0], ptrs->dst, 1, ptrs->src, (int)j.n, v, n, j.aligned != 0,
                         make_coef(j.n, a.lr, a.momentum), tid, nthr);
    bar_sync(BAR_RANGE, nthr);  // the range's new values (global, this CTA) before the fan-out
    for (uint32_t i = tid; i < n; i += nthr) {
      const float p = __ldcg(j.m + e0 + i);
      asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(j.dst[0] + e0 + i), "f"(p) : "memory");
    }
    bar_sync(BAR_RANGE, nthr);
    return;
  }
  if (bf)
    cta_update_bf16(ptrs->dst, (int)j.ndst, ptrs->src, (int)j.n, own, v, n, make_coef(j.n, a.lr, a.momentum), tid, nthr);
  else
    cta_update_generic(ptrs->dst[0], ptrs->dst, (int)j.ndst, ptrs->src, (int)j.n, v, n, j.aligned != 0,
                       make_coef(j.n, a.lr, a.momentum), tid, nthr);
  bar_sync(BAR_RANGE, nthr);  // the scratch may be rewritten by the next range
}

// TMA staging. A stage holds one tile of every source of a job (reduce: the N contributions,
// the master copy p and the momentum v; push: the gradient) — `tile` elements each, at
// 4-byte pitch. The producer warp streams tiles of consecutive jobs into the stage ring
// with cp.async.bulk (no registers, up to P3_STAGES tiles in flight per SM, running ahead
// across job boundaries); the consumer warps compute from shared memory and store.
#ifndef P3_STAGES
#define P3_STAGES 3
#endif
#ifndef P3_STAGE_BYTES
#define P3_STAGE_BYTES (64 * 1024)
#endif
#define ST_LAST 1u    // last stage of its job
#define ST_EXIT 2u    // no more jobs
#define ST_DIRECT 4u  // consumers take the range straight from global memory
struct StageDesc {
  uint32_t b;      // job slot
  uint32_t e0, n;  // element range of the job
  uint32_t flags;
  uint32_t tile;   // elements per source tile (pitch)
};
__device__ __forceinline__ uint32_t job_sources(const Job& j) {
  return j.kind == JOB_PUSH ? 1u : j.n + 1u + (j.v ? 1u : 0u);
}
__device__ __forceinline__ uint32_t job_tile(const Job& j) {
  return (P3_STAGE_BYTES / (4u * job_sources(j))) & ~7u;
}
// 16-byte aligned sources (TMA requirement; bf16 receive slots at 2-byte pitch)
__device__ __forceinline__ bool job_tma_ok(const Job& j) {
  if (j.kind == JOB_PUSH)  // and the vector stores of the consumers (float4, or 4 x bf16)
    return ((uintptr_t)j.src[0] & 15) == 0 && ((uintptr_t)j.dst[0] & (j.bf16 == 1 ? 7 : 15)) == 0;
  uintptr_t al = (uintptr_t)j.dst[0] | (uintptr_t)j.v | (uintptr_t)j.m;
  for (uint32_t q = 0; q < j.n; ++q) al |= (uintptr_t)j.src[q];
  return (al & 15) == 0 && j.aligned;
}

// Consumers, staged path: one tile range [e0, e0 + n) (n a multiple of 8) from shared memory.
// Specialised on the rank count and the mode so the inner loop keeps its pointers in
// registers (no reloads of the shared job slot per element) and unrolls the rank-ordered sum.
template <int NW, bool BF, bool MOM>
__device__ __forceinline__ void consume_reduce(const uint8_t* st, uint32_t pitch, uint32_t n4, uint32_t e4,
                                               float* const* dstp, float* vp, int own, const UpdCoef& c,
                                               uint32_t tid, uint32_t nthr, int tosmem, int ndst, bool mc = false) {
  float4* dst[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) dst[q] = reinterpret_cast<float4*>(dstp[q]) + e4;
  float4* v = MOM ? reinterpret_cast<float4*>(vp) + e4 : nullptr;
  const float4* tp = reinterpret_cast<const float4*>(st + NW * pitch);
  const float4* tv = reinterpret_cast<const float4*>(st + (NW + 1) * pitch);
  for (uint32_t k = tid; k < n4; k += nthr) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < NW; ++q) {  // ascending rank order from +0.0
      float4 x;
      if (!BF) {
        x = reinterpret_cast<const float4*>(st + q * pitch)[k];
      } else if (q == own) {
        const float4 f = reinterpret_cast<const float4*>(st + q * pitch)[k];
        x = make_float4(bf16_round(f.x), bf16_round(f.y), bf16_round(f.z), bf16_round(f.w));
      } else {
        x = from_bf16x4(reinterpret_cast<const uint2*>(st + q * pitch)[k]);
      }
      acc.x = __fadd_rn(acc.x, x.x);
      acc.y = __fadd_rn(acc.y, x.y);
      acc.z = __fadd_rn(acc.z, x.z);
      acc.w = __fadd_rn(acc.w, x.w);
    }
    float4 vv = MOM ? tv[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 r = sgd4(tp[k], acc, c, MOM ? &vv : nullptr);
    if (tosmem) {  // results back into the stage (p tile), stored by TMA afterwards
      const_cast<float4*>(tp)[k] = r;
      if (tosmem == 1) {  // every replica and v by TMA
        if (MOM) const_cast<float4*>(tv)[k] = vv;
        continue;
      }
    }
    if (MOM) v[k] = vv;
    if (mc) {  // nvls: every replica at once
      asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst[0] + k), "f"(r.x), "f"(r.y),
                   "f"(r.z), "f"(r.w)
                   : "memory");
      continue;
    }
#pragma unroll
    for (int q = 0; q < NW; ++q)  // (tosmem 2: the local replica here, the remote ones by TMA)
      if (q < ndst && (tosmem != 2 || q == 0)) dst[q][k] = r;
  }
}

// param_bf16 reduce of one staged tile: the N bf16 contributions summed in fp32 in ascending
// rank order, the fp32 master updated (the same sgd4 as the fp32 path) and stored, and every
// replica written as bf16(master), round to nearest even. Out of line: an opt-in mode.
__device__ __noinline__ void consume_reduce_pb16(const CommArgs& a, const Job& j, const StageDesc& d,
                                                 const uint8_t* st, uint32_t tid, uint32_t nthr) {
  const uint32_t N = j.n, n4 = d.n / 4, e4 = d.e0 / 4, pitch = d.tile * 4;
  const UpdCoef c = make_coef(N, a.lr, a.momentum);
  const float4* tp = reinterpret_cast<const float4*>(st + N * pitch);
  const float4* tv = reinterpret_cast<const float4*>(st + (N + 1) * pitch);
  float4* m = reinterpret_cast<float4*>(j.m) + e4;
  float4* v = j.v ? reinterpret_cast<float4*>(j.v) + e4 : nullptr;
  for (uint32_t k = tid; k < n4; k += nthr) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t q = 0; q < N; ++q) {
      const float4 x = from_bf16x4(reinterpret_cast<const uint2*>(st + q * pitch)[k]);
      acc.x = __fadd_rn(acc.x, x.x);
      acc.y = __fadd_rn(acc.y, x.y);
      acc.z = __fadd_rn(acc.z, x.z);
      acc.w = __fadd_rn(acc.w, x.w);
    }
    float4 vv = v ? tv[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 r = sgd4(tp[k], acc, c, v ? &vv : nullptr);
    if (v) v[k] = vv;
    m[k] = r;
    const uint2 h = to_bf16x4(r);
    for (uint32_t q = 0; q < j.ndst; ++q) reinterpret_cast<uint2*>(j.dst[q])[e4 + k] = h;
  }
}

__device__ __noinline__ void move_range_pb16(const CommArgs& a, const Job& j, uint32_t e0, uint32_t n, uint32_t tid,
                                             uint32_t nthr) {
  const UpdCoef c = make_coef(j.n, a.lr, a.momentum);
  for (uint32_t i = e0 + tid; i < e0 + n; i += nthr) {
    if (j.kind == JOB_PUSH) {  // bf16 copy
      reinterpret_cast<__nv_bfloat16*>(j.dst[0])[i] = reinterpret_cast<const __nv_bfloat16*>(j.src[0])[i];
      continue;
    }
    float acc = 0.f;
    for (uint32_t q = 0; q < j.n; ++q)
      acc = __fadd_rn(acc, __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(j.src[q])[i]));
    const float p = sgd_step(j.m[i], acc, c, j.v ? j.v + i : nullptr);
    j.m[i] = p;
    const __nv_bfloat16 h = __float2bfloat16_rn(p);
    for (uint32_t q = 0; q < j.ndst; ++q) reinterpret_cast<__nv_bfloat16*>(j.dst[q])[i] = h;
  }
}

template <bool ONE>
__device__ void consume_tile(const CommArgs& a, const Job& j, const StageDesc& d, const uint8_t* st, uint32_t tid,
                             uint32_t nthr, int tosmem = 0) {
  const uint32_t n4 = d.n / 4, e4 = d.e0 / 4, pitch = d.tile * 4;
  if (j.kind == JOB_PUSH) {
    const float4* t0 = reinterpret_cast<const float4*>(st);
    if (j.bf16 == 2) {  // bf16 copy: 8 bf16 per 16 bytes
      float4* out = reinterpret_cast<float4*>(reinterpret_cast<__nv_bfloat16*>(j.dst[0]) + d.e0);
      for (uint32_t k = tid; k < d.n / 8; k += nthr) out[k] = t0[k];
    } else if (j.bf16) {
      uint2* out = reinterpret_cast<uint2*>(j.dst[0]) + e4;  // 4 bf16 per 8 bytes
      for (uint32_t k = tid; k < n4; k += nthr) out[k] = to_bf16x4(t0[k]);
    } else {
      float4* out = reinterpret_cast<float4*>(j.dst[0]) + e4;
      for (uint32_t k = tid; k < n4; k += nthr) out[k] = t0[k];
    }
    return;
  }
  if (!ONE && j.pb16) {
    consume_reduce_pb16(a, j, d, st, tid, nthr);
    return;
  }
  const uint32_t N = ONE ? 1u : j.n;
  const int nd = (int)j.ndst;
  const bool bf = j.bf16 != 0, mom = j.v != nullptr;
  const int own = bf ? (int)j.bf16 - 1 : -1;
  const UpdCoef c = make_coef(N, a.lr, a.momentum);
  float* const* dst = j.dst;
  float* v = j.v;
  const bool mc = !ONE && j.mc;
#define P3_CONSUME(K)                                                                                   \
  case K:                                                                                               \
    if (bf) {                                                                                           \
      if (mom) consume_reduce<K, true, true>(st, pitch, n4, e4, dst, v, own, c, tid, nthr, tosmem, nd, mc);     \
      else consume_reduce<K, true, false>(st, pitch, n4, e4, dst, v, own, c, tid, nthr, tosmem, nd, mc);        \
    } else {                                                                                            \
      if (mom) consume_reduce<K, false, true>(st, pitch, n4, e4, dst, v, own, c, tid, nthr, tosmem, nd, mc);    \
      else consume_reduce<K, false, false>(st, pitch, n4, e4, dst, v, own, c, tid, nthr, tosmem, nd, mc);       \
    }                                                                                                   \
    return;
  if (ONE) {
    switch (N) { P3_CONSUME(1) default: break; }
  } else {
    switch (N) {
      P3_CONSUME(1) P3_CONSUME(2) P3_CONSUME(3) P3_CONSUME(4) P3_CONSUME(5) P3_CONSUME(6) P3_CONSUME(7)
      P3_CONSUME(8)
      default: break;
    }
  }
#undef P3_CONSUME
  // more than 8 ranks: runtime rank loop
  for (uint32_t k = tid; k < n4; k += nthr) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t q = 0; q < N; ++q) {
      float4 x;
      if (!bf) {
        x = reinterpret_cast<const float4*>(st + q * pitch)[k];
      } else if ((int)q == own) {
        const float4 f = reinterpret_cast<const float4*>(st + q * pitch)[k];
        x = make_float4(bf16_round(f.x), bf16_round(f.y), bf16_round(f.z), bf16_round(f.w));
      } else {
        x = from_bf16x4(reinterpret_cast<const uint2*>(st + q * pitch)[k]);
      }
      acc.x = __fadd_rn(acc.x, x.x);
      acc.y = __fadd_rn(acc.y, x.y);
      acc.z = __fadd_rn(acc.z, x.z);
      acc.w = __fadd_rn(acc.w, x.w);
    }
    float4 vv = mom ? reinterpret_cast<const float4*>(st + (N + 1) * pitch)[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 r = sgd4(reinterpret_cast<const float4*>(st + N * pitch)[k], acc, c, mom ? &vv : nullptr);
    if (mom) reinterpret_cast<float4*>(v)[e4 + k] = vv;
    if (mc) {
      asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(reinterpret_cast<float4*>(dst[0]) + e4 + k),
                   "f"(r.x), "f"(r.y), "f"(r.z), "f"(r.w)
                   : "memory");
      continue;
    }
    for (int q = 0; q < nd; ++q) reinterpret_cast<float4*>(dst[q])[e4 + k] = r;
  }
}

// Signaler (one thread, after the consumers' barrier): publish the job's completion with
// release semantics at system scope when a peer lives on another GPU. Push: count the
// arrival at the owner (and the owner's layer hint when it completes the slice). Reduce:
// bump every replica's done[layer] (the forward gate, worker.py:262-269).
__device__ P3_COLD void signal_job(const CommArgs& a, const Job& j) {
  const PlanDev& P = a.plan;
  const LocalDev& L = a.loc[j.li];
  // one fence releases every store the consumers made (ordered before it by the DONE barrier);
  // the counter updates after it are plain relaxed reductions (fire and forget)
  if (a.remote) fence_acq_rel_sys(); else fence_acq_rel_gpu();
  if (j.kind == JOB_PUSH && j.answer) {
    // notify mode: the pulled slice is in the requester's replica (the BCAST answer of
    // server.py:240-247; on_bcast, worker.py:241-269)
    red_add_relaxed_sys(a.peers.done[j.rank] + j.layer, 1u);
    red_add_relaxed_sys(a.peers.gdone[j.rank] + P.layer_group[j.layer], 1u);
    atomicAdd(L.pcount + 1, 1u);
    atomicAdd(L.bytes + 1, (j.bf16 == 2 ? 2ull : 4ull) * j.len);
    if (L.trace_cap) trace_append(L, a.k, j.layer, j.g - P.layer_first[j.layer], j.rank, P3_EV_BCAST);
    return;
  }
  if (j.kind == JOB_PUSH) {
    // the last arriver completes the slice and tells the owner's scheduler (hint)
    const uint32_t old = atom_add_relaxed_sys(a.peers.arrivals[j.rank] + j.opos, 1u);
    P3_CHECK(old >= a.k * P.world && old < (a.k + 1) * P.world);  // one push per rank and slice
    red_add_relaxed_sys(a.peers.tally[j.rank], 1u);
    if (old + 1 == (a.k + 1) * P.world) {
      red_add_relaxed_sys(a.peers.hint[j.rank] + j.layer, 1u);
      red_add_relaxed_sys(a.peers.tally[j.rank] + 1, 1u);
      if (L.trace_cap) {  // COMPLETE once the completion is visible to the owner's picks
        fence_acq_rel_sys();
        trace_append(L, a.k, j.layer, j.g - P.layer_first[j.layer], j.rank, P3_EV_COMPLETE);
      }
    }
    atomicAdd(L.bytes + 1, (j.bf16 ? 2ull : 4ull) * j.len);
    return;
  }
  if (P3_EXP && j.pieces > 1) {
    // a piece of a slice reduced in pieces: only the last one to finish signals the slice,
    // after acquiring the other pieces' releases
    atomicAdd(L.bytes + 0, (j.bf16 || j.pb16 ? 2ull : 4ull) * j.len * (j.n - 1));
    if (!a.notify) atomicAdd(L.bytes + 1, (j.pb16 ? 2ull : 4ull) * j.len * (j.n - 1));
    if (atomicAdd(L.piece_done + j.opos, 1u) + 1 < j.pieces) return;
    fence_acq_rel_sys();
  }
  if (a.notify) {
    // notify mode: the owner's replica holds the update; NOTIFY every other rank, which will
    // PULL it (server.py:227-239)
    const uint32_t grp = P.layer_group[j.layer];
    red_add_relaxed_sys(a.peers.done[j.rank] + j.layer, j.run);
    red_add_relaxed_sys(a.peers.gdone[j.rank] + grp, j.run);
    for (uint32_t q = 0; q < j.n; ++q) {
      if (q == j.rank) continue;
      for (uint32_t i = 0; i < j.run; ++i) {
        const uint32_t pos = atom_add_relaxed_sys(a.peers.ntf_tail[q], 1u);
        *(volatile unsigned long long*)(a.peers.ntf_ring[q] + pos % a.ntf_cap) =
            ((unsigned long long)(a.k + 1) << 32) | (j.g + i);
        if (L.trace_cap) trace_append(L, a.k, j.layer, j.g + i - P.layer_first[j.layer], q, P3_EV_NOTIFY);
      }
    }
    if (!P3_EXP || j.pieces <= 1) atomicAdd(L.bytes + 0, (j.bf16 || j.pb16 ? 2ull : 4ull) * j.len * (j.n - 1));  // pushes received
  } else {
    const uint32_t grp = P.layer_group[j.layer];
    for (uint32_t q = 0; q < j.n; ++q) {
      red_add_relaxed_sys(a.peers.done[q] + j.layer, j.run);
      red_add_relaxed_sys(a.peers.gdone[q] + grp, j.run);
    }
    if (!P3_EXP || j.pieces <= 1) {
      atomicAdd(L.bytes + 0, (j.bf16 || j.pb16 ? 2ull : 4ull) * j.len * (j.n - 1));  // pushes received
      atomicAdd(L.bytes + 1, (j.pb16 ? 2ull : 4ull) * j.len * (j.n - 1));  // broadcasts sent
    }
    if (L.trace_cap)
      for (uint32_t i = 0; i < j.run; ++i)
        trace_append(L, a.k, j.layer, j.g + i - P.layer_first[j.layer], a.trace_cta ? blockIdx.x : j.rank, P3_EV_BCAST);
  }
}

// Next stashed claim (one warp; the stash is in layer order).
__device__ uint32_t take_stash(Stash* st, Popped* out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t g = st->g[0];
  out->run = st->run[0];
  out->layer = st->layer[0];
  out->word = st->word[0];
  out->t0 = st->t0[0];
  __syncwarp();
  if (lane == 0) {
    for (uint32_t i = 1; i < st->n; ++i) {
      st->g[i - 1] = st->g[i];
      st->run[i - 1] = st->run[i];
      st->layer[i - 1] = st->layer[i];
      st->word[i - 1] = st->word[i];
      st->t0[i - 1] = st->t0[i];
    }
    st->n -= 1;
  }
  __syncwarp();
  return g;
}

// Notify mode, owner side: claim the next PULL request of this rank's pull ring (one warp;
// lane 0 decides). Returns the slice and the requester, or P3_NONE.
__device__ P3_COLD uint32_t warp_answer_pick(const CommArgs& a, const LocalDev& L, uint32_t* layer, uint32_t* requester) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t g = P3_NONE, q = 0;
  if (lane == 0) {
    const uint32_t o = L.rank;
    const uint32_t h = ld_relaxed_gpu(L.pull_head), t = ld_relaxed_sys(a.peers.pull_tail[o]);
    if ((int32_t)(t - h) > 0 && atomicCAS(L.pull_head, h, h + 1) == h) {
      const volatile unsigned long long* e = a.peers.pull_ring[o] + h % a.pull_cap;
      unsigned long long v = *e;
      const uint64_t t0 = globaltimer();
      while ((uint32_t)(v >> 40) != ((a.k + 1) & 0xffffffu)) {  // reserved, entry still on its way
        if (globaltimer() - t0 > a.timeout_ns) break;
        __nanosleep(64);
        v = *e;
      }
      fence_acq_rel_sys();  // acquire: the request came after the NOTIFY of the updated slice
      q = (uint32_t)(v >> 32) & 0xffu;
      g = (uint32_t)v;
    }
  }
  g = __shfl_sync(FULL_MASK, g, 0);
  q = __shfl_sync(FULL_MASK, q, 0);
  if (g != P3_NONE) {
    *layer = a.plan.slice_layer[g];
    *requester = q;
  }
  return g;
}

// Notify mode, worker side: turn the next NOTIFY of this rank into a PULL request queued at
// the slice's owner (worker.py:226-239). Returns whether one was sent.
__device__ P3_COLD bool warp_issue_pull(const CommArgs& a, const LocalDev& L) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t sent = 0;
  if (lane == 0) {
    const uint32_t r = L.rank;
    const uint32_t h = ld_relaxed_gpu(L.ntf_head), t = ld_relaxed_sys(a.peers.ntf_tail[r]);
    if ((int32_t)(t - h) > 0 && atomicCAS(L.ntf_head, h, h + 1) == h) {
      const volatile unsigned long long* e = a.peers.ntf_ring[r] + h % a.ntf_cap;
      unsigned long long v = *e;
      const uint64_t t0 = globaltimer();
      while ((uint32_t)(v >> 32) != a.k + 1) {
        if (globaltimer() - t0 > a.timeout_ns) break;
        __nanosleep(64);
        v = *e;
      }
      const uint32_t g = (uint32_t)v;
      const uint32_t o = a.plan.slice_owner[g];
      const uint32_t pos = atom_add_relaxed_sys(a.peers.pull_tail[o], 1u);
      *(volatile unsigned long long*)(a.peers.pull_ring[o] + pos % a.pull_cap) =
          ((unsigned long long)((a.k + 1) & 0xffffffu) << 40) | ((unsigned long long)r << 32) | g;
      atomicAdd(L.pcount, 1u);
      const uint32_t l = a.plan.slice_layer[g];
      if (L.trace_cap) trace_append(L, a.k, l, g - a.plan.layer_first[l], o, P3_EV_PULL);
      sent = 1;
    }
  }
  return __shfl_sync(FULL_MASK, sent, 0) != 0;
}

// Broadcast-pull mode (notify 2), worker side: take the next NOTIFY of this rank; the
// scheduler turns it into a fetch of the owner's updated slice (one NVLink read, no request).
__device__ P3_COLD uint32_t warp_take_notify(const CommArgs& a, const LocalDev& L, uint32_t* layer) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t g = P3_NONE;
  if (lane == 0) {
    const uint32_t r = L.rank;
    const uint32_t h = ld_relaxed_gpu(L.ntf_head), t = ld_relaxed_sys(a.peers.ntf_tail[r]);
    if ((int32_t)(t - h) > 0 && atomicCAS(L.ntf_head, h, h + 1) == h) {
      const volatile unsigned long long* e = a.peers.ntf_ring[r] + h % a.ntf_cap;
      unsigned long long v = *e;
      const uint64_t t0 = globaltimer();
      while ((uint32_t)(v >> 32) != a.k + 1) {  // reserved, entry still on its way
        if (globaltimer() - t0 > a.timeout_ns) break;
        __nanosleep(64);
        v = *e;
      }
      fence_acq_rel_sys();  // acquire: the owner's replica stores came before its NOTIFY
      g = (uint32_t)v;
      if (L.trace_cap) {
        const uint32_t l = a.plan.slice_layer[g];
        trace_append(L, a.k, l, g - a.plan.layer_first[l], a.plan.slice_owner[g], P3_EV_PULL);
      }
    }
  }
  g = __shfl_sync(FULL_MASK, g, 0);
  if (g != P3_NONE) *layer = a.plan.slice_layer[g];
  return g;
}

// Notify mode: the answer to a PULL — the owner's updated slice copied into the requester's
// replica (a push-shaped job: TMA-staged, bulk-stored over NVLink).
// Broadcast pull (fetch = true): the same copy run by the requester q itself, from the owner's
// replica into its own.
__device__ P3_COLD void prepare_answer(const CommArgs& a, uint32_t li, uint32_t g, uint32_t l, uint32_t q, Job* job,
                                       bool fetch = false) {
  const PlanDev& P = a.plan;
  const LocalDev& L = a.loc[li];
  if ((threadIdx.x & 31) == 0) {
    const uint64_t woff = P.layer_woff[l] + P.slice_off[g];
    const uint32_t from = fetch ? P.slice_owner[g] : L.rank;
    job->kind = JOB_PUSH;
    job->answer = fetch ? 2u : 1u;
    job->pb16 = 0;
    job->ndst = 1;
    job->run = 1;
    job->n = 1;
    job->li = li;
    job->g = g;
    job->layer = l;
    job->rank = q;
    job->len = P.slice_len[g];
    if (a.pb16) {  // bf16 replicas: a 2-byte copy
      job->bf16 = 2;
      job->src[0] = reinterpret_cast<const float*>(reinterpret_cast<const __nv_bfloat16*>(a.peers.W[from]) + woff);
      job->dst[0] = reinterpret_cast<float*>(reinterpret_cast<__nv_bfloat16*>(a.peers.W[q]) + woff);
    } else {
      job->bf16 = 0;
      job->src[0] = a.peers.W[from] + woff;
      job->dst[0] = a.peers.W[q] + woff;
    }
  }
}

// Comm kernel. Warp 0 of every CTA is the scheduler, warp 1 the signaler, warp 2 the TMA
// producer, warps 3.. the consumers; two job slots and a 3-stage ring in shared memory. At
// N > 1 (k_comm<false>) each job slot has its own signaler: warps 1 and 3, consumers from 4.
//   scheduler: pick the next job — server work first (a reduced slice unblocks the next
//   forward pass), then the most urgent published slice of the local worker queues — and
//   prepare its pointers while the previous job is still moving;
//   producer: cut the job into tiles and stream its sources into the ring (cp.async.bulk),
//   running ahead into the next job;
//   consumers: compute / store each staged tile (push tiles leave as TMA bulk stores);
//   signaler: once a job's last tile is done, fence and publish the completion
//   (arrival / done counters), then release the slot to the scheduler.
// The queue is re-read for every pick, so a layer published while the kernel runs
// preempts less urgent slices at slice granularity. DRAIN launches (one per published
// batch of layers) exit as soon as nothing is available: a kernel spinning on unpublished
// gradients would hold SMs that the compute producing them may need (co-residency-bound
// library kernels, lazy module loading). The FINISH launch of an iteration ends once every
// local slice is pushed and every owned slice reduced; it waits only for peers' pushes.
// ONE: the single-rank instantiation (no peers, no server role, fp32 replicas): the N>1,
// notify and bf16-replica paths are compiled out, so the scheduler and movers run a smaller
// kernel (measured: the general kernel is ~5% slower at N=1 than this one).
template <bool ONE>
__global__ void __launch_bounds__(P3_COMM_MAX_THREADS, 1) k_comm(const __grid_constant__ CommArgs a) {
  __shared__ Job slots[P3_SLOTS];  // a ring: the scheduler fills ahead while earlier jobs move
  __shared__ StageDesc sdesc[P3_STAGES];
  __shared__ __align__(8) uint64_t full_bar[P3_STAGES], empty_bar[P3_STAGES];
  __shared__ RangePtrs rptrs;
  extern __shared__ __align__(128) uint8_t stage_mem[];  // P3_STAGES x P3_STAGE_BYTES
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nthr = blockDim.x;
  // NSIG signaler warps: with one per job slot, slot b's jobs are signalled by their own warp
  // (1, then 3, 4, ...), so a slow system-scope release of one job does not hold back the next
  // job's slot (measured at N=2: ResNet-50 sync -8%)
  constexpr uint32_t NSIG = ONE ? 1u : P3_NSIG;
  static_assert(NSIG == 1 || NSIG == P3_SLOTS, "signalers: one, or one per job slot");
  const uint32_t cw = 2 + NSIG;          // first consumer warp
  const uint32_t ncons = nthr - 32 * cw;  // consumer threads
  IterState* stats = a.loc[0].it;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < P3_STAGES; ++i) {
      mbar_init(&full_bar[i], 1);              // the producer's arrive (+ the tile bytes)
      mbar_init(&empty_bar[i], ncons / 32);    // one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (a.trace_cta && threadIdx.x == 0)  // diagnostics: CTA start (event 16)
    trace_append(a.loc[0], a.k, 0, 0, blockIdx.x, 16);
  if (warp == 0) {
    uint32_t* phase = (lane == 0 && blockIdx.x < P3_DBG_CTAS) ? a.loc[0].cta_phase + blockIdx.x : nullptr;
    const uint64_t t0 = globaltimer();
    uint64_t t_pick = 0, t_wait = 0;
    uint32_t backoff = 0, b = 0;
    uint64_t idle_since = 0;  // DRAIN linger start (lane 0)
    __shared__ Stash stash;   // slices claimed by this CTA's scheduler, not yet dispatched
    __shared__ uint32_t stash_li;
    if (lane == 0) stash.n = 0;
    __syncwarp();
    bool pending[P3_SLOTS];
#pragma unroll
    for (uint32_t i = 0; i < P3_SLOTS; ++i) pending[i] = false;
    bool pops_done = false;  // FINISH, N > 1: every local slice claimed (see the pop phase)
    bool last_push = false;  // the most recently filled slot holds a push
    for (uint32_t iter = 0;; ++iter) {
      if (phase) *(volatile uint32_t*)phase = (a.k << 24) | (1u << 20) | (iter & 0xfffff);
      const uint64_t tp = stat_clock();
      uint32_t kind = JOB_NONE, li = 0, g = P3_NONE;
      Popped pp;
      pp.run = 1;
      pp.piece = 0;
      pp.layer = 0;
      pp.word = 0;
      pp.t0 = 0;
      if (ONE || a.plan.world == 1) {
        // single rank: a popped slice is complete the moment it is popped (the owner's own
        // contribution is read in place), so the pop claims the reduction directly — no
        // arrival counting, no server role — and takes up to pop_run consecutive slices of
        // the layer (contiguous in memory) as one job
        const LocalDev& L = a.loc[0];
        if (stash.n) {
          g = take_stash(&stash, &pp);
        } else {
          g = warp_pop(queue_of(a, L), a.k + 1, phase, (L.V || L.M) ? 1u : a.pop_run, &pp, &stash);
        }
        if (g != P3_NONE) {
          if (lane == 0) {
            // (the acquire of the publication word is the fence in prepare_reduce)
            atomicAdd(&L.it->pushed, pp.run);
            atomicAdd(&L.it->reduced, pp.run);
            if (L.trace_cap)
              for (uint32_t i = 0; i < pp.run; ++i)
                trace_append(L, a.k, pp.layer, g + i - a.plan.layer_first[pp.layer], a.trace_cta ? blockIdx.x : L.rank,
                             P3_EV_PUSH, pp.t0);
          }
          kind = JOB_REDUCE;
        }
      }
      // Server work (reduce + broadcast of a completed owned slice) and worker pushes both
      // progress, like the reference's server and sender threads: `push_split` > 0 makes
      // every push_split-th CTA look for pushes first, the others for server work first.
      const bool push_first = a.push_split && (blockIdx.x % a.push_split) == a.push_split - 1;
      // push_ctas: split roles (FINISH) — the first push_ctas CTAs only push, the rest only reduce
      const bool split = P3_EXP && a.push_ctas && a.mode == P3_COMM_FINISH;
      const bool push_only = split && blockIdx.x < a.push_ctas, srv_only = split && blockIdx.x >= a.push_ctas;
      if (!ONE && P3_EXP && a.lazy_pick && pops_done) {
        // late binding: a job picked now would wait behind the one moving; with no pushes left,
        // leave it to an idle CTA unless this one's movers are done too
        const uint32_t pb = (b + P3_SLOTS - 1) % P3_SLOTS;
        if (pending[pb]) {
          bar_sync(BAR_EMPTY(pb), 64);
          pending[pb] = false;
        }
      }
      uint32_t ans_q = 0;
      bool pulled = false, was_capped = false, token = false;
      for (uint32_t round = 0; round < 2 && kind == JOB_NONE && !ONE && a.plan.world > 1; ++round) {
        if ((round == 0) != push_first) {
          for (uint32_t t = 0; t < a.n_local && kind == JOB_NONE && !push_only; ++t) {
            li = (blockIdx.x + t) % a.n_local;
            g = warp_server_pick(a, a.loc[li], &pp.layer, phase, &pp.piece);
            if (g != P3_NONE) kind = JOB_REDUCE;
          }
          for (uint32_t t = 0; t < a.n_local && kind == JOB_NONE && a.notify == 1; ++t) {
            li = (blockIdx.x + t) % a.n_local;
            g = warp_answer_pick(a, a.loc[li], &pp.layer, &ans_q);
            if (g != P3_NONE) kind = JOB_ANSWER;
          }
          for (uint32_t t = 0; t < a.n_local && kind == JOB_NONE && P3_EXP && a.notify == 2; ++t) {
            li = (blockIdx.x + t) % a.n_local;
            g = warp_take_notify(a, a.loc[li], &pp.layer);
            if (g != P3_NONE) kind = JOB_FETCH;
          }
        } else {
          // server-reserved CTAs (srv_reserve > 0: every srv_reserve-th CTA) never take pushes,
          // so a completed slice is reduced while the other CTAs' pipelines hold pushes
          const bool reserved = srv_only || (a.srv_reserve && (blockIdx.x % a.srv_reserve) == 0) ||
                                (a.push_max == 1 && a.mode == P3_COMM_FINISH && last_push && backoff < 512u &&
                                 pending[(b + P3_SLOTS - 1) % P3_SLOTS]);  // (an idle scheduler pushes anyway)
          // push_cap: a pop takes one of push_cap tokens of the rank (returned by the push's
          // signal, or at once when the pop yields no remote push), so the first pushes
          // complete (and their reductions start) early instead of every CTA's pushes sharing
          // the link at once
          bool capped = false;
          if (P3_EXP && a.push_cap && (stash.n || (!pops_done && !reserved))) {
            uint32_t ok = 0;
            if (lane == 0) {
              ok = atomicAdd(&a.loc[0].it->push_live, 1u) < a.push_cap;
              if (!ok) atomicSub(&a.loc[0].it->push_live, 1u);
            }
            token = __shfl_sync(FULL_MASK, ok, 0) != 0;
            capped = was_capped = !token;
          }
          if (stash.n && !capped) {
            li = stash_li;
            g = take_stash(&stash, &pp);
            if (lane == 0) atomicAdd(&a.loc[li].it->pushed, 1u);
            kind = JOB_PUSH;
          }
          for (uint32_t t = 0; t < a.n_local && kind == JOB_NONE && !pops_done && !reserved && !capped && !stash.n; ++t) {
            li = (blockIdx.x + t) % a.n_local;
            g = warp_pop(queue_of(a, a.loc[li]), a.k + 1, phase, 1u, &pp, &stash);
            if (lane == 0) stash_li = li;
            __syncwarp();
            if (g != P3_NONE) {
              if (lane == 0) atomicAdd(&a.loc[li].it->pushed, 1u);
              kind = JOB_PUSH;
            }
          }
          if (token && kind != JOB_PUSH) {  // nothing popped: give the token back
            if (lane == 0) atomicSub(&a.loc[0].it->push_live, 1u);
            token = false;
          }
          // notify mode: PULLs wait behind the pushes (the baseline's per-server FIFO outbox)
          for (uint32_t t = 0; t < a.n_local && kind == JOB_NONE && a.notify == 1; ++t)
            pulled |= warp_issue_pull(a, a.loc[(blockIdx.x + t) % a.n_local]);
          if (kind == JOB_NONE && !pops_done && a.mode == P3_COMM_FINISH) {
            // FINISH runs after every publication of the iteration: once every local slice
            // is claimed there is nothing left to pop — idle picks then only poll the server
            // gate (one round trip), so they can poll often
            uint32_t all = 1;
            if (lane == 0)
              for (uint32_t t = 0; t < a.n_local; ++t)
                all &= ld_relaxed_gpu(&a.loc[t].it->pushed) >= a.plan.total_slices;
            pops_done = __shfl_sync(FULL_MASK, all, 0) != 0;
          }
        }
      }
      if (!ONE && kind == JOB_NONE && pulled) continue;  // progress (requests sent): look again at once
      if (kind == JOB_NONE) {
        // decided by lane 0 and broadcast: a per-lane decision could split the warp
        uint32_t verdict = 0;  // 0 keep looking, 1 leave, 2 timed out
        if (lane == 0) {
          if (a.mode == P3_COMM_DRAIN && ONE) {
            verdict = 1;  // single rank: nothing arrives from peers
          } else if (a.mode == P3_COMM_DRAIN) {
            // Nothing to do. Linger (bounded) while some owned slice has part of its pushes:
            // the rest come from peers' comm kernels, never from this rank's compute, and
            // reducing it now keeps it off the post-backward tail.
            bool partial = false;
            for (uint32_t t = 0; t < a.n_local && !partial; ++t) {
              const uint32_t o = a.loc[t].rank, ot = a.plan.own_total[o], N = a.plan.world;
              const uint32_t arrived = ld_relaxed_sys(a.peers.tally[o]) - a.k * N * ot;
              const uint32_t completed = ld_relaxed_sys(a.peers.tally[o] + 1) - a.k * ot;
              partial = (int32_t)(arrived - N * completed) > 0;
            }
            if (!partial || idle_since == 0 || globaltimer() - idle_since > a.linger_ns) verdict = 1;
            if (idle_since == 0) idle_since = globaltimer();
          } else {
            bool fin = true;
            for (uint32_t t = 0; t < a.n_local; ++t) {
              const LocalDev& L = a.loc[t];
              const uint32_t own = a.plan.own_total[L.rank];
              fin = fin && ld_relaxed_gpu(&L.it->pushed) >= a.plan.total_slices &&
                    ld_relaxed_gpu(&L.it->reduced) >= own;
              if (!ONE && a.notify == 1)  // every NOTIFY pulled, every PULL of an owned slice answered
                fin = fin && ld_relaxed_gpu(L.pcount) >= a.plan.total_slices - own &&
                      ld_relaxed_gpu(L.pcount + 1) >= own * (a.plan.world - 1);
              if (!ONE && P3_EXP && a.notify == 2)  // every other owner's slice fetched
                fin = fin && ld_relaxed_gpu(L.pcount + 1) >= a.plan.total_slices - own;
            }
            verdict = (fin || ld_relaxed_gpu(a.err) != 0) ? 1u : (globaltimer() - t0 > a.timeout_ns ? 2u : 0u);
          }
          if (verdict == 2 && atomicCAS(a.err, 0u, (uint32_t)P3_ETIMEOUT) == 0u) {
            // diagnostics for the host (p3_sync_all), then release every forward gate of
            // the local ranks so the compute streams drain
            a.err[1] = a.k;
            for (uint32_t t = 0; t < a.n_local; ++t) {
              a.err[2 + 2 * t] = ld_relaxed_gpu(&a.loc[t].it->pushed);
              a.err[3 + 2 * t] = ld_relaxed_gpu(&a.loc[t].it->reduced);
            }
            for (uint32_t t = 0; t < a.n_local; ++t)
              for (uint32_t l = 0; l < a.plan.n_layers; ++l) {
                atomicAdd(a.peers.done[a.loc[t].rank] + l, 0x40000000u);
                atomicAdd(a.peers.gdone[a.loc[t].rank] + a.plan.layer_group[l], 0x40000000u);
              }
          }
        }
        verdict = __shfl_sync(FULL_MASK, verdict, 0);
        if (verdict == 0) {
          // FINISH runs after the iteration's last publication: what it waits for is near
          // (the ingest of the ring, a peer's push), so it polls at most every 0.5 us; a DRAIN
          // launch may wait for the backward pass and backs off up to 4 us
          backoff = min(2u * backoff + 64u, (a.mode == P3_COMM_FINISH || pops_done || was_capped) ? 512u : 4096u);
          __nanosleep(backoff);
          continue;
        }
        kind = JOB_EXIT;
      }
      backoff = 0;
      idle_since = 0;
      if (lane == 0 && (kind == JOB_PUSH || kind == JOB_REDUCE)) {
        P3_CHECK(g < a.plan.total_slices && pp.layer < a.plan.n_layers);
        P3_CHECK(a.plan.slice_layer[g] == pp.layer);  // the pop's layer is the slice's layer
        P3_CHECK(pp.run >= 1 && g + pp.run <= a.plan.layer_first[pp.layer] + a.plan.layer_nslices[pp.layer]);
        P3_CHECK(kind == JOB_PUSH || a.plan.slice_owner[g] == a.loc[li].rank);  // reduce only what it owns
      }
      if (kind == JOB_PUSH) {
        const uint32_t how = prepare_push(a, li, g, pp.layer, pp.word, nullptr, pp.t0);
        if (token && how != PUSH_REMOTE && lane == 0) atomicSub(&a.loc[0].it->push_live, 1u);  // (no link use)
        if (how == PUSH_DONE) continue;  // own slice, still waiting for peers: counted in place
        if (how == PUSH_REDUCE) kind = JOB_REDUCE;  // own slice completed it: reduce right away
      }
      if (!ONE && (kind == JOB_PUSH || kind == JOB_REDUCE || kind == JOB_ANSWER || kind == JOB_FETCH) && a.ns_per_byte != 0.f &&
          a.plan.world > 1) {
        // egress bytes of this job on the rank's link (K7): a push, an answer to a PULL, or the
        // N-1 broadcast copies of a reduce (none in notify mode: the peers pull)
        const bool two = a.pb16 || (kind == JOB_PUSH && a.push_bf16);  // 2-byte elements on the link
        const uint64_t bytes = (two ? 2ull : 4ull) * a.plan.slice_len[g] *
                               (kind == JOB_REDUCE ? (a.notify ? 0u : a.plan.world - 1u) : 1u);
        if (lane == 0) pace(a, a.loc[li], bytes);
        __syncwarp();
      }
      const uint64_t tw = stat_clock();
      t_pick += tw - tp;
      if (pending[b]) bar_sync(BAR_EMPTY(b), 64);  // the signaler released this slot
      if (kind == JOB_PUSH) {
        prepare_push(a, li, g, pp.layer, pp.word, &slots[b]);
      } else if (kind == JOB_ANSWER) {
        prepare_answer(a, li, g, pp.layer, ans_q, &slots[b]);
      } else if (kind == JOB_FETCH) {
        prepare_answer(a, li, g, pp.layer, a.loc[li].rank, &slots[b], true);
      } else if (kind == JOB_REDUCE) {
        prepare_reduce(a, li, g, pp.layer, pp.word, &slots[b], pp.run, pp.piece);
      } else {
        for (uint32_t i = 1; i < P3_SLOTS; ++i) {  // leave every barrier balanced
          const uint32_t bi = (b + i) % P3_SLOTS;
          if (pending[bi]) bar_sync(BAR_EMPTY(bi), 64);
        }
        if (lane == 0) slots[b].kind = JOB_EXIT;
      }
      t_wait += stat_clock() - tw;
      __syncwarp();
      bar_arrive(BAR_FULL(b), 96);  // producer + signaler wait on it
      if (kind == JOB_EXIT) {
        for (uint32_t i = 1; NSIG > 1 && i < P3_SLOTS; ++i) {  // every slot's signaler leaves
          const uint32_t bi = (b + i) % P3_SLOTS;  // (empty: synced above)
          if (lane == 0) slots[bi].kind = JOB_EXIT;
          __syncwarp();
          bar_arrive(BAR_FULL(bi), 96);
        }
        break;
      }
      pending[b] = true;
      last_push = kind == JOB_PUSH || kind == JOB_ANSWER || kind == JOB_FETCH;
      b = (b + 1) % P3_SLOTS;
      if (lane == 0) atomicAdd(&stats->jobs, 1u);
    }
    if (lane == 0) {
      atomicAdd(&stats->t_pick, (unsigned long long)t_pick);
      atomicAdd(&stats->t_slot_wait, (unsigned long long)t_wait);
      if (a.mode == P3_COMM_FINISH) atomicAdd(&stats->exited, 1u);
    }
    if (phase) *(volatile uint32_t*)phase = (a.k << 24) | (5u << 20);
    if (a.trace_cta && lane == 0) trace_append(a.loc[0], a.k, 0, 0, blockIdx.x, 17);  // diagnostics: scheduler exit
  } else if (warp == 1 || (warp >= 3 && warp < 2 + NSIG)) {
    // signaler: in job order, once the consumers are done with a job, fence and publish
    uint64_t t_sig = 0;
    for (uint32_t b = warp == 1 ? 0u : warp - 2;; b = (b + NSIG) % P3_SLOTS) {
      bar_sync(BAR_FULL(b), 96);
      const Job& j = slots[b];
      if (j.kind == JOB_EXIT) break;
      bar_sync(BAR_DONE(b), ncons + 32);
      Job mine;  // what the signal needs, so the slot can be refilled right away
      mine.kind = j.kind;
      mine.li = j.li;
      mine.g = j.g;
      mine.layer = j.layer;
      mine.opos = j.opos;
      mine.rank = j.rank;
      mine.len = j.len;
      mine.n = j.n;
      mine.run = j.run;
      mine.bf16 = j.bf16;
      mine.ndst = j.ndst;
      mine.answer = j.answer;
      mine.pb16 = j.pb16;
      mine.pieces = j.pieces;
      // push_cap: the token goes back once the data has moved (before the signal's fence)
      if (P3_EXP && a.push_cap && lane == 0 && mine.kind == JOB_PUSH && !mine.answer)
        atomicSub(&a.loc[0].it->push_live, 1u);
      __syncwarp();
      bar_arrive(BAR_EMPTY(b), 64);
      if (lane == 0) {
        const uint64_t ts = stat_clock();
        if (ONE) {  // single rank: the update is in the replica; open its gate
          const PlanDev& P = a.plan;
          const LocalDev& L = a.loc[0];
          fence_acq_rel_gpu();
          red_add_relaxed_sys(a.peers.done[L.rank] + mine.layer, mine.run);
          red_add_relaxed_sys(a.peers.gdone[L.rank] + P.layer_group[mine.layer], mine.run);
          if (L.trace_cap)
            for (uint32_t i = 0; i < mine.run; ++i)
              trace_append(L, a.k, mine.layer, mine.g + i - P.layer_first[mine.layer], L.rank, P3_EV_BCAST);
        } else {
          signal_job(a, mine);
        }
        t_sig += stat_clock() - ts;
      }
      __syncwarp();
    }
    if (lane == 0) atomicAdd(&stats->t_signal, (unsigned long long)t_sig);
  } else if (warp == 2) {
    // producer: cut each job into stage tiles and stream them in with TMA bulk copies
    uint32_t it = 0;  // stages issued (ring position and phase)
    auto next_stage = [&](uint32_t& sidx) {
      sidx = it % P3_STAGES;
      if (it >= P3_STAGES) mbar_wait_bounded(&empty_bar[sidx], ((it / P3_STAGES) - 1) & 1u, a);
      ++it;
    };
    for (uint32_t b = 0;; b = (b + 1) % P3_SLOTS) {
      bar_sync(BAR_FULL(b), 96);
      const Job& j = slots[b];
      if (lane == 0) {
        uint32_t sidx;
        if (j.kind == JOB_EXIT) {
          next_stage(sidx);
          sdesc[sidx].flags = ST_EXIT;
          mbar_arrive(&full_bar[sidx]);
        } else {
          // the job's sources were published to this CTA through generic-proxy acquires
          // (scheduler); order them before the async-proxy (TMA) reads
          asm volatile("fence.proxy.async.global;" ::: "memory");
          const uint32_t len = j.len;
          const bool tma = a.use_tma && job_tma_ok(j);
          const uint32_t tile = job_tile(j), main = tma ? (len & ~7u) : 0u;
          const uint32_t nsrc = job_sources(j);
          P3_CHECK(j.n >= 1 && j.n <= P3_MAX_RANKS && len > 0);
          for (uint32_t e0 = 0; e0 < main; e0 += tile) {
            const uint32_t n = min(tile, main - e0);
            P3_CHECK(n > 0 && n <= tile && (n & 7u) == 0);
            next_stage(sidx);
            StageDesc& d = sdesc[sidx];
            d.b = b;
            d.e0 = e0;
            d.n = n;
            d.tile = tile;
            d.flags = (e0 + n == len) ? ST_LAST : 0u;
            uint8_t* st = stage_mem + (size_t)sidx * P3_STAGE_BYTES;
            uint32_t bytes = 0;
            for (uint32_t q = 0; q < nsrc; ++q) {
              const bool half = j.kind == JOB_PUSH ? j.bf16 == 2
                                                   : q < j.n && (j.pb16 || (j.bf16 && (int)q != (int)j.bf16 - 1));
              bytes += n * (half ? 2u : 4u);
            }
            mbar_arrive_expect_tx(&full_bar[sidx], bytes);
            for (uint32_t q = 0; q < nsrc; ++q) {
              const void* g;
              uint32_t esz = 4;
              if (j.kind == JOB_PUSH) {
                esz = j.bf16 == 2 ? 2u : 4u;  // (2: a bf16 copy)
                g = j.bf16 == 2 ? (const void*)(reinterpret_cast<const __nv_bfloat16*>(j.src[0]) + e0)
                                : (const void*)(j.src[0] + e0);
              } else if (q < j.n) {
                const bool half = j.pb16 || (j.bf16 && (int)q != (int)j.bf16 - 1);
                esz = half ? 2u : 4u;
                g = half ? (const void*)(reinterpret_cast<const __nv_bfloat16*>(j.src[q]) + e0)
                         : (const void*)(j.src[q] + e0);
              } else if (q == j.n) {
                g = (j.pb16 || j.mc) ? j.m + e0 : j.dst[0] + e0;  // master copy p
              } else {
                g = j.v + e0;
              }
              tma_load_1d(st + q * tile * 4, g, n * esz, &full_bar[sidx]);
            }
          }
          if (main < len) {  // unaligned job or the residue: consumers read global memory
            next_stage(sidx);
            StageDesc& d = sdesc[sidx];
            d.b = b;
            d.e0 = main;
            d.n = len - main;
            d.tile = 0;
            d.flags = ST_LAST | ST_DIRECT;
            mbar_arrive(&full_bar[sidx]);
          }
        }
      }
      __syncwarp();
      if (j.kind == JOB_EXIT) {
        for (uint32_t i = 1; NSIG > 1 && i < P3_SLOTS; ++i) bar_sync(BAR_FULL((b + i) % P3_SLOTS), 96);
        break;
      }
    }
  } else {
    // consumers: compute each stage from shared memory, release it, report finished jobs.
    // A stage that leaves by TMA bulk store is released once the engine has read it; with
    // P3_EXP the first consumer warp defers that wait to the next bulk stage (all groups but
    // the newest), so the next tile computes while the store drains (measured: helps only the
    // TMA-stored reduce variants, ~1% slower in the default configuration).
    const uint32_t tid = threadIdx.x - 32 * cw;
    const bool w0 = warp == cw;  // the first consumer warp (tid 0 issues the bulk stores)
    uint32_t pend = P3_NONE;    // (w0) stage whose release waits for its bulk store's read
    // (P3_EXP, w0) job slot of a push whose completion wait — and w0's DONE arrival — moved to
    // w0's next stage, so the next job's stores start while this one's drain
    uint32_t done_pend = P3_NONE;
    uint64_t t_move = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t sidx = it % P3_STAGES;
      if (P3_EXP && w0 && done_pend != P3_NONE) {
        // no next stage soon (e.g. the scheduler waits for work that this push's signal
        // unblocks): complete the push now
        const uint64_t tw = globaltimer();
        bool ready = false;
        while (!(ready = mbar_try_wait(&full_bar[sidx], (it / P3_STAGES) & 1u)) && globaltimer() - tw < 2000) {
        }
        if (!ready) {
          if (lane == 0) tma_store_wait_all();
          __syncwarp();
          bar_arrive(BAR_DONE(done_pend), ncons + 32);
          done_pend = P3_NONE;
        }
      }
      mbar_wait_bounded(&full_bar[sidx], (it / P3_STAGES) & 1u, a);
      const StageDesc d = sdesc[sidx];
      if (d.flags & ST_EXIT) {
        if (P3_EXP && w0 && done_pend != P3_NONE) {
          if (lane == 0) tma_store_wait_all();
          __syncwarp();
          bar_arrive(BAR_DONE(done_pend), ncons + 32);
        }
        if (w0 && pend != P3_NONE) {
          if (lane == 0) tma_store_wait_read();
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[pend]);
        }
        break;
      }
      P3_CHECK(d.b < P3_SLOTS);
      const uint64_t tm = tid == 0 ? stat_clock() : 0;
      const Job& j = slots[d.b];
      if (P3_TRACE && a.trace_cta && tid == 0 && d.e0 == 0)  // diagnostics: a job's first stage (18)
        trace_append(a.loc[j.li], a.k, j.layer, j.g - a.plan.layer_first[j.layer], blockIdx.x, 18, j.kind);
      const bool bulk_push = a.tma_store && j.kind == JOB_PUSH && j.bf16 != 1 && !(d.flags & ST_DIRECT);
      bool bulk = false;  // this stage leaves by TMA bulk store (one group)
      if (bulk_push) {
        // the staged gradient tile goes out as one TMA bulk store (over NVLink to the
        // owner's receive slot)
        if (tid == 0) {
          if (j.bf16 == 2)  // bf16 copy (param_bf16 push / answer)
            tma_store_1d_nc(reinterpret_cast<__nv_bfloat16*>(j.dst[0]) + d.e0,
                            stage_mem + (size_t)sidx * P3_STAGE_BYTES, d.n * 2u);
          else
            tma_store_1d_nc(j.dst[0] + d.e0, stage_mem + (size_t)sidx * P3_STAGE_BYTES, d.n * 4u);
          bulk_commit();
        }
        bulk = true;
      } else if (d.flags & ST_DIRECT) {
        move_range(a, j, d.e0, d.n, &rptrs, tid, ncons);
      } else if (!ONE && a.tma_store_red && j.kind == JOB_REDUCE && j.n <= 8 && !j.pb16 && j.bf16 == 0 &&
                 (a.tma_store_red == 1 || j.ndst > 1)) {
        // results go back into the stage, then TMA bulk stores: every replica and the momentum
        // (tma_store_red 1), or only the remote replicas over NVLink while the consumers store
        // the local one (2)
        uint8_t* st = stage_mem + (size_t)sidx * P3_STAGE_BYTES;
        const int mode = (int)a.tma_store_red;
        consume_tile<ONE>(a, j, d, st, tid, ncons, mode);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_sync(BAR_RANGE, ncons);
        if (tid == 0) {
          const uint32_t pitch = d.tile * 4;
          for (uint32_t q = mode == 2 ? 1u : 0u; q < j.ndst; ++q) tma_store_1d_nc(j.dst[q] + d.e0, st + j.n * pitch, d.n * 4u);
          if (j.v && mode == 1) tma_store_1d_nc(j.v + d.e0, st + (j.n + 1) * pitch, d.n * 4u);
          bulk_commit();
        }
        bulk = true;
      } else {
        consume_tile<ONE>(a, j, d, stage_mem + (size_t)sidx * P3_STAGE_BYTES, tid, ncons);
      }
      const bool last = (d.flags & ST_LAST) != 0;
      const bool defer_done = P3_EXP && last && bulk_push;
      if (!P3_EXP && bulk && !last && tid == 0) tma_store_wait_read();  // (default: release at once)
      if (last && tid == 0 && (a.tma_store || a.tma_store_red)) {
        if (defer_done) tma_store_wait_read();  // (completion: at w0's next stage)
        else tma_store_wait_all();  // every bulk store of the job complete before its signal
      }
      __syncwarp();
      if (P3_EXP && w0 && done_pend != P3_NONE) {  // the previous push: complete, then DONE
        if (lane == 0) {
          if (bulk) asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");  // all but this stage's
          else tma_store_wait_all();
        }
        __syncwarp();
        bar_arrive(BAR_DONE(done_pend), ncons + 32);
        done_pend = P3_NONE;
      }
      if (P3_EXP && w0 && bulk && !last) {  // release the previous deferred stage, defer this one
        if (pend != P3_NONE) {
          if (lane == 0) tma_store_wait_read_all_but_one();
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[pend]);
        }
        pend = sidx;
      } else {
        if (w0 && pend != P3_NONE) {
          if (lane == 0 && !last) tma_store_wait_read();  // (at a job end the wait above covered it)
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[pend]);
          pend = P3_NONE;
        }
        if (lane == 0) mbar_arrive(&empty_bar[sidx]);
      }
      if (tid == 0) t_move += stat_clock() - tm;
      if (P3_TRACE && a.trace_cta && tid == 0 && (d.flags & ST_LAST))  // ... and its last one done (19)
        trace_append(a.loc[j.li], a.k, j.layer, j.g - a.plan.layer_first[j.layer], blockIdx.x, 19, j.kind);
      if (d.flags & ST_LAST) {
        if (P3_EXP && w0 && defer_done) done_pend = d.b;
        else bar_arrive(BAR_DONE(d.b), ncons + 32);
      }
    }
    if (tid == 0) atomicAdd(&stats->t_move, (unsigned long long)t_move);
  }
}

// p3_trace_mark: one stream-ordered trace record (iteration start / synced) on the device clock.
__global__ void k_mark(const LocalDev L, uint32_t k, uint32_t ev) {
  if (threadIdx.x == 0) trace_append(L, k, 0, 0, L.rank, ev);
}

// p3_apply_slice: count a host-applied slice towards its layer's and gate group's forward gate
// (system-scope release: the values copied before it on the stream are visible first).
__global__ void k_bump(uint32_t* done, uint32_t* gdone, uint32_t v) {
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    red_add_relaxed_sys(done, v);
    red_add_relaxed_sys(gdone, v);
  }
}

// param_bf16: the fp32 master of every owned slice from the (bf16) replica, once at start.
__global__ void k_master_init(const __grid_constant__ CommArgs a) {
  const PlanDev& P = a.plan;
  const LocalDev& L = a.loc[0];
  const uint32_t o = L.rank, base = P.own_base[o];
  for (uint32_t i = blockIdx.x; i < P.own_total[o]; i += gridDim.x) {
    const uint32_t g = P.own_list[base + i];
    const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(a.peers.W[o]) + P.layer_woff[P.slice_layer[g]] +
                             P.slice_off[g];
    float* m = L.M + P.slice_slot[g];
    for (uint32_t e = threadIdx.x; e < P.slice_len[g]; e += blockDim.x) m[e] = __bfloat162float(w[e]);
  }
}

int launch_master_init(const CommArgs& a, void* stream) {
  k_master_init<<<296, 256, 0, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

int launch_bump(uint32_t* done, uint32_t* gdone, uint32_t v, void* stream) {
  k_bump<<<1, 32, 0, (cudaStream_t)stream>>>(done, gdone, v);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

int launch_mark(const LocalDev& L, uint32_t k, uint32_t ev, void* stream) {
  k_mark<<<1, 32, 0, (cudaStream_t)stream>>>(L, k, ev);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

// ------------------------------------------------------------------ single-rank FINISH

// With one rank there is nothing to exchange: once every layer is published (no DRAIN launch
// ran, so the FINISH launch is the only consumer) the iteration's sync is the fused update
// p -= lr * (0 + g) / 1 (server.py:55-68 with N = 1) of every slice, in priority order so the
// next forward's gates open layer by layer. As one streaming kernel: tiles of P3_STREAM_TILE
// elements of the priority-ordered element space (layers back to back, each padded to 8) go to
// the CTAs round-robin, so round r of the grid covers the r-th stretch of the model; a tile is
// cut at layer and slice ends, and a slice is complete when all its elements are (its gate
// counters then advance, exactly as the comm kernel's broadcast signal does).
#ifndef P3_STREAM_TILE
#define P3_STREAM_TILE 4096u
#endif
#ifndef P3_STREAM_THREADS
#define P3_STREAM_THREADS 512
#endif
#ifndef P3_STREAM_CTAS_PER_SM
#define P3_STREAM_CTAS_PER_SM 1
#endif
#ifndef P3_STREAM_U
#define P3_STREAM_U 4  // float4s of each stream in flight per lane (8: register spills)
#endif

// Largest l < n_layers with layer_flat[l] <= pos (one warp, 32-ary search).
__device__ uint32_t warp_find_layer(const PlanDev& P, uint64_t pos) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = P.n_layers;
  while (hi - lo > 1) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t idx = lo + lane * step;
    const uint32_t m = __ballot_sync(FULL_MASK, idx < hi && P.layer_flat[idx] <= pos);
    lo += (31 - __clz(m)) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// One warp updates elements [0, n) of a piece: g the gradient, p the replica (read, then
// written), v the momentum; U float4s of each stream in flight per lane.
template <bool MOM>
__device__ __forceinline__ void warp_stream_piece(const float* __restrict__ g, float* __restrict__ p,
                                                  float* __restrict__ v, uint32_t n, const UpdCoef& c, bool bf,
                                                  uint32_t lane) {
  constexpr int U = P3_STREAM_U;
  uint32_t done = 0;
  if ((((uintptr_t)g | (uintptr_t)p | (uintptr_t)v) & 15) == 0) {
    const uint32_t n4 = n / 4;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    float4* p4 = reinterpret_cast<float4*>(p);
    float4* v4 = reinterpret_cast<float4*>(v);
    for (uint32_t j = lane; j < n4; j += U * 32) {
      float4 gg[U], pp[U], vv[MOM ? U : 1];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // every load of the round before any use
        const uint32_t i = j + u * 32 < n4 ? j + u * 32 : j;
        gg[u] = __ldcs(g4 + i);  // read once: evict first
        pp[u] = __ldcg(p4 + i);
        if (MOM) vv[MOM ? u : 0] = __ldcg(v4 + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = j + u * 32;
        if (i >= n4) continue;
        float4 x = gg[u];
        if (bf) x = make_float4(bf16_round(x.x), bf16_round(x.y), bf16_round(x.z), bf16_round(x.w));
        // the rank-ordered sum from +0.0 of one contribution, then / 1, * lr, - (server.py:60-65)
        const float4 acc = make_float4(__fadd_rn(0.f, x.x), __fadd_rn(0.f, x.y), __fadd_rn(0.f, x.z),
                                       __fadd_rn(0.f, x.w));
        const float4 r = sgd4(pp[u], acc, c, MOM ? &vv[MOM ? u : 0] : nullptr);
        if (MOM) v4[i] = vv[MOM ? u : 0];
        p4[i] = r;
      }
    }
    done = 4 * n4;
  }
  for (uint32_t i = done + lane; i < n; i += 32) {
    float x = __ldcs(g + i);
    if (bf) x = bf16_round(x);
    p[i] = sgd_step(__ldcg(p + i), __fadd_rn(0.f, x), c, MOM ? v + i : nullptr);
  }
}

// Work units are warp tiles of the element space, claimed in order with one atomic (strict
// priority order at tile granularity, balanced over all warps): P3_STREAM_TILE elements, and
// P3_STREAM_TAIL-element tiles over the last stretch (the last wave stays short).
#ifndef P3_STREAM_TAIL
#define P3_STREAM_TAIL 1024u
#endif
#ifndef P3_STREAM_TAIL_TILES
#define P3_STREAM_TAIL_TILES 2u  // tail tiles per warp
#endif

__global__ void __launch_bounds__(P3_STREAM_THREADS, P3_STREAM_CTAS_PER_SM)
    k_update_stream(const __grid_constant__ CommArgs a) {
  const PlanDev& P = a.plan;
  const LocalDev& L = a.loc[0];
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t total = P.layer_flat[P.n_layers];
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x / 32);
  // tiles [0, t1) are big, the rest small (P3_STREAM_TAIL_TILES per warp at the end); models of
  // 32M+ parameters take tiles twice as big (measured: ResNet-50 / seq2seq / VGG-19 sweeps)
  const uint64_t big = total >= (32ull << 20) ? 2ull * P3_STREAM_TILE : (uint64_t)P3_STREAM_TILE;
  const uint64_t small = big * P3_STREAM_TAIL / P3_STREAM_TILE;
  const uint64_t tail = min(total, nwarps * P3_STREAM_TAIL_TILES * small);
  const uint64_t t1 = (total - tail) / big;
  const uint64_t big_end = t1 * big;
  const UpdCoef c = make_coef(1, a.lr, a.momentum);
  float* const W = a.peers.W[L.rank];
  uint32_t lc = P3_NONE;  // cached layer and its metadata (warp-uniform)
  uint64_t lstart = 0, lnext = 0, count = 0, unit = 1, woff = 0, word = 0;
  uint32_t first = 0, ns = 0, grp = 0;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(L.stream_next, 1ull);
    t = __shfl_sync(FULL_MASK, t, 0);
    uint64_t pos = t < t1 ? t * big : big_end + (t - t1) * small;
    if (pos >= total) break;
    const uint64_t end = min(pos + (t < t1 ? big : small), total);
    while (pos < end) {
      if (lc == P3_NONE || pos < lstart || pos >= lnext) {  // the layer holding pos
        lc = warp_find_layer(P, pos);
        lstart = P.layer_flat[lc];
        lnext = P.layer_flat[lc + 1];
        first = P.layer_first[lc];
        ns = P.layer_nslices[lc];
        unit = P.slice_len[first];
        count = P.slice_off[first + ns - 1] + P.slice_len[first + ns - 1];
        woff = P.layer_woff[lc];
        grp = P.layer_group[lc];
        word = ld_relaxed_gpu64(L.pub + lc);
        if (!pub_ready(word, a.k + 1)) {  // published before this launch; maybe not yet ingested
          const uint64_t t0 = globaltimer();
          while (!pub_ready(word, a.k + 1)) {
            ingest_lanes(L);  // (single rank: priority discipline, no FIFO keys)
            __nanosleep(128);
            word = ld_relaxed_gpu64(L.pub + lc);
            if (globaltimer() - t0 > a.timeout_ns) {
              if (lane == 0) atomicCAS(a.err, 0u, (uint32_t)P3_ETIMEOUT);
              return;
            }
          }
        }
        if (lane == 0) fence_acq_rel_gpu();  // acquire of the gradient (ingest released it)
        __syncwarp();
      }
      const uint64_t e0 = pos - lstart;
      if (e0 >= count) {  // the layer's padding
        pos = min(lnext, end);
        continue;
      }
      const uint32_t g = first + (uint32_t)min(e0 / unit, (uint64_t)(ns - 1));
      const uint64_t soff = P.slice_off[g], send = soff + P.slice_len[g];
      const uint64_t e1 = min(end - lstart, send);  // cut at the slice end (and the tile end)
      float* v = L.V ? L.V + P.slice_slot[g] + (e0 - soff) : nullptr;
      if (v)
        warp_stream_piece<true>(pub_ptr(word) + e0, W + woff + e0, v, (uint32_t)(e1 - e0), c, a.push_bf16 != 0, lane);
      else
        warp_stream_piece<false>(pub_ptr(word) + e0, W + woff + e0, v, (uint32_t)(e1 - e0), c, a.push_bf16 != 0, lane);
      __syncwarp();
      if (lane == 0) {
        if (e0 == soff) {  // the slice's first element: its pop
          atomicAdd(&L.it->pushed, 1u);
          if (L.trace_cap) trace_append(L, a.k, lc, g - first, L.rank, P3_EV_PUSH);
        }
        fence_acq_rel_gpu();  // release this piece (and acquire the other pieces' releases)
        const uint32_t part = (uint32_t)(e1 - e0);
        if (atomicAdd(L.slice_elems + g, part) + part == send - soff) {
          fence_acq_rel_gpu();
          red_add_relaxed_sys(a.peers.done[L.rank] + lc, 1u);
          red_add_relaxed_sys(a.peers.gdone[L.rank] + grp, 1u);
          atomicAdd(&L.it->reduced, 1u);
          if (L.trace_cap) trace_append(L, a.k, lc, g - first, L.rank, P3_EV_BCAST);
        }
      }
      __syncwarp();
      pos = min(e1 >= count ? lnext : lstart + e1, end);
    }
  }
}

int launch_update_stream(const CommArgs& a, uint32_t sms, void* stream) {
  k_update_stream<<<sms * P3_STREAM_CTAS_PER_SM, P3_STREAM_THREADS, 0, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

// With lazy module loading (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default) the first launch
// of a kernel loads it, and loading waits for the kernels already running on the device.
// A comm kernel that waited for work of the compute streams would block them, so every kernel those
// streams may launch must be loaded before the comm kernel starts: query them all here.
int preload_kernels() {
  if (cudaFuncSetAttribute(k_comm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, P3_STAGES * P3_STAGE_BYTES) !=
          cudaSuccess ||
      cudaFuncSetAttribute(k_comm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P3_STAGES * P3_STAGE_BYTES) !=
          cudaSuccess)
    return P3_ECUDA;
  cudaFuncAttributes fa;
  const void* fns[] = {(const void*)k_comm<false>, (const void*)k_comm<true>, (const void*)k_gradgen, (const void*)k_sleep,
                       (const void*)k_shard_update, (const void*)k_queue_pop, (const void*)k_mark, (const void*)k_bump,
                       (const void*)k_master_init, (const void*)k_update_stream};
  for (const void* f : fns)
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return P3_ECUDA;
  return P3_OK;
}

int launch_comm(const CommArgs& a, uint32_t ctas, uint32_t threads, void* stream) {
  if (a.plan.world == 1 && !a.pb16)
    k_comm<true><<<ctas, threads, P3_STAGES * P3_STAGE_BYTES, (cudaStream_t)stream>>>(a);
  else
    k_comm<false><<<ctas, threads, P3_STAGES * P3_STAGE_BYTES, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

}  // namespace p3

extern "C" int p3_emulate_compute(uint64_t duration_us, void* stream) {
  if (duration_us == 0) return P3_OK;
  p3::k_sleep<<<1, 32, 0, (cudaStream_t)stream>>>(duration_us * 1000ull);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    p3::set_thread_error(cudaGetErrorString(e));
    return P3_ECUDA;
  }
  return P3_OK;
}
