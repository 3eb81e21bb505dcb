// sm_100a kernels of the P3 sync path.
//
//   K1 k_gradgen       gradient_block / _materialize          hashing.py:55-63, worker.py:166-171
//   K4 k_shard_update  ShardState.aggregate_and_update        server.py:55-68
//   K3 k_comm          persistent per-iteration comm kernel:
//        worker role   FrameQueue.poll + _priority_sender     queues.py:52-62, worker.py:184-190
//        server role   ShardState.on_push/aggregate/bcast     server.py:36-88, 208-226
//        apply role    on_bcast -> flags[layer]               worker.py:241-269 (remote stores +
//                                                             per-layer counters)
//   k_queue_pop        one FrameQueue.poll on the device queue (scripted tick replay)
//   k_sleep            TrainingWorker._emulate                worker.py:299-310
//
// All traffic is bandwidth-bound streaming: 16-byte vector loads/stores, no tensor cores.
// Floating point follows the reference's numpy fp32 semantics exactly: the sum is taken in
// ascending rank order starting from +0.0, then divided by N, then p - lr*g with the multiply
// and the subtract rounded separately (explicit _rn intrinsics: no FMA contraction).
#include <cuda_runtime.h>
#include <stdint.h>

#include "p3_internal.h"

namespace p3 {

#define FULL_MASK 0xffffffffu
#define P3_NONE 0xffffffffu

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
__device__ __forceinline__ void red_add_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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
template <int NW, int U>
__device__ void cta_update_vec(const float* p_src, float* const* dst, int ndst, const float* const* src,
                               float* v, uint64_t n4, const UpdCoef& c) {
  const uint64_t stride = blockDim.x;
  uint64_t j = threadIdx.x;
  for (; j + (U - 1) * stride < n4; j += U * stride) {
    float4 g[U][NW], p[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = 4 * (j + u * stride);
#pragma unroll
      for (int q = 0; q < NW; ++q) g[u][q] = __ldcg(reinterpret_cast<const float4*>(src[q] + i));
      p[u] = __ldcg(reinterpret_cast<const float4*>(p_src + i));
      if (v) vv[u] = __ldcg(reinterpret_cast<const float4*>(v + i));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = 4 * (j + u * stride);
      const float4 r = sgd4(p[u], sum_in_rank_order<NW>(g[u]), c, v ? &vv[u] : nullptr);
      if (v) *reinterpret_cast<float4*>(v + i) = vv[u];
      for (int d = 0; d < ndst; ++d) *reinterpret_cast<float4*>(dst[d] + i) = r;
    }
  }
  for (; j < n4; j += stride) {
    const uint64_t i = 4 * j;
    float4 g1[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) g1[q] = __ldcg(reinterpret_cast<const float4*>(src[q] + i));
    float4 vv1 = v ? __ldcg(reinterpret_cast<const float4*>(v + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 r = sgd4(__ldcg(reinterpret_cast<const float4*>(p_src + i)), sum_in_rank_order<NW>(g1), c,
                          v ? &vv1 : nullptr);
    if (v) *reinterpret_cast<float4*>(v + i) = vv1;
    for (int d = 0; d < ndst; ++d) *reinterpret_cast<float4*>(dst[d] + i) = r;
  }
}

__device__ void cta_update_generic(const float* p_src, float* const* dst, int ndst, const float* const* src,
                                   int nw, float* v, uint64_t n, bool aligned, const UpdCoef& c) {
  uint64_t done = 0;
  if (aligned) {
    const uint64_t n4 = n / 4;
    switch (nw) {
#define P3_CASE(K) \
  case K: cta_update_vec<K, (K <= 1 ? 4 : K <= 2 ? 2 : 1)>(p_src, dst, ndst, src, v, n4, c); break;
      P3_CASE(1) P3_CASE(2) P3_CASE(3) P3_CASE(4) P3_CASE(5) P3_CASE(6) P3_CASE(7) P3_CASE(8)
#undef P3_CASE
      default: aligned = false; break;
    }
    if (aligned) done = 4 * n4;
  }
  for (uint64_t i = done + threadIdx.x; i < n; i += blockDim.x) {
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
                     make_coef(nw, lr, mu));
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

// ------------------------------------------------------------------ device slice queue

// The outbox of one worker: per layer an iteration tag (ready), a publish sequence
// (fifo_key) and a claim cursor. The minimum under the FrameQueue order is the lowest ready
// layer with unclaimed slices (priority == layer index, plan.py:112, ties by slice index
// through the ascending cursor), or the earliest-published such layer in FIFO mode.
struct QueueView {
  uint32_t n_layers;
  uint32_t sched;
  const uint32_t* nslices;
  const uint32_t* first;
  const uint32_t* ready;
  const uint32_t* fifo_key;
  uint32_t* cursor;
};

// Executed by one full warp; returns the popped global slice id or P3_NONE.
// Priority discipline: layers are examined in ascending order 32 at a time (lane i owns
// layer base+i); each lane first loads the availability of all its layers (independent
// loads, one memory round trip), then the warp walks the availability ballots in layer
// order and claims the first slice it wins. A lost race moves on to the next candidate
// without rescanning. FIFO discipline: arg-min of the publish sequence, then claim.
__device__ uint32_t warp_pop(const QueueView& q, uint32_t tag, uint32_t* dbg = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
  if (q.sched == P3_SCHED_PRIORITY) {
    for (uint32_t group = 0; group < q.n_layers; group += 32 * 32) {
      uint32_t bits = 0;  // bit c: layer group + 32*c + lane is poppable
#pragma unroll 4
      for (uint32_t c = 0; c < 32; ++c) {
        const uint32_t l = group + 32 * c + lane;
        if (l >= q.n_layers) break;
        const bool ok = (int32_t)(ld_acquire_gpu(q.ready + l) - tag) >= 0 &&
                        ld_relaxed_gpu(q.cursor + l) < q.nslices[l];
        bits |= (uint32_t)ok << c;
      }
      const uint32_t nchunk = min(32u, (q.n_layers - group + 31) / 32);
      for (uint32_t c = 0; c < nchunk; ++c) {
        uint32_t m = __ballot_sync(FULL_MASK, (bits >> c) & 1u);
        while (m) {
          const uint32_t j = __ffs(m) - 1;
          const uint32_t l = group + 32 * c + j;
          uint32_t s = 0;
          if (lane == j) s = atomicAdd(q.cursor + l, 1u);
          s = __shfl_sync(FULL_MASK, s, j);
          if (s < q.nslices[l]) return q.first[l] + s;
          m &= m - 1;  // lost the race for the layer's last slice: next candidate
        }
      }
    }
    return P3_NONE;
  }
  for (uint32_t retry = 0;; ++retry) {
    if (dbg && lane == 0) *(volatile uint32_t*)dbg = (6u << 20) | (retry & 0xfffff);
    uint32_t best_key = P3_NONE, best_l = P3_NONE;
    for (uint32_t l = lane; l < q.n_layers; l += 32) {
      const uint32_t r = ld_acquire_gpu(q.ready + l);
      if ((int32_t)(r - tag) < 0) continue;
      if (ld_relaxed_gpu(q.cursor + l) >= q.nslices[l]) continue;
      const uint32_t key = ld_relaxed_gpu(q.fifo_key + l);
      if (key < best_key || (key == best_key && l < best_l)) {
        best_key = key;
        best_l = l;
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const uint32_t ok = __shfl_xor_sync(FULL_MASK, best_key, off);
      const uint32_t ol = __shfl_xor_sync(FULL_MASK, best_l, off);
      if (ok < best_key || (ok == best_key && ol < best_l)) {
        best_key = ok;
        best_l = ol;
      }
    }
    if (best_l == P3_NONE) return P3_NONE;
    uint32_t s = 0;
    if (lane == 0) s = atomicAdd(q.cursor + best_l, 1u);
    s = __shfl_sync(FULL_MASK, s, 0);
    if (s < q.nslices[best_l]) return q.first[best_l] + s;
    // lost the race for the last slice of that layer: rescan
  }
}

__global__ void k_queue_pop(QueueView q, uint32_t tag, uint32_t* result) {
  const uint32_t g = warp_pop(q, tag);
  if (threadIdx.x == 0) *result = g;
}

int launch_queue_pop(const uint32_t* nslices, const uint32_t* first, const uint32_t* ready,
                     const uint32_t* fifo_key, uint32_t* cursor, uint32_t n_layers, uint32_t sched,
                     uint32_t tag, uint32_t* result, void* stream) {
  QueueView q{n_layers, sched, nslices, first, ready, fifo_key, cursor};
  k_queue_pop<<<1, 32, 0, (cudaStream_t)stream>>>(q, tag, result);
  return cudaGetLastError() == cudaSuccess ? P3_OK : P3_ECUDA;
}

// ------------------------------------------------------------------ K3: comm kernel

// Server role pick (one warp): the lowest layer with a completed, unclaimed owned slice,
// then the first such slice of that layer (ascending slice index). The inbox of
// ServerEngine is priority ordered (server.py:118), so the same order is used here.
__device__ uint32_t warp_server_pick(const CommArgs& a, const LocalDev& L, uint32_t* dbg = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
  const PlanDev& P = a.plan;
  const uint32_t o = L.rank, nl = P.n_layers, k = a.k;
  const uint32_t* hint = a.peers.hint[o];
  const uint32_t* arrivals = a.peers.arrivals[o];
  const uint32_t* lcount = P.own_lcount + (uint64_t)o * nl;
  const uint32_t need = (k + 1) * P.world;
  for (uint32_t group = 0; group < nl; group += 32 * 32) {
    // candidate layers: an owned slice completed this iteration and not yet claimed
    uint32_t bits = 0;
#pragma unroll 4
    for (uint32_t c = 0; c < 32; ++c) {
      const uint32_t l = group + 32 * c + lane;
      if (l >= nl) break;
      const uint32_t oc = lcount[l];
      bool ok = false;
      if (oc) {
        const uint32_t completed = ld_acquire_sys(hint + l) - k * oc;
        ok = (int32_t)(completed - ld_relaxed_gpu(L.srv_taken + l)) > 0;
      }
      bits |= (uint32_t)ok << c;
    }
    const uint32_t nchunk = min(32u, (nl - group + 31) / 32);
    for (uint32_t c = 0; c < nchunk; ++c) {
      uint32_t lm = __ballot_sync(FULL_MASK, (bits >> c) & 1u);
      while (lm) {
        const uint32_t l = group + 32 * c + (__ffs(lm) - 1);
        lm &= lm - 1;
        const uint32_t lf = P.own_lfirst[(uint64_t)o * nl + l], cnt = lcount[l];
        // lanes are not guaranteed to execute this load together (independent thread
        // scheduling) and other CTAs move the watermark: take lane 0's value so the trip
        // count — and every warp-synchronous call inside — is uniform across the warp
        uint32_t lo = 0;
        if (lane == 0) lo = ld_relaxed_gpu(L.srv_lo + l);
        lo = __shfl_sync(FULL_MASK, lo, 0);
        for (uint32_t i0 = lo; i0 < cnt; i0 += 32) {
          if (dbg && lane == 0) *(volatile uint32_t*)dbg = (8u << 20) | ((l & 0x3ff) << 10) | (i0 & 0x3ff);
          const uint32_t i = i0 + lane;
          uint32_t g = P3_NONE;
          bool ok = false, claimed = true;
          if (i < cnt) {
            g = P.own_list[lf + i];
            claimed = ld_relaxed_gpu(L.claim + g) != k;
            ok = !claimed && (int32_t)(ld_acquire_sys(arrivals + g) - need) >= 0;
          }
          if (__all_sync(FULL_MASK, claimed) && lane == 0) atomicMax(L.srv_lo + l, i0 + 32);
          uint32_t m = __ballot_sync(FULL_MASK, ok);
          while (m) {
            const int j = __ffs(m) - 1;
            const uint32_t gj = __shfl_sync(FULL_MASK, g, j);
            uint32_t won = 0;
            if (lane == 0) {
              won = atomicCAS(L.claim + gj, k, k + 1) == k;
              if (won) {
                atomicAdd(L.srv_taken + l, 1u);
                atomicAdd(&L.it->reduced, 1u);
              }
            }
            won = __shfl_sync(FULL_MASK, won, 0);
            if (won) return gj;
            m &= m - 1;
          }
        }
      }
    }
  }
  return P3_NONE;
}

__device__ __forceinline__ void trace_append(const LocalDev& L, uint32_t k, uint32_t layer, uint32_t slice,
                                             uint32_t rank, uint32_t ev) {
  if (!L.trace_cap) return;
  const unsigned long long idx = atomicAdd(L.trace_n, 1ull);
  if (idx < L.trace_cap) {
    p3_trace_rec_t r;
    r.t_ns = globaltimer();
    r.iteration = k;
    r.layer = layer;
    r.slice = slice;
    r.rank = (uint16_t)rank;
    r.event = (uint16_t)ev;
    L.trace[idx] = r;
  }
}

__device__ void cta_copy(float* dst, const float* src, uint32_t n) {
  constexpr int U = 8;  // 8 independent 16-byte loads in flight per thread
  uint32_t done = 0;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const uint32_t n4 = n / 4, stride = blockDim.x;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    uint32_t j = threadIdx.x;
    for (; j + (U - 1) * stride < n4; j += U * stride) {
      float4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = __ldcg(s4 + j + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u) d4[j + u * stride] = r[u];
    }
    for (; j < n4; j += stride) d4[j] = __ldcg(s4 + j);
    done = 4 * n4;
  }
  for (uint32_t i = done + threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcg(src + i);
}

struct PushSmem {
  const float* src;
};

// Worker role: store one slice of this rank's gradient into the owner's receive slot
// over NVLink (or nothing when the owner is local), then count the arrival.
__device__ void do_push(const CommArgs& a, const LocalDev& L, uint32_t g, PushSmem* sm) {
  const PlanDev& P = a.plan;
  const uint32_t r = L.rank, o = P.slice_owner[g], l = P.slice_layer[g];
  const uint32_t len = P.slice_len[g];
  if (o == r) {
    // the owner reads its own contribution from the gradient in place: only count it
    if (threadIdx.x == 0) {
      (void)ld_acquire_gpu(L.ready + l);  // gradient published -> visible to the reducer
      const uint32_t old = atom_add_release_sys(a.peers.arrivals[o] + g, 1u);
      if (old + 1 == (a.k + 1) * P.world) red_add_release_sys(a.peers.hint[o] + l, 1u);
    }
    return;
  }
  if (threadIdx.x == 0) {
    (void)ld_acquire_gpu(L.ready + l);
    sm->src = reinterpret_cast<const float*>(ld_relaxed_gpu64(L.gptr + l)) + P.slice_off[g];
  }
  __syncthreads();
  float* dst = a.peers.R[o] + (uint64_t)r * P.own_stride[o] + P.slice_slot[g];
  cta_copy(dst, sm->src, len);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (a.remote) __threadfence_system(); else __threadfence();
    atomicAdd(L.bytes + 1, 4ull * len);
    const uint32_t old = atom_add_release_sys(a.peers.arrivals[o] + g, 1u);
    if (old + 1 == (a.k + 1) * P.world) red_add_release_sys(a.peers.hint[o] + l, 1u);
  }
}

struct ReduceSmem {
  const float* src[P3_MAX_RANKS];
  float* dst[P3_MAX_RANKS];
  int aligned;
};

// Server role: aggregate the N pushes of an owned slice in rank order, apply SGD to the
// master (the owner's replica), store the result into every replica, bump done[layer].
__device__ void do_reduce(const CommArgs& a, const LocalDev& L, uint32_t g, ReduceSmem* sm) {
  const PlanDev& P = a.plan;
  const uint32_t o = L.rank, l = P.slice_layer[g], N = P.world;
  const uint32_t len = P.slice_len[g];
  const uint64_t woff = P.layer_woff[l] + P.slice_off[g];
  if (threadIdx.x < N) {
    const uint32_t q = threadIdx.x;
    if (q == o) {
      (void)ld_acquire_sys(a.peers.arrivals[o] + g);
      sm->src[q] = reinterpret_cast<const float*>(ld_relaxed_gpu64(L.gptr + l)) + P.slice_off[g];
    } else {
      sm->src[q] = a.peers.R[o] + (uint64_t)q * P.own_stride[o] + P.slice_slot[g];
    }
    // the owner's own replica goes first: it is also the master copy read below
    const uint32_t d = q == o ? 0 : (q < o ? q + 1 : q);
    sm->dst[d] = a.peers.W[q] + woff;
  }
  if (threadIdx.x == 0) (void)ld_acquire_sys(a.peers.arrivals[o] + g);
  __syncthreads();
  if (threadIdx.x == 0) {
    uintptr_t al = 0;
    for (uint32_t q = 0; q < N; ++q) al |= (uintptr_t)sm->src[q] | (uintptr_t)sm->dst[q];
    if (L.V) al |= (uintptr_t)(L.V + P.slice_slot[g]);
    sm->aligned = (al & 15) == 0;
  }
  __syncthreads();
  cta_update_generic(sm->dst[0], sm->dst, (int)N, sm->src, (int)N, L.V ? L.V + P.slice_slot[g] : nullptr,
                     len, sm->aligned != 0, make_coef(N, a.lr, a.momentum));
  __syncthreads();
  if (threadIdx.x == 0) {
    if (a.remote) __threadfence_system(); else __threadfence();
    for (uint32_t q = 0; q < N; ++q) red_add_release_sys(a.peers.done[q] + l, 1u);
    atomicAdd(L.bytes + 0, 4ull * len * (N - 1));  // pushes received
    atomicAdd(L.bytes + 1, 4ull * len * (N - 1));  // broadcasts sent
    trace_append(L, a.k, l, g - P.layer_first[l], o, P3_EV_BCAST);
  }
}

__device__ __forceinline__ QueueView queue_of(const CommArgs& a, const LocalDev& L) {
  QueueView q;
  q.n_layers = a.plan.n_layers;
  q.sched = a.sched;
  q.nslices = a.plan.layer_nslices;
  q.first = a.plan.layer_first;
  q.ready = L.ready;
  q.fifo_key = L.fifo_key;
  q.cursor = L.cursor;
  return q;
}

// Comm kernel. Every CTA loops: warp 0 picks a job (server work first, since a finished
// slice unblocks the next forward pass; then the most urgent ready slice of the local
// worker queues), the whole CTA executes it. The queue is re-read before every job, so a
// layer published while the kernel runs preempts less urgent slices at slice granularity.
// DRAIN launches (one per published layer) exit when no job is available: a kernel that
// spun on not-yet-published gradients would hold SMs that the compute producing them may
// need (co-residency-bound library kernels, lazy module loading). The FINISH launch of an
// iteration ends once every local slice is pushed and every owned slice reduced; it waits
// only for peers' pushes, never for local compute.
__global__ void __launch_bounds__(512, 1) k_comm(const __grid_constant__ CommArgs a) {
  __shared__ uint32_t s_job, s_li, s_g;
  __shared__ PushSmem s_push;
  __shared__ ReduceSmem s_red;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t t0 = globaltimer();
  uint32_t backoff = 0;
  uint32_t* phase = (threadIdx.x == 0 && blockIdx.x < P3_DBG_CTAS) ? a.loc[0].cta_phase + blockIdx.x : nullptr;
  for (uint32_t iter = 0;; ++iter) {
    if (phase) *(volatile uint32_t*)phase = (a.k << 24) | (1u << 20) | (iter & 0xfffff);
    if (warp == 0) {
      if (backoff) __nanosleep(backoff);
      uint32_t job = 0, li = 0, g = P3_NONE;
      for (uint32_t t = 0; t < a.n_local && job == 0; ++t) {
        li = (blockIdx.x + t) % a.n_local;
        if (phase) *(volatile uint32_t*)phase = (7u << 20);
        g = warp_server_pick(a, a.loc[li], phase);
        if (g != P3_NONE) job = 1;
      }
      for (uint32_t t = 0; t < a.n_local && job == 0; ++t) {
        li = (blockIdx.x + t) % a.n_local;
        g = warp_pop(queue_of(a, a.loc[li]), a.k + 1, phase);
        if (g != P3_NONE) {
          job = 2;
          if (lane == 0) {
            // the transmission sequence is the pop order (the moment _priority_sender
            // hands a slice to the link, worker.py:184-190)
            const LocalDev& L = a.loc[li];
            atomicAdd(&L.it->pushed, 1u);
            const uint32_t l = a.plan.slice_layer[g];
            trace_append(L, a.k, l, g - a.plan.layer_first[l], L.rank, P3_EV_PUSH);
          }
        }
      }
      if (job == 0 && a.mode == P3_COMM_DRAIN) {
        job = 3;  // nothing published is pending: leave the SMs to compute
      } else if (job == 0) {
        // decided by lane 0 and broadcast: a per-lane decision could split the warp
        uint32_t verdict = 0;  // 0 keep waiting, 1 done or failed elsewhere, 2 timed out
        if (lane == 0) {
          bool fin = true;
          for (uint32_t t = 0; t < a.n_local; ++t) {
            const LocalDev& L = a.loc[t];
            fin = fin && ld_relaxed_gpu(&L.it->pushed) >= a.plan.total_slices &&
                  ld_relaxed_gpu(&L.it->reduced) >= a.plan.own_total[L.rank];
          }
          verdict = (fin || ld_relaxed_gpu(a.err) != 0) ? 1u : (globaltimer() - t0 > a.timeout_ns ? 2u : 0u);
        }
        verdict = __shfl_sync(FULL_MASK, verdict, 0);
        if (verdict == 1) {
          job = 3;
        } else if (verdict == 2) {
          job = 3;
          if (lane == 0 && atomicCAS(a.err, 0u, (uint32_t)P3_ETIMEOUT) == 0u) {
            // diagnostics for the host (p3_sync_all), then release every forward gate of the
            // local ranks so the compute streams drain
            a.err[1] = a.k;
            for (uint32_t t = 0; t < a.n_local; ++t) {
              a.err[2 + 2 * t] = ld_relaxed_gpu(&a.loc[t].it->pushed);
              a.err[3 + 2 * t] = ld_relaxed_gpu(&a.loc[t].it->reduced);
            }
            for (uint32_t t = 0; t < a.n_local; ++t)
              for (uint32_t l = 0; l < a.plan.n_layers; ++l)
                atomicAdd(a.peers.done[a.loc[t].rank] + l, 0x40000000u);
          }
        }
      }
      if (lane == 0) {
        s_job = job;
        s_li = li;
        s_g = g;
      }
      backoff = job == 0 ? min(2u * backoff + 64u, 4096u) : 0u;
    }
    __syncthreads();
    const uint32_t job = s_job;
    if (job == 3) break;
    if (phase) *(volatile uint32_t*)phase = (a.k << 24) | ((1u + job) << 20) | (iter & 0xfffff);
    if (job == 1) do_reduce(a, a.loc[s_li], s_g, &s_red);
    else if (job == 2) do_push(a, a.loc[s_li], s_g, &s_push);
    if (job && threadIdx.x == 0) atomicAdd(&a.loc[0].it->jobs, 1u);
    __syncthreads();
  }
  if (phase) *(volatile uint32_t*)phase = (a.k << 24) | (5u << 20);
  if (threadIdx.x == 0 && a.mode == P3_COMM_FINISH) atomicAdd(&a.loc[0].it->exited, 1u);
}

// With lazy module loading (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default) the first launch
// of a kernel loads it, and loading waits for the kernels already running on the device.
// A persistent comm kernel waits for work of the compute streams, so every kernel those
// streams may launch must be loaded before the comm kernel starts: query them all here.
int preload_kernels() {
  cudaFuncAttributes fa;
  const void* fns[] = {(const void*)k_comm, (const void*)k_gradgen, (const void*)k_sleep,
                       (const void*)k_shard_update, (const void*)k_queue_pop};
  for (const void* f : fns)
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return P3_ECUDA;
  return P3_OK;
}

int launch_comm(const CommArgs& a, uint32_t ctas, uint32_t threads, void* stream) {
  k_comm<<<ctas, threads, 0, (cudaStream_t)stream>>>(a);
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
