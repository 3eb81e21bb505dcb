// Wire frames for sync traffic that leaves the NVSwitch domain.
//
//   p3_frame_encode / p3_frame_decode   encode_frame / try_decode   proto.py:61-120
//   p3_frames_pack / p3_frames_unpack   the same frames built / parsed on the device, so a
//                                       NIC (GPUDirect RDMA) can send slices straight from
//                                       the gradient / parameter arenas
//
// Layout (proto.py:18-21): 39-byte little-endian header "<4sBIQHIIQI" — magic "P3W1",
// msg_type u8, priority u32, iteration u64, worker_rank u16, layer u32, slice u32, offset
// u64, payload_len u32 — then payload_len bytes of float32 (PUSH and BCAST only).
// The payload therefore starts 39 bytes into the frame: device copies move 16-byte words
// between a float-aligned side and a byte-shifted side with funnel shifts.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "p3_internal.h"

namespace p3 {
namespace {

constexpr uint32_t kHeader = P3_FRAME_HEADER_BYTES;
__host__ __device__ inline uint8_t magic(uint32_t i) {  // "P3W1"
  return i == 0 ? 'P' : i == 1 ? '3' : i == 2 ? 'W' : '1';
}

__host__ __device__ inline bool has_payload(uint32_t t) { return t == P3_MSG_PUSH || t == P3_MSG_BCAST; }

// Byte b of the header of f (field offsets 0,4,5,9,17,19,23,27,35).
__host__ __device__ inline uint8_t header_byte(const p3_frame_t& f, uint32_t b) {
  auto le = [](uint64_t v, uint32_t i) { return (uint8_t)(v >> (8 * i)); };
  if (b < 4) return magic(b);
  if (b < 5) return (uint8_t)f.msg_type;
  if (b < 9) return le(f.priority, b - 5);
  if (b < 17) return le(f.iteration, b - 9);
  if (b < 19) return le(f.worker_rank, b - 17);
  if (b < 23) return le(f.layer, b - 19);
  if (b < 27) return le(f.slice, b - 23);
  if (b < 35) return le(f.offset, b - 27);
  return le(f.payload_len, b - 35);
}

template <typename T>
__host__ __device__ inline T read_le(const uint8_t* p, uint32_t n) {
  uint64_t v = 0;
  for (uint32_t i = 0; i < n; ++i) v |= (uint64_t)p[i] << (8 * i);
  return (T)v;
}

// Decode + validate a header (try_decode, proto.py:97-109). Returns 0 or a reason code:
// 1 magic, 2 msg_type, 3 payload over max, 4 payload on a control frame.
__host__ __device__ inline uint32_t parse_header(const uint8_t* h, uint64_t max_payload, p3_frame_t* f) {
  f->msg_type = h[4];
  f->priority = read_le<uint32_t>(h + 5, 4);
  f->iteration = read_le<uint64_t>(h + 9, 8);
  f->worker_rank = read_le<uint32_t>(h + 17, 2);
  f->layer = read_le<uint32_t>(h + 19, 4);
  f->slice = read_le<uint32_t>(h + 23, 4);
  f->offset = read_le<uint64_t>(h + 27, 8);
  f->payload_len = read_le<uint32_t>(h + 35, 4);
  f->reserved = 0;
  if (h[0] != magic(0) || h[1] != magic(1) || h[2] != magic(2) || h[3] != magic(3)) return 1;
  if (f->msg_type > P3_MSG_FIN) return 2;
  if (f->payload_len > max_payload) return 3;
  if (!has_payload(f->msg_type) && f->payload_len != 0) return 4;
  return 0;
}

// ------------------------------------------------------------------ device pack / unpack

constexpr uint32_t kThreads = 256;
constexpr uint32_t kBlocksPerFrame = 16;

// Bytes [0, n) of src to dst, any alignment of either: byte-wise until dst is 16-byte
// aligned, then 16-byte stores, each assembled from the two aligned 16-byte source chunks
// that cover it (funnel shifts by the — per-call uniform — source misalignment), then the
// tail byte-wise. A chunk load may touch up to 15 bytes past the last byte it needs; the
// chunk is 16-byte aligned, so it never leaves the allocation granule.
template <int WO>
__device__ __forceinline__ uint4 shifted16(const uint4& A, const uint4& B, uint32_t r) {
  const uint32_t w[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
  uint4 o;
  o.x = r ? __funnelshift_r(w[WO + 0], w[WO + 1], 8 * r) : w[WO + 0];
  o.y = r ? __funnelshift_r(w[WO + 1], w[WO + 2], 8 * r) : w[WO + 1];
  o.z = r ? __funnelshift_r(w[WO + 2], w[WO + 3], 8 * r) : w[WO + 2];
  o.w = r ? __funnelshift_r(w[WO + 3], w[WO + 4], 8 * r) : w[WO + 3];
  return o;
}

__device__ void copy_bytes(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint32_t t, uint32_t nt) {
  const uint32_t head = min(bytes, (uint32_t)((16 - ((uintptr_t)dst & 15)) & 15));
  if (t < head) dst[t] = src[t];
  const uint32_t chunks = (bytes - head) / 16;
  const uint8_t* s = src + head;
  const uint32_t q = (uint32_t)((uintptr_t)s & 15), wo = q / 4, r = q % 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(s - q);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (uint32_t k = t; k < chunks; k += nt) {
    const uint4 A = __ldg(s4 + k);
    const uint4 B = q ? __ldg(s4 + k + 1) : A;
    uint4 o;
    switch (wo) {  // uniform across the grid: no divergence
      case 0: o = shifted16<0>(A, B, r); break;
      case 1: o = shifted16<1>(A, B, r); break;
      case 2: o = shifted16<2>(A, B, r); break;
      default: o = shifted16<3>(A, B, r); break;
    }
    d4[k] = o;
  }
  for (uint32_t i = head + 16 * chunks + t; i < bytes; i += nt) dst[i] = src[i];
}

__global__ void __launch_bounds__(kThreads) k_frames_pack(const p3_frame_t* frames, const float* const* src,
                                                        const uint64_t* out_off, uint32_t first, uint8_t* out) {
  const uint32_t i = first + blockIdx.y;
  const p3_frame_t f = frames[i];
  uint8_t* base = out + out_off[i];
  if (blockIdx.x == 0 && threadIdx.x < kHeader) base[threadIdx.x] = header_byte(f, threadIdx.x);
  const uint8_t* s = reinterpret_cast<const uint8_t*>(src[i]);
  if (!has_payload(f.msg_type) || !s || f.payload_len == 0) return;
  copy_bytes(base + kHeader, s, f.payload_len, blockIdx.x * kThreads + threadIdx.x, gridDim.x * kThreads);
}

__global__ void __launch_bounds__(kThreads) k_frames_unpack(const uint8_t* in, const uint64_t* in_off, uint32_t first,
                                                          uint64_t max_payload, float* const* dst,
                                                          p3_frame_t* frames_out, uint32_t* err) {
  const uint32_t i = first + blockIdx.y;
  const uint8_t* base = in + in_off[i];
  __shared__ uint8_t h[kHeader];
  if (threadIdx.x < kHeader) h[threadIdx.x] = base[threadIdx.x];
  __syncthreads();
  p3_frame_t f;
  const uint32_t why = parse_header(h, max_payload, &f);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (frames_out) frames_out[i] = f;
    if (why && atomicCAS(err, 0u, (uint32_t)P3_EPROTOCOL) == 0u) {
      err[1] = i;
      err[2] = why;
    }
  }
  if (why || !dst || !dst[i] || f.payload_len == 0) return;
  copy_bytes(reinterpret_cast<uint8_t*>(dst[i]), base + kHeader, f.payload_len, blockIdx.x * kThreads + threadIdx.x,
             gridDim.x * kThreads);
}

}  // namespace
}  // namespace p3

using namespace p3;

extern "C" int p3_frame_encode(const p3_frame_t* f, const void* payload, uint8_t* out, uint64_t cap,
                               uint64_t* n_out) {
  if (!f || !n_out) {
    set_thread_error("null frame or size pointer");
    return P3_EUSAGE;
  }
  if (f->msg_type > P3_MSG_FIN || f->worker_rank > 0xffffu) {
    set_thread_error("msg_type or worker_rank out of range");
    return P3_EUSAGE;
  }
  if (has_payload(f->msg_type)) {
    if (f->payload_len % 4) {
      set_thread_error(std::string(f->msg_type == P3_MSG_PUSH ? "PUSH" : "BCAST") + " payload not a float32 array");
      return P3_EPROTOCOL;
    }
  } else if (f->payload_len) {
    static const char* names[] = {"PUSH", "BCAST", "PULL", "NOTIFY", "HELLO", "FIN"};
    set_thread_error(std::string(names[f->msg_type]) + " frames carry no payload");
    return P3_EPROTOCOL;
  }
  const uint64_t total = kHeader + (uint64_t)f->payload_len;
  *n_out = total;
  if (!out) return P3_OK;
  if (cap < total || (f->payload_len && !payload)) {
    set_thread_error("output buffer too small or payload missing");
    return P3_EUSAGE;
  }
  for (uint32_t b = 0; b < kHeader; ++b) out[b] = header_byte(*f, b);
  if (f->payload_len) std::memcpy(out + kHeader, payload, f->payload_len);
  return P3_OK;
}

extern "C" int p3_frame_decode(const uint8_t* buf, uint64_t n, uint64_t max_payload, p3_frame_t* f,
                               uint64_t* n_out) {
  if (!f || !n_out || (n && !buf)) {
    set_thread_error("null argument");
    return P3_EUSAGE;
  }
  if (n < kHeader) {
    *n_out = kHeader - n;
    return P3_EMORE;
  }
  const uint32_t why = parse_header(buf, max_payload, f);
  if (why) {
    static const char* names[] = {"PUSH", "BCAST", "PULL", "NOTIFY", "HELLO", "FIN"};
    std::string m;
    if (why == 1) {
      m = "bad magic b'";
      for (int i = 0; i < 4; ++i) m += (char)buf[i];
      m += "'";
    } else if (why == 2) {
      m = "unknown msg_type " + std::to_string(buf[4]);
    } else if (why == 3) {
      m = "payload_len " + std::to_string(f->payload_len) + " exceeds max " + std::to_string(max_payload);
    } else {
      m = std::string(names[f->msg_type]) + " frame with nonzero payload_len " + std::to_string(f->payload_len);
    }
    set_thread_error(m);
    return P3_EPROTOCOL;
  }
  const uint64_t total = kHeader + (uint64_t)f->payload_len;
  if (n < total) {
    *n_out = total - n;
    return P3_EMORE;
  }
  *n_out = total;
  return P3_OK;
}

extern "C" int p3_frames_pack(const p3_frame_t* frames_dev, const float* const* src_dev, const uint64_t* out_off_dev,
                              uint32_t n, uint8_t* out_dev, void* stream) {
  for (uint32_t first = 0; first < n; first += 65535) {
    const dim3 grid(kBlocksPerFrame, std::min<uint32_t>(65535, n - first));
    k_frames_pack<<<grid, kThreads, 0, (cudaStream_t)stream>>>(frames_dev, src_dev, out_off_dev, first, out_dev);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_thread_error(cudaGetErrorString(e));
    return P3_ECUDA;
  }
  return P3_OK;
}

extern "C" int p3_frames_unpack(const uint8_t* in_dev, const uint64_t* in_off_dev, uint32_t n, uint64_t max_payload,
                                float* const* dst_dev, p3_frame_t* frames_out_dev, uint32_t* err_dev, void* stream) {
  if (!err_dev) {
    set_thread_error("err_dev is required");
    return P3_EUSAGE;
  }
  for (uint32_t first = 0; first < n; first += 65535) {
    const dim3 grid(kBlocksPerFrame, std::min<uint32_t>(65535, n - first));
    k_frames_unpack<<<grid, kThreads, 0, (cudaStream_t)stream>>>(in_dev, in_off_dev, first, max_payload, dst_dev,
                                                                frames_out_dev, err_dev);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_thread_error(cudaGetErrorString(e));
    return P3_ECUDA;
  }
  return P3_OK;
}
