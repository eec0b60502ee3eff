// bsg_api.cu -- the C ABI (include/bsg.h): argument semantics of the
// reference API, device workspace management, host<->device staging and
// dispatch to the sm_100a kernels.  No CPU fallback exists: every shuffle,
// gather and bijection evaluation of the public API runs on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bsg.h"
#include "bsg_internal.h"
#include "bsg_partition.h"

namespace {

using bsg::BijParams;

thread_local std::string t_err;

bsg_status fail(bsg_status s, const std::string& msg) {
  t_err = msg;
  return s;
}

#define BSG_CUDA(expr)                                                                                \
  do {                                                                                                \
    cudaError_t _e = (expr);                                                                          \
    if (_e != cudaSuccess) {                                                                          \
      if (_e == cudaErrorMemoryAllocation) {                                                          \
        cudaGetLastError();                                                                           \
        return fail(BSG_ENOMEM, std::string(#expr) + ": " + cudaGetErrorString(_e));                  \
      }                                                                                               \
      return fail(BSG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));                    \
    }                                                                                                 \
  } while (0)

#define BSG_TRY(expr)                    \
  do {                                   \
    bsg_status _s = (expr);              \
    if (_s != BSG_OK) return _s;         \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  // Set when a captured CUDA graph references the buffer: growing it then retires the old allocation instead of
  // freeing it, so the graph stays valid (retired buffers are freed with the buffer's owner).
  bool captured = false;
  std::vector<void*> retired;
  cudaError_t ensure(size_t n, bool zero = false) {
    if (bytes >= n && p) return cudaSuccess;
    if (captured && p) {
      retired.push_back(p);
      p = nullptr;
      bytes = 0;
      captured = false;
    }
    release();
    size_t want = std::max<size_t>(n, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      p = nullptr;
      return e;
    }
    bytes = want;
    if (zero) e = cudaMemset(p, 0, want);
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void release_all() {  // also the retired allocations (bsg_release_workspace: no graph may replay afterwards)
    release();
    for (void* q : retired) cudaFree(q);
    retired.clear();
    captured = false;
  }
};

// Per-device state: look-back workspace, generic-round keys and staging
// buffers.  All kernels of one device context are ordered through `ws_done`
// (wait before, record after), so concurrent callers on different streams
// never share the look-back status words or the key buffer.
struct DeviceCtx {
  int device = 0;
  std::mutex mu;
  DevBuf status;   // look-back status words (u64 per tile)
  DevBuf scratch;  // [0] tile counter (u32), [8] count (u64)
  uint32_t epoch = 0;
  DevBuf keys;     // round keys for non-24-round Philox
  DevBuf st_in, st_out, st_idx, st_tmp;  // host-pointer staging / temporaries
  DevBuf part;                           // partitioned-path workspace
  std::deque<std::vector<uint32_t>> captured_keys;  // host key schedules read by captured graphs
  cudaEvent_t ws_done = nullptr;
  // staged host-pointer calls: copy streams and events of the chunked H2D / D2H (created on first use)
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  std::vector<cudaEvent_t> stage_ev;
  bool ready = false;
};

// Host buffers a synchronous host-pointer call hands to run_range: the partitioned path overlaps their copies
// with its first and last passes (chunks); any other path copies them whole around the kernel on the stream.
struct StageIO {
  const void* h_in = nullptr;
  void* h_out = nullptr;
  size_t in_bytes = 0, out_bytes = 0;
};
constexpr int kStageChunks = 8;

std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DeviceCtx>> g_ctx;
int g_force_compact = 0;
// 0 auto, 1 single-pass only, 2 partitioned whenever eligible; BSG_PATH overrides at load.
int g_path = [] {
  const char* e = std::getenv("BSG_PATH");
  return (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
}();
// Auto mode uses the partitioned path for power-of-two shuffles whose payload
// exceeds this many bytes (below it the single pass is L2-resident and faster).
uint64_t g_partition_min_bytes = 256ULL << 20;
// Auto mode: the partitioned path for payloads of at least g_partition_min_bytes with elements of at most
// 8 bytes.  16-byte records move 108 B/element through the three passes against one random 16-B read per
// element in the single pass, which wins there (C5: 23.9 vs 25.5 ms for 2^30 records).
bool auto_partition(uint64_t n, uint64_t elem_bytes) {
  return g_path == 2 || (n * elem_bytes >= g_partition_min_bytes && elem_bytes <= 8);
}

bsg_status current_ctx(DeviceCtx** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(BSG_ENODEV, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (static_cast<int>(g_ctx.size()) <= dev) g_ctx.resize(dev + 1);
  if (!g_ctx[dev]) {
    g_ctx[dev] = std::make_unique<DeviceCtx>();
    g_ctx[dev]->device = dev;
  }
  DeviceCtx* c = g_ctx[dev].get();
  if (!c->ready) {
    BSG_CUDA(cudaEventCreateWithFlags(&c->ws_done, cudaEventDisableTiming));
    BSG_CUDA(c->scratch.ensure(64, true));
    c->ready = true;
  }
  *out = c;
  return BSG_OK;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  const char* x = static_cast<const char*>(a);
  const char* y = static_cast<const char*>(b);
  return an && bn && x < y + bn && y < x + an;
}

bsg_config resolve_cfg(const bsg_config* cfg) { return cfg ? *cfg : bsg_config_default(); }

// make_lcg / make_philox checks (bijection.hpp:26-27, 75-78), message text
// following the reference exceptions.
bsg_status build_params(int variant, int bits, uint64_t seed, int rounds, BijParams& p) {
  if (variant != bsg::kLcg && variant != bsg::kPhilox) return fail(BSG_EINVAL, "unknown bijection variant");
  if (bsg::make_params(variant, bits, seed, rounds, p) != 0) {
    if (variant == bsg::kLcg) return fail(BSG_EINVAL, "modulus_bits must be in [1, 63]");
    if (bits < 2 || bits > 63) return fail(BSG_EINVAL, "total_bits must be in [2, 63]");
    return fail(BSG_EINVAL, "num_rounds must be >= 3");
  }
  return BSG_OK;
}

// Orders this call after every earlier kernel of the context (any stream).
// True while `s` is being captured into a CUDA graph.  Captured calls skip the cross-stream workspace
// ordering (a graph replays on one stream; replays must not overlap other calls on the same device) and every
// host synchronisation; the workspaces must already be sized by one uncaptured call of the same shape.
bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return s != nullptr && cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}

bsg_status ws_begin(DeviceCtx* c, cudaStream_t s) {
  if (capturing(s)) return BSG_OK;
  BSG_CUDA(cudaStreamWaitEvent(s, c->ws_done, 0));
  return BSG_OK;
}
bsg_status ws_end(DeviceCtx* c, cudaStream_t s) {
  if (capturing(s)) return BSG_OK;
  BSG_CUDA(cudaEventRecord(c->ws_done, s));
  return BSG_OK;
}

// Sizes a workspace buffer for a call on stream s.  While s is being captured nothing may be allocated: the
// buffer must already be large enough (one uncaptured call of the same shape), and it is marked captured so a
// later larger uncaptured call retires it instead of freeing memory a graph still references.
bsg_status ensure_ws(DevBuf& b, size_t n, cudaStream_t s) {
  if (capturing(s)) {
    if (!b.p || b.bytes < n) return fail(BSG_EINVAL, "graph capture: run this call once uncaptured first");
    b.captured = true;
    return BSG_OK;
  }
  BSG_CUDA(b.ensure(n));
  return BSG_OK;
}

// Uploads the key schedule for generic-round Philox kernels.
bsg_status upload_keys(DeviceCtx* c, BijParams& p, uint64_t seed, cudaStream_t s) {
  if (p.variant != bsg::kPhilox || p.rounds == 24) return BSG_OK;
  std::vector<uint32_t> k(static_cast<size_t>(p.rounds));
  for (int i = 0; i < p.rounds; ++i) k[i] = bsg::round_key(seed, i);
  if (capturing(s)) {
    // the graph's copy node reads this host array at every replay: keep it for the context's lifetime
    if (c->keys.bytes < k.size() * 4) return fail(BSG_EINVAL, "graph capture: run this call once uncaptured first");
    c->keys.captured = true;
    c->captured_keys.push_back(std::move(k));
    const std::vector<uint32_t>& kk = c->captured_keys.back();
    BSG_CUDA(cudaMemcpyAsync(c->keys.p, kk.data(), kk.size() * 4, cudaMemcpyHostToDevice, s));
  } else {
    BSG_CUDA(c->keys.ensure(k.size() * 4));
    BSG_CUDA(cudaMemcpyAsync(c->keys.p, k.data(), k.size() * 4, cudaMemcpyHostToDevice, s));
    BSG_CUDA(cudaStreamSynchronize(s));  // k is a stack temporary
  }
  p.gkeys = static_cast<const uint32_t*>(c->keys.p);
  return BSG_OK;
}

// Prepares the look-back workspace for a compacting launch over `tiles`.
bsg_status lookback_prepare(DeviceCtx* c, uint64_t tiles, cudaStream_t s, bsg::Lookback& lb) {
  const size_t need = std::max<uint64_t>(tiles, 1) * sizeof(unsigned long long);
  lb.status = static_cast<unsigned long long*>(c->status.p);
  lb.tile_counter = static_cast<unsigned int*>(c->scratch.p);
  if (capturing(s)) {
    // A replayed graph cannot advance the epoch: it clears its status words and uses epoch 1, which
    // uncaptured launches never use.
    if (c->status.bytes < need) return fail(BSG_EINVAL, "graph capture: run this call once uncaptured first");
    c->status.captured = true;
    BSG_CUDA(cudaMemsetAsync(c->status.p, 0, need, s));
    lb.epoch = 1;
    return BSG_OK;
  }
  if (c->status.bytes < need) {
    BSG_CUDA(cudaStreamSynchronize(s));
    BSG_CUDA(c->status.ensure(need, true));
    lb.status = static_cast<unsigned long long*>(c->status.p);
    c->epoch = 1;
  }
  if (++c->epoch >= (1u << 22) || c->epoch < 2) {  // wrap: clear stale words once (epoch 1 is the graphs')
    BSG_CUDA(cudaMemsetAsync(c->status.p, 0, c->status.bytes, s));
    c->epoch = 2;
  }
  lb.epoch = c->epoch;
  return BSG_OK;
}

int native_code(uint32_t eb, const void* a, const void* b) {
  if (eb != 1 && eb != 2 && eb != 4 && eb != 8 && eb != 16) return -1;
  const uintptr_t al = eb;
  if ((reinterpret_cast<uintptr_t>(a) % al) || (reinterpret_cast<uintptr_t>(b) % al)) return -1;
  return static_cast<int>(eb);
}

// Device-pointer core: range [c0, c1) of an m >= 3 shuffle.  elem_code 0 =
// indices.  count_dev (device) receives the survivor count when non-null.
bsg_status stage_streams(DeviceCtx* c) {
  if (!c->cs_in) BSG_CUDA(cudaStreamCreateWithFlags(&c->cs_in, cudaStreamNonBlocking));
  if (!c->cs_out) BSG_CUDA(cudaStreamCreateWithFlags(&c->cs_out, cudaStreamNonBlocking));
  while (c->stage_ev.size() < 2 * kStageChunks + 2) {
    cudaEvent_t e;
    BSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->stage_ev.push_back(e);
  }
  return BSG_OK;
}

bsg_status run_range(DeviceCtx* c, uint64_t m, const bsg_config& cfg, uint64_t c0, uint64_t c1, const bsg::Src& src,
                     void* out, int elem_code, unsigned long long* count_dev, cudaStream_t s,
                     const StageIO* io = nullptr) {
  const int bits = bsg::domain_bits(m);
  BijParams p;
  BSG_TRY(build_params(cfg.variant, bits, cfg.seed, cfg.num_rounds, p));
  BSG_TRY(ws_begin(c, s));
  BSG_TRY(upload_keys(c, p, cfg.seed, s));
  const bool pow2 = (m == (1ULL << bits));
  // Partitioned path: whole power-of-two domains, and whole non-power-of-two domains with elements <= 8 B
  // (routed by counter, compacted by counter rank in the last pass).
  if (!g_force_compact && g_path != 1 && elem_code > 0 && src.nshards == 0 && c0 == 0 && c1 == (1ULL << bits) &&
      (pow2 || elem_code <= 8) && bsg::partition_eligible(elem_code, bits, !pow2) &&
      auto_partition(m, static_cast<uint64_t>(elem_code))) {
    const size_t need = bsg::partition_workspace_bytes(elem_code, bits, !pow2);
    // while capturing, never allocate (it would invalidate the capture): use the workspace only if it is sized
    const bool cap = capturing(s);
    const cudaError_t ae = cap ? (c->part.p && c->part.bytes >= need ? cudaSuccess : cudaErrorNotReady)
                               : c->part.ensure(need);
    if (ae == cudaSuccess) {
      if (cap) c->part.captured = true;
      bsg::PartitionLaunch P;
      bsg::partition_layout(elem_code, bits, !pow2, c->part.p, P);
      P.in = src.base;
      P.out = out;
      P.m = m;
      P.p = p;
      if (io) {
        BSG_TRY(stage_streams(c));
        P.h_in = io->h_in;
        P.h_out = pow2 ? io->h_out : nullptr;  // padded outputs leave by one copy after the rank placement
        P.cs_in = c->cs_in;
        P.cs_out = c->cs_out;
        P.ev = c->stage_ev.data();
        P.chunks = kStageChunks;
      }
      BSG_CUDA(bsg::launch_partition(elem_code, P, s));
      if (io && io->h_out && !P.h_out)
        BSG_CUDA(cudaMemcpyAsync(io->h_out, out, io->out_bytes, cudaMemcpyDeviceToHost, s));
      if (count_dev) BSG_CUDA(bsg::launch_store_u64(count_dev, m, s));
      return ws_end(c, s);
    }
    cudaGetLastError();  // workspace did not fit: the single-pass kernel needs none
  }
  bsg::ShuffleLaunch L;
  L.src = src;
  L.out = out;
  L.m = m;
  L.c0 = c0;
  L.c1 = c1;
  L.p = p;
  L.compact = !pow2 || g_force_compact;
  L.count_out = count_dev;
  if (L.compact) {
    const uint64_t tile = bsg::kCompactTileMin;  // sizes the status words for the smallest tile
    BSG_TRY(lookback_prepare(c, (c1 - c0 + tile - 1) / tile, s, L.lb));
  }
  if (io && io->h_in)
    BSG_CUDA(cudaMemcpyAsync(const_cast<void*>(src.base), io->h_in, io->in_bytes, cudaMemcpyHostToDevice, s));
  if (c1 > c0) BSG_CUDA(bsg::launch_shuffle(elem_code, L, s));
  if (io && io->h_out) BSG_CUDA(cudaMemcpyAsync(io->h_out, out, io->out_bytes, cudaMemcpyDeviceToHost, s));
  if (count_dev && (!L.compact || c1 == c0)) BSG_CUDA(bsg::launch_store_u64(count_dev, c1 - c0, s));
  return ws_end(c, s);
}

// Device-pointer shuffle of m elements (all sizes, m >= 0).
bsg_status shuffle_device(DeviceCtx* c, const void* in, void* out, uint64_t m, uint32_t eb, const bsg_config& cfg,
                          cudaStream_t s) {
  if (m == 0) return BSG_OK;
  const bool idx = (in == nullptr);
  const size_t ob = idx ? 8 : eb;
  if (m <= 2) {  // shuffle.hpp:228-240 / 249-259: variant and rounds ignored
    const uint64_t bit = (m == 2) ? (bsg::mix64(cfg.seed) & 1) : 0;
    if (idx) {
      uint64_t* o = static_cast<uint64_t*>(out);
      BSG_CUDA(bsg::launch_store_u64(reinterpret_cast<unsigned long long*>(o), bit, s));
      if (m == 2) BSG_CUDA(bsg::launch_store_u64(reinterpret_cast<unsigned long long*>(o + 1), bit ^ 1, s));
    } else {
      for (uint64_t k = 0; k < m; ++k)
        BSG_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + k * ob, static_cast<const char*>(in) + (k ^ bit) * eb, eb,
                                 cudaMemcpyDeviceToDevice, s));
    }
    return BSG_OK;
  }
  bsg::Src src;
  src.base = in;
  const int bits = bsg::domain_bits(m);
  const uint64_t n = (bits >= 64) ? 0 : (1ULL << bits);
  if (bits > 63) return fail(BSG_EINVAL, cfg.variant == bsg::kLcg ? "modulus_bits must be in [1, 63]"
                                                                     : "total_bits must be in [2, 63]");
  if (idx) return run_range(c, m, cfg, 0, n, src, out, 0, nullptr, s);
  const int code = native_code(eb, in, out);
  if (code > 0) return run_range(c, m, cfg, 0, n, src, out, code, nullptr, s);
  // Other element sizes: permutation first, then a record gather.
  BSG_TRY(ensure_ws(c->st_idx, m * 8, s));
  BSG_TRY(run_range(c, m, cfg, 0, n, bsg::Src{}, c->st_idx.p, 0, nullptr, s));
  BSG_TRY(ws_begin(c, s));
  BSG_CUDA(bsg::launch_gather_bytes(in, static_cast<const uint64_t*>(c->st_idx.p), out, m, eb, s));
  return ws_end(c, s);
}

template <typename Fn>
bsg_status with_ctx(Fn&& fn) {
  DeviceCtx* c = nullptr;
  BSG_TRY(current_ctx(&c));
  std::lock_guard<std::mutex> lk(c->mu);
  t_err.clear();
  return fn(c);
}

}  // namespace

extern "C" {

bsg_config bsg_config_default(void) {
  bsg_config c;
  c.seed = 0;
  c.variant = BSG_VARIABLE_PHILOX;
  c.num_rounds = 24;
  c.workers = 0;
  c.reserved = 0;
  return c;
}

uint64_t bsg_mix64(uint64_t z) { return bsg::mix64(z); }

bsg_status bsg_derive_round_keys(uint64_t seed, int32_t rounds, uint32_t* keys_out) {
  if (rounds < 1) return fail(BSG_EINVAL, "num_rounds must be >= 1");
  for (int i = 0; i < rounds; ++i) keys_out[i] = bsg::round_key(seed, i);
  return BSG_OK;
}

int32_t bsg_domain_bits(uint64_t m) { return bsg::domain_bits(m); }

bsg_status bsg_make_lcg(int32_t bits, uint64_t seed, uint64_t* a, uint64_t* c) {
  BijParams p;
  BSG_TRY(build_params(bsg::kLcg, bits, seed, 0, p));
  *a = p.lcg_a;
  *c = p.lcg_c;
  return BSG_OK;
}

bsg_status bsg_lcg_apply(int32_t bits, uint64_t a, uint64_t c, uint64_t x, uint64_t* y) {
  const uint64_t mask = bits >= 64 ? ~0ULL : ((1ULL << bits) - 1);  // LcgParams::domain_mask
  if (x > mask) return fail(BSG_ERANGE, "lcg_apply: x outside [0, 2^bits)");
  *y = (a * x + c) & mask;
  return BSG_OK;
}

bsg_status bsg_philox_apply(int32_t bits, uint64_t seed, int32_t rounds, uint64_t x, uint64_t* y) {
  BijParams p;
  BSG_TRY(build_params(bsg::kPhilox, bits, seed, rounds, p));
  if ((x >> bits) != 0) return fail(BSG_ERANGE, "philox_apply: x outside [0, 2^total_bits)");
  *y = bsg::host_apply(p, seed, x, false);
  return BSG_OK;
}

bsg_status bsg_philox_invert(int32_t bits, uint64_t seed, int32_t rounds, uint64_t y, uint64_t* x) {
  BijParams p;
  BSG_TRY(build_params(bsg::kPhilox, bits, seed, rounds, p));
  if ((y >> bits) != 0) return fail(BSG_ERANGE, "philox_invert: y outside [0, 2^total_bits)");
  *x = bsg::host_apply(p, seed, y, true);
  return BSG_OK;
}

// philox_apply / philox_invert over caller-held parameters (bijection.hpp:94-143), host scalar, 64-bit state as
// in the reference so that any field combination it accepts gives its result.
static bsg_status check_philox_params(const bsg_philox_params* p) {
  if (!p) return fail(BSG_EINVAL, "null params");
  if (p->left_side_bits < 0 || p->left_side_bits > 63 || p->right_side_bits < 0 || p->right_side_bits > 63 ||
      p->right_side_bits < p->left_side_bits)
    return fail(BSG_EINVAL, "side widths must satisfy 0 <= left_side_bits <= right_side_bits <= 63");
  if (p->num_rounds > 0 && (!p->round_keys || p->num_keys < static_cast<uint64_t>(p->num_rounds)))
    return fail(BSG_EINVAL, "round_keys holds fewer keys than num_rounds");
  return BSG_OK;
}

bsg_status bsg_philox_apply_params(const bsg_philox_params* p, uint64_t x, uint64_t* y) {
  BSG_TRY(check_philox_params(p));
  if (p->total_bits < 64 && p->total_bits >= 0 && (x >> p->total_bits) != 0)
    return fail(BSG_ERANGE, "philox_apply: x outside [0, 2^total_bits)");
  const int L = p->left_side_bits, R = p->right_side_bits, d = R - L;
  uint64_t a = x >> R, b = x & p->right_side_mask;
  for (int i = 0; i < p->num_rounds; ++i) {
    const uint64_t w = bsg::kM0 * a;  // 64-bit product: high word feeds the left side, low word the right
    const uint64_t nb = ((w & 0xFFFFFFFFULL) << d) | (b >> L);
    a = ((w >> 32) ^ p->round_keys[i] ^ b) & p->left_side_mask;
    b = nb & p->right_side_mask;
  }
  *y = (a << R) | b;
  return BSG_OK;
}

bsg_status bsg_philox_invert_params(const bsg_philox_params* p, uint64_t y, uint64_t* x) {
  BSG_TRY(check_philox_params(p));
  if (p->total_bits < 64 && p->total_bits >= 0 && (y >> p->total_bits) != 0)
    return fail(BSG_ERANGE, "philox_invert: y outside [0, 2^total_bits)");
  const int L = p->left_side_bits, R = p->right_side_bits, d = R - L;
  uint64_t a = y >> R, b = y & p->right_side_mask;
  for (int i = p->num_rounds - 1; i >= 0; --i) {
    // b = (lo << d | spare) & right_mask with lo = M0 * prev_a mod 2^32: recover prev_a from lo mod 2^L through
    // M0^-1, then the previous right side from the round's XOR (its top d bits are the spare bits)
    const uint64_t prev_a = (bsg::kM0Inv * ((b >> d) & p->left_side_mask)) & p->left_side_mask;
    const uint64_t hi = (bsg::kM0 * prev_a) >> 32;
    const uint64_t prev_b = ((hi ^ p->round_keys[i] ^ a) & p->left_side_mask) | ((b & ((1ULL << d) - 1)) << L);
    a = prev_a;
    b = prev_b;
  }
  *x = (a << R) | b;
  return BSG_OK;
}

bsg_status bsg_bijection_apply(int32_t variant, int32_t bits, uint64_t seed, int32_t rounds, int32_t inverse,
                               const uint64_t* x, uint64_t start, uint64_t* y, uint64_t n, void* stream) {
  BijParams p;
  BSG_TRY(build_params(variant, bits, seed, rounds, p));
  if (n == 0) return BSG_OK;
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    const bool xd = x && is_device_ptr(x), yd = is_device_ptr(y);
    if (x && !xd) {
      for (uint64_t i = 0; i < n; ++i)
        if (x[i] > p.mask) return fail(BSG_ERANGE, "bijection_apply: x outside [0, 2^bits)");
    } else if (!x && (start > p.mask || n - 1 > p.mask - start)) {
      return fail(BSG_ERANGE, "bijection_apply: counters outside [0, 2^bits)");
    }
    const uint64_t* dx = x;
    uint64_t* dy = y;
    // staging buffers may still be read by an earlier asynchronous call of this context on another stream
    BSG_TRY(ws_begin(c, s));
    if (x && !xd) {
      BSG_CUDA(c->st_in.ensure(n * 8));
      BSG_CUDA(cudaMemcpyAsync(c->st_in.p, x, n * 8, cudaMemcpyHostToDevice, s));
      dx = static_cast<const uint64_t*>(c->st_in.p);
    }
    if (!yd) {
      BSG_CUDA(c->st_out.ensure(n * 8));
      dy = static_cast<uint64_t*>(c->st_out.p);
    }
    BSG_TRY(ws_begin(c, s));
    BSG_TRY(upload_keys(c, p, seed, s));
    BSG_CUDA(bsg::launch_map(dx, dy, n, start, p, inverse != 0, s));
    BSG_TRY(ws_end(c, s));
    if (!yd) {
      BSG_CUDA(cudaMemcpyAsync(y, dy, n * 8, cudaMemcpyDeviceToHost, s));
      BSG_CUDA(cudaStreamSynchronize(s));
    }
    return BSG_OK;
  });
}

bsg_status bsg_shuffle_indices(uint64_t m, const bsg_config* cfg_in, uint64_t* out, void* stream) {
  const bsg_config cfg = resolve_cfg(cfg_in);
  if (m == 0) return BSG_OK;
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    if (is_device_ptr(out)) return shuffle_device(c, nullptr, out, m, 8, cfg, s);
    BSG_CUDA(c->st_out.ensure(m * 8));
    BSG_TRY(shuffle_device(c, nullptr, c->st_out.p, m, 8, cfg, s));
    BSG_CUDA(cudaMemcpyAsync(out, c->st_out.p, m * 8, cudaMemcpyDeviceToHost, s));
    BSG_CUDA(cudaStreamSynchronize(s));
    return BSG_OK;
  });
}

bsg_status bsg_shuffle_values(const void* in, void* out, uint64_t m, uint32_t elem_bytes, const bsg_config* cfg_in,
                              void* stream) {
  const bsg_config cfg = resolve_cfg(cfg_in);
  if (in != nullptr && in == out) return fail(BSG_EALIAS, "shuffle_values_into: out aliases input");
  if (m == 0) return BSG_OK;
  if (elem_bytes == 0) return fail(BSG_EINVAL, "elem_bytes must be >= 1");
  if (!in || !out) return fail(BSG_EINVAL, "null pointer");
  const size_t bytes = m * static_cast<size_t>(elem_bytes);
  if (overlaps(in, bytes, out, bytes)) return fail(BSG_EALIAS, "shuffle_values_into: out aliases input");
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    const bool din = is_device_ptr(in), dout = is_device_ptr(out);
    if (din && dout) return shuffle_device(c, in, out, m, elem_bytes, cfg, s);
    const void* di = in;
    void* dO = out;
    BSG_TRY(ws_begin(c, s));  // order the staging writes after earlier asynchronous users of st_*
    const int code = native_code(elem_bytes, in, out);
    if (!din && !dout && m >= 3 && code > 0) {
      // both buffers on the host: the copies travel with the shuffle (chunked under the partitioned passes)
      BSG_CUDA(c->st_in.ensure(bytes));
      BSG_CUDA(c->st_out.ensure(bytes));
      StageIO io;
      io.h_in = in;
      io.h_out = out;
      io.in_bytes = io.out_bytes = bytes;
      bsg::Src src;
      src.base = c->st_in.p;
      BSG_TRY(run_range(c, m, cfg, 0, 1ULL << bsg::domain_bits(m), src, c->st_out.p, code, nullptr, s, &io));
      BSG_CUDA(cudaStreamSynchronize(s));
      return BSG_OK;
    }
    if (!din) {
      BSG_CUDA(c->st_in.ensure(bytes));
      BSG_CUDA(cudaMemcpyAsync(c->st_in.p, in, bytes, cudaMemcpyHostToDevice, s));
      di = c->st_in.p;
    }
    if (!dout) {
      BSG_CUDA(c->st_out.ensure(bytes));
      dO = c->st_out.p;
    }
    BSG_TRY(shuffle_device(c, di, dO, m, elem_bytes, cfg, s));
    if (!dout) BSG_CUDA(cudaMemcpyAsync(out, dO, bytes, cudaMemcpyDeviceToHost, s));
    BSG_CUDA(cudaStreamSynchronize(s));
    return BSG_OK;
  });
}

namespace {
// Device part of bsg_shuffle_values_batched (device pointers, stream-ordered): row b shuffled with seed + b.
bsg_status batched_device(DeviceCtx* c, const void* di, void* dO, uint64_t batch, uint64_t m, uint32_t elem_bytes,
                          const bsg_config& cfg, cudaStream_t s) {
  const int bits = bsg::domain_bits(m);
  const int code = native_code(elem_bytes, di, dO);
  if (m >= 3 && code > 0 && bsg::batched_supported(code, static_cast<uint32_t>(m), bits, cfg.num_rounds)) {
    bsg::BatchedLaunch B;
    B.in = di;
    B.out = dO;
    B.batch = batch;
    B.m = static_cast<uint32_t>(m);
    B.seed = cfg.seed;
    BSG_TRY(build_params(cfg.variant, bits, cfg.seed, cfg.num_rounds, B.p));
    BSG_TRY(ws_begin(c, s));
    BSG_CUDA(bsg::launch_batched(code, B, s));
    BSG_TRY(ws_end(c, s));
    return BSG_OK;
  }
  const size_t row = m * static_cast<size_t>(elem_bytes);
  for (uint64_t b = 0; b < batch; ++b) {
    bsg_config cb = cfg;
    cb.seed = cfg.seed + b;
    BSG_TRY(shuffle_device(c, static_cast<const char*>(di) + b * row, static_cast<char*>(dO) + b * row, m,
                           elem_bytes, cb, s));
  }
  return BSG_OK;
}
}  // namespace

bsg_status bsg_shuffle_values_batched(const void* in, void* out, uint64_t batch, uint64_t m, uint32_t elem_bytes,
                                      const bsg_config* cfg_in, void* stream) {
  const bsg_config cfg = resolve_cfg(cfg_in);
  if (in != nullptr && in == out) return fail(BSG_EALIAS, "shuffle_values_batched: out aliases input");
  if (m == 0 || batch == 0) return BSG_OK;
  if (elem_bytes == 0) return fail(BSG_EINVAL, "elem_bytes must be >= 1");
  if (!in || !out) return fail(BSG_EINVAL, "null pointer");
  const size_t bytes = batch * m * static_cast<size_t>(elem_bytes);
  if (overlaps(in, bytes, out, bytes)) return fail(BSG_EALIAS, "shuffle_values_batched: out aliases input");
  const int bits = bsg::domain_bits(m);
  if (m >= 3) {
    BijParams p;
    BSG_TRY(build_params(cfg.variant, bits, cfg.seed, cfg.num_rounds, p));
  }
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    const bool din = is_device_ptr(in), dout = is_device_ptr(out);
    const void* di = in;
    void* dO = out;
    if (!din || !dout) BSG_TRY(ws_begin(c, s));  // staging writes after earlier asynchronous users of st_*
    if (!din) {
      BSG_CUDA(c->st_in.ensure(bytes));
      BSG_CUDA(cudaMemcpyAsync(c->st_in.p, in, bytes, cudaMemcpyHostToDevice, s));
      di = c->st_in.p;
    }
    if (!dout) {
      BSG_CUDA(c->st_out.ensure(bytes));
      dO = c->st_out.p;
    }
    BSG_TRY(batched_device(c, di, dO, batch, m, elem_bytes, cfg, s));
    if (!dout) BSG_CUDA(cudaMemcpyAsync(out, dO, bytes, cudaMemcpyDeviceToHost, s));
    if (!din || !dout) BSG_CUDA(cudaStreamSynchronize(s));
    return BSG_OK;
  });
}

bsg_status bsg_gather(const void* src, uint64_t src_len, const uint64_t* idx, void* out, uint64_t n,
                      uint32_t elem_bytes, void* stream) {
  if (out != nullptr && (out == src || out == static_cast<const void*>(idx)))
    return fail(BSG_EALIAS, "gather_into: out aliases an input");
  if (n == 0) return BSG_OK;
  if (elem_bytes == 0 || !src || !idx || !out) return fail(BSG_EINVAL, "invalid gather arguments");
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    const bool ds = is_device_ptr(src), di = is_device_ptr(idx), dout = is_device_ptr(out);
    const void* S = src;
    const uint64_t* I = idx;
    void* O = out;
    const size_t sb = src_len * static_cast<size_t>(elem_bytes), ob = n * static_cast<size_t>(elem_bytes);
    if (!ds || !di || !dout) BSG_TRY(ws_begin(c, s));  // staging writes after earlier asynchronous users of st_*
    if (!ds) {
      BSG_CUDA(c->st_in.ensure(sb));
      BSG_CUDA(cudaMemcpyAsync(c->st_in.p, src, sb, cudaMemcpyHostToDevice, s));
      S = c->st_in.p;
    }
    if (!di) {
      BSG_CUDA(c->st_idx.ensure(n * 8));
      BSG_CUDA(cudaMemcpyAsync(c->st_idx.p, idx, n * 8, cudaMemcpyHostToDevice, s));
      I = static_cast<const uint64_t*>(c->st_idx.p);
    }
    if (!dout) {
      BSG_CUDA(c->st_out.ensure(ob));
      O = c->st_out.p;
    }
    BSG_TRY(ws_begin(c, s));
    const int code = native_code(elem_bytes, S, O);
    if (code > 0) BSG_CUDA(bsg::launch_gather(code, S, I, O, n, s));
    else BSG_CUDA(bsg::launch_gather_bytes(S, I, O, n, elem_bytes, s));
    BSG_TRY(ws_end(c, s));
    if (!dout) BSG_CUDA(cudaMemcpyAsync(out, O, ob, cudaMemcpyDeviceToHost, s));
    if (!ds || !di || !dout) BSG_CUDA(cudaStreamSynchronize(s));
    return BSG_OK;
  });
}

static bsg_status make_src(const void* in, const bsg_shards* sh, uint64_t m, bsg::Src& src) {
  src = bsg::Src{};
  if (sh && sh->count > 0) {
    if (sh->count > bsg::kMaxShards) return fail(BSG_EINVAL, "at most 16 input shards");
    if (sh->shard_elems == 0 || static_cast<uint64_t>(sh->count) * sh->shard_elems < m)
      return fail(BSG_EINVAL, "input shards do not cover m elements");
    for (int g = 0; g < sh->count; ++g) src.shard[g] = sh->ptrs[g];
    src.nshards = sh->count;
    src.shard_elems = sh->shard_elems;
    src.shard_shift = -1;
    if ((sh->shard_elems & (sh->shard_elems - 1)) == 0) {
      int sft = 0;
      while ((1ULL << sft) < sh->shard_elems) ++sft;
      src.shard_shift = sft;
    }
  } else {
    src.base = in;
  }
  return BSG_OK;
}

bsg_status bsg_shuffle_range(uint64_t m, const bsg_config* cfg_in, uint64_t counter_begin, uint64_t counter_end,
                             const void* in, const bsg_shards* in_shards, void* out, uint32_t elem_bytes,
                             uint64_t* count_out, void* stream) {
  const bsg_config cfg = resolve_cfg(cfg_in);
  if (m < 3) return fail(BSG_EINVAL, "shuffle_range needs m >= 3 (m <= 2 has no padded domain)");
  const int bits = bsg::domain_bits(m);
  BijParams p;
  BSG_TRY(build_params(cfg.variant, bits, cfg.seed, cfg.num_rounds, p));
  const uint64_t n = 1ULL << bits;
  if (counter_begin > counter_end || counter_end > n) return fail(BSG_ERANGE, "counter range outside [0, 2^bits)");
  const bool indices = (in == nullptr) && (in_shards == nullptr || in_shards->count == 0);
  bsg::Src src;
  BSG_TRY(make_src(in, in_shards, m, src));
  int code = 0;
  if (!indices) {
    code = native_code(elem_bytes, src.nshards ? src.shard[0] : in, out);
    if (code < 0) return fail(BSG_EUNSUPPORTED, "shuffle_range: elem_bytes must be 1, 2, 4, 8 or 16 (aligned)");
  }
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    if (!is_device_ptr(out)) return fail(BSG_EINVAL, "shuffle_range: out must be device memory");
    const bool count_dev = count_out && is_device_ptr(count_out);
    unsigned long long* cd =
        count_dev ? reinterpret_cast<unsigned long long*>(count_out)
                  : reinterpret_cast<unsigned long long*>(static_cast<char*>(c->scratch.p) + 8);
    BSG_TRY(run_range(c, m, cfg, counter_begin, counter_end, src, out, code, cd, s));
    if (count_out && !count_dev) {
      BSG_CUDA(cudaMemcpyAsync(count_out, cd, 8, cudaMemcpyDeviceToHost, s));
      BSG_CUDA(cudaStreamSynchronize(s));
    }
    return BSG_OK;
  });
}

bsg_status bsg_range_count(uint64_t m, const bsg_config* cfg_in, uint64_t counter_begin, uint64_t counter_end,
                           uint64_t* count, void* stream) {
  const bsg_config cfg = resolve_cfg(cfg_in);
  if (m < 3) return fail(BSG_EINVAL, "range_count needs m >= 3");
  const int bits = bsg::domain_bits(m);
  BijParams p;
  BSG_TRY(build_params(cfg.variant, bits, cfg.seed, cfg.num_rounds, p));
  const uint64_t n = 1ULL << bits;
  if (counter_begin > counter_end || counter_end > n) return fail(BSG_ERANGE, "counter range outside [0, 2^bits)");
  if (m == n) {
    *count = counter_end - counter_begin;
    return BSG_OK;
  }
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    auto* cd = reinterpret_cast<unsigned long long*>(static_cast<char*>(c->scratch.p) + 8);
    BSG_TRY(ws_begin(c, s));
    BSG_TRY(upload_keys(c, p, cfg.seed, s));
    BSG_CUDA(bsg::launch_count(m, counter_begin, counter_end, p, cd, s));
    BSG_TRY(ws_end(c, s));
    BSG_CUDA(cudaMemcpyAsync(count, cd, 8, cudaMemcpyDeviceToHost, s));
    BSG_CUDA(cudaStreamSynchronize(s));
    return BSG_OK;
  });
}

bsg_status bsg_dist_counter_range(uint64_t m, int32_t rank, int32_t world, uint64_t* begin, uint64_t* end) {
  if (world < 1 || rank < 0 || rank >= world) return fail(BSG_EINVAL, "rank/world out of range");
  if (m < 3) return fail(BSG_EINVAL, "distributed shuffle needs m >= 3");
  const int bits = bsg::domain_bits(m);
  if (bits > 63) return fail(BSG_EINVAL, "total_bits must be in [2, 63]");
  const uint64_t n = 1ULL << bits;
  const uint64_t base = n / world, rem = n % world;
  *begin = rank * base + std::min<uint64_t>(rank, rem);
  *end = *begin + base + (static_cast<uint64_t>(rank) < rem ? 1 : 0);
  return BSG_OK;
}

bsg_status bsg_dist_shuffle_values(uint64_t m, const bsg_config* cfg_in, int32_t rank, int32_t world, const void* in,
                                   const bsg_shards* in_shards, void* out, uint32_t elem_bytes,
                                   bsg_allgather_u64_fn allgather, void* user, uint64_t* global_offset,
                                   uint64_t* local_count, void* stream) {
  if (!allgather) return fail(BSG_EINVAL, "allgather callback required");
  uint64_t b = 0, e = 0;
  BSG_TRY(bsg_dist_counter_range(m, rank, world, &b, &e));
  uint64_t cnt = 0;
  BSG_TRY(bsg_shuffle_range(m, cfg_in, b, e, in, in_shards, out, elem_bytes, &cnt, stream));
  std::vector<uint64_t> all(static_cast<size_t>(world), 0);
  if (allgather(&cnt, all.data(), user) != 0) return fail(BSG_ECUDA, "allgather callback failed");
  uint64_t off = 0, tot = 0;
  for (int r = 0; r < world; ++r) {
    if (r < rank) off += all[r];
    tot += all[r];
  }
  if (tot != m) return fail(BSG_ECUDA, "survivor counts do not sum to m (inconsistent ranks?)");
  *global_offset = off;
  *local_count = cnt;
  return BSG_OK;
}

bsg_status bsg_route_by_dest(const void* in, uint64_t n_local, uint64_t global_offset, uint64_t m,
                             const bsg_config* cfg_in, int32_t nparts, void* out_values, uint32_t* out_dest,
                             uint64_t* part_counts, uint32_t elem_bytes, void* stream) {
  const bsg_config cfg = resolve_cfg(cfg_in);
  if (m < 16 || (m & (m - 1))) return fail(BSG_EINVAL, "route_by_dest: m must be a power of two >= 16");
  const int bits = bsg::domain_bits(m);
  if (bits > 32) return fail(BSG_EUNSUPPORTED, "route_by_dest: m <= 2^32");
  if (nparts < 1 || nparts > 64 || (nparts & (nparts - 1)) || m % static_cast<uint64_t>(nparts))
    return fail(BSG_EINVAL, "route_by_dest: nparts must be a power of two <= 64 dividing m");
  if (global_offset > m || n_local > m - global_offset) return fail(BSG_ERANGE, "route_by_dest: local range outside m");
  if (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16)
    return fail(BSG_EUNSUPPORTED, "route_by_dest: elem_bytes must be 4, 8 or 16");
  BijParams p;
  BSG_TRY(build_params(cfg.variant, bits, cfg.seed, cfg.num_rounds, p));
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    if (!is_device_ptr(in) || !is_device_ptr(out_values) || !is_device_ptr(out_dest))
      return fail(BSG_EINVAL, "route_by_dest: device pointers only");
    BSG_TRY(ensure_ws(c->st_idx, std::max<uint64_t>(n_local, 1) * 4 + 2 * 64 * 8, s));
    char* w = static_cast<char*>(c->st_idx.p);
    bsg::RouteLaunch R;
    R.in = in;
    R.n = n_local;
    R.offset = global_offset;
    R.part_size = m / nparts;
    R.nparts = nparts;
    R.p = p;
    R.counts = reinterpret_cast<unsigned long long*>(w);
    R.cursors = reinterpret_cast<unsigned long long*>(w + 64 * 8);
    R.tmp_dest = reinterpret_cast<uint32_t*>(w + 2 * 64 * 8);
    R.out_values = out_values;
    R.out_dest = out_dest;
    BSG_TRY(ws_begin(c, s));
    BSG_TRY(upload_keys(c, R.p, cfg.seed, s));
    if (n_local) BSG_CUDA(bsg::launch_route(static_cast<int>(elem_bytes), R, s));
    else BSG_CUDA(cudaMemsetAsync(R.counts, 0, 64 * 8, s));
    BSG_TRY(ws_end(c, s));
    if (part_counts) {
      BSG_CUDA(cudaMemcpyAsync(part_counts, R.counts, sizeof(uint64_t) * nparts, cudaMemcpyDeviceToHost, s));
      BSG_CUDA(cudaStreamSynchronize(s));
    }
    return BSG_OK;
  });
}

namespace {
bsg_status xpart_check(uint64_t m, uint32_t elem_bytes, int32_t world, int* G) {
  if (m < 16 || (m & (m - 1))) return fail(BSG_EINVAL, "xpart: m must be a power of two >= 16");
  *G = bsg::domain_bits(m);
  if (!bsg::xpart_eligible(static_cast<int>(elem_bytes), *G, world))
    return fail(BSG_EUNSUPPORTED, "xpart: two ranks, 4- or 8-byte elements, 2^16 <= m <= 2^32");
  return BSG_OK;
}
}  // namespace

bsg_status bsg_xpart_workspace_bytes(uint64_t m, uint32_t elem_bytes, int32_t world, uint64_t* bytes) {
  int G = 0;
  BSG_TRY(xpart_check(m, elem_bytes, world, &G));
  if (!bytes) return fail(BSG_EINVAL, "null pointer");
  *bytes = bsg::xpart_workspace_bytes(static_cast<int>(elem_bytes), G);
  return BSG_OK;
}

bsg_status bsg_xpart_route(const void* in_half, uint64_t m, uint32_t elem_bytes, const bsg_config* cfg_in,
                           int32_t rank, int32_t world, void* const* workspaces, void* stream) {
  const bsg_config cfg = resolve_cfg(cfg_in);
  int G = 0;
  BSG_TRY(xpart_check(m, elem_bytes, world, &G));
  if (rank < 0 || rank >= world) return fail(BSG_EINVAL, "xpart: rank outside [0, world)");
  if (!in_half || !workspaces || !workspaces[0] || !workspaces[1]) return fail(BSG_EINVAL, "null pointer");
  BijParams p;
  BSG_TRY(build_params(cfg.variant, G, cfg.seed, cfg.num_rounds, p));
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    if (!is_device_ptr(in_half)) return fail(BSG_EINVAL, "xpart_route: device pointers only");
    bsg::XpartLaunch X;
    X.in = in_half;
    X.ws[0] = workspaces[0];
    X.ws[1] = workspaces[1];
    X.G = G;
    X.rank = rank;
    X.p = p;
    BSG_TRY(ws_begin(c, s));
    BSG_TRY(upload_keys(c, X.p, cfg.seed, s));
    BSG_CUDA(bsg::launch_xpart_route(static_cast<int>(elem_bytes), X, s));
    BSG_TRY(ws_end(c, s));
    return BSG_OK;
  });
}

bsg_status bsg_xpart_place(uint64_t m, uint32_t elem_bytes, int32_t rank, int32_t world, void* const* workspaces,
                           void* out_half, void* stream) {
  int G = 0;
  BSG_TRY(xpart_check(m, elem_bytes, world, &G));
  if (rank < 0 || rank >= world) return fail(BSG_EINVAL, "xpart: rank outside [0, world)");
  if (!out_half || !workspaces || !workspaces[0] || !workspaces[1]) return fail(BSG_EINVAL, "null pointer");
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    if (!is_device_ptr(out_half)) return fail(BSG_EINVAL, "xpart_place: device pointers only");
    bsg::XpartLaunch X;
    X.out = out_half;
    X.ws[0] = workspaces[0];
    X.ws[1] = workspaces[1];
    X.G = G;
    X.rank = rank;
    BSG_CUDA(bsg::launch_xpart_place(static_cast<int>(elem_bytes), X, s));
    return BSG_OK;
  });
}

bsg_status bsg_scatter_permutation(const void* values, const uint32_t* dest, uint64_t n, void* out,
                                   uint32_t elem_bytes, void* stream) {
  if (n == 0) return BSG_OK;
  if (values == out) return fail(BSG_EALIAS, "scatter_permutation: out aliases input");
  if (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16)
    return fail(BSG_EUNSUPPORTED, "scatter_permutation: elem_bytes must be 4, 8 or 16");
  if (n > (1ULL << 32)) return fail(BSG_EUNSUPPORTED, "scatter_permutation: n <= 2^32");
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    if (!is_device_ptr(values) || !is_device_ptr(dest) || !is_device_ptr(out))
      return fail(BSG_EINVAL, "scatter_permutation: device pointers only");
    const int code = static_cast<int>(elem_bytes);
    int bits = 0;
    while ((1ULL << bits) < n) ++bits;
    BSG_TRY(ws_begin(c, s));
    const bool pow2 = (1ULL << bits) == n;
    if (pow2 && g_path != 1 && bsg::partition_eligible(code, bits) &&
        (g_path == 2 || n * static_cast<uint64_t>(elem_bytes) >= g_partition_min_bytes) &&
        (capturing(s) ? (c->part.p && c->part.bytes >= bsg::partition_workspace_bytes(code, bits))
                      : c->part.ensure(bsg::partition_workspace_bytes(code, bits)) == cudaSuccess)) {
      if (capturing(s)) c->part.captured = true;
      bsg::PartitionLaunch P;
      bsg::partition_layout(code, bits, false, c->part.p, P);
      P.in = values;
      P.out = out;
      P.dest_in = dest;
      P.p.bits = bits;
      BSG_CUDA(bsg::launch_partition(code, P, s));
    } else {
      cudaGetLastError();
      BSG_CUDA(bsg::launch_scatter_simple(code, values, dest, n, out, s));
    }
    return ws_end(c, s);
  });
}

// Base of the allocation containing p (driver cuMemGetAddressRange through the runtime's entry-point query, so
// libbsg does not link libcuda directly).
static bsg_status alloc_base(const void* p, uintptr_t* base) {
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  static GetRange fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<GetRange>(f);
  }();
  if (!fn) return fail(BSG_ECUDA, "cuMemGetAddressRange unavailable");
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0) return fail(BSG_EINVAL, "not a device allocation");
  *base = static_cast<uintptr_t>(b);
  return BSG_OK;
}

static std::mutex g_ipc_mu;
static std::vector<std::pair<void*, void*>> g_ipc_open;  // (returned pointer, mapped allocation base)

bsg_status bsg_ipc_export(const void* dev_ptr, unsigned char handle_out[BSG_IPC_HANDLE_BYTES]) {
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) + 8 <= BSG_IPC_HANDLE_BYTES, "ipc handle size");
  uintptr_t base = 0;
  BSG_TRY(alloc_base(dev_ptr, &base));
  BSG_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  const uint64_t off = reinterpret_cast<uintptr_t>(dev_ptr) - base;
  std::memset(handle_out, 0, BSG_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  std::memcpy(handle_out + sizeof(h), &off, 8);
  return BSG_OK;
}

bsg_status bsg_ipc_open(const unsigned char handle[BSG_IPC_HANDLE_BYTES], void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  uint64_t off = 0;
  std::memcpy(&h, handle, sizeof(h));
  std::memcpy(&off, handle + sizeof(h), 8);
  void* base = nullptr;
  BSG_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr_out = static_cast<char*>(base) + off;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_open.emplace_back(*dev_ptr_out, base);
  return BSG_OK;
}

bsg_status bsg_ipc_close(void* dev_ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (auto it = g_ipc_open.begin(); it != g_ipc_open.end(); ++it)
      if (it->first == dev_ptr) {
        base = it->second;
        g_ipc_open.erase(it);
        break;
      }
  }
  if (!base) return fail(BSG_EINVAL, "ipc_close: pointer was not returned by bsg_ipc_open");
  BSG_CUDA(cudaIpcCloseMemHandle(base));
  return BSG_OK;
}

bsg_status bsg_sort_shuffle_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t seed, void* stream) {
  if (n == 0) return BSG_OK;
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    cudaStream_t s = as_stream(stream);
    if (!is_device_ptr(in) || !is_device_ptr(out)) return fail(BSG_EINVAL, "sort_shuffle: device pointers only");
    size_t need = 0;
    BSG_CUDA(bsg::sort_shuffle_u64(in, out, n, seed, nullptr, &need, s));
    BSG_CUDA(c->st_tmp.ensure(need));
    size_t have = c->st_tmp.bytes;
    BSG_TRY(ws_begin(c, s));
    BSG_CUDA(bsg::sort_shuffle_u64(in, out, n, seed, c->st_tmp.p, &have, s));
    return ws_end(c, s);
  });
}

}  // extern "C"

struct bsg_pipeline {
  struct Slot {
    DevBuf din, dout;
    cudaEvent_t h2d_done = nullptr, kernel_done = nullptr, d2h_done = nullptr;
    uint64_t ticket = ~0ULL;
  };
  int device = 0;
  uint64_t max_m = 0;
  uint32_t eb = 0;
  std::vector<Slot> slots;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  uint64_t next = 0;
};

extern "C" {

bsg_status bsg_pipeline_create(uint64_t max_m, uint32_t elem_bytes, int32_t depth, bsg_pipeline** out) {
  if (!out || elem_bytes == 0 || depth < 1 || depth > 8) return fail(BSG_EINVAL, "pipeline: bad arguments");
  DeviceCtx* c = nullptr;
  BSG_TRY(current_ctx(&c));
  auto p = std::make_unique<bsg_pipeline>();
  p->device = c->device;
  p->max_m = max_m;
  p->eb = elem_bytes;
  p->slots.resize(static_cast<size_t>(depth));
  const size_t bytes = std::max<uint64_t>(max_m, 1) * elem_bytes;
  for (auto& s : p->slots) {
    BSG_CUDA(s.din.ensure(bytes));
    BSG_CUDA(s.dout.ensure(bytes));
    BSG_CUDA(cudaEventCreateWithFlags(&s.h2d_done, cudaEventDisableTiming));
    BSG_CUDA(cudaEventCreateWithFlags(&s.kernel_done, cudaEventDisableTiming));
    BSG_CUDA(cudaEventCreateWithFlags(&s.d2h_done, cudaEventDisableTiming));
  }
  BSG_CUDA(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
  BSG_CUDA(cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking));
  BSG_CUDA(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
  *out = p.release();
  return BSG_OK;
}

bsg_status bsg_pipeline_submit(bsg_pipeline* p, const void* host_in, void* host_out, uint64_t m,
                               const bsg_config* cfg_in, uint64_t* ticket) {
  if (!p) return fail(BSG_EINVAL, "pipeline: null handle");
  if (m > p->max_m) return fail(BSG_EINVAL, "pipeline: m exceeds the capacity given at creation");
  if (host_in != nullptr && host_in == host_out) return fail(BSG_EALIAS, "shuffle_values_into: out aliases input");
  const bsg_config cfg = resolve_cfg(cfg_in);
  const uint64_t t = p->next++;
  auto& s = p->slots[t % p->slots.size()];
  const size_t bytes = m * static_cast<size_t>(p->eb);
  if (ticket) *ticket = t;
  s.ticket = t;
  if (m == 0) return BSG_OK;
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    // H2D into the slot once the slot's previous shuffle has consumed its input.
    BSG_CUDA(cudaStreamWaitEvent(p->s_h2d, s.kernel_done, 0));
    BSG_CUDA(cudaMemcpyAsync(s.din.p, host_in, bytes, cudaMemcpyHostToDevice, p->s_h2d));
    BSG_CUDA(cudaEventRecord(s.h2d_done, p->s_h2d));
    // Shuffle once the input landed and the slot's previous output left.
    BSG_CUDA(cudaStreamWaitEvent(p->s_comp, s.h2d_done, 0));
    BSG_CUDA(cudaStreamWaitEvent(p->s_comp, s.d2h_done, 0));
    BSG_TRY(shuffle_device(c, s.din.p, s.dout.p, m, p->eb, cfg, p->s_comp));
    BSG_CUDA(cudaEventRecord(s.kernel_done, p->s_comp));
    // D2H of the result.
    BSG_CUDA(cudaStreamWaitEvent(p->s_d2h, s.kernel_done, 0));
    BSG_CUDA(cudaMemcpyAsync(host_out, s.dout.p, bytes, cudaMemcpyDeviceToHost, p->s_d2h));
    BSG_CUDA(cudaEventRecord(s.d2h_done, p->s_d2h));
    return BSG_OK;
  });
}

bsg_status bsg_pipeline_submit_batched(bsg_pipeline* p, const void* host_in, void* host_out, uint64_t batch,
                                       uint64_t m, const bsg_config* cfg_in, uint64_t* ticket) {
  if (!p) return fail(BSG_EINVAL, "pipeline: null handle");
  if (batch != 0 && m > p->max_m / batch) return fail(BSG_EINVAL, "pipeline: batch * m exceeds the capacity");
  if (host_in != nullptr && host_in == host_out) return fail(BSG_EALIAS, "shuffle_values_batched: out aliases input");
  const bsg_config cfg = resolve_cfg(cfg_in);
  if (m >= 3) {
    BijParams bp;
    BSG_TRY(build_params(cfg.variant, bsg::domain_bits(m), cfg.seed, cfg.num_rounds, bp));
  }
  const uint64_t t = p->next++;
  auto& s = p->slots[t % p->slots.size()];
  const size_t bytes = batch * m * static_cast<size_t>(p->eb);
  if (ticket) *ticket = t;
  s.ticket = t;
  if (bytes == 0) return BSG_OK;
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    BSG_CUDA(cudaStreamWaitEvent(p->s_h2d, s.kernel_done, 0));
    BSG_CUDA(cudaMemcpyAsync(s.din.p, host_in, bytes, cudaMemcpyHostToDevice, p->s_h2d));
    BSG_CUDA(cudaEventRecord(s.h2d_done, p->s_h2d));
    BSG_CUDA(cudaStreamWaitEvent(p->s_comp, s.h2d_done, 0));
    BSG_CUDA(cudaStreamWaitEvent(p->s_comp, s.d2h_done, 0));
    BSG_TRY(batched_device(c, s.din.p, s.dout.p, batch, m, p->eb, cfg, p->s_comp));
    BSG_CUDA(cudaEventRecord(s.kernel_done, p->s_comp));
    BSG_CUDA(cudaStreamWaitEvent(p->s_d2h, s.kernel_done, 0));
    BSG_CUDA(cudaMemcpyAsync(host_out, s.dout.p, bytes, cudaMemcpyDeviceToHost, p->s_d2h));
    BSG_CUDA(cudaEventRecord(s.d2h_done, p->s_d2h));
    return BSG_OK;
  });
}

bsg_status bsg_pipeline_wait(bsg_pipeline* p, uint64_t ticket) {
  if (!p) return fail(BSG_EINVAL, "pipeline: null handle");
  if (ticket >= p->next) return fail(BSG_EINVAL, "pipeline: unknown ticket");
  if (p->next - ticket > p->slots.size()) {  // slot reused since: its latest D2H completes later
    BSG_CUDA(cudaStreamSynchronize(p->s_d2h));
    return BSG_OK;
  }
  BSG_CUDA(cudaEventSynchronize(p->slots[ticket % p->slots.size()].d2h_done));
  return BSG_OK;
}

bsg_status bsg_pipeline_destroy(bsg_pipeline* p) {
  if (!p) return BSG_OK;
  cudaStreamSynchronize(p->s_h2d);
  cudaStreamSynchronize(p->s_comp);
  cudaStreamSynchronize(p->s_d2h);
  for (auto& s : p->slots) {
    s.din.release();
    s.dout.release();
    cudaEventDestroy(s.h2d_done);
    cudaEventDestroy(s.kernel_done);
    cudaEventDestroy(s.d2h_done);
  }
  cudaStreamDestroy(p->s_h2d);
  cudaStreamDestroy(p->s_comp);
  cudaStreamDestroy(p->s_d2h);
  delete p;
  return BSG_OK;
}

const char* bsg_status_string(bsg_status s) {
  switch (s) {
    case BSG_OK: return "ok";
    case BSG_EINVAL: return "invalid argument";
    case BSG_ERANGE: return "out of range";
    case BSG_EALIAS: return "output aliases input";
    case BSG_ENOMEM: return "out of memory";
    case BSG_ECUDA: return "CUDA error";
    case BSG_ENODEV: return "no CUDA device";
    case BSG_EUNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* bsg_last_error(void) { return t_err.c_str(); }

int32_t bsg_version(void) { return 100; }

uint64_t bsg_kernel_launches(void) { return bsg::launches(); }

int32_t bsg_set_path(int32_t path) {
  const int old = g_path;
  g_path = (path >= 0 && path <= 2) ? path : 0;
  return old;
}

uint32_t bsg_set_rank_stage_cap(uint32_t cap) { return bsg::set_rank_stage_cap(cap); }

int32_t bsg_set_bulk_stores(int32_t on) { return bsg::set_bulk_stores(on); }

int32_t bsg_set_force_compact(int32_t on) {
  const int old = g_force_compact;
  g_force_compact = on ? 1 : 0;
  return old;
}

bsg_status bsg_workspace_bytes(uint64_t* bytes) {
  if (!bytes) return fail(BSG_EINVAL, "null pointer");
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    uint64_t t = 0;
    for (const DevBuf* b : {&c->status, &c->scratch, &c->keys, &c->st_in, &c->st_out, &c->st_idx, &c->st_tmp,
                            &c->part})
      t += b->bytes;
    *bytes = t;
    return BSG_OK;
  });
}

bsg_status bsg_release_workspace(void) {
  return with_ctx([&](DeviceCtx* c) -> bsg_status {
    BSG_CUDA(cudaDeviceSynchronize());
    c->status.release_all();  // graphs captured earlier must not be replayed after this
    c->keys.release_all();
    c->st_in.release_all();
    c->st_out.release_all();
    c->st_idx.release_all();
    c->st_tmp.release_all();
    c->part.release_all();
    c->epoch = 0;
    return BSG_OK;
  });
}

}  // extern "C"
