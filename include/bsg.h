/*
 * bsg.h -- C ABI of the B200-native bijective shuffle (libbsg.so).
 *
 * Drop-in boundary for the CPU path of the reference library `bijshuf`
 * (proj/include/bijshuf/ headers).  The reference has no FFI of its own: its
 * surface is header-only C++ templates.  Each entry point below replaces the
 * reference function cited beside it, with plain pointers and sizes, no C++
 * or torch types, and status codes instead of exceptions.  The C++ shim
 * include/bijshuf_gpu/shuffle.hpp re-exposes the reference's exact names and
 * signatures (std::vector, ShuffleConfig, exceptions) on top of this ABI.
 *
 * Pointers: every data pointer may be host memory (pageable or pinned) or
 * device memory of the current CUDA device.  Device pointers run
 * asynchronously on `stream` (a cudaStream_t; NULL = the legacy default
 * stream).  Host pointers are staged through device buffers owned by the
 * library and the call returns when the result is back in host memory.
 * Results are bit-identical to the reference for the same (m, seed, variant,
 * rounds), independent of `workers` and of any launch geometry.
 */
#ifndef BSG_H_
#define BSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* Mirrors the reference's exception classes (SURVEY.md 8b "Errors"). */
typedef enum {
  BSG_OK = 0,
  BSG_EINVAL = 1,      /* std::invalid_argument: rounds < 3, bits outside [2,63], derive_round_keys(r<1) */
  BSG_ERANGE = 2,      /* std::out_of_range: x outside [0, 2^bits) in *_apply / philox_invert */
  BSG_EALIAS = 3,      /* std::invalid_argument("... out aliases input"), shuffle.hpp:311-312, 356-358 */
  BSG_ENOMEM = 4,      /* std::bad_alloc */
  BSG_ECUDA = 5,       /* CUDA runtime error (detail in bsg_last_error()) */
  BSG_ENODEV = 6,      /* no CUDA device */
  BSG_EUNSUPPORTED = 7 /* shape this build does not handle (detail in bsg_last_error()) */
} bsg_status;

/* BijectionVariant, shuffle.hpp:20 */
typedef enum { BSG_LCG = 0, BSG_VARIABLE_PHILOX = 1 } bsg_variant;

/* ShuffleConfig, shuffle.hpp:25-30.  `workers` is accepted and ignored: the
 * output never depends on it (shuffle.hpp:22-24). */
typedef struct {
  uint64_t seed;
  int32_t variant;
  int32_t num_rounds;
  int32_t workers;
  int32_t reserved;
} bsg_config;

/* Default ShuffleConfig{} (seed 0, VariablePhilox, 24 rounds, workers 0). */
bsg_config bsg_config_default(void);

/* ------------------------------------------------------------ bijections --- */
/* splitmix.hpp:11-15 */
uint64_t bsg_mix64(uint64_t z);
/* splitmix.hpp:22-31 (EINVAL if rounds < 1) */
bsg_status bsg_derive_round_keys(uint64_t seed, int32_t rounds, uint32_t* keys_out);
/* shuffle.hpp:49-52 (m >= 2) */
int32_t bsg_domain_bits(uint64_t m);
/* make_lcg, bijection.hpp:25-34 */
bsg_status bsg_make_lcg(int32_t bits, uint64_t seed, uint64_t* a, uint64_t* c);
/* lcg_apply, bijection.hpp:36-40 (host scalar) */
bsg_status bsg_lcg_apply(int32_t bits, uint64_t a, uint64_t c, uint64_t x, uint64_t* y);
/* make_philox + philox_apply / philox_invert, bijection.hpp:73-143 (host scalar) */
bsg_status bsg_philox_apply(int32_t bits, uint64_t seed, int32_t rounds, uint64_t x, uint64_t* y);
bsg_status bsg_philox_invert(int32_t bits, uint64_t seed, int32_t rounds, uint64_t y, uint64_t* x);
/* VariablePhiloxParams (bijection.hpp:45-53) exactly as the caller holds
 * them -- from make_philox or assembled field by field (the reference's
 * ZeroRoundsIsIdentity tests set num_rounds = 0 by hand).  The two calls below
 * evaluate philox_apply / philox_invert (bijection.hpp:94-143) from these
 * fields alone: caller-edited round_keys and round counts are honoured.
 * ERANGE for an input outside [0, 2^total_bits) (total_bits < 64); EINVAL
 * for fields the reference's arithmetic is undefined on (side widths outside
 * [0, 63], right_side_bits < left_side_bits, fewer keys than rounds). */
typedef struct {
  int32_t total_bits;
  int32_t left_side_bits;
  int32_t right_side_bits;
  int32_t num_rounds;
  uint64_t left_side_mask;
  uint64_t right_side_mask;
  const uint32_t* round_keys; /* num_keys entries; may be NULL when num_rounds <= 0 */
  uint64_t num_keys;
} bsg_philox_params;
bsg_status bsg_philox_apply_params(const bsg_philox_params* p, uint64_t x, uint64_t* y);
bsg_status bsg_philox_invert_params(const bsg_philox_params* p, uint64_t y, uint64_t* x);
/* Batched evaluation on the GPU: y[i] = f(x[i]) (inverse != 0: f^-1).
 * x == NULL evaluates the counters start .. start+n-1.  ERANGE if an input
 * lies outside the domain (checked on the host for host inputs only). */
bsg_status bsg_bijection_apply(int32_t variant, int32_t bits, uint64_t seed, int32_t rounds, int32_t inverse,
                               const uint64_t* x, uint64_t start, uint64_t* y, uint64_t n, void* stream);

/* --------------------------------------------------------------- shuffle --- */
/* shuffle_indices / shuffle_indices_into, shuffle.hpp:280-293:
 * out[k] = sigma(k), the k-th in-range image in counter order. */
bsg_status bsg_shuffle_indices(uint64_t m, const bsg_config* cfg, uint64_t* out, void* stream);
/* shuffle_values / shuffle_values_into, shuffle.hpp:298-315:
 * out[k] = in[sigma(k)] for trivially copyable elements of elem_bytes bytes
 * (1, 2, 4, 8, 16 natively; any other size through an index pass + byte gather).
 * EALIAS when out overlaps in. */
bsg_status bsg_shuffle_values(const void* in, void* out, uint64_t m, uint32_t elem_bytes, const bsg_config* cfg,
                              void* stream);
/* `batch` independent shuffles of m elements laid out row-major; shuffle b is
 * keyed by seed + b (BijectiveShuffleSampler, stats.hpp:314-324). */
bsg_status bsg_shuffle_values_batched(const void* in, void* out, uint64_t batch, uint64_t m, uint32_t elem_bytes,
                                      const bsg_config* cfg, void* stream);
/* gather / gather_into, shuffle.hpp:319-362: out[i] = src[idx[i]] for
 * i < n; src holds src_len elements.  Indices are not validated (as in the
 * reference).  EALIAS when out is src or idx (shuffle.hpp:356-358). */
bsg_status bsg_gather(const void* src, uint64_t src_len, const uint64_t* idx, void* out, uint64_t n,
                      uint32_t elem_bytes, void* stream);

/* ------------------------------------------- partitioned / multi-GPU path --- */
/* Up to 16 equally sized input shards (shard g = elements [g*shard_elems,
 * (g+1)*shard_elems)); pointers may be peer mappings from bsg_ipc_open. */
typedef struct {
  const void* ptrs[16];
  int32_t count;
  int32_t reserved;
  uint64_t shard_elems;
} bsg_shards;

/* One contiguous counter range [counter_begin, counter_end) of the padded
 * domain of an m-element shuffle: writes the survivors' payload (or images
 * when in == NULL and in_shards == NULL) to out[0 .. count) in counter order
 * and stores count to *count_out (device or host pointer; may be NULL).
 * Concatenating the ranges of a partition of [0, 2^bits) in order yields the
 * full shuffle: the unit of the multi-GPU scheme. m >= 3. */
bsg_status bsg_shuffle_range(uint64_t m, const bsg_config* cfg, uint64_t counter_begin, uint64_t counter_end,
                             const void* in, const bsg_shards* in_shards, void* out, uint32_t elem_bytes,
                             uint64_t* count_out, void* stream);
/* Exact number of survivors in [counter_begin, counter_end) (count-only pass;
 * closed form when m == 2^bits). Host result. */
bsg_status bsg_range_count(uint64_t m, const bsg_config* cfg, uint64_t counter_begin, uint64_t counter_end,
                           uint64_t* count, void* stream);

/* All-gather of one u64 per rank (an 8-byte ncclAllGather in practice). */
typedef int (*bsg_allgather_u64_fn)(const uint64_t* send_one, uint64_t* recv_world, void* user);

/* Rank `rank` of `world` shuffles its contiguous share of the counter domain
 * (the north-star partition), exchanges survivor counts with `allgather`, and
 * reports where its piece lands: out[0 .. *local_count) holds global output
 * positions [*global_offset, *global_offset + *local_count).  Input is either
 * replicated (`in`, all m elements local) or sharded (`in_shards`, peer
 * pointers).  Device pointers only. */
bsg_status bsg_dist_shuffle_values(uint64_t m, const bsg_config* cfg, int32_t rank, int32_t world, const void* in,
                                   const bsg_shards* in_shards, void* out, uint32_t elem_bytes,
                                   bsg_allgather_u64_fn allgather, void* user, uint64_t* global_offset,
                                   uint64_t* local_count, void* stream);
/* Counter range [begin, end) owned by `rank` of `world` for an m-element shuffle. */
bsg_status bsg_dist_counter_range(uint64_t m, int32_t rank, int32_t world, uint64_t* begin, uint64_t* end);

/* Exchange-partitioned shuffle over two ranks (one process per GPU; DESIGN.md
 * section 7): the power-of-two domain m = 2^G (2^16..2^32, 4- or 8-byte
 * elements) is sharded in halves, rank r holding input elements and output
 * positions [r*m/2, (r+1)*m/2).  Replaces shuffle_values_into
 * (shuffle.hpp:308-315) for that layout: the concatenated output halves equal
 * the single-GPU shuffle of the m elements.  Each rank allocates
 * bsg_xpart_workspace_bytes of device memory, maps its peer's workspace
 * (bsg_ipc_export/open) and passes both as workspaces[0..1] (rank order).
 * bsg_xpart_route streams the rank's input half through the inverse cipher
 * and appends every element to its destination bucket in the owner rank's
 * workspace, rank 0 from the front and rank 1 from the back (peer stores over
 * NVLink, no remote atomics).  After BOTH
 * ranks' route completed (host barrier), bsg_xpart_place partitions and
 * places the rank's own buckets into out_half.  Device pointers; both calls
 * asynchronous on `stream`. */
bsg_status bsg_xpart_workspace_bytes(uint64_t m, uint32_t elem_bytes, int32_t world, uint64_t* bytes);
bsg_status bsg_xpart_route(const void* in_half, uint64_t m, uint32_t elem_bytes, const bsg_config* cfg,
                           int32_t rank, int32_t world, void* const* workspaces, void* stream);
bsg_status bsg_xpart_place(uint64_t m, uint32_t elem_bytes, int32_t rank, int32_t world,
                           void* const* workspaces, void* out_half, void* stream);

/* Sharded power-of-two shuffle by destination routing: the
 * local elements global_offset .. global_offset+n_local-1 of an m-element
 * shuffle (m = 2^bits <= 2^32) are grouped by the part owning their output
 * position f^-1(j) (nparts contiguous output shards of m/nparts); out_dest
 * holds the position inside the part; part_counts (host, nparts) the group
 * sizes.  An all-to-all of the groups followed by bsg_scatter_permutation on
 * each part completes the shuffle with bulk transfers only.  Device pointers. */
bsg_status bsg_route_by_dest(const void* in, uint64_t n_local, uint64_t global_offset, uint64_t m,
                             const bsg_config* cfg, int32_t nparts, void* out_values, uint32_t* out_dest,
                             uint64_t* part_counts, uint32_t elem_bytes, void* stream);
/* out[dest[i]] = values[i] where dest is a permutation of [0, n): the
 * partitioned three-pass placement for large power-of-two n, a direct scatter
 * otherwise.  elem_bytes 4, 8 or 16; device pointers. */
bsg_status bsg_scatter_permutation(const void* values, const uint32_t* dest, uint64_t n, void* out,
                                   uint32_t elem_bytes, void* stream);

/* CUDA IPC helpers for sharded inputs across processes (one process per GPU).
 * The exported handle carries the CUDA IPC handle of the allocation that
 * contains dev_ptr plus dev_ptr's offset inside it (pointers from a caching
 * allocator such as PyTorch's usually sit inside a larger segment), so
 * bsg_ipc_open returns the peer's address of dev_ptr itself.  bsg_ipc_close
 * takes that returned pointer. */
#define BSG_IPC_HANDLE_BYTES 80
bsg_status bsg_ipc_export(const void* dev_ptr, unsigned char handle_out[BSG_IPC_HANDLE_BYTES]);
bsg_status bsg_ipc_open(const unsigned char handle[BSG_IPC_HANDLE_BYTES], void** dev_ptr_out);
bsg_status bsg_ipc_close(void* dev_ptr);

/* ------------------------------------------------- host-buffer pipeline --- */
/* Streaming form of bsg_shuffle_values for HOST buffers: each submitted
 * shuffle is H2D-copied, shuffled and D2H-copied on three internal streams
 * with `depth` device staging slots, so the H2D of shuffle i+1 overlaps the
 * D2H of shuffle i (PCIe is full duplex).  Host buffers should be pinned
 * (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous, and
 * must stay untouched until bsg_pipeline_wait(ticket) returns.  Results are
 * identical to bsg_shuffle_values. */
typedef struct bsg_pipeline bsg_pipeline;
bsg_status bsg_pipeline_create(uint64_t max_m, uint32_t elem_bytes, int32_t depth, bsg_pipeline** out);
bsg_status bsg_pipeline_submit(bsg_pipeline* p, const void* host_in, void* host_out, uint64_t m,
                               const bsg_config* cfg, uint64_t* ticket);
/* Batched form (bsg_shuffle_values_batched, stats.hpp:314-324): batch rows of
 * m elements, row b shuffled with seed + b; batch * m <= the pipeline's max_m. */
bsg_status bsg_pipeline_submit_batched(bsg_pipeline* p, const void* host_in, void* host_out, uint64_t batch,
                                       uint64_t m, const bsg_config* cfg, uint64_t* ticket);
bsg_status bsg_pipeline_wait(bsg_pipeline* p, uint64_t ticket);
bsg_status bsg_pipeline_destroy(bsg_pipeline* p);

/* ------------------------------------------------------------ baselines --- */
/* The paper's SortShuffle (bench.hpp:109-156): random 64-bit
 * keys mix64(mix64(seed) + i*gamma) and a CUB radix sort of (key, value). */
bsg_status bsg_sort_shuffle_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t seed, void* stream);

/* --------------------------------------------------------------- utility --- */
const char* bsg_status_string(bsg_status s);
/* Detail of the last failure on this thread ("" if none). */
const char* bsg_last_error(void);
int32_t bsg_version(void);
/* Number of kernels this library has launched since load (bench evidence). */
uint64_t bsg_kernel_launches(void);
/* Testing knob: 0 = automatic path choice, 1 = always use the compacting
 * (look-back) kernel even when every image survives. Returns the old value. */
int32_t bsg_set_force_compact(int32_t on);
/* Path selection for whole-domain shuffles: 0 = automatic (the partitioned
 * kernels for payloads >= 256 MiB with elements of at most 8 bytes -- power of
 * two or not -- and the single fused pass otherwise), 1 = always the single
 * fused pass, 2 = partitioned whenever eligible (domains of 2^14..2^32
 * counters).  Outputs are identical; returns the old value. */
int32_t bsg_set_path(int32_t path);
/* Testing knob: survivors per counter window that the persistent last pass of
 * padded partitioned shuffles stages in shared memory (default and maximum
 * 9216); windows holding more take the round-based pass.  Lower it to exercise
 * that path; outputs are identical.  Returns the old value. */
uint32_t bsg_set_rank_stage_cap(uint32_t cap);
/* Testing knob: the partitioned path's last passes write their placed windows
 * with bulk shared->global copies (1, default) or plain stores (0).  Outputs
 * are identical; compute-sanitizer's initcheck does not model bulk-copy
 * writes.  Returns the old value. */
int32_t bsg_set_bulk_stores(int32_t on);
/* Bytes of device memory the library currently holds as cached workspaces on
 * the current device (the partitioned path keeps ~14 B per counter for power-of-two
 * domains and ~22 B per counter for padded ones between calls: 7.5 GB after a
 * 2^29-element u64 shuffle).  bsg_release_workspace() returns them. */
bsg_status bsg_workspace_bytes(uint64_t* bytes);
/* Release cached device/host workspaces of the current device.  CUDA graphs
 * captured from libbsg calls reference these workspaces and must not be
 * replayed afterwards (growing a workspace, by contrast, keeps the old one
 * alive for such graphs). */
bsg_status bsg_release_workspace(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* BSG_H_ */
