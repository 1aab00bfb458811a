/* lpp_b200.h — C ABI of the B200-native LPP-SGD hot path.
 *
 * This is the drop-in boundary that replaces the reference's only native
 * component, the CPython module `asyncsgd._atomics`
 * (/root/reference/pkg/src/asyncsgd/_atomics.c:394-412), and the numpy
 * work the engine does around it (engine.py:199-229, 343-355, 418-421).
 *
 * Conventions (mirroring _atomics.c:1-7 and :20-39):
 *   - plain pointers and sizes only; no torch / CUDA types in signatures
 *     (streams are passed as `void*` = cudaStream_t);
 *   - the caller owns every buffer it passes in; functions never keep them;
 *   - every function returns 0 on success and a negative LPP_E* code on
 *     error; lpp_last_error() returns the thread-local message of the most
 *     recent failure (the reference raises ValueError/IndexError instead);
 *   - device functions are asynchronous on the given stream; they are safe
 *     to call concurrently from many host threads on different streams;
 *   - element order inside one call is unspecified (the GPU has no
 *     "ascending" order), but every element update is a single atomic
 *     read-modify-write in atomic modes, so concurrent updates at the same
 *     index are never lost, and every 32-bit element is read/written
 *     untorn (_atomics.c:58-74 guarantees the same for fp64).
 */
#ifndef LPP_B200_H
#define LPP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPP_ABI_VERSION 4

/* error codes */
#define LPP_OK 0
#define LPP_E_VALUE -1   /* bad size / alignment / argument  (ref: ValueError) */
#define LPP_E_INDEX -2   /* index or range out of bounds     (ref: IndexError) */
#define LPP_E_CUDA -3    /* CUDA runtime error                                */
#define LPP_E_NOMEM -4   /* allocation failed                                 */

/* apply modes (K1/K2, K4) */
#define LPP_MODE_PLAIN 0 /* ld/st read-modify-write: Hogwild "classic", may lose
                            concurrent updates; for single-writer use only     */
#define LPP_MODE_RED 1   /* red.global.add.v4.f32: element-atomic, default      */
#define LPP_MODE_BULK 2  /* cp.reduce.async.bulk .add.f32 from shared memory   */

int lpp_abi_version(void);
const char* lpp_last_error(void);
/* number of kernels this library has launched so far (process-wide) */
unsigned long long lpp_launch_count(void);

/* ------------------------------------------------------------------ */
/* host atomics (K6) — replace _atomics.{load,store,fetch_add}_i64     */
/* (_atomics.c:125-183).  Operate on caller-owned host int64 cells,    */
/* e.g. numpy buffers or a POSIX shared-memory control block.          */
/* Memory order: acquire loads, release stores, acq_rel RMW.           */
int64_t lpp_atomic_load_i64(const int64_t* p);
void lpp_atomic_store_i64(int64_t* p, int64_t v);
int64_t lpp_atomic_fetch_add_i64(int64_t* p, int64_t delta);
/* returns 1 if *p was `expected` and is now `desired`, else 0 */
int lpp_atomic_cas_i64(int64_t* p, int64_t expected, int64_t desired);
/* Spin (with exponential back-off sleeps up to max_sleep_us) until
 * *p >= target; returns the value seen, or INT64_MIN if *abort_flag != 0
 * first (abort_flag may be NULL).  Releases no locks: call from a thread
 * that may block (the Python binding drops the GIL around it). */
int64_t lpp_atomic_wait_ge_i64(const int64_t* p, int64_t target,
                               const int64_t* abort_flag, int max_sleep_us);

/* Host memory the kernels read and write directly (cudaHostAlloc mapped +
 * portable, zero-filled): round-stamp cells, sampled-tag index rings and
 * classification records.  *dev is the device view (== *host under UVA). */
int lpp_host_alloc(size_t bytes, void** host, void** dev);
int lpp_host_free(void* host);

/* ------------------------------------------------------------------ */
/* arenas: flat fp32 parameter vectors in device memory (a1)           */
/* replace ParamStore.values (paramstore.py:59-77)                     */
typedef struct lpp_arena* lpp_arena_t;

/* cudaMalloc'd, 256-byte aligned, zero-filled, IPC-exportable */
int lpp_arena_create(int device, size_t n_elems, lpp_arena_t* out);
int lpp_arena_destroy(lpp_arena_t arena);
float* lpp_arena_data(lpp_arena_t arena);
size_t lpp_arena_size(lpp_arena_t arena);
int lpp_arena_device(lpp_arena_t arena);

/* Element access — replaces _atomics.load_f64 / store_f64 (_atomics.c:41-56,
 * method table :395-396; ParamStore.read / write, paramstore.py:79-86): one
 * untorn element of a device arena of `len` elements, acquire load / release
 * store at system scope, ordered on `stream` and synchronous (returns after
 * the element was read / written).  i >= len -> LPP_E_INDEX (ref IndexError). */
int lpp_load_f32(const float* arena, size_t len, size_t i, float* out, void* stream);
int lpp_store_f32(float* arena, size_t len, size_t i, float v, void* stream);

/* Multi-process peer mapping (one process per GPU, NVLink P2P).
 * export writes LPP_IPC_HANDLE_BYTES bytes to handle_out. */
#define LPP_IPC_HANDLE_BYTES 64
int lpp_arena_export_ipc(lpp_arena_t arena, void* handle_out);
int lpp_ipc_open(int device, const void* handle, float** ptr_out);
int lpp_ipc_close(int device, float* ptr);
/* Single-process peer access: device `device` may load/store/red into
 * memory of `peer`.  Returns 0 if enabled (or already enabled). */
int lpp_enable_peer_access(int device, int peer);
int lpp_can_access_peer(int device, int peer, int* out);

/* ------------------------------------------------------------------ */
/* K1/K2 apply — replaces ParamStore.sub_assign -> accum_cas_f64        */
/* (paramstore.py:121-136, _atomics.c:312-344; call site engine.py:355)*/
/*
 *   for e in [0, n):
 *     g' = g[e] + wd * x[e]                (wd != 0 only)
 *     m[e] = mu * m[e] + g'                (mu != 0 only; m is per-stream)
 *     x[e] += -(lr * (mu != 0 ? m[e] : g'))  atomically per element
 *
 * x, g and m are already offset to the block start (x = arena + lo).
 * lr: if lr_dev != NULL the learning rate is *lr_dev (device scalar, so a
 * captured CUDA graph can replay with a fresh value), else `lr`.
 * x, g, m must share the same address alignment modulo 16 bytes.
 */
int lpp_apply_sgd(float* x, const float* g, float* m, size_t n, float lr,
                  const float* lr_dev, float mu, float wd, int mode,
                  void* stream);

/* K1+K3 fused: apply the block [lo, hi) of this step (as lpp_apply_sgd on
 * x + lo, g + lo, m + lo, with tags[e] = stamp when tags != NULL) and write
 * replica[e] for every e in [0, n): inside the block, x[e] re-read after this
 * step's vector reduction landed (a value the arena really held; old + delta
 * when no other writer raced), an untorn copy of x outside it.  x, g, m, replica, tags are arena BASES (16-byte aligned). */
int lpp_apply_snapshot(float* x, const float* g, float* m, float* replica,
                       int32_t* tags, size_t n, size_t lo, size_t hi, float lr,
                       const float* lr_dev, float mu, float wd, int32_t stamp,
                       void* stream);

/* K5 inside the fused launch, in the reference updater's order
 * (engine.py:343-362: sampled tags at the snapshot, k_claim after the
 * gradient, then the apply), with per-BLOCK write stamps: every update
 * writes one whole block range, so an element's tag is the newest stamp of
 * the blocks covering it (block 0 = all, and its partial block).
 *   block_stamps[block_id] is NOT written here: call lpp_publish_stamp
 *       after it, ordered on a stream (once every element reduction is
 *       performed)
 *   cur_claim[0..1] = (k_claim, clean): k_claim = *avg_cell read when the
 *       kernel starts (after this step's gradient), clean = all of this
 *       step's k tags cur_dev[j] >= k_claim              (cur_claim may be NULL)
 *   next_dev[j] (and next_host[j]) = the next step's sampled tag j, read by
 *       the thread that refreshes the replica element next_idx[j] BEFORE it
 *       reads the value and after this launch's own reduction there:
 *       max(*avg_cell, block_stamps[0], block_stamps[b(e)], stamp if e is in
 *       [lo, hi)); *avg_cell (the worker's last completed round stamp, a
 *       device cell) is the floor a round writes into every element
 *       (engine.py:421)                              (next_idx may be NULL)
 * next_idx and block_bounds (num_blocks + 1 boundaries, 0 ... n) are HOST
 * pointers: the k indices and their partial blocks are computed into the
 * launch parameters; k <= 32, num_blocks <= 127; next_host and cur_claim
 * may point into lpp_host_alloc memory. */
typedef struct lpp_tag_plan {
  const int64_t* next_idx;
  int32_t* next_dev;
  int32_t* next_host;
  const int32_t* cur_dev;
  int64_t* cur_claim;
  const int64_t* avg_cell;
  int32_t* block_stamps;
  const int64_t* block_bounds;
  int32_t num_blocks;
  int32_t block_id;
  int32_t k;
} lpp_tag_plan;
int lpp_apply_snapshot_plan(float* x, const float* g, float* m, float* replica,
                            int32_t* tags, size_t n, size_t lo, size_t hi, float lr,
                            const float* lr_dev, float mu, float wd, int32_t stamp,
                            const lpp_tag_plan* plan, void* stream);

/* Reference-shaped accumulate: dst[start + e] += scale * delta[e],
 * e in [0, n), with dst of length dst_len (range-checked like
 * _atomics.c:328-333).  fp32 mirror of accum_cas_f64. */
int lpp_accum(float* dst, size_t dst_len, size_t start, const float* delta,
              size_t n, float scale, int mode, void* stream);

/* ------------------------------------------------------------------ */
/* K3 snapshot — replaces ParamStore.snapshot -> snapshot_f64           */
/* (paramstore.py:97-117, _atomics.c:186-215; call site engine.py:343) */
/* out[e] = src[e] for e in [0, n), per-element untorn loads.           */
int lpp_snapshot(const float* src, float* out, size_t n, void* stream);

/* ------------------------------------------------------------------ */
/* K4 averaging — replaces _averager_body's snapshot + _MeanAllReduce   */
/* + add_assign(mean - snap) (engine.py:199-229, 418-421).              */
/*
 * Owner-computes over the shard [lo, hi) of Q arenas (arenas[q] is the
 * base of worker q's arena; remote ones are peer / IPC mappings):
 *   v_q  = arenas[q][e]                        (q = 0..Q-1, loads)
 *   mean = (((v_0 + v_1) + v_2) + ...) / Q     (fixed order, as np.mean(axis=0))
 *   arenas[q][e] += mean - v_q                 (atomic per element, mode RED;
 *                                               plain store of mean-correction
 *                                               in mode PLAIN)
 *   mean_out[e - lo] = mean                    (mean_out may be NULL)
 * Updaters may keep writing the arenas concurrently: their updates are
 * preserved (the correction is added, not stored).  Q <= LPP_MAX_WORKERS.
 * `arenas` is a HOST array of Q device pointers.  Mode BULK stages the
 * round through shared memory with the bulk-copy (TMA) engine: bulk loads
 * of the Q shard tiles on an mbarrier, the correction written in place,
 * cp.reduce.async.bulk .add.f32 back into every arena (same values as RED;
 * the tagged variant serves BULK as RED).
 */
#define LPP_MAX_WORKERS 8
int lpp_average_shard(float* const* arenas, int Q, size_t lo, size_t hi,
                      float* mean_out, int mode, void* stream);

/* ------------------------------------------------------------------ */
/* K5 write tags — replace the tagged _atomics ops (_atomics.c:217-310,  */
/* 346-392).  Tags are int32 update-order stamps, one per element, in a  */
/* buffer with the same alignment as the values.  Writers update the     */
/* value first and the tag second; readers load the tag first and the    */
/* value second, so a tag never claims a newer write than the value it   */
/* is read with (paramstore.py:47-53).                                   */

/* lpp_apply_sgd + tags[e] = stamp (mode BULK is served as RED) */
int lpp_apply_sgd_tagged(float* x, const float* g, float* m, size_t n, float lr,
                         const float* lr_dev, float mu, float wd, int mode,
                         int32_t* tags, int32_t stamp, void* stream);
/* accum_cas_tagged_f64(dst, tags, start, delta, scale, stamp) */
int lpp_accum_tagged(float* dst, int32_t* tags, size_t dst_len, size_t start,
                     const float* delta, size_t n, float scale, int32_t stamp,
                     int mode, void* stream);
/* snapshot_tagged_f64: out / out_tags may be NULL; if min_tag_out != NULL
 * the minimum tag seen is atomicMin-ed into *min_tag_out (init INT32_MAX) */
int lpp_snapshot_tagged(const float* src, const int32_t* tags, float* out,
                        int32_t* out_tags, size_t n, int32_t* min_tag_out,
                        void* stream);
/* gather_i64(tags, idx, out): out[k] = tags[idx[k]] (device idx, caller
 * guarantees 0 <= idx[k] < len(tags)) */
int lpp_gather_tags(const int32_t* tags, const int64_t* idx, size_t k, int32_t* out,
                    void* stream);
/* the sampled-tag gather of an unfused snapshot with the round floor:
 * out[j] = max(tags[idx[j]], *floor_cell) (floor_cell may be NULL = 0);
 * idx / floor_cell / out_host may be lpp_host_alloc memory */
int lpp_gather_tags_floor(const int32_t* tags, const int64_t* idx, size_t k,
                          const int64_t* floor_cell, int32_t* out_dev, int32_t* out_host,
                          void* stream);
/* the sampled tags of a fused run's first snapshot from the block stamps:
 * out[j] = max(*floor_cell, stamps[0], stamps[b(idx[j])]) */
int lpp_gather_block_stamps(const int32_t* stamps, const int64_t* bounds, int nb,
                            const int64_t* idx, size_t k, const int64_t* floor_cell,
                            int32_t* out_dev, int32_t* out_host, void* stream);
/* stamps[block_id] = stamp, in stream order after all prior work on the
 * stream and a system-wide memory barrier (a stream memory operation, no
 * kernel): issued after an update's lpp_apply_snapshot_plan, ordered after
 * it.  The last write wins, like the reference's per-element tags. */
int lpp_publish_stamp(int32_t* stamps, int block_id, int32_t stamp, void* stream);
/* *dev = v in stream order (the round-stamp cell the apply kernels read) */
int lpp_set_i64(int64_t* dev, int64_t v, void* stream);
/* classification at apply time (engine.py:353-362) for the unfused paths:
 * out[0] = *claim_cell read when the kernel runs, out[1] = all k tags >= it */
int lpp_classify(const int32_t* tags, size_t k, const int64_t* claim_cell, int64_t* out,
                 void* stream);
/* K4 + tags_q[e] = stamps[q] after the correction (host arrays of Q) */
int lpp_average_shard_tagged(float* const* arenas, int32_t* const* tags,
                             const int32_t* stamps, int Q, size_t lo, size_t hi,
                             float* mean_out, int mode, void* stream);

/* ------------------------------------------------------------------ */
/* NVLS averaging: VMM buffers bound to a multicast  */
/* object; the owner reduces its shard IN the NVSwitch and broadcasts    */
/* the mean (multimem.ld_reduce / multimem.st), each worker then adds    */
/* (mean - snapshot) locally — the reference round snapshot -> mean      */
/* all-reduce -> add_assign(mean - snap) (engine.py:418-421).            */
typedef struct lpp_vmm* lpp_vmm_t;
typedef struct lpp_mc* lpp_mc_t;
int lpp_mc_supported(int device, int* out);
/* allocation granularity for a multicast object over num_devices */
int lpp_mc_granularity(int device, int num_devices, size_t* out);
/* device memory from cuMemCreate (size rounded up to the granularity),
 * mapped read/write on `device`, zero-filled */
int lpp_vmm_create(int device, size_t bytes, lpp_vmm_t* out);
float* lpp_vmm_ptr(lpp_vmm_t v);
size_t lpp_vmm_size(lpp_vmm_t v);
int lpp_vmm_destroy(lpp_vmm_t v);
/* multicast object lifecycle: create (one process) -> export/import the
 * POSIX fd (others) -> every process adds its device -> (group barrier) ->
 * every process binds its VMM buffer -> map the multicast VA */
int lpp_mc_create(int num_devices, size_t bytes, lpp_mc_t* out);
int lpp_mc_export_fd(lpp_mc_t mc, int* fd_out);
int lpp_mc_import_fd(int fd, size_t bytes, lpp_mc_t* out);
int lpp_mc_add_device(lpp_mc_t mc, int device);
int lpp_mc_bind(lpp_mc_t mc, lpp_vmm_t mem, size_t mc_offset);
int lpp_mc_map(lpp_mc_t mc, int device, float** mc_ptr_out);
int lpp_mc_destroy(lpp_mc_t mc);
/* owner: mc_mean[e] = (sum over workers of mc_stage[e]) / Q for e in
 * [lo, hi) (lo a multiple of 4); both pointers are multicast addresses */
int lpp_nvls_mean_shard(const float* mc_stage, float* mc_mean, size_t lo, size_t hi,
                        int Q, void* stream);
/* local: x[e] += mean[e] - stage[e] atomically, tags[e] = stamp (tags may
 * be NULL); 16-byte aligned buffers */
int lpp_nvls_apply(float* x, const float* stage, const float* mean, size_t n,
                   int32_t* tags, int32_t stamp, void* stream);

/* ------------------------------------------------------------------ */
/* utilities */
/* Stream-ordered copy between any two of {pinned host, device} buffers
 * (cudaMemcpyAsync, kind inferred): the per-step index / tag H2D and D2H
 * without a framework dispatch. */
int lpp_copy_async(void* dst, const void* src, size_t n_bytes, void* stream);
/* Host row gather for the end-to-end input path: dst row i = src row
 * idx[i] (row_bytes each) for i in [0, n_idx); LPP_E_INDEX if any idx is
 * outside [0, n_rows).  Single-threaded memcpy per row, called from each
 * updater thread with the GIL released (a framework CPU index_select fans
 * out to an intra-op thread pool per call: 4 updater threads oversubscribe
 * the host, measured 151k vs 160k images/s end to end). */
int lpp_host_gather_rows(void* dst, const void* src, size_t n_rows, size_t row_bytes,
                         const int64_t* idx, size_t n_idx);
/* Launch an instantiated CUDA graph (cudaGraphExec_t) on a stream: the
 * captured fwd/bwd step replayed without a framework wrapper. */
int lpp_graph_launch(void* graph_exec, void* stream);
/* Write a buffer of n_bytes (>= L2 size to flush it) on the stream. */
int lpp_l2_flush(void* scratch, size_t n_bytes, void* stream);
/* number of SMs of `device` */
int lpp_sm_count(int device, int* out);

/* ------------------------------------------------------------------ */
/* Native updater loop (a10: _updater_loop / _updater_body,
 * engine.py:289-383) and its pure helpers.
 *
 * lpp_lr_at: lr_at (schedules.py:56-68), bit-identical to the Python
 * restatement (same IEEE operation order, libm cos/pow): kind 0 = cosine,
 * 1 = multistep.  lpp_select_block: select_block (partition.py:132-145),
 * returns the block id, or LPP_E_VALUE for a rank outside [1, num_blocks]. */
double lpp_lr_at(int kind, double alpha0, double peak, int64_t warmup, int64_t total,
                 const int64_t* milestones, int n_milestones, double gamma, int64_t s);
int lpp_select_block(int64_t s, int64_t warm_start, int num_blocks, int rank);

/* Device-side uniform batch sampling for captured steps: idx[i] =
 * floor(h(key, step, i) * n / 2^64) for i in [0, batch), h a splitmix64
 * chain, step read from the device counter *step which the kernel then
 * increments — so a CUDA graph that captured this launch draws a fresh
 * batch on every replay with no host involvement.  The host twin computes
 * the same indices for a given step (tests). */
int lpp_sample_indices(int64_t* idx, int64_t* step, int32_t batch, int64_t n, uint64_t key,
                       void* stream);
int lpp_sample_indices_host(int64_t* out, int32_t batch, int64_t n, uint64_t key, int64_t step);

/* The reference's host sampling stream in native code (csrc/nprng.cu):
 * numpy.random.default_rng(SeedSequence(entropy)) restated bit for bit —
 * integers(0, n, b), choice(pop, k, replace=False), permutation(m) — so the
 * native updater loop draws exactly the reference's batches and sampled tag
 * indices (engine.py:293, 343-351).  A handle is one generator's state. */
int lpp_nprng_create(const uint64_t* entropy, int n, void** out);
int lpp_nprng_destroy(void* h);
int lpp_nprng_integers(void* h, int64_t n, int32_t b, int64_t* out);
int lpp_nprng_choice(void* h, int64_t pop, int32_t k, int64_t* out);
int lpp_nprng_permutation(void* h, int64_t m, int64_t* out);

/* Device-side epoch-partition sampling (f4; EpochSampler, objectives.py:
 * 77-104): position step * batch + i of the stream is element
 * perm_e(pos mod shard_len) of the shard {shard_base + p * shard_stride},
 * epoch e = pos / shard_len, perm_e a keyed Feistel bijection — each
 * epoch visits every shard element exactly once in a fresh order.  Same
 * device step counter protocol as lpp_sample_indices; host twin for tests
 * and for the native loop's end-to-end input. */
int lpp_sample_epoch(int64_t* idx, int64_t* step, int32_t batch, int64_t shard_base,
                     int64_t shard_stride, int64_t shard_len, uint64_t key, void* stream);
int lpp_sample_epoch_host(int64_t* out, int32_t batch, int64_t shard_base, int64_t shard_stride,
                          int64_t shard_len, uint64_t key, int64_t step);

/* One updater's whole asynchronous loop in native code (GIL-free): claim
 * s = C^q++ (host cell), lr = lr_at(s), b = select_block(s, ...), u = the
 * write stamp, then on the updater's stream
 *   [sampled tags: H2D of k sorted distinct indices, K5 gather, D2H]
 *   K3 snapshot (or, fused, only before the first step)
 *   cudaGraphLaunch(graph_exec[b])          -- the captured fwd/bwd
 *   K1/K2 apply (+K5 tags) or the fused K1+K3 apply_snapshot
 * with in_flight steps outstanding (an event per slot); a step's sampled
 * tags are classified clean iff all >= the averaging stamp read at claim
 * time (engine.py:357-362) once its event completed.  Stops at the claim
 * rule of engine.py:336 (each updater processes exactly one slot >= budget)
 * or when *stop becomes non-zero.  Pointers to host int64 cells are shared
 * with the averager thread (host atomics K6). */
typedef struct {
  int64_t* sample_counter;        /* C^q (read_and_inc) */
  int64_t* update_order;          /* write stamps: u = fetch_add + 1 */
  const int64_t* stop;            /* non-zero: stop claiming */
  const int64_t* last_avg_stamp;  /* k_claim */
  int64_t budget;
  /* lr_at */
  int32_t lr_kind;
  int32_t n_milestones;
  double alpha0, peak, gamma;
  int64_t warmup, total;
  const int64_t* milestones;
  /* select_block */
  int32_t lpp;                    /* 1: lpp_sgd block rule, 0: always block 0 */
  int32_t num_blocks;
  int32_t rank;                   /* 1-based */
  int32_t fused;                  /* 1: K1+K3 fused apply_snapshot */
  int64_t warm_start;
  const int64_t* block_lo;        /* [num_blocks + 1] element ranges per block id */
  const int64_t* block_hi;
  void* const* graph_exec;        /* cudaGraphExec_t [block id][input buffer 0/1] */
  const int64_t* flops_of;        /* per block id */
  /* arenas (bases) */
  float* x;
  float* g;
  float* m;                       /* NULL without momentum */
  float* replica;
  int32_t* tags;                  /* NULL: no write tags */
  size_t n;
  float mu, wd;
  int32_t apply_mode;
  int32_t in_flight;
  /* sampled tags (K5); ignored when tags == NULL or tag_pick == 0 */
  int32_t tag_pick;
  int32_t time_apply;             /* 1: CUDA events around every apply */
  uint64_t tag_seed;
  int64_t* tag_idx_pinned;        /* [in_flight + 2][tag_pick] */
  int64_t* tag_idx_dev;           /* [tag_pick] */
  int64_t* classified;            /* host counters (+= per classified step) */
  int64_t* clean;
  double apply_bytes_per_elem;    /* algorithmic bytes per block element */
  void* stream;
  void* apply_stream;             /* NULL: apply on `stream`; else a (high-priority) stream
                                     ordered after the step's graph by events */
  /* end-to-end input: when host_feats != NULL every step draws its batch
   * indices on the host (the device sampler's stream, lpp_sample_indices_host
   * keyed by sample_key), gathers the rows from pinned host memory into a
   * pinned staging slot and copies them on copy_stream into the graph's
   * input buffer t % 2 (double-buffered: the copy for step t+1 overlaps
   * step t, ordered by events) */
  const void* host_feats;         /* pinned [n_rows][row_bytes] */
  const void* host_labels;        /* pinned [n_rows][label_bytes] */
  int64_t n_rows;
  int64_t row_bytes;
  int64_t label_bytes;
  int32_t batch;
  int32_t read_loss;              /* 1: D2H of each step's loss, logged in loss_log */
  uint64_t sample_key;
  void* feat_pinned;              /* [in_flight + 2][batch * row_bytes] */
  void* label_pinned;             /* [in_flight + 2][batch * label_bytes] */
  void* xbuf[2];                  /* the captured graphs' input buffers */
  void* ybuf[2];
  void* copy_stream;
  const float* loss_dev[2];       /* the graphs' loss scalars (per input buffer) */
  float* loss_pinned;             /* [in_flight + 2] */
  float* loss_log;                /* [loss_cap] losses in step order */
  int64_t loss_cap;
  int64_t* loss_count;
  int64_t sample_step0;           /* host draws use steps sample_step0, sample_step0 + 1, ... */
  int64_t epoch_base;             /* epoch_len > 0: host draws follow lpp_sample_epoch_host */
  int64_t epoch_stride;
  int64_t epoch_len;
  /* per-update records (record_mode "light", UpdateRecord, engine.py:74-92):
   * row t = (s, u, k_claim, block_id, reason 0 warm_start / 1 alternate_full
   * / 2 alternate_partial, clean -1 unknown / 0 / 1), its lr, and its
   * sampled tag indices and tag values; NULL rec_i64 = no records */
  int64_t* rec_i64;               /* [rec_cap][6] */
  double* rec_lr;                 /* [rec_cap] */
  int64_t* rec_tag_idx;           /* [rec_cap][tag_pick] or NULL */
  int32_t* rec_tags;              /* [rec_cap][tag_pick] or NULL */
  int64_t rec_cap;
  int64_t* rec_count;
  /* the reference's host sampling stream (sampling="host"): every step
   * draws, from numpy's default_rng(SeedSequence(rng_entropy)) restated in
   * csrc/nprng.cu, first the sampled tag indices (sorted choice(n, tag_pick),
   * when tags are sampled) and then the batch — integers(0, n_rows, batch),
   * or with epoch_seed >= 0 the EpochSampler walk over the shard (epoch e
   * permuted by default_rng(SeedSequence([epoch_seed, e]))) — exactly the
   * reference updater's draws (engine.py:293-296, 343-351).  Without host
   * batches the indices are copied into idx_dev (the captured graph gathers
   * from the device dataset) through the pinned ring idx_pinned. */
  int32_t host_rng;
  int32_t n_entropy;
  uint64_t rng_entropy[4];
  int64_t epoch_seed;             /* < 0: i.i.d. draws */
  int64_t* idx_pinned;            /* [in_flight + 2][batch] */
  int64_t* idx_dev;               /* [batch] */
  /* K5 in the reference's order (lpp_tag_plan): the sampled-tag indices are
   * drawn into the pinned ring tag_idx_pinned and copied (stream-ordered,
   * before the step's graph) into the device ring tag_idx_dev, both
   * [in_flight + 2][tag_pick].  Step records, per in-flight slot s, in
   * rec_cols int64 cells: {k_claim, clean, tags[tag_pick] as int32} — on the
   * device (rec_dev, written by the kernels: the step's tags at its
   * snapshot, its (k_claim, clean) by its apply), copied into rec_pinned[s]
   * after the apply; k_claim is read from the worker's device round-stamp
   * cell avg_cell_dev.  (Host-mapped outputs measured +1.5 us each on the
   * kernel: its completion waits for the system-scope write flush.) */
  int64_t* rec_dev;
  int64_t* rec_pinned;
  int32_t rec_cols;
  const int64_t* avg_cell_dev;
  /* fused runs: the worker's per-block write stamps [num_blocks + 1] and the
   * block boundaries [num_blocks + 1] on the device (lpp_tag_plan) */
  int32_t* block_stamps;
  const int64_t* block_bounds_dev;
  /* time_apply: each timed apply's CUDA-event ms, in step order (NULL: sum only) */
  float* apply_ms_log;
  int64_t apply_ms_cap;
  /* per block id: kernels of this library inside the step graph
   * (csrc/conv_f32.cu's convolutions), summed into stats->graph_kernels per
   * launch (NULL: not counted) */
  const int64_t* graph_kernels_of;
} lpp_updater_cfg;

typedef struct {
  int64_t steps;                  /* minibatches processed */
  int64_t flops;                  /* sum of flops_of over the steps */
  int64_t apply_launches;         /* timed applies (time_apply) */
  double apply_ms;                /* summed CUDA-event time of the applies */
  double apply_bytes;             /* summed algorithmic bytes of the applies */
  int64_t graph_kernels;          /* sum of graph_kernels_of over the steps */
} lpp_updater_stats;

int lpp_updater_run(const lpp_updater_cfg* cfg, lpp_updater_stats* stats);

/* One worker's averager (a11: _averager_body, engine.py:385-453) in native
 * code: the round protocol of paper_2203_06638_b200/rounds.py over the
 * shared int64 control block (RoundControl layout: [0] round_calls, [1]
 * stop, [2] abort, [3] drained workers, [8, 8+Q) round stamps, then the
 * vote / final-vote / fence0 / fence1 arrays of RING = 8 cells indexed by
 * round mod 8, each round's cells zeroed once all votes of the next round
 * are in — no limit on the number of rounds) and the owner-computes K4
 * round on its own stream:
 *   open (CAS on round_calls when this worker's sync_every period is due,
 *   or every worker drained) -> vote -> u = stamp; [tags: publish u,
 *   fence 0] -> K4 over the owned shard (+ the mean on the final round)
 *   -> stream sync -> [tags / floor / eval: fence 1] -> last_avg_stamp = u
 *   -> wait for all Q votes -> release the previous round's cells -> stop
 *   after the unanimous final round.
 * One record per joined round (round, u, s_cur, k_delta, unanimous,
 * wall ms since t0) for RunResult.stamps. */
typedef struct {
  int64_t* ctrl;                  /* RoundControl buffer */
  int64_t max_rounds;             /* unused (the control block is a ring); kept for layout */
  int32_t workers;                /* Q */
  int32_t q;                      /* this worker */
  int32_t updaters;               /* U: this worker drained when *exited == U */
  int32_t tagged;                 /* stamp the tags (K5) with the round's stamps */
  const int64_t* sample_counter;  /* C^q */
  int64_t* update_order;          /* u = fetch_add + 1 */
  const int64_t* exited;
  int64_t* last_avg_stamp;
  int64_t* synced_at;
  int64_t switch_point;           /* sync_every: 1 before, period after */
  int64_t period;
  int64_t stop_after;             /* round budget (0: none) */
  float* const* arenas;           /* [Q] local or peer-mapped arena bases */
  int32_t* const* tags;           /* [Q] or NULL */
  size_t lo, hi;                  /* owned shard */
  size_t n;                       /* arena length */
  float* mean_out;                /* final round: the mean (shard [lo, hi); all of it at Q = 1) */
  void* stream;
  double t0;                      /* CLOCK_MONOTONIC seconds at the run start */
  int64_t* rec;                   /* [max_records][5] round, u, s_cur, k_delta, unanimous */
  double* rec_wall_ms;            /* [max_records] */
  int64_t max_records;
  /* eval points (engine.py:445-451, worker 0): with eval_interval > 0 every
   * round writes its mean and is fenced; at the first non-final round with
   * s_cur past the next multiple of eval_interval worker 0 copies the round
   * mean (the owners' mean_out shards, or — mean_parts == NULL, one process
   * per GPU — its own arena) into eval_buf and records the point */
  int64_t eval_interval;
  float* const* mean_parts;       /* [Q] every owner's mean_out base, or NULL */
  const int64_t* shard_bounds;    /* [Q + 1] owner shard boundaries */
  float* eval_buf;                /* [eval_cap][n] */
  int64_t eval_cap;
  int64_t* eval_rec;              /* [eval_cap][5] s_cur, round, flops, classified, clean */
  double* eval_wall_ms;           /* [eval_cap] */
  int64_t* eval_count;
  const int64_t* flops_cell;
  const int64_t* classified_cell;
  const int64_t* clean_cell;
  /* in-situ K4 timing (CUDA events around every round's launch) */
  int32_t time_rounds;
  double* k4_ms;                  /* summed */
  int64_t* k4_rounds;             /* timed rounds */
  /* the updaters classify with the round floor (lpp_tag_plan): the round
   * counts as applied (last_avg_stamp) only after every owner is done with
   * this worker's arena (fence 1), with no per-element tag writes */
  int32_t stamp_floor;
  /* the worker's device round-stamp cell (lpp_set_i64 before last_avg_stamp
   * moves; NULL: none) */
  int64_t* round_cell;
} lpp_averager_cfg;

int lpp_averager_run(const lpp_averager_cfg* cfg, int64_t* rounds_out);

/* p[i] = v for i in [0, n) (int32, stream-ordered) */
int lpp_fill_i32(int32_t* p, size_t n, int32_t v, void* stream);

/* ---- fp32 3x3 / stride-1 / pad-1 C->C convolutions (csrc/conv_f32.cu) ----
 * The gradient step of SURVEY §8 a6 on the GPU: the CNN forward/backward.
 * Replaces, for CIFAR ResNet-20's 3x3 stride-1 C->C convolutions in fp32
 * (TF32 off), the cuDNN calls torch's F.conv2d / convolution_backward make
 * (the reference computes these in fp64 numpy/torch-CPU on its objectives'
 * grad_block, objectives.py:33-63).  Activations NHWC [n][hw][hw][c]
 * (torch channels_last), weights and their gradient OHWI [c][3][3][c] (the
 * arena's channels_last view).  Shapes with a kernel: (c, hw) in
 * {(16, 32), (32, 16), (64, 8)}. */
int lpp_conv3x3_supported(int c, int hw);
/* measurement utility: blocks x 256 threads x iters x 128 dependent-chain
 * FFMAs (8 chains per thread), no memory traffic — the fp32 FMA peak the
 * convolutions' roofline divides by (2 flops per FFMA) */
int lpp_fma_probe(float* out, int blocks, int iters, void* stream);
/* dgrad = 0: y = conv(x, w); dgrad = 1: y = dX of conv for dY = x;
 * dgrad = 2: y = conv(x, w) with w tap-major (lpp_conv3x3_tapmajor).
 * Forward only, stat_sums != NULL: also the BatchNorm statistics of y,
 * stat_sums[c][2] = (sum, sum of squares) over the n x hw x hw pixels, fused
 * into the epilogue and reduced in the same launch (fixed order, as
 * lpp_conv3x3_wgrad_f32), with stat_ws (lpp_conv3x3_stats_workspace bytes)
 * and LPP_CONV_ARRIVALS zeroed stat_arrivals cells.  dgrad = 1 with
 * stat_ws != NULL: y = dX + stat_ws (an NHWC addend of stat_ws_bytes >= the
 * output's: the residual branch's gradient of the same activation). */
int lpp_conv3x3_f32(const float* x, const float* w, float* y, int n, int c, int hw, int dgrad,
                    float* stat_ws, size_t stat_ws_bytes, float* stat_sums, uint32_t* stat_arrivals,
                    void* stream);
size_t lpp_conv3x3_stats_workspace(int n, int c, int hw);
/* wt[t][ci][co] = w[co][t][ci]: tap-major weights for lpp_conv3x3_f32's
 * dgrad = 2 (a forward whose weights need no per-CTA transpose) */
int lpp_conv3x3_tapmajor(const float* w, float* wt, int c, void* stream);
/* bytes of workspace lpp_conv3x3_wgrad_f32 needs (per-cluster partial sums) */
size_t lpp_conv3x3_wgrad_workspace(int n, int c, int hw);
/* dw = sum over pixels of x (*) dy in ONE launch, deterministic: CTA
 * partials summed over thread-block-cluster DSMEM in rank order, cluster
 * partials summed in cluster order by the last cluster to arrive.
 * arrivals: LPP_CONV_ARRIVALS uint32 device cells, zero before the first
 * call and left zero by every call; one set per stream (launches sharing a
 * set must be stream-ordered). */
#define LPP_CONV_ARRIVALS 8

/* 1x1 stride-2 projection shortcuts (ci -> co, hw_in -> hw_in / 2) at
 * CIFAR ResNet-20's shapes {(16, 32, 32), (32, 64, 16)}.
 * mode 0: out = y  of (a = x [n][hw][hw][ci], b = w [co][ci]);
 * mode 1: out = dX of (a = dY [n][hw/2][hw/2][co], b = w);
 * mode 2: out = dW of (a = x, b = dY), one launch, deterministic (as
 *         lpp_conv3x3_wgrad_f32; ws / arrivals used only here). */
int lpp_conv1x1s2_supported(int ci, int co, int hw_in);
/* 3x3 stride-2 pad-1 convolutions (ci -> co, hw_in -> hw_in / 2) at the
 * same shapes, same modes and arguments (w [co][3][3][ci]); dgrad per 2x2
 * quad of dX pixels (no products with inserted zeros) */
int lpp_conv3x3s2_supported(int ci, int co, int hw_in);
size_t lpp_conv3x3s2_wgrad_workspace(int n, int ci, int co, int hw_in);
int lpp_conv3x3s2_f32(const float* a, const float* b, float* out, int n, int ci, int co, int hw_in, int mode,
                      float* ws, size_t ws_bytes, uint32_t* arrivals, float* stat_sums, void* stream);
size_t lpp_conv3x3s2_stats_workspace(int n, int ci, int co, int hw_in);

/* BatchNorm in training mode from the fused statistics (sums[c][2] of the
 * npix pixels, NHWC x of c in {16, 32, 64} channels):
 * y = [relu](x * gamma * invstd + beta - mean * gamma * invstd [+ resid]);
 * writes save_mean / save_invstd (the backward's inputs, as
 * torch.native_batch_norm) and, when given, moves running_mean /
 * running_var by momentum (unbiased variance) — BatchNorm2d.forward
 * (+ the block's residual add and ReLU) in one memory pass.  relu: also
 * relu_mask, 1 bit per element (npix * c / 32 words), for the backward. */
int lpp_bn_apply_f32(const float* x, const float* sums, const float* gamma, const float* beta,
                     const float* resid, float* y, float* save_mean, float* save_invstd,
                     float* running_mean, float* running_var, uint32_t* relu_mask, int64_t npix, int c,
                     float eps, float momentum, int relu, void* stream);
/* its backward in two launches (a cluster-reduced per-channel sum, then
 * the elementwise pass): g = gy [* relu_mask]; dx = gamma * invstd * (g -
 * mean(g) - xhat * mean(g xhat)); gres = g (the residual branch, NULL:
 * none); ggamma / gbeta = sum g xhat / sum g (NULL: not wanted); dx NULL:
 * not wanted.  ws: lpp_bn_backward_workspace bytes; arrivals as
 * lpp_conv3x3_wgrad_f32. */
size_t lpp_bn_backward_workspace(int64_t npix, int c);
/* The CIFAR stem (3 -> 16, 3x3, 32 x 32) reading the input batch in NCHW:
 * mode 0 y = conv(a = x, b = w) (+ BatchNorm statistics into stat_sums);
 * mode 2 dW [16][3][3][3] (OHWI) of (a = x, b = dY); ws of
 * lpp_stem_workspace bytes, arrivals as lpp_conv3x3_wgrad_f32. */
size_t lpp_stem_workspace(int n);
int lpp_stem_f32(const float* a, const float* b, float* out, int n, int mode, float* ws, size_t ws_bytes,
                 uint32_t* arrivals, float* stat_sums, void* stream);
int lpp_bn_backward_f32(const float* gy, const uint32_t* relu_mask, const float* x, const float* mean,
                        const float* invstd,
                        const float* gamma, float* dx, float* gres, float* ggamma, float* gbeta, float* ws,
                        size_t ws_bytes, uint32_t* arrivals, int64_t npix, int c, int relu, void* stream);
size_t lpp_conv1x1s2_wgrad_workspace(int n, int ci, int co, int hw_in);
int lpp_conv1x1s2_f32(const float* a, const float* b, float* out, int n, int ci, int co, int hw_in, int mode,
                      float* ws, size_t ws_bytes, uint32_t* arrivals, float* stat_sums, void* stream);
/* mode 0 with stat_sums: the fused BatchNorm statistics of y (as
 * lpp_conv3x3_f32; ws of lpp_conv1x1s2_stats_workspace bytes) */
size_t lpp_conv1x1s2_stats_workspace(int n, int ci, int co, int hw_in);
int lpp_conv3x3_wgrad_f32(const float* x, const float* dy, float* dw, float* ws, size_t ws_bytes,
                          uint32_t* arrivals, int n, int c, int hw, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LPP_B200_H */
