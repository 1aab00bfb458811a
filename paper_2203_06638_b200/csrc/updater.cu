// updater.cu — the native updater loop, the native
// averager (a11) and device-side batch sampling for captured steps.
//
// lpp_updater_run is the reference's _updater_loop / _updater_body
// (engine.py:289-383) for one updater stream, with the per-step host work
// (claim, lr_at, select_block, stamp, tag draw, launches, in-flight window,
// clean classification) in C++: the Python engine calls it once per updater
// thread through ctypes, which drops the GIL for the whole run, so U
// updater threads issue their steps truly concurrently and the averager
// thread (Python, host atomics) runs beside them.  The CUDA work it
// enqueues per step is exactly the Python loop's: the K5 gather, K3 (or
// nothing, fused), the captured fwd/bwd graph of the step's block, and the
// K1/K2 (or fused K1+K3) apply — through the same C-ABI entry points.
//
// lpp_averager_run is _averager_body (engine.py:385-453) restated over the
// round-control block of rounds.py: the same open / vote / fence / stamp
// protocol, so native and Python averagers interoperate across processes.

#include "common.cuh"

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <ctime>
#include <thread>
#include <vector>

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ int64_t sample_one(uint64_t key, int64_t step, int i,
                                                       uint64_t n) {
  uint64_t base = mix64(key ^ mix64((uint64_t)step));
  uint64_t r = mix64(base + (uint64_t)i * 0xD1B54A32D192ED03ull);
#ifdef __CUDA_ARCH__
  return (int64_t)__umul64hi(r, n);
#else
  return (int64_t)(((unsigned __int128)r * n) >> 64);
#endif
}

// epoch-partition sampling (f4: EpochSampler, objectives.py:77-104, on the
// device): position pos = step * B + i of an updater's stream is element
// perm_e(pos mod m) of its worker's shard (base + p * stride, the
// reference's arange(n)[q::Q]), epoch e = pos / m, perm_e a keyed bijection
// of [0, m): a 4-round balanced Feistel network on the next even power of two,
// cycle-walked back into [0, m).  Every epoch visits each shard element
// exactly once, in a fresh order, with no stored permutation.
__host__ __device__ __forceinline__ uint64_t feistel_perm(uint64_t j, uint64_t m, uint64_t key) {
  int bits = 2;
  while ((1ull << bits) < m) ++bits;
  if (bits & 1) ++bits;
  const int half = bits / 2;
  const uint64_t mask = (1ull << half) - 1;
  uint64_t x = j;
  do {
    uint64_t l = x >> half, r = x & mask;
#pragma unroll
    for (int round = 0; round < 4; ++round) {
      uint64_t f = mix64(key ^ (0x9E3779B97F4A7C15ull * (uint64_t)(round + 1)) ^ r) & mask;
      uint64_t nl = r;
      r = l ^ f;
      l = nl;
    }
    x = (l << half) | r;
  } while (x >= m);
  return x;
}

__host__ __device__ __forceinline__ int64_t epoch_one(uint64_t key, int64_t step, int i, int batch,
                                                      int64_t base, int64_t stride, uint64_t m) {
  uint64_t pos = (uint64_t)step * (uint64_t)batch + (uint64_t)i;
  uint64_t e = pos / m, j = pos % m;
  uint64_t p = feistel_perm(j, m, mix64(key ^ mix64(e + 0x632BE59BD9B4E019ull)));
  return base + (int64_t)p * stride;
}

__global__ void k_sample_epoch(int64_t* idx, int64_t* step, int b, int64_t base, int64_t stride,
                               uint64_t m, uint64_t key) {
  const int64_t t = *step;
  for (int i = threadIdx.x; i < b; i += blockDim.x) idx[i] = epoch_one(key, t, i, b, base, stride, m);
  __syncthreads();
  if (threadIdx.x == 0) *step = t + 1;
}

__global__ void k_sample_indices(int64_t* idx, int64_t* step, int b, uint64_t n, uint64_t key) {
  const int64_t t = *step;
  for (int i = threadIdx.x; i < b; i += blockDim.x) idx[i] = sample_one(key, t, i, n);
  __syncthreads();
  if (threadIdx.x == 0) *step = t + 1;
}

}  // namespace

extern "C" int lpp_sample_indices(int64_t* idx, int64_t* step, int32_t batch, int64_t n,
                                  uint64_t key, void* stream) {
  if (batch <= 0) return LPP_OK;
  if (!idx || !step) return set_err(LPP_E_VALUE, "sample_indices: null buffer");
  if (n <= 0) return set_err(LPP_E_VALUE, "sample_indices: empty population");
  int threads = std::min(1024, ((batch + 31) / 32) * 32);
  k_sample_indices<<<1, threads, 0, (cudaStream_t)stream>>>(idx, step, batch, (uint64_t)n, key);
  LAUNCH_CHECK("sample_indices");
  return LPP_OK;
}

extern "C" int lpp_sample_indices_host(int64_t* out, int32_t batch, int64_t n, uint64_t key,
                                       int64_t step) {
  if (batch <= 0) return LPP_OK;
  if (!out) return set_err(LPP_E_VALUE, "sample_indices_host: null buffer");
  if (n <= 0) return set_err(LPP_E_VALUE, "sample_indices_host: empty population");
  for (int i = 0; i < batch; ++i) out[i] = sample_one(key, step, i, (uint64_t)n);
  return LPP_OK;
}

extern "C" int lpp_sample_epoch(int64_t* idx, int64_t* step, int32_t batch, int64_t shard_base,
                                int64_t shard_stride, int64_t shard_len, uint64_t key,
                                void* stream) {
  if (batch <= 0) return LPP_OK;
  if (!idx || !step) return set_err(LPP_E_VALUE, "sample_epoch: null buffer");
  if (shard_len <= 0 || shard_stride <= 0 || shard_base < 0)
    return set_err(LPP_E_VALUE, "sample_epoch: empty or invalid shard");
  int threads = std::min(1024, ((batch + 31) / 32) * 32);
  k_sample_epoch<<<1, threads, 0, (cudaStream_t)stream>>>(idx, step, batch, shard_base, shard_stride,
                                                          (uint64_t)shard_len, key);
  LAUNCH_CHECK("sample_epoch");
  return LPP_OK;
}

extern "C" int lpp_sample_epoch_host(int64_t* out, int32_t batch, int64_t shard_base,
                                     int64_t shard_stride, int64_t shard_len, uint64_t key,
                                     int64_t step) {
  if (batch <= 0) return LPP_OK;
  if (!out) return set_err(LPP_E_VALUE, "sample_epoch_host: null buffer");
  if (shard_len <= 0 || shard_stride <= 0 || shard_base < 0)
    return set_err(LPP_E_VALUE, "sample_epoch_host: empty or invalid shard");
  for (int i = 0; i < batch; ++i)
    out[i] = epoch_one(key, step, i, batch, shard_base, shard_stride, (uint64_t)shard_len);
  return LPP_OK;
}

// lr_at (schedules.py:56-68): the operations and their order follow the
// Python restatement exactly so that the two agree bit for bit
extern "C" double lpp_lr_at(int kind, double alpha0, double peak, int64_t warmup, int64_t total,
                            const int64_t* milestones, int n_milestones, double gamma,
                            int64_t s) {
  if (s < warmup) return alpha0 + (peak - alpha0) * (double)s / (double)warmup;
  if (kind == 0) {
    if (s >= total) return 0.0;
    int64_t span = total - warmup;
    return peak * 0.5 * (1.0 + std::cos(M_PI * (double)(s - warmup) / (double)span));
  }
  int drops = 0;
  for (int i = 0; i < n_milestones; ++i)
    if (s >= milestones[i]) ++drops;
  return peak * std::pow(gamma, (double)drops);
}

// select_block (partition.py:132-145)
extern "C" int lpp_select_block(int64_t s, int64_t warm_start, int num_blocks, int rank) {
  if (rank < 1 || rank > num_blocks)
    return set_err(LPP_E_VALUE, "select_block: rank %d outside [1, %d]", rank, num_blocks);
  if (s <= warm_start) return 0;
  if ((s - warm_start) & 1) return 0;
  return rank;
}

// the reference's numpy sampling stream (csrc/nprng.cu)
namespace nprng {
struct Pcg64;
}
nprng::Pcg64* lpp_nprng_new_impl(const uint64_t* ints, int n);
void lpp_nprng_free_impl(nprng::Pcg64* g);
void lpp_nprng_integers_impl(nprng::Pcg64* g, int64_t n, int32_t b, int64_t* out);
void lpp_nprng_choice_impl(nprng::Pcg64* g, int64_t pop, int32_t k, int64_t* out);
void lpp_nprng_permutation_impl(nprng::Pcg64* g, int64_t m, int64_t* out);

namespace {

struct NpRngOwner {
  nprng::Pcg64* g = nullptr;
  ~NpRngOwner() {
    if (g) lpp_nprng_free_impl(g);
  }
};

struct Events {
  std::vector<cudaEvent_t> ev;
  ~Events() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
  int make(int count, unsigned flags) {
    for (int i = 0; i < count; ++i) {
      cudaEvent_t e = nullptr;
      CUDA_TRY(cudaEventCreateWithFlags(&e, flags));
      ev.push_back(e);
    }
    return LPP_OK;
  }
};

// k sorted distinct indices in [0, d) from a splitmix64 stream (the
// sampled-tag draw; the Python loop draws the reference's numpy stream)
void draw_tags(uint64_t* state, int64_t d, int k, int64_t* out) {
  int got = 0;
  while (got < k) {
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t r = mix64(*state);
    int64_t v = (int64_t)(((unsigned __int128)r * (uint64_t)d) >> 64);
    bool dup = false;
    for (int j = 0; j < got; ++j) dup |= (out[j] == v);
    if (!dup) out[got++] = v;
  }
  std::sort(out, out + k);
}

}  // namespace

extern "C" int lpp_updater_run(const lpp_updater_cfg* c, lpp_updater_stats* st) {
  if (!c || !st) return set_err(LPP_E_VALUE, "updater_run: null cfg/stats");
  if (!c->sample_counter || !c->update_order || !c->stop || !c->last_avg_stamp)
    return set_err(LPP_E_VALUE, "updater_run: null control cell");
  if (!c->block_lo || !c->block_hi || !c->graph_exec || !c->flops_of)
    return set_err(LPP_E_VALUE, "updater_run: null block tables");
  if (!c->x || !c->g || !c->replica || c->n == 0)
    return set_err(LPP_E_VALUE, "updater_run: null arena");
  if (c->lpp && (c->rank < 1 || c->rank > c->num_blocks))
    return set_err(LPP_E_VALUE, "updater_run: rank %d outside [1, %d]", c->rank, c->num_blocks);
  const bool tagged = c->tags != nullptr;
  const int K = tagged ? c->tag_pick : 0;
  if (K > 0 && (!c->tag_idx_pinned || !c->tag_idx_dev || !c->rec_dev || !c->rec_pinned ||
                c->rec_cols < 2 + (K + 1) / 2 || !c->avg_cell_dev || !c->classified || !c->clean ||
                (c->fused && (!c->block_stamps || !c->block_bounds_dev))))
    return set_err(LPP_E_VALUE, "updater_run: tag sampling buffers missing");
  const int F = c->in_flight < 1 ? 1 : c->in_flight;
  const int depth = F + 2;
  cudaStream_t stream = (cudaStream_t)c->stream;
  const bool host = c->host_feats != nullptr;
  if (host && (!c->host_labels || !c->feat_pinned || !c->label_pinned || !c->xbuf[0] ||
               !c->xbuf[1] || !c->ybuf[0] || !c->ybuf[1] || !c->copy_stream || c->batch <= 0 ||
               c->n_rows <= 0 || c->row_bytes <= 0 || c->label_bytes <= 0))
    return set_err(LPP_E_VALUE, "updater_run: host-batch buffers missing");
  if (c->read_loss && (!c->loss_dev[0] || !c->loss_dev[1] || !c->loss_pinned || !c->loss_log ||
                       !c->loss_count))
    return set_err(LPP_E_VALUE, "updater_run: loss read-back buffers missing");

  cudaStream_t astream = c->apply_stream ? (cudaStream_t)c->apply_stream : stream;
  const bool side = astream != stream;
  cudaStream_t cstream = host ? (cudaStream_t)c->copy_stream : stream;
  Events done, t0, t1, order, copied, buf_free;
  int rc;
  if ((rc = done.make(F, cudaEventDisableTiming)) != LPP_OK) return rc;
  if (side && (rc = order.make(2, cudaEventDisableTiming)) != LPP_OK) return rc;
  if (host && (rc = copied.make(depth, cudaEventDisableTiming)) != LPP_OK) return rc;
  if (host && (rc = buf_free.make(2, cudaEventDisableTiming)) != LPP_OK) return rc;
  std::vector<int64_t> idx((host || c->host_rng) ? c->batch : 0);
  // the reference's host stream: one generator per updater, plus the
  // EpochSampler's per-epoch generators (objectives.py:77-104)
  NpRngOwner rng;
  if (c->host_rng) {
    if (c->n_entropy < 1 || c->n_entropy > 4 || c->batch <= 0 || c->n_rows <= 0)
      return set_err(LPP_E_VALUE, "updater_run: host_rng needs entropy, batch and n_rows");
    if (!host && (!c->idx_pinned || !c->idx_dev))
      return set_err(LPP_E_VALUE, "updater_run: host_rng index ring missing");
    rng.g = lpp_nprng_new_impl(c->rng_entropy, c->n_entropy);
  }
  std::vector<int64_t> ep_order, ep_perm;
  int64_t ep_pos = 0, ep_epoch = -1;
  auto epoch_batch = [&](int64_t* out) {
    int got = 0;
    while (got < c->batch) {
      if (ep_pos >= (int64_t)ep_order.size()) {
        ++ep_epoch;
        const uint64_t ent[2] = {(uint64_t)c->epoch_seed, (uint64_t)ep_epoch};
        NpRngOwner eg;
        eg.g = lpp_nprng_new_impl(ent, 2);
        ep_perm.resize(c->epoch_len);
        lpp_nprng_permutation_impl(eg.g, c->epoch_len, ep_perm.data());
        ep_order.resize(c->epoch_len);
        for (int64_t i = 0; i < c->epoch_len; ++i)
          ep_order[i] = c->epoch_base + ep_perm[i] * c->epoch_stride;
        ep_pos = 0;
      }
      int64_t take = std::min<int64_t>(c->batch - got, (int64_t)ep_order.size() - ep_pos);
      for (int64_t i = 0; i < take; ++i) out[got + i] = ep_order[ep_pos + i];
      ep_pos += take;
      got += (int)take;
    }
  };
  auto draw_ref_tags = [&](int slot) {
    int64_t* h = c->tag_idx_pinned + (size_t)slot * K;
    lpp_nprng_choice_impl(rng.g, (int64_t)c->n, K, h);
    std::sort(h, h + K);
  };
  if (c->time_apply) {
    if ((rc = t0.make(F, cudaEventDefault)) != LPP_OK) return rc;
    if ((rc = t1.make(F, cudaEventDefault)) != LPP_OK) return rc;
  }
  std::vector<char> used(F, 0);
  std::vector<int64_t> claim_of(F, 0);
  std::vector<int> slot_of(F, 0);
  std::vector<double> bytes_of(F, 0.0);
  std::vector<int64_t> step_of(F, 0);
  uint64_t tag_state = c->tag_seed;
  *st = lpp_updater_stats{};

  // a step's sampled tags live in slot t % depth (indices drawn into the
  // pinned ring; unfused gathers read them from the device ring, the fused
  // apply takes them by value).  Unfused steps (and the first fused
  // one) gather them before their snapshot values are read
  // (paramstore.py:108-112); fused steps get them from the previous step's
  // apply kernel, after that apply landed (engine.py:343-362 order)
  // draw (device-sampling runs; host_rng runs drew them in step order)
  // and copy one slot of indices to the device ring, on the updater stream
  auto draw_idx = [&](int slot) -> int {
    const size_t o = (size_t)slot * K;
    if (!c->host_rng) draw_tags(&tag_state, (int64_t)c->n, K, c->tag_idx_pinned + o);
    return lpp_copy_async(c->tag_idx_dev + o, c->tag_idx_pinned + o, 8 * (size_t)K, stream);
  };
  // step records: slot s = {k_claim, clean, tags[K] (int32)} in rec_cols cells
  auto rec_tags = [&](int slot) -> int32_t* {
    return reinterpret_cast<int32_t*>(c->rec_dev + (size_t)slot * c->rec_cols + 2);
  };
  auto rec_claim = [&](int slot) -> int64_t* { return c->rec_dev + (size_t)slot * c->rec_cols; };
  auto gather = [&](int slot) -> int {
    const size_t o = (size_t)slot * K;
    if (c->fused)  // fused runs stamp blocks, not elements
      return lpp_gather_block_stamps(c->block_stamps, c->block_bounds_dev, c->num_blocks,
                                     c->tag_idx_dev + o, (size_t)K, c->avg_cell_dev,
                                     rec_tags(slot), nullptr, stream);
    return lpp_gather_tags_floor(c->tags, c->tag_idx_dev + o, (size_t)K, c->avg_cell_dev,
                                 rec_tags(slot), nullptr, stream);
  };
  // the step's record to the host once its apply wrote (k_claim, clean)
  auto copy_rec = [&](int slot, cudaStream_t st_) -> int {
    const size_t o = (size_t)slot * c->rec_cols;
    return lpp_copy_async(c->rec_pinned + o, c->rec_dev + o, 8 * (size_t)c->rec_cols, st_);
  };
  // once a step's event completed: classify its tags, collect its apply time
  auto retire = [&](int k) -> int {
    if (c->read_loss) {
      int64_t i = *c->loss_count;
      if (i < c->loss_cap) c->loss_log[i] = c->loss_pinned[slot_of[k]];
      *c->loss_count = i + 1;
    }
    if (K > 0) {
      // (k_claim, clean) as the step's apply kernel saw them
      const int64_t* row = c->rec_pinned + (size_t)slot_of[k] * c->rec_cols;
      const int32_t* tg = reinterpret_cast<const int32_t*>(row + 2);
      const int64_t kc = row[0];
      const bool clean = row[1] != 0;
      __atomic_fetch_add(c->classified, 1, __ATOMIC_ACQ_REL);
      if (clean) __atomic_fetch_add(c->clean, 1, __ATOMIC_ACQ_REL);
      const int64_t ts = step_of[k];
      if (c->rec_i64 && ts < c->rec_cap) {
        c->rec_i64[6 * ts + 2] = kc;
        c->rec_i64[6 * ts + 5] = clean ? 1 : 0;
        if (c->rec_tags)
          for (int j = 0; j < K; ++j) c->rec_tags[(size_t)ts * K + j] = tg[j];
        if (c->rec_tag_idx) {
          const int64_t* ti = c->tag_idx_pinned + (size_t)slot_of[k] * K;
          for (int j = 0; j < K; ++j) c->rec_tag_idx[(size_t)ts * K + j] = ti[j];
        }
      }
    }
    if (c->time_apply) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, t0.ev[k], t1.ev[k]));
      st->apply_ms += ms;
      if (c->apply_ms_log && st->apply_launches < c->apply_ms_cap)
        c->apply_ms_log[st->apply_launches] = ms;
      st->apply_bytes += bytes_of[k];
      st->apply_launches += 1;
    }
    return LPP_OK;
  };

  int64_t s = 0, t = 0;
  while (s < c->budget && __atomic_load_n(c->stop, __ATOMIC_ACQUIRE) == 0) {
    s = __atomic_fetch_add(c->sample_counter, 1, __ATOMIC_ACQ_REL);               // engine.py:336
    const double lr = lpp_lr_at(c->lr_kind, c->alpha0, c->peak, c->warmup, c->total,
                                c->milestones, c->n_milestones, c->gamma, s);
    const int b = c->lpp ? lpp_select_block(s, c->warm_start, c->num_blocks, c->rank) : 0;
    const int k = (int)(t % F);
    if (used[k]) {
      CUDA_TRY(cudaEventSynchronize(done.ev[k]));
      if ((rc = retire(k)) != LPP_OK) return rc;
    }
    const int slot = (int)(t % depth), next_slot = (int)((t + 1) % depth);
    // untagged runs record k_claim at enqueue; tagged ones take it from
    // the apply kernel, which reads it after the gradient (engine.py:353)
    const int64_t k_claim = K > 0 ? -1 : __atomic_load_n(c->last_avg_stamp, __ATOMIC_ACQUIRE);
    const int64_t u = __atomic_fetch_add(c->update_order, 1, __ATOMIC_ACQ_REL) + 1;
    if (c->rec_i64 && t < c->rec_cap) {
      int64_t* row = c->rec_i64 + 6 * t;
      int reason = 0;  // select_block's reason (partition.py:132-145)
      if (c->lpp && s > c->warm_start) reason = ((s - c->warm_start) & 1) ? 1 : 2;
      row[0] = s, row[1] = u, row[2] = k_claim, row[3] = b, row[4] = reason, row[5] = -1;
      c->rec_lr[t] = lr;
    }
    const int64_t lo = c->block_lo[b], hi = c->block_hi[b], len = hi - lo;
    const float lr32 = (float)lr;
    const int buf = host ? (int)(t & 1) : 0;
    if (c->host_rng) {
      // the reference updater's draw order: sampled tag indices, then the
      // batch (engine.py:343-351); fused, the next step's tag indices follow
      if (K > 0 && (!c->fused || t == 0)) draw_ref_tags(slot);
      if (c->epoch_seed >= 0)
        epoch_batch(idx.data());
      else
        lpp_nprng_integers_impl(rng.g, c->n_rows, c->batch, idx.data());
      if (K > 0 && c->fused) draw_ref_tags(next_slot);
      if (!host) {
        int64_t* hp = c->idx_pinned + (size_t)slot * c->batch;
        std::memcpy(hp, idx.data(), sizeof(int64_t) * (size_t)c->batch);
        if ((rc = lpp_copy_async(c->idx_dev, hp, sizeof(int64_t) * (size_t)c->batch, stream)) != LPP_OK)
          return rc;
      }
    }
    if (host) {
      // end-to-end input: host draw + pinned row gather + H2D on the copy
      // stream into input buffer `buf` once the step that last read it is done
      if (!c->host_rng)
        for (int i = 0; i < c->batch; ++i)
          idx[i] = c->epoch_len > 0
                       ? epoch_one(c->sample_key, c->sample_step0 + t, i, c->batch, c->epoch_base,
                                   c->epoch_stride, (uint64_t)c->epoch_len)
                       : sample_one(c->sample_key, c->sample_step0 + t, i, (uint64_t)c->n_rows);
      char* fdst = static_cast<char*>(c->feat_pinned) + (size_t)slot * c->batch * c->row_bytes;
      char* ldst = static_cast<char*>(c->label_pinned) + (size_t)slot * c->batch * c->label_bytes;
      if ((rc = lpp_host_gather_rows(fdst, c->host_feats, (size_t)c->n_rows, (size_t)c->row_bytes,
                                     idx.data(), (size_t)c->batch)) != LPP_OK)
        return rc;
      if ((rc = lpp_host_gather_rows(ldst, c->host_labels, (size_t)c->n_rows,
                                     (size_t)c->label_bytes, idx.data(), (size_t)c->batch)) != LPP_OK)
        return rc;
      CUDA_TRY(cudaStreamWaitEvent(cstream, buf_free.ev[buf], 0));
      CUDA_TRY(cudaMemcpyAsync(c->xbuf[buf], fdst, (size_t)c->batch * c->row_bytes,
                               cudaMemcpyHostToDevice, cstream));
      CUDA_TRY(cudaMemcpyAsync(c->ybuf[buf], ldst, (size_t)c->batch * c->label_bytes,
                               cudaMemcpyHostToDevice, cstream));
      CUDA_TRY(cudaEventRecord(copied.ev[slot], cstream));
      CUDA_TRY(cudaStreamWaitEvent(stream, copied.ev[slot], 0));
    }
    if (!c->fused || t == 0) {
      if (K > 0) {
        if ((rc = draw_idx(slot)) != LPP_OK) return rc;
        if ((rc = gather(slot)) != LPP_OK) return rc;                               // K5
      }
      if ((rc = lpp_snapshot(c->x, c->replica, c->n, stream)) != LPP_OK) return rc;   // K3
    }
    // the next step's tag indices (host ring; the apply launch takes them by value)
    if (c->fused && K > 0 && !c->host_rng)
      draw_tags(&tag_state, (int64_t)c->n, K, c->tag_idx_pinned + (size_t)next_slot * K);
    if ((rc = lpp_graph_launch(c->graph_exec[2 * b + buf], stream)) != LPP_OK) return rc;  // fwd+bwd
    if (host) CUDA_TRY(cudaEventRecord(buf_free.ev[buf], stream));
    if (c->read_loss)
      CUDA_TRY(cudaMemcpyAsync(c->loss_pinned + slot, c->loss_dev[buf], sizeof(float),
                               cudaMemcpyDeviceToHost, stream));
    if (side) {  // the apply on its own (high-priority) stream, after the graph
      CUDA_TRY(cudaEventRecord(order.ev[0], stream));
      CUDA_TRY(cudaStreamWaitEvent(astream, order.ev[0], 0));
    }
    if (c->time_apply) CUDA_TRY(cudaEventRecord(t0.ev[k], astream));
    if (c->fused && K > 0) {
      // K1+K3 + K5: classify this step, read the next step's tags (block_hi
      // serves as the boundaries: block_hi[b] = end of partial block b)
      const size_t on = (size_t)next_slot * K;
      lpp_tag_plan plan{c->tag_idx_pinned + on, rec_tags(next_slot), nullptr, rec_tags(slot),
                        rec_claim(slot),       c->avg_cell_dev,      c->block_stamps,
                        c->block_hi,           c->num_blocks,        b,           K};
      rc = lpp_apply_snapshot_plan(c->x, c->g, c->m, c->replica, nullptr, c->n, (size_t)lo,
                                   (size_t)hi, lr32, nullptr, c->mu, c->wd, (int32_t)u, &plan,
                                   astream);
      bytes_of[k] = c->apply_bytes_per_elem * (double)len + 4.0 * (double)(c->n - len) +
                    4.0 * (double)c->n;
    } else if (c->fused) {
      rc = lpp_apply_snapshot(c->x, c->g, c->m, c->replica, tagged ? c->tags : nullptr, c->n,
                              (size_t)lo, (size_t)hi, lr32, nullptr, c->mu, c->wd, (int32_t)u,
                              astream);                                               // K1+K3
      bytes_of[k] = c->apply_bytes_per_elem * (double)len + 4.0 * (double)(c->n - len) +
                    4.0 * (double)c->n;
    } else if (tagged) {
      if (K > 0) {  // k_claim after the gradient, on the apply's stream
        rc = lpp_classify(rec_tags(slot), (size_t)K, c->avg_cell_dev, rec_claim(slot), astream);
        if (rc != LPP_OK) return rc;
      }
      rc = lpp_apply_sgd_tagged(c->x + lo, c->g + lo, c->m ? c->m + lo : nullptr, (size_t)len,
                                lr32, nullptr, c->mu, c->wd, c->apply_mode, c->tags + lo,
                                (int32_t)u, astream);                                 // K1/K2+K5
      bytes_of[k] = c->apply_bytes_per_elem * (double)len;
    } else {
      rc = lpp_apply_sgd(c->x + lo, c->g + lo, c->m ? c->m + lo : nullptr, (size_t)len, lr32,
                         nullptr, c->mu, c->wd, c->apply_mode, astream);              // K1/K2
      bytes_of[k] = c->apply_bytes_per_elem * (double)len;
    }
    if (rc != LPP_OK) return rc;
    if (c->time_apply) CUDA_TRY(cudaEventRecord(t1.ev[k], astream));

    if (side) {
      CUDA_TRY(cudaEventRecord(order.ev[1], astream));
      CUDA_TRY(cudaStreamWaitEvent(stream, order.ev[1], 0));
    }
    // K5 bookkeeping on the updater stream, ordered after the apply: this
    // update's block stamp, then the step's record to the host (queued
    // behind the apply on the high-priority apply stream, the copy measured
    // +5 us on the apply's in-situ time, tools/exp_insitu_variants.py)
    if (c->fused && K > 0 &&
        (rc = lpp_publish_stamp(c->block_stamps, b, (int32_t)u, stream)) != LPP_OK)
      return rc;
    if (K > 0 && (rc = copy_rec(slot, stream)) != LPP_OK) return rc;
    CUDA_TRY(cudaEventRecord(done.ev[k], stream));
    used[k] = 1;
    claim_of[k] = k_claim;
    slot_of[k] = slot;
    step_of[k] = t;
    st->flops += c->flops_of[b];
    if (c->graph_kernels_of) st->graph_kernels += c->graph_kernels_of[b];
    ++t;
  }
  CUDA_TRY(cudaStreamSynchronize(stream));
  for (int64_t tt = t - F < 0 ? 0 : t - F; tt < t; ++tt)   // the last steps, in step order
    if ((rc = retire((int)(tt % F))) != LPP_OK) return rc;
  st->steps = t;
  if (c->rec_count) *c->rec_count = t < c->rec_cap ? t : c->rec_cap;
  return LPP_OK;
}

// ---------------------------------------------------------------------------
// native averager (a11)

namespace {

__global__ void k_fill_i32(int32_t* p, size_t n, int32_t v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}

inline double now_s() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

// RoundControl layout (rounds.py)
constexpr int64_t kHeader = 16, kStamps = 8, kRing = 8;   // rounds.RoundControl.RING
inline int64_t* cell(const lpp_averager_cfg* c, int64_t i) { return c->ctrl + i; }
inline int64_t* vote_cell(const lpp_averager_cfg* c, int64_t r) { return cell(c, kHeader + r % kRing); }
inline int64_t* final_cell(const lpp_averager_cfg* c, int64_t r) {
  return cell(c, kHeader + kRing + r % kRing);
}
inline int64_t* fence_cell(const lpp_averager_cfg* c, int which, int64_t r) {
  return cell(c, kHeader + (2 + which) * kRing + r % kRing);
}
inline int64_t ld(const int64_t* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
inline void st(int64_t* p, int64_t v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }
inline int64_t add(int64_t* p, int64_t d) { return __atomic_fetch_add(p, d, __ATOMIC_ACQ_REL); }

}  // namespace

extern "C" int lpp_fill_i32(int32_t* p, size_t n, int32_t v, void* stream) {
  if (n == 0) return LPP_OK;
  if (!p) return set_err(LPP_E_VALUE, "fill_i32: null buffer");
  size_t want = (n + 255) / 256;
  unsigned grid = (unsigned)(want < 2368 ? want : 2368);
  k_fill_i32<<<grid, 256, 0, (cudaStream_t)stream>>>(p, n, v);
  LAUNCH_CHECK("fill_i32");
  return LPP_OK;
}

extern "C" int lpp_averager_run(const lpp_averager_cfg* c, int64_t* rounds_out) {
  if (!c || !rounds_out) return set_err(LPP_E_VALUE, "averager_run: null cfg");
  if (!c->ctrl || !c->sample_counter || !c->update_order || !c->exited || !c->last_avg_stamp ||
      !c->synced_at || !c->arenas || !c->mean_out)
    return set_err(LPP_E_VALUE, "averager_run: null pointer");
  if (c->workers < 1 || c->workers > LPP_MAX_WORKERS || c->q < 0 || c->q >= c->workers)
    return set_err(LPP_E_VALUE, "averager_run: worker %d of %d", c->q, c->workers);
  if (c->tagged && !c->tags) return set_err(LPP_E_VALUE, "averager_run: tagged without tags");
  const int Q = c->workers;
  int64_t* round_calls = cell(c, 0);
  int64_t* stop = cell(c, 1);
  int64_t* abort_ = cell(c, 2);
  int64_t* drained = cell(c, 3);
  cudaStream_t stream = (cudaStream_t)c->stream;
  int64_t s_pre = 0, round_no = 0;
  double backoff = 0.0;
  *rounds_out = 0;
  const bool evalm = c->eval_interval > 0;
  if (evalm && (!c->eval_buf || !c->eval_rec || !c->eval_wall_ms || !c->eval_count ||
                !c->shard_bounds || !c->flops_cell || !c->classified_cell || !c->clean_cell))
    return set_err(LPP_E_VALUE, "averager_run: eval buffers missing");
  int64_t next_eval = c->eval_interval;
  if (evalm) *c->eval_count = 0;
  // fence 0: every worker's stamp is published before owners write tags;
  // fence 1: every owner is done with this worker's arena before the round
  // counts as applied (last_avg_stamp: the updaters' k_claim and tag floor)
  const bool fenced0 = c->tagged;
  const bool fenced1 = c->tagged || evalm || c->stamp_floor;
  const bool timed = c->time_rounds && c->k4_ms && c->k4_rounds && Q > 1;
  cudaEvent_t k4a = nullptr, k4b = nullptr;
  struct EvPair {
    cudaEvent_t* a;
    cudaEvent_t* b;
    ~EvPair() {
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
    }
  } k4ev{&k4a, &k4b};
  if (timed) {
    CUDA_TRY(cudaEventCreate(&k4a));
    CUDA_TRY(cudaEventCreate(&k4b));
    *c->k4_ms = 0.0;
    *c->k4_rounds = 0;
  }
  auto wait_ge = [&](const int64_t* p, int64_t target) -> bool {
    return lpp_atomic_wait_ge_i64(p, target, abort_, 200) != INT64_MIN;
  };
  auto fail = [&](int code) {
    st(abort_, 1);
    st(stop, 1);
    return code;
  };
  for (;;) {
    if (ld(abort_)) break;
    const int64_t s_cur = ld(c->sample_counter);
    const bool drain = ld(c->exited) == c->updaters;
    const bool pending = ld(round_calls) > round_no;
    const int64_t period = s_cur < c->switch_point ? 1 : c->period;      // sync_every
    const bool fresh = s_cur - s_pre >= period;
    if (!pending) {
      if (fresh || (drain && ld(drained) == Q)) {
        int64_t expected = round_no;
        __atomic_compare_exchange_n(round_calls, &expected, round_no + 1, false, __ATOMIC_ACQ_REL,
                                    __ATOMIC_ACQUIRE);
      } else {
        std::this_thread::sleep_for(std::chrono::duration<double>(backoff));
        backoff = std::min(2e-4, backoff * 2 + 1e-5);
        continue;
      }
    }
    backoff = 0.0;
    const int64_t r = round_no + 1;
    // vote (rounds.RoundControl.vote)
    if (drain) add(final_cell(c, r), 1);
    add(vote_cell(c, r), 1);
    // do_round: this worker's share of round r
    const int64_t u = add(c->update_order, 1) + 1;
    bool ok = true;
    int32_t stamps[LPP_MAX_WORKERS] = {0};
    if (fenced0) {
      st(cell(c, kStamps + c->q), u);
      add(fence_cell(c, 0, r), 1);
      ok = wait_ge(fence_cell(c, 0, r), Q);
      for (int i = 0; ok && i < Q; ++i) stamps[i] = (int32_t)ld(cell(c, kStamps + i));
    }
    const bool with_mean = drain || evalm;   // eval points need every round's mean
    if (ok) {
      int rc = LPP_OK;
      if (Q == 1) {
        // a single worker's mean is itself (test_engine.py:169-182)
        if (with_mean) rc = lpp_snapshot(c->arenas[0], c->mean_out, c->n, stream);
        if (rc == LPP_OK && c->tagged) rc = lpp_fill_i32(c->tags[0], c->n, stamps[0], stream);
      } else {
        float* mean = with_mean ? c->mean_out + c->lo : nullptr;
        if (timed) cudaEventRecord(k4a, stream);
        rc = c->tagged ? lpp_average_shard_tagged(c->arenas, c->tags, stamps, Q, c->lo, c->hi, mean,
                                                  LPP_MODE_RED, stream)
                       : lpp_average_shard(c->arenas, Q, c->lo, c->hi, mean, LPP_MODE_RED, stream);
        if (timed) cudaEventRecord(k4b, stream);
      }
      if (rc != LPP_OK) return fail(rc);
      cudaError_t e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) {
        fail(LPP_E_CUDA);
        return set_err(LPP_E_CUDA, "averager: stream sync failed: %s", cudaGetErrorString(e));
      }
      if (timed) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, k4a, k4b) == cudaSuccess) {
          *c->k4_ms += ms;
          *c->k4_rounds += 1;
        }
      }
      if (fenced1) {
        add(fence_cell(c, 1, r), 1);
        ok = wait_ge(fence_cell(c, 1, r), Q);
      }
      if (ok && c->round_cell) {
        // the device round-stamp cell the updaters' apply kernels read as
        // k_claim and tag floor (stream-ordered; no wait: the host cell
        // below serves host readers, the kernels read the device one)
        int rc2 = lpp_set_i64(c->round_cell, u, stream);
        if (rc2 != LPP_OK) return fail(rc2);
      }
      if (ok) {
        st(c->last_avg_stamp, u);
        st(c->synced_at, s_cur);
      }
    }
    // wait for every worker's vote (rounds.RoundControl.wait_votes)
    if (!wait_ge(vote_cell(c, r), Q)) break;
    const bool unanimous = ld(final_cell(c, r)) == Q;
    if (r > 1) {  // rounds.RoundControl.release: round r - 1's cells are free
      st(vote_cell(c, r - 1), 0);
      st(final_cell(c, r - 1), 0);
      st(fence_cell(c, 0, r - 1), 0);
      st(fence_cell(c, 1, r - 1), 0);
    }
    round_no = r;
    if (c->stop_after > 0 && round_no >= c->stop_after) st(stop, 1);
    if (c->rec && round_no <= c->max_records) {
      int64_t* row = c->rec + 5 * (round_no - 1);
      row[0] = r, row[1] = u, row[2] = s_cur, row[3] = s_cur - s_pre, row[4] = unanimous;
      if (c->rec_wall_ms) c->rec_wall_ms[round_no - 1] = 1e3 * (now_s() - c->t0);
    }
    *rounds_out = round_no;
    // eval point (worker 0): this round's mean, assembled from the owners
    if (evalm && ok && c->q == 0 && !unanimous && s_cur >= next_eval &&
        *c->eval_count < c->eval_cap) {
      const int64_t i = *c->eval_count;
      float* dst = c->eval_buf + (size_t)i * c->n;
      if (c->mean_parts) {
        for (int o = 0; o < Q; ++o) {
          const int64_t a = c->shard_bounds[o], b = c->shard_bounds[o + 1];
          if (b > a)
            CUDA_TRY(cudaMemcpyAsync(dst + a, c->mean_parts[o] + a, 4 * (size_t)(b - a),
                                     cudaMemcpyDeviceToDevice, stream));
        }
      } else {
        CUDA_TRY(cudaMemcpyAsync(dst, c->arenas[c->q], 4 * c->n, cudaMemcpyDeviceToDevice, stream));
      }
      CUDA_TRY(cudaStreamSynchronize(stream));
      int64_t* row = c->eval_rec + 5 * i;
      row[0] = s_cur, row[1] = r, row[2] = ld(c->flops_cell);
      row[3] = ld(c->classified_cell), row[4] = ld(c->clean_cell);
      c->eval_wall_ms[i] = 1e3 * (now_s() - c->t0);
      *c->eval_count = i + 1;
      while (next_eval <= s_cur) next_eval += c->eval_interval;
    }
    s_pre = s_cur;
    if (unanimous) break;
  }
  return LPP_OK;
}
