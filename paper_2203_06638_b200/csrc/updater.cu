// updater.cu — the native updater loop and device-side
// batch sampling for captured steps.
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

#include "common.cuh"

#include <algorithm>
#include <cmath>
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

namespace {

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
  if (K > 0 && (!c->tag_idx_pinned || !c->tag_idx_dev || !c->tag_out_dev || !c->tag_out_pinned ||
                !c->classified || !c->clean))
    return set_err(LPP_E_VALUE, "updater_run: tag sampling buffers missing");
  const int F = c->in_flight < 1 ? 1 : c->in_flight;
  const int depth = F + 2;
  cudaStream_t stream = (cudaStream_t)c->stream;

  Events done, t0, t1;
  int rc;
  if ((rc = done.make(F, cudaEventDisableTiming)) != LPP_OK) return rc;
  if (c->time_apply) {
    if ((rc = t0.make(F, cudaEventDefault)) != LPP_OK) return rc;
    if ((rc = t1.make(F, cudaEventDefault)) != LPP_OK) return rc;
  }
  std::vector<char> used(F, 0);
  std::vector<int64_t> claim_of(F, 0);
  std::vector<int> slot_of(F, 0);
  std::vector<double> bytes_of(F, 0.0);
  uint64_t tag_state = c->tag_seed;
  *st = lpp_updater_stats{};

  // a step's sampled tags live in slot t % depth; the gather for step t runs
  // before its snapshot values are read (paramstore.py:108-112)
  auto gather = [&](int slot) -> int {
    int64_t* hidx = c->tag_idx_pinned + (size_t)slot * K;
    draw_tags(&tag_state, (int64_t)c->n, K, hidx);
    int r;
    if ((r = lpp_copy_async(c->tag_idx_dev, hidx, 8 * (size_t)K, stream)) != LPP_OK) return r;
    if ((r = lpp_gather_tags(c->tags, c->tag_idx_dev, (size_t)K, c->tag_out_dev + (size_t)slot * K,
                             stream)) != LPP_OK)
      return r;
    return lpp_copy_async(c->tag_out_pinned + (size_t)slot * K, c->tag_out_dev + (size_t)slot * K,
                          4 * (size_t)K, stream);
  };
  // once a step's event completed: classify its tags, collect its apply time
  auto retire = [&](int k) -> int {
    if (K > 0) {
      const int32_t* tg = c->tag_out_pinned + (size_t)slot_of[k] * K;
      bool clean = true;
      for (int j = 0; j < K; ++j) clean &= ((int64_t)tg[j] >= claim_of[k]);
      __atomic_fetch_add(c->classified, 1, __ATOMIC_ACQ_REL);
      if (clean) __atomic_fetch_add(c->clean, 1, __ATOMIC_ACQ_REL);
    }
    if (c->time_apply) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, t0.ev[k], t1.ev[k]));
      st->apply_ms += ms;
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
    const int64_t k_claim = __atomic_load_n(c->last_avg_stamp, __ATOMIC_ACQUIRE);
    const int64_t u = __atomic_fetch_add(c->update_order, 1, __ATOMIC_ACQ_REL) + 1;
    const int64_t lo = c->block_lo[b], hi = c->block_hi[b], len = hi - lo;
    const float lr32 = (float)lr;
    if (!c->fused || t == 0) {
      if (K > 0 && (rc = gather(slot)) != LPP_OK) return rc;
      if ((rc = lpp_snapshot(c->x, c->replica, c->n, stream)) != LPP_OK) return rc;   // K3
    }
    if ((rc = lpp_graph_launch(c->graph_exec[b], stream)) != LPP_OK) return rc;       // fwd+bwd
    if (c->fused && K > 0 && (rc = gather(next_slot)) != LPP_OK) return rc;          // K5 (next)
    if (c->time_apply) CUDA_TRY(cudaEventRecord(t0.ev[k], stream));
    if (c->fused) {
      rc = lpp_apply_snapshot(c->x, c->g, c->m, c->replica, tagged ? c->tags : nullptr, c->n,
                              (size_t)lo, (size_t)hi, lr32, nullptr, c->mu, c->wd, (int32_t)u,
                              stream);                                                // K1+K3
      bytes_of[k] = c->apply_bytes_per_elem * (double)len + 4.0 * (double)(c->n - len) +
                    4.0 * (double)c->n;
    } else if (tagged) {
      rc = lpp_apply_sgd_tagged(c->x + lo, c->g + lo, c->m ? c->m + lo : nullptr, (size_t)len,
                                lr32, nullptr, c->mu, c->wd, c->apply_mode, c->tags + lo,
                                (int32_t)u, stream);                                  // K1/K2+K5
      bytes_of[k] = c->apply_bytes_per_elem * (double)len;
    } else {
      rc = lpp_apply_sgd(c->x + lo, c->g + lo, c->m ? c->m + lo : nullptr, (size_t)len, lr32,
                         nullptr, c->mu, c->wd, c->apply_mode, stream);               // K1/K2
      bytes_of[k] = c->apply_bytes_per_elem * (double)len;
    }
    if (rc != LPP_OK) return rc;
    if (c->time_apply) CUDA_TRY(cudaEventRecord(t1.ev[k], stream));
    CUDA_TRY(cudaEventRecord(done.ev[k], stream));
    used[k] = 1;
    claim_of[k] = k_claim;
    slot_of[k] = slot;
    st->flops += c->flops_of[b];
    ++t;
  }
  CUDA_TRY(cudaStreamSynchronize(stream));
  for (int64_t j = 1; j <= F; ++j) {
    int64_t tt = t - j;
    if (tt < 0) break;
    if ((rc = retire((int)(tt % F))) != LPP_OK) return rc;
  }
  st->steps = t;
  return LPP_OK;
}
