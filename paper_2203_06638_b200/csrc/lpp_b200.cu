// lpp_b200.cu — sm_100a kernels and the C ABI declared in include/lpp_b200.h.
//
// Kernels (ids from SURVEY.md §2):
//   K1/K2  k_apply / k_apply_bulk : Hogwild SGD apply into the shared arena,
//          replaces ParamStore.sub_assign -> _atomics.accum_cas_f64
//          (paramstore.py:121-136, _atomics.c:312-344, call site engine.py:355)
//   K3     k_snapshot             : replica refresh,
//          replaces ParamStore.snapshot -> snapshot_f64 (_atomics.c:186-215)
//   K1+K3  k_apply_snapshot       : the async default — one step's apply
//          fused with the next step's replica refresh (engine.py:343-355);
//          with a lpp_tag_plan also the updater's K5 bookkeeping in the
//          reference's order (this step's classification, the next step's
//          sampled tags before their values), per-block write stamps
//          published by a stream write after it (engine.py:343-362)
//   K4     k_average              : owner-computes in-place model averaging,
//          replaces _averager_body + _MeanAllReduce + add_assign(mean - snap)
//          (engine.py:199-229, 418-421); k_average_bulk: the TMA-staged
//          variant (bulk loads on an mbarrier, bulk reductions)
//   K5     tagged variants / k_gather_tags / k_gather_tags_floor /
//          k_gather_block_stamps / k_classify / lpp_publish_stamp : write
//          stamps, the sampled-tag gather, the clean classification
//          (_atomics.c:217-310, 346-392; engine.py:353-362)
//   K6     host atomics           : _atomics.{load,store,fetch_add}_i64
//          (_atomics.c:125-183)
//   NVLS   k_nvls_mean / k_nvls_apply : the averaging round in the switch
//          (multimem.ld_reduce / multimem.st)
// The native updater / averager loops and the device samplers live in
// updater.cu, the reference's numpy sampling stream in nprng.cu.
//
// All of them are HBM- (or NVLink-) bound streaming kernels: 128-bit
// vectorised, grid-stride with several independent 16-byte loads in flight
// per thread, grid sized in multiples of the SM count.  Element-atomic
// updates use the sm_90+ vector reduction red.global.add.v4.f32 (SASS
// REDG.E.ADD.F32x4) or the bulk-async reduction cp.reduce.async.bulk
// .add.f32 (SASS UBLKRED) issued from shared memory.

#include "common.cuh"

#include <atomic>
#include <climits>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>

// ---------------------------------------------------------------------------
// errors and the launch counter (shared with updater.cu through common.cuh)

static thread_local char g_err[512] = "";

int lpp_set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// every successful kernel launch of this library is counted (the bench's
// gpu_launches is the delta of this counter over the timed region)
static std::atomic<unsigned long long> g_launches{0};

void lpp_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" int lpp_abi_version(void) { return LPP_ABI_VERSION; }
extern "C" unsigned long long lpp_launch_count(void) { return g_launches.load(); }
extern "C" const char* lpp_last_error(void) { return g_err; }

// ---------------------------------------------------------------------------
// K6: host atomics on caller-owned int64 cells

extern "C" int64_t lpp_atomic_load_i64(const int64_t* p) {
  return __atomic_load_n(p, __ATOMIC_ACQUIRE);
}
extern "C" void lpp_atomic_store_i64(int64_t* p, int64_t v) {
  __atomic_store_n(p, v, __ATOMIC_RELEASE);
}
extern "C" int64_t lpp_atomic_fetch_add_i64(int64_t* p, int64_t delta) {
  return __atomic_fetch_add(p, delta, __ATOMIC_ACQ_REL);
}
extern "C" int lpp_atomic_cas_i64(int64_t* p, int64_t expected, int64_t desired) {
  return __atomic_compare_exchange_n(p, &expected, desired, 0, __ATOMIC_ACQ_REL,
                                     __ATOMIC_ACQUIRE)
             ? 1
             : 0;
}
extern "C" int64_t lpp_atomic_wait_ge_i64(const int64_t* p, int64_t target,
                                          const int64_t* abort_flag,
                                          int max_sleep_us) {
  int spins = 0;
  int sleep_us = 1;
  for (;;) {
    int64_t v = __atomic_load_n(p, __ATOMIC_ACQUIRE);
    if (v >= target) return v;
    if (abort_flag && __atomic_load_n(abort_flag, __ATOMIC_ACQUIRE) != 0)
      return INT64_MIN;
    if (++spins < 64) continue;
    std::this_thread::sleep_for(std::chrono::microseconds(sleep_us));
    if (sleep_us < max_sleep_us) sleep_us *= 2;
    if (sleep_us > max_sleep_us) sleep_us = max_sleep_us > 0 ? max_sleep_us : 1;
  }
}

// ---------------------------------------------------------------------------
// device helpers

static int sm_count_cached(int device) {
  static std::atomic<int> cache[64];
  if (device < 0 || device >= 64) return 148;
  int v = cache[device].load(std::memory_order_relaxed);
  if (v > 0) return v;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
    n = 148;
  cache[device].store(n, std::memory_order_relaxed);
  return n;
}

static int current_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return sm_count_cached(dev);
}

constexpr int kThreads = 256;
constexpr int kUnroll = 4;       // independent 16-byte loads in flight per thread
constexpr int kBlocksPerSM = 16;  // 2 waves of 8 x 256 threads: better tail than 1 wave

static unsigned grid_for(size_t nvec, int sms) {
  size_t want = (nvec + kThreads - 1) / kThreads;
  size_t cap = (size_t)sms * kBlocksPerSM;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (unsigned)want;
}

// number of leading scalar elements before p is 16-byte aligned
static inline size_t head_elems(const void* p, size_t n) {
  size_t mis = ((uintptr_t)p & 15u);
  size_t h = mis ? (16u - mis) / 4u : 0u;
  return h < n ? h : n;
}

__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
  asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// L2-coherent loads for data other agents may be writing concurrently
// release/acquire fences for the value -> tag message passing (K5).  The
// pattern only needs acq_rel (MEMBAR.ALL), not sequential consistency
// (MEMBAR.SC + L1 invalidate, which __threadfence() emits).
__device__ __forceinline__ void fence_ar_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_ar_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ float4 ld_cg4(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float ld_cg(const float* p) { return __ldcg(p); }

// K5 write tags: value first, tag second (accum_cas_tagged_f64,
// _atomics.c:346-392).  One gpu-scope fence per unrolled group orders the
// preceding value reductions before the tag stores; a reader loads tags
// first, fences, then values (snapshot_tagged_f64, _atomics.c:217-266), so a
// tag can only under-report how fresh the value it describes is.
__device__ __forceinline__ void st_tag4(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_tag(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_tag4_sys(int* p, int v) {
  asm volatile("st.relaxed.sys.global.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_tag_sys(int* p, int v) {
  asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int4 ld_tag4(const int* p) {
  int4 r;
  asm volatile("ld.relaxed.sys.global.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ int ld_tag(const int* p) {
  int r;
  asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

// The per-element SGD arithmetic, written with explicit round-to-nearest
// intrinsics so that ptxas cannot contract it into FMAs; oracle/apply_ref.c
// restates exactly this sequence.
template <bool WD, bool MOM>
__device__ __forceinline__ float sgd_delta(float g, float x, float& m, float lr, float mu,
                                           float wd) {
  float gp = g;
  if (WD) gp = __fadd_rn(gp, __fmul_rn(wd, x));
  if (MOM) {
    float mm = __fadd_rn(__fmul_rn(mu, m), gp);
    m = mm;
    gp = mm;
  }
  return -__fmul_rn(lr, gp);
}

// ---------------------------------------------------------------------------
// K1/K2: apply (modes PLAIN and RED)

template <int MODE, bool WD, bool MOM>
__global__ void __launch_bounds__(kThreads)
    k_apply(float* x, const float* __restrict__ g, float* m, size_t n, size_t head,
            size_t nvec, float lr, const float* __restrict__ lr_dev, float mu, float wd,
            int* tags, int stamp) {
  if (lr_dev) lr = *lr_dev;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  float* xb = x + head;
  const float* gb = g + head;
  float* mb = MOM ? m + head : nullptr;

  for (size_t i0 = tid; i0 < nvec; i0 += stride * kUnroll) {
    float4 gr[kUnroll], xr[kUnroll], mr[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
        gr[u] = __ldg(reinterpret_cast<const float4*>(gb) + i);
        if (WD || MODE == LPP_MODE_PLAIN) xr[u] = ld_cg4(xb + 4 * i);
        if (MOM) mr[u] = reinterpret_cast<const float4*>(mb)[i];
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
        float4 d;
        d.x = sgd_delta<WD, MOM>(gr[u].x, xr[u].x, mr[u].x, lr, mu, wd);
        d.y = sgd_delta<WD, MOM>(gr[u].y, xr[u].y, mr[u].y, lr, mu, wd);
        d.z = sgd_delta<WD, MOM>(gr[u].z, xr[u].z, mr[u].z, lr, mu, wd);
        d.w = sgd_delta<WD, MOM>(gr[u].w, xr[u].w, mr[u].w, lr, mu, wd);
        if (MOM) reinterpret_cast<float4*>(mb)[i] = mr[u];
        if (MODE == LPP_MODE_PLAIN) {
          float4 o;
          o.x = __fadd_rn(xr[u].x, d.x);
          o.y = __fadd_rn(xr[u].y, d.y);
          o.z = __fadd_rn(xr[u].z, d.z);
          o.w = __fadd_rn(xr[u].w, d.w);
          __stcg(reinterpret_cast<float4*>(xb) + i, o);
        } else {
          red_add_v4(xb + 4 * i, d);
        }
      }
    }
    if (tags) {
      fence_ar_gpu();
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        size_t i = i0 + (size_t)u * stride;
        if (i < nvec) st_tag4(tags + head + 4 * i, stamp);
      }
    }
  }
  // scalar head [0, head) and tail [head + 4*nvec, n): first block only
  if (blockIdx.x == 0) {
    size_t tail0 = head + 4 * nvec;
    size_t nscalar = head + (n - tail0);
    for (size_t k = threadIdx.x; k < nscalar; k += blockDim.x) {
      size_t e = k < head ? k : tail0 + (k - head);
      float xv = (WD || MODE == LPP_MODE_PLAIN) ? ld_cg(x + e) : 0.f;
      float mv = MOM ? m[e] : 0.f;
      float d = sgd_delta<WD, MOM>(g[e], xv, mv, lr, mu, wd);
      if (MOM) m[e] = mv;
      if (MODE == LPP_MODE_PLAIN)
        __stcg(x + e, __fadd_rn(xv, d));
      else
        red_add_f32(x + e, d);
      if (tags) {
        fence_ar_gpu();
        st_tag(tags + e, stamp);
      }
    }
  }
}

// K1/K2 mode BULK: the CTA computes a 16 KB tile of deltas into shared memory
// and one thread hands it to the bulk-copy engine as an element-wise atomic
// add (cp.reduce.async.bulk .add.f32), STAGES tiles in flight per CTA.
constexpr int kBulkTileV = kThreads * 4;  // float4 per tile (16 KB)
constexpr int kBulkStages = 3;

template <bool WD, bool MOM>
__global__ void __launch_bounds__(kThreads)
    k_apply_bulk(float* x, const float* __restrict__ g, float* m, size_t n, size_t head,
                 size_t nvec, float lr, const float* __restrict__ lr_dev, float mu,
                 float wd) {
  extern __shared__ __align__(128) float4 s_tile[];  // kBulkStages * kBulkTileV
  if (lr_dev) lr = *lr_dev;
  float* xb = x + head;
  const float4* gb = reinterpret_cast<const float4*>(g + head);
  float4* mb = MOM ? reinterpret_cast<float4*>(m + head) : nullptr;
  const size_t ntiles = (nvec + kBulkTileV - 1) / kBulkTileV;
  int stage = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x == 0)
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBulkStages - 1) : "memory");
    __syncthreads();
    const size_t base = t * kBulkTileV;
    const int cnt = (int)((nvec - base) < (size_t)kBulkTileV ? (nvec - base) : kBulkTileV);
    float4* buf = s_tile + stage * kBulkTileV;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int j = threadIdx.x + u * kThreads;
      if (j < cnt) {
        float4 gv = __ldg(gb + base + j);
        float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 mv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (WD) xv = ld_cg4(xb + 4 * (base + j));
        if (MOM) mv = mb[base + j];
        float4 d;
        d.x = sgd_delta<WD, MOM>(gv.x, xv.x, mv.x, lr, mu, wd);
        d.y = sgd_delta<WD, MOM>(gv.y, xv.y, mv.y, lr, mu, wd);
        d.z = sgd_delta<WD, MOM>(gv.z, xv.z, mv.z, lr, mu, wd);
        d.w = sgd_delta<WD, MOM>(gv.w, xv.w, mv.w, lr, mu, wd);
        if (MOM) mb[base + j] = mv;
        buf[j] = d;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t saddr = (uint32_t)__cvta_generic_to_shared(buf);
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
              xb + 4 * base),
          "r"(saddr), "r"(cnt * 16)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    stage = (stage + 1) % kBulkStages;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (blockIdx.x == 0) {
    size_t tail0 = head + 4 * nvec;
    size_t nscalar = head + (n - tail0);
    for (size_t k = threadIdx.x; k < nscalar; k += blockDim.x) {
      size_t e = k < head ? k : tail0 + (k - head);
      float xv = WD ? ld_cg(x + e) : 0.f;
      float mv = MOM ? m[e] : 0.f;
      float d = sgd_delta<WD, MOM>(g[e], xv, mv, lr, mu, wd);
      if (MOM) m[e] = mv;
      red_add_f32(x + e, d);
    }
  }
}

template <int MODE, bool WD, bool MOM>
static void launch_apply_t(float* x, const float* g, float* m, size_t n, size_t head,
                           size_t nvec, float lr, const float* lr_dev, float mu, float wd,
                           int* tags, int stamp, cudaStream_t st) {
  int sms = current_sms();
  if (MODE == LPP_MODE_BULK) {
    size_t ntiles = (nvec + kBulkTileV - 1) / kBulkTileV;
    size_t cap = (size_t)sms * 4;  // 3 x 16 KB smem per CTA -> 4 CTAs/SM
    unsigned grid = (unsigned)(ntiles < cap ? (ntiles ? ntiles : 1) : cap);
    size_t smem = (size_t)kBulkStages * kBulkTileV * sizeof(float4);
    k_apply_bulk<WD, MOM><<<grid, kThreads, smem, st>>>(x, g, m, n, head, nvec, lr, lr_dev,
                                                       mu, wd);
  } else {
    k_apply<MODE, WD, MOM><<<grid_for(nvec, sms), kThreads, 0, st>>>(x, g, m, n, head, nvec,
                                                                    lr, lr_dev, mu, wd, tags,
                                                                    stamp);
  }
}

template <int MODE>
static void launch_apply_mode(float* x, const float* g, float* m, size_t n, size_t head,
                              size_t nvec, float lr, const float* lr_dev, float mu, float wd,
                              int* tags, int stamp, cudaStream_t st) {
  bool WD = wd != 0.f, MOM = mu != 0.f;
  if (WD && MOM)
    launch_apply_t<MODE, true, true>(x, g, m, n, head, nvec, lr, lr_dev, mu, wd, tags, stamp, st);
  else if (WD)
    launch_apply_t<MODE, true, false>(x, g, m, n, head, nvec, lr, lr_dev, mu, wd, tags, stamp, st);
  else if (MOM)
    launch_apply_t<MODE, false, true>(x, g, m, n, head, nvec, lr, lr_dev, mu, wd, tags, stamp, st);
  else
    launch_apply_t<MODE, false, false>(x, g, m, n, head, nvec, lr, lr_dev, mu, wd, tags, stamp,
                                       st);
}

static int apply_impl(float* x, const float* g, float* m, size_t n, float lr, const float* lr_dev,
                      float mu, float wd, int mode, int32_t* tags, int32_t stamp, void* stream);

extern "C" int lpp_apply_sgd(float* x, const float* g, float* m, size_t n, float lr,
                             const float* lr_dev, float mu, float wd, int mode,
                             void* stream) {
  return apply_impl(x, g, m, n, lr, lr_dev, mu, wd, mode, nullptr, 0, stream);
}

extern "C" int lpp_apply_sgd_tagged(float* x, const float* g, float* m, size_t n, float lr,
                                    const float* lr_dev, float mu, float wd, int mode,
                                    int32_t* tags, int32_t stamp, void* stream) {
  if (!tags) return set_err(LPP_E_VALUE, "apply_sgd_tagged: null tags");
  if (mode == LPP_MODE_BULK) mode = LPP_MODE_RED;  // tags need the value update done in-thread
  if ((((uintptr_t)x) ^ ((uintptr_t)tags)) & 15u)
    return set_err(LPP_E_VALUE, "apply_sgd_tagged: tags must share x's alignment modulo 16");
  return apply_impl(x, g, m, n, lr, lr_dev, mu, wd, mode, tags, stamp, stream);
}

static int apply_impl(float* x, const float* g, float* m, size_t n, float lr, const float* lr_dev,
                      float mu, float wd, int mode, int32_t* tags, int32_t stamp, void* stream) {
  if (n == 0) return LPP_OK;
  if (!x || !g) return set_err(LPP_E_VALUE, "apply_sgd: null x or g");
  if (mu != 0.f && !m) return set_err(LPP_E_VALUE, "apply_sgd: momentum needs a buffer");
  if (mode < LPP_MODE_PLAIN || mode > LPP_MODE_BULK)
    return set_err(LPP_E_VALUE, "apply_sgd: unknown mode %d", mode);
  if (((uintptr_t)x & 3u) || ((uintptr_t)g & 3u) || (m && ((uintptr_t)m & 3u)))
    return set_err(LPP_E_VALUE, "apply_sgd: buffers must be 4-byte aligned");
  if ((((uintptr_t)x ^ (uintptr_t)g) & 15u) || (m && (((uintptr_t)x ^ (uintptr_t)m) & 15u)))
    return set_err(LPP_E_VALUE,
                   "apply_sgd: x, g, m must share their alignment modulo 16 bytes");
  size_t head = head_elems(x, n);
  size_t nvec = (n - head) / 4;
  cudaStream_t st = (cudaStream_t)stream;
  switch (mode) {
    case LPP_MODE_PLAIN:
      launch_apply_mode<LPP_MODE_PLAIN>(x, g, m, n, head, nvec, lr, lr_dev, mu, wd, tags, stamp,
                                        st);
      break;
    case LPP_MODE_RED:
      launch_apply_mode<LPP_MODE_RED>(x, g, m, n, head, nvec, lr, lr_dev, mu, wd, tags, stamp,
                                      st);
      break;
    default:
      launch_apply_mode<LPP_MODE_BULK>(x, g, m, n, head, nvec, lr, lr_dev, mu, wd, tags, stamp,
                                       st);
      break;
  }
  LAUNCH_CHECK("apply_sgd");
  return LPP_OK;
}

// ---------------------------------------------------------------------------
// K1+K3 fused: apply this step's block gradient AND refresh the stream's
// replica for its next step in one pass over the arena.  Inside [lo, hi)
// the element update is the K1 vector reduction (red.add.v4.f32) followed
// by a re-read of the same 16 bytes: the replica receives the value the
// element held after this update landed (an untorn value that was really in
// the arena, exactly what K3 would copy after the apply); the re-read hits
// the L2 line the reduction just wrote.  Outside the block the replica is a
// plain copy.  It replaces the next step's K3 launch (the step's snapshot is
// taken when the previous step's apply lands, which on the updater's stream
// is when K3 would have run anyway) and saves the block's second DRAM read.
// (A returning atom.add.v4.f32 — old + delta — measured 4-8 % slower at
// d18/d50: tools/bench_fused.py.)
//
// K5 inside the same launch (``lpp_tag_plan``), in the reference's order
// (engine.py:343-362: snapshot tags -> gradient -> k_claim -> apply):
//   * write stamps per BLOCK, not per element: every update writes one
//     whole block range, so an element's tag is the newest stamp of the (at
//     most two) blocks covering it — block 0 (full) and its partial block.
//     The stamp is written by lpp_publish_stamp, a stream memory operation
//     after the apply, so it is visible only once every element reduction
//     of its update is performed (value before tag, _atomics.c:346-392) — at no
//     per-element cost and with no CTA barrier or fence in this kernel
//     (in situ, among convolution CTAs, a completion counter + fence per
//     CTA measured 4x the apply's latency: the CTAs run in many small waves);
//   * classification of THIS step: block 0 reads k_claim from the worker's
//     device round-stamp cell when the kernel starts, i.e. after the step's
//     gradient, and compares the step's sampled tags with it;
//   * the NEXT step's sampled tags, element by element in snapshot order
//     (paramstore.py:108-112: tag before value): the thread that refreshes
//     the replica vector holding a sampled element acquire-reads the stamps
//     and the round floor BEFORE it re-reads the value, after its own
//     reduction of that vector; the effective tag is
//     max(floor, stamp[0], stamp[b(e)], this update's stamp if e is in its
//     block).  The floor is the worker's last completed round stamp (rounds
//     stamp every element, engine.py:421 add_assign(..., stamp=u_avg)).

struct TagPlanDev {
  int64_t idx[32];          // the next step's k sampled indices, by value (constant bank)
  int8_t blk[32];           // ... and the partial block b(e) holding each (from host bounds)
  uint32_t owner[32];       // owning thread of each, ascending (computed at launch)
  int8_t owner_j[32];       // ... and which sampled element it is
  int has_next;
  int* next_dev;            // -> the next step's effective tags (device ring slot)
  int* next_host;           // -> and a host-mapped copy for the records (may be null)
  const int* cur_dev;       // this step's effective tags (read at its snapshot)
  int64_t* cur_claim;       // -> this step's (k_claim, clean) (host-mapped; may be null)
  const int64_t* avg_cell;  // the worker's last completed round stamp (device cell)
  int* block_stamps;        // [nb + 1] newest stamp per block (device)
  int nb;
  int bid;                  // this update's block id
  int k;                    // <= 32
};

__device__ __forceinline__ int64_t ld_sys_i64(const int64_t* p) {
  int64_t r;
  asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_acq_i32(const int* p) {
  int r;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

// effective tag of sampled element j (element e), read before its value:
// three independent loads (one round trip), b(e) precomputed at launch
__device__ __forceinline__ int plan_tag_of(const TagPlanDev& plan, int j, int64_t e, size_t lo,
                                           size_t hi, int stamp) {
  int t = ld_acq_i32(plan.block_stamps);
  int tb = ld_acq_i32(plan.block_stamps + plan.blk[j]);
  const int fl = (int)ld_sys_i64(plan.avg_cell);
  t = t > tb ? t : tb;
  t = t > fl ? t : fl;
  if ((size_t)e >= lo && (size_t)e < hi && stamp > t) t = stamp;
  return t;
}

template <bool WD, bool MOM>
__device__ __forceinline__ void fused_elem(float* x, const float* g, float* m, float* rep, size_t e,
                                           size_t lo, size_t hi, float lr, float mu, float wd) {
  if (e >= lo && e < hi) {
    float xv = WD ? ld_cg(x + e) : 0.f;
    float mv = MOM ? m[e] : 0.f;
    float d = sgd_delta<WD, MOM>(g[e], xv, mv, lr, mu, wd);
    red_add_f32(x + e, d);
    float nv = ld_cg(x + e);
    if (MOM) m[e] = mv;
    rep[e] = nv;
  } else {
    rep[e] = ld_cg(x + e);
  }
}

template <bool WD, bool MOM, bool TAGS, bool PLAN, int UNR = 1>
__global__ void __launch_bounds__(kThreads)
    k_apply_snapshot(float* x, const float* __restrict__ g, float* m, float* __restrict__ rep,
                     int* tags, size_t n, size_t lo, size_t hi, float lr,
                     const float* __restrict__ lr_dev, float mu, float wd, int stamp,
                     TagPlanDev plan) {
  // k_claim of this step (engine.py:353: read after the gradient), issued
  // first and consumed at the end
  const bool classifier = PLAN && blockIdx.x == 0 && threadIdx.x == 0 && plan.cur_claim != nullptr;
  int64_t k_claim = 0;
  if (classifier) k_claim = plan.avg_cell ? ld_sys_i64(plan.avg_cell) : 0;
  if (lr_dev) lr = *lr_dev;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nvec = n / 4;
  // which of the next step's sampled elements this thread refreshes: vector
  // v belongs to thread v mod stride, a tail element e >= 4 nvec to block 0,
  // thread (e - 4 nvec) mod blockDim.  The launcher computes the owners and
  // passes them in the launch parameters (constant bank): a load from
  // memory here, once per CTA, doubled the in-situ latency of the launch,
  // whose CTAs run in many small waves among the convolutions' CTAs, and
  // per-thread modulo arithmetic cost ~8 us of it
  unsigned own = 0;
  if (PLAN && plan.has_next) {
    // fully unrolled: each compare takes its operand straight from the
    // constant bank (no load, no divergence)
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < plan.k && plan.owner[j] == (uint32_t)tid) own |= 1u << plan.owner_j[j];
  }
  // vectors fully inside [lo, hi) take the apply path, vectors fully outside
  // the copy path; the (at most two) straddling vectors go per element
  const size_t vlo = (lo + 3) / 4, vhi = hi / 4;
  // UNR vectors per thread per round (v = i0 + u * stride keeps the owner
  // rule): every load of the round is issued before the first reduction,
  // then the reductions, then the re-reads — more bytes in flight per
  // resident thread, which is what matters when the launch only gets the
  // SM slots the convolutions leave (in situ)
  for (size_t i0 = tid; i0 < nvec; i0 += stride * UNR) {
    float4 gr[UNR], xr[UNR], mr[UNR];
    int kind[UNR];  // 0 none, 1 inside the block, 2 outside, 3 straddling
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const size_t i = i0 + (size_t)u * stride;
      kind[u] = 0;
      gr[u] = xr[u] = mr[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i >= nvec) continue;
      if (PLAN && own) {  // sampled elements of this vector: tags before values
        for (unsigned bits = own; bits; bits &= bits - 1) {
          const int j = __ffs(bits) - 1;
          const int64_t e = plan.idx[j];
          if ((size_t)e / 4 == i) {
            const int t = plan_tag_of(plan, j, e, lo, hi, stamp);
            plan.next_dev[j] = t;
            if (plan.next_host) plan.next_host[j] = t;
          }
        }
      }
      if (i >= vlo && i < vhi) {
        kind[u] = 1;
        gr[u] = __ldg(reinterpret_cast<const float4*>(g) + i);
        if (WD) xr[u] = ld_cg4(x + 4 * i);
        if (MOM) mr[u] = reinterpret_cast<const float4*>(m)[i];
      } else if (4 * i + 4 <= lo || 4 * i >= hi) {
        kind[u] = 2;
        xr[u] = ld_cg4(x + 4 * i);
      } else {
        kind[u] = 3;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (kind[u] != 1) continue;
      const size_t i = i0 + (size_t)u * stride;
      float4 dr;
      dr.x = sgd_delta<WD, MOM>(gr[u].x, xr[u].x, mr[u].x, lr, mu, wd);
      dr.y = sgd_delta<WD, MOM>(gr[u].y, xr[u].y, mr[u].y, lr, mu, wd);
      dr.z = sgd_delta<WD, MOM>(gr[u].z, xr[u].z, mr[u].z, lr, mu, wd);
      dr.w = sgd_delta<WD, MOM>(gr[u].w, xr[u].w, mr[u].w, lr, mu, wd);
      // vector reduction, then (below) the re-read: the replica gets the
      // arena value after this step's add (plus any concurrent adds that
      // landed first), i.e. what a K3 snapshot right after the apply copies
      red_add_v4(x + 4 * i, dr);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const size_t i = i0 + (size_t)u * stride;
      if (kind[u] == 1) {
        const float4 nv = ld_cg4(x + 4 * i);
        if (MOM) reinterpret_cast<float4*>(m)[i] = mr[u];
        reinterpret_cast<float4*>(rep)[i] = nv;
      } else if (kind[u] == 2) {
        reinterpret_cast<float4*>(rep)[i] = xr[u];
      } else if (kind[u] == 3) {
        for (size_t e = 4 * i; e < 4 * i + 4; ++e)
          fused_elem<WD, MOM>(x, g, m, rep, e, lo, hi, lr, mu, wd);
      }
    }
  }
  if (blockIdx.x == 0)
    for (size_t e = 4 * nvec + threadIdx.x; e < n; e += blockDim.x) {
      if (PLAN && own)
        for (unsigned bits = own; bits; bits &= bits - 1) {
          const int j = __ffs(bits) - 1;
          if ((size_t)plan.idx[j] == e) {
            const int t = plan_tag_of(plan, j, (int64_t)e, lo, hi, stamp);
            plan.next_dev[j] = t;
            if (plan.next_host) plan.next_host[j] = t;
          }
        }
      fused_elem<WD, MOM>(x, g, m, rep, e, lo, hi, lr, mu, wd);
    }
  if (TAGS) {
    // per-element tags (ParamStore-level API): one fence per thread, then
    // the tags of exactly the elements it updated
    fence_ar_gpu();
    for (size_t i = tid; i < nvec; i += stride) {
      if (i >= vlo && i < vhi) {
        st_tag4(tags + 4 * i, stamp);
      } else if (!(4 * i + 4 <= lo || 4 * i >= hi)) {
        for (size_t e = 4 * i; e < 4 * i + 4; ++e)
          if (e >= lo && e < hi) st_tag(tags + e, stamp);
      }
    }
    if (blockIdx.x == 0)
      for (size_t e = 4 * nvec + threadIdx.x; e < n; e += blockDim.x)
        if (e >= lo && e < hi) st_tag(tags + e, stamp);
  }
  if (PLAN) {
    if (classifier) {
      int clean = 1;
      for (int j = 0; j < plan.k; ++j) clean &= ((int64_t)plan.cur_dev[j] >= k_claim);
      plan.cur_claim[0] = k_claim;
      plan.cur_claim[1] = clean;
    }
  }
}

static int apply_snapshot_launch(float* x, const float* g, float* m, float* replica, int32_t* tags,
                                 size_t n, size_t lo, size_t hi, float lr, const float* lr_dev,
                                 float mu, float wd, int32_t stamp, const lpp_tag_plan* plan,
                                 void* stream) {
  if (n == 0) return LPP_OK;
  if (!x || !g || !replica) return set_err(LPP_E_VALUE, "apply_snapshot: null buffer");
  if (lo > hi || hi > n) return set_err(LPP_E_INDEX, "apply_snapshot: block outside [0, n)");
  if (mu != 0.f && !m) return set_err(LPP_E_VALUE, "apply_snapshot: momentum needs a buffer");
  uintptr_t a = (uintptr_t)x | (uintptr_t)g | (uintptr_t)replica | (m ? (uintptr_t)m : 0) |
                (tags ? (uintptr_t)tags : 0);
  if (a & 15u)
    return set_err(LPP_E_VALUE, "apply_snapshot: arena bases must be 16-byte aligned");
  TagPlanDev pd{};
  if (plan) {
    if (plan->k < 0 || plan->k > 32)
      return set_err(LPP_E_VALUE, "apply_snapshot: tag count %d outside [0, 32]", plan->k);
    if (!plan->block_stamps || !plan->block_bounds || !plan->avg_cell)
      return set_err(LPP_E_VALUE, "apply_snapshot: a tag plan needs stamps, bounds, round cell");
    if (plan->num_blocks > 127)
      return set_err(LPP_E_VALUE, "apply_snapshot: at most 127 blocks with a tag plan");
    if (plan->num_blocks < 1 || plan->block_id < 0 || plan->block_id > plan->num_blocks)
      return set_err(LPP_E_VALUE, "apply_snapshot: block %d outside [0, %d]", plan->block_id,
                     plan->num_blocks);
    if (plan->k > 0 && plan->next_idx && !plan->next_dev)
      return set_err(LPP_E_VALUE, "apply_snapshot: next-step tags need an output");
    if (plan->cur_claim && plan->k > 0 && !plan->cur_dev)
      return set_err(LPP_E_VALUE, "apply_snapshot: classification needs this step's tags");
    pd.has_next = plan->next_idx != nullptr && plan->k > 0;
    for (int j = 0; pd.has_next && j < plan->k; ++j) {  // host memory, copied into the launch
      if (plan->next_idx[j] < 0 || (size_t)plan->next_idx[j] >= n)
        return set_err(LPP_E_INDEX, "apply_snapshot: sampled index %lld outside [0, %zu)",
                       (long long)plan->next_idx[j], n);
      pd.idx[j] = plan->next_idx[j];
      int b = 1;  // the partial block holding the element (host bounds)
      while (b < plan->num_blocks && plan->next_idx[j] >= plan->block_bounds[b]) ++b;
      pd.blk[j] = (int8_t)b;
    }
    pd.next_dev = plan->next_dev;
    pd.next_host = plan->next_host;
    pd.cur_dev = plan->cur_dev;
    pd.cur_claim = plan->cur_claim;
    pd.avg_cell = plan->avg_cell;
    pd.block_stamps = plan->block_stamps;
    pd.nb = plan->num_blocks;
    pd.bid = plan->block_id;
    pd.k = plan->k;
  }
  size_t nvec = n / 4;
  // vectors per thread per round of the plan kernel: 2 (LPP_FUSED_UNR
  // overrides: 1, 2, 4).  In situ (bf16 ResNet-18 / ResNet-50 steps,
  // tools/exp_fused_insitu.py) 2 reaches 0.72 / 0.79-0.81 of HBM vs 0.70 /
  // 0.75-0.76 with 1 and 0.63 / 0.73-0.75 with 4 (84 registers); standalone
  // and at d20 in situ the three are within noise
  static const int unr = [] {
    const char* e = std::getenv("LPP_FUSED_UNR");
    const int v = e ? std::atoi(e) : 2;
    return (v == 1 || v == 2 || v == 4) ? v : 2;
  }();
  // grid: one round of `unr` vectors per thread (the plain kernels: one vector);
  // at d20 the plan launch then needs 134 CTAs instead of 267 — fewer SM slots
  // to wait for among the convolutions' CTAs
  const size_t per_thread = plan ? (size_t)unr : 1;
  unsigned grid = grid_for(nvec ? (nvec + per_thread - 1) / per_thread : 1, current_sms());
  // experiment hook: LPP_FUSED_CTAS caps the grid (tools/exp_insitu_grid.py)
  static const long cap_env = [] {
    const char* e = std::getenv("LPP_FUSED_CTAS");
    return e ? std::atol(e) : 0L;
  }();
  if (cap_env > 0 && grid > (unsigned)cap_env) grid = (unsigned)cap_env;
  if (plan && pd.has_next) {  // owning thread of each sampled element, sorted
    const size_t stride = (size_t)grid * kThreads;
    for (int j = 0; j < pd.k; ++j) {
      const size_t e = (size_t)pd.idx[j], v = e / 4;
      pd.owner[j] = (uint32_t)(v < nvec ? v % stride : (e - 4 * nvec) % kThreads);
      pd.owner_j[j] = (int8_t)j;
    }
    for (int j = 1; j < pd.k; ++j)  // insertion sort of <= 32 (owner, j) pairs
      for (int i = j; i > 0 && pd.owner[i - 1] > pd.owner[i]; --i) {
        uint32_t t = pd.owner[i]; pd.owner[i] = pd.owner[i - 1]; pd.owner[i - 1] = t;
        int8_t u = pd.owner_j[i]; pd.owner_j[i] = pd.owner_j[i - 1]; pd.owner_j[i - 1] = u;
      }
  }
  cudaStream_t st = (cudaStream_t)stream;
  bool WD = wd != 0.f, MOM = mu != 0.f;
  // one vector per thread per grid stride: unrolling (2, 4 vectors with all
  // loads hoisted) measured no faster at d20/d50 and 4-10 % slower at d18
  // (with both the returning-atomic and the reduction + re-read bodies); 64-
  // or 128-thread CTAs (easier to fit between other streams' CTAs) changed
  // neither the in-situ d20 time nor images/s
#define FUSED_LAUNCH(W, M)                                                                      \
  if (plan && unr == 4)                                                                         \
    k_apply_snapshot<W, M, false, true, 4><<<grid, kThreads, 0, st>>>(                         \
        x, g, m, replica, tags, n, lo, hi, lr, lr_dev, mu, wd, stamp, pd);                     \
  else if (plan && unr == 2)                                                                    \
    k_apply_snapshot<W, M, false, true, 2><<<grid, kThreads, 0, st>>>(                         \
        x, g, m, replica, tags, n, lo, hi, lr, lr_dev, mu, wd, stamp, pd);                     \
  else if (plan)                                                                                \
    k_apply_snapshot<W, M, false, true><<<grid, kThreads, 0, st>>>(                            \
        x, g, m, replica, tags, n, lo, hi, lr, lr_dev, mu, wd, stamp, pd);                     \
  else if (tags)                                                                                \
    k_apply_snapshot<W, M, true, false><<<grid, kThreads, 0, st>>>(                            \
        x, g, m, replica, tags, n, lo, hi, lr, lr_dev, mu, wd, stamp, pd);                     \
  else                                                                                          \
    k_apply_snapshot<W, M, false, false><<<grid, kThreads, 0, st>>>(                           \
        x, g, m, replica, tags, n, lo, hi, lr, lr_dev, mu, wd, stamp, pd);
  if (WD && MOM) {
    FUSED_LAUNCH(true, true)
  } else if (WD) {
    FUSED_LAUNCH(true, false)
  } else if (MOM) {
    FUSED_LAUNCH(false, true)
  } else {
    FUSED_LAUNCH(false, false)
  }
#undef FUSED_LAUNCH
  LAUNCH_CHECK("apply_snapshot");
  return LPP_OK;
}

extern "C" int lpp_apply_snapshot(float* x, const float* g, float* m, float* replica,
                                  int32_t* tags, size_t n, size_t lo, size_t hi, float lr,
                                  const float* lr_dev, float mu, float wd, int32_t stamp,
                                  void* stream) {
  return apply_snapshot_launch(x, g, m, replica, tags, n, lo, hi, lr, lr_dev, mu, wd, stamp,
                               nullptr, stream);
}

extern "C" int lpp_apply_snapshot_plan(float* x, const float* g, float* m, float* replica,
                                       int32_t* tags, size_t n, size_t lo, size_t hi, float lr,
                                       const float* lr_dev, float mu, float wd, int32_t stamp,
                                       const lpp_tag_plan* plan, void* stream) {
  if (!plan) return set_err(LPP_E_VALUE, "apply_snapshot_plan: null plan");
  return apply_snapshot_launch(x, g, m, replica, tags, n, lo, hi, lr, lr_dev, mu, wd, stamp, plan,
                               stream);
}

// K5 gather with the round floor, for a step whose snapshot is a separate
// K3 (the first step of a fused run, the unfused paths): out = max(tag, floor)
__global__ void k_gather_tags_floor(const int* tags, const int64_t* idx, int k,
                                    const int64_t* floor_cell, int* out_dev, int* out_host) {
  const int floor_ = floor_cell ? (int)ld_sys_i64(floor_cell) : 0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    int t = ld_tag(tags + ld_sys_i64(idx + j));
    t = t > floor_ ? t : floor_;
    if (out_dev) out_dev[j] = t;
    if (out_host) out_host[j] = t;
  }
}

extern "C" int lpp_gather_tags_floor(const int32_t* tags, const int64_t* idx, size_t k,
                                     const int64_t* floor_cell, int32_t* out_dev,
                                     int32_t* out_host, void* stream) {
  if (k == 0) return LPP_OK;
  if (!tags || !idx || (!out_dev && !out_host))
    return set_err(LPP_E_VALUE, "gather_tags_floor: null buffer");
  if (k > (1u << 20)) return set_err(LPP_E_VALUE, "gather_tags_floor: k too large");
  k_gather_tags_floor<<<1, kThreads, 0, (cudaStream_t)stream>>>(tags, idx, (int)k, floor_cell,
                                                                 out_dev, out_host);
  LAUNCH_CHECK("gather_tags_floor");
  return LPP_OK;
}

// the first step of a fused run: its sampled tags from the block stamps
// (tag before value: the K3 snapshot that follows on the stream reads values)
__global__ void k_gather_block_stamps(const int* stamps, const int64_t* bounds, int nb,
                                      const int64_t* idx, int k, const int64_t* floor_cell,
                                      int* out_dev, int* out_host) {
  const int fl = floor_cell ? (int)ld_sys_i64(floor_cell) : 0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const int64_t e = idx[j];
    int b = 1;
    while (b < nb && e >= bounds[b]) ++b;
    int t = ld_acq_i32(stamps), tb = ld_acq_i32(stamps + b);
    t = t > tb ? t : tb;
    t = t > fl ? t : fl;
    if (out_dev) out_dev[j] = t;
    if (out_host) out_host[j] = t;
  }
}

extern "C" int lpp_gather_block_stamps(const int32_t* stamps, const int64_t* bounds, int nb,
                                       const int64_t* idx, size_t k, const int64_t* floor_cell,
                                       int32_t* out_dev, int32_t* out_host, void* stream) {
  if (k == 0) return LPP_OK;
  if (!stamps || !bounds || !idx || nb < 1 || (!out_dev && !out_host))
    return set_err(LPP_E_VALUE, "gather_block_stamps: null buffer or no blocks");
  if (k > (1u << 20)) return set_err(LPP_E_VALUE, "gather_block_stamps: k too large");
  k_gather_block_stamps<<<1, kThreads, 0, (cudaStream_t)stream>>>(stamps, bounds, nb, idx, (int)k,
                                                                   floor_cell, out_dev, out_host);
  LAUNCH_CHECK("gather_block_stamps");
  return LPP_OK;
}

// K5 classification at apply time for the unfused paths (engine.py:353-362):
// out[0] = k_claim read now from the round-stamp cell, out[1] = all tags >= it
__global__ void k_classify(const int* tags, int k, const int64_t* claim_cell, int64_t* out) {
  if (threadIdx.x != 0) return;
  const int64_t kc = claim_cell ? ld_sys_i64(claim_cell) : 0;
  int clean = 1;
  for (int j = 0; j < k; ++j) clean &= ((int64_t)tags[j] >= kc);
  out[0] = kc;
  out[1] = clean;
}

extern "C" int lpp_classify(const int32_t* tags, size_t k, const int64_t* claim_cell,
                            int64_t* out, void* stream) {
  if (!out || (k > 0 && !tags)) return set_err(LPP_E_VALUE, "classify: null buffer");
  if (k > (1u << 20)) return set_err(LPP_E_VALUE, "classify: k too large");
  k_classify<<<1, 32, 0, (cudaStream_t)stream>>>(tags, (int)k, claim_cell, out);
  LAUNCH_CHECK("classify");
  return LPP_OK;
}

// a device int64 cell set in stream order (the worker's round-stamp cell,
// written by its averager once a round is applied to its arena)
__global__ void k_set_i64(int64_t* p, int64_t v) {
  asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

extern "C" int lpp_set_i64(int64_t* dev, int64_t v, void* stream) {
  if (!dev) return set_err(LPP_E_VALUE, "set_i64: null cell");
  k_set_i64<<<1, 1, 0, (cudaStream_t)stream>>>(dev, v);
  LAUNCH_CHECK("set_i64");
  return LPP_OK;
}

// element access (_atomics.load_f64 / store_f64, _atomics.c:41-56)
__global__ void k_load_f32(const float* p, float* out) {
  float v;
  asm volatile("ld.acquire.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  *out = v;
}
__global__ void k_store_f32(float* p, float v) {
  asm volatile("st.release.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

namespace {
struct HostScratch {  // per host thread: 16 bytes of mapped host memory
  void* h = nullptr;
  void* d = nullptr;
  ~HostScratch() {
    if (h) cudaFreeHost(h);
  }
};
thread_local HostScratch g_scratch;
}  // namespace

extern "C" int lpp_load_f32(const float* arena, size_t len, size_t i, float* out, void* stream) {
  if (!arena || !out) return set_err(LPP_E_VALUE, "load_f32: null buffer");
  if (i >= len) return set_err(LPP_E_INDEX, "index %zu out of range [0, %zu)", i, len);
  if (!g_scratch.h) {
    CUDA_TRY(cudaHostAlloc(&g_scratch.h, 16, cudaHostAllocMapped | cudaHostAllocPortable));
    CUDA_TRY(cudaHostGetDevicePointer(&g_scratch.d, g_scratch.h, 0));
  }
  k_load_f32<<<1, 1, 0, (cudaStream_t)stream>>>(arena + i, static_cast<float*>(g_scratch.d));
  LAUNCH_CHECK("load_f32");
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  *out = *static_cast<volatile float*>(g_scratch.h);
  return LPP_OK;
}

extern "C" int lpp_store_f32(float* arena, size_t len, size_t i, float v, void* stream) {
  if (!arena) return set_err(LPP_E_VALUE, "store_f32: null buffer");
  if (i >= len) return set_err(LPP_E_INDEX, "index %zu out of range [0, %zu)", i, len);
  k_store_f32<<<1, 1, 0, (cudaStream_t)stream>>>(arena + i, v);
  LAUNCH_CHECK("store_f32");
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return LPP_OK;
}

// host memory the kernels read and write directly (mapped, portable)
extern "C" int lpp_host_alloc(size_t bytes, void** host, void** dev) {
  if (!host || !dev) return set_err(LPP_E_VALUE, "host_alloc: null out");
  *host = *dev = nullptr;
  if (bytes == 0) bytes = 16;
  CUDA_TRY(cudaHostAlloc(host, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(*host, 0, bytes);
  cudaError_t e = cudaHostGetDevicePointer(dev, *host, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(*host);
    *host = nullptr;
    return set_err(LPP_E_CUDA, "cudaHostGetDevicePointer failed: %s", cudaGetErrorString(e));
  }
  return LPP_OK;
}

extern "C" int lpp_host_free(void* host) {
  if (host) CUDA_TRY(cudaFreeHost(host));
  return LPP_OK;
}

// reference-shaped accumulate: dst[start+e] += scale*delta[e]
__global__ void __launch_bounds__(kThreads)
    k_accum(float* d, const float* __restrict__ s, size_t n, size_t head, size_t nvec,
            float scale, int mode, int* tags, int stamp) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (size_t i = tid; i < nvec; i += stride) {
    float4 v = __ldg(reinterpret_cast<const float4*>(s + head) + i);
    v.x = __fmul_rn(scale, v.x);
    v.y = __fmul_rn(scale, v.y);
    v.z = __fmul_rn(scale, v.z);
    v.w = __fmul_rn(scale, v.w);
    if (mode == LPP_MODE_PLAIN) {
      float4 o = ld_cg4(d + head + 4 * i);
      o.x = __fadd_rn(o.x, v.x);
      o.y = __fadd_rn(o.y, v.y);
      o.z = __fadd_rn(o.z, v.z);
      o.w = __fadd_rn(o.w, v.w);
      __stcg(reinterpret_cast<float4*>(d + head) + i, o);
    } else {
      red_add_v4(d + head + 4 * i, v);
    }
    if (tags) {
      fence_ar_gpu();
      st_tag4(tags + head + 4 * i, stamp);
    }
  }
  if (blockIdx.x == 0) {
    size_t tail0 = head + 4 * nvec;
    size_t nscalar = head + (n - tail0);
    for (size_t k = threadIdx.x; k < nscalar; k += blockDim.x) {
      size_t e = k < head ? k : tail0 + (k - head);
      float v = __fmul_rn(scale, s[e]);
      if (mode == LPP_MODE_PLAIN)
        __stcg(d + e, __fadd_rn(ld_cg(d + e), v));
      else
        red_add_f32(d + e, v);
      if (tags) {
        fence_ar_gpu();
        st_tag(tags + e, stamp);
      }
    }
  }
}

static int accum_impl(float* dst, int32_t* tags, size_t dst_len, size_t start,
                      const float* delta, size_t n, float scale, int32_t stamp, int mode,
                      void* stream);

extern "C" int lpp_accum(float* dst, size_t dst_len, size_t start, const float* delta,
                         size_t n, float scale, int mode, void* stream) {
  return accum_impl(dst, nullptr, dst_len, start, delta, n, scale, 0, mode, stream);
}

extern "C" int lpp_accum_tagged(float* dst, int32_t* tags, size_t dst_len, size_t start,
                                const float* delta, size_t n, float scale, int32_t stamp,
                                int mode, void* stream) {
  if (!tags) return set_err(LPP_E_VALUE, "accum_tagged: null tags");
  if ((((uintptr_t)dst) ^ ((uintptr_t)tags)) & 15u)
    return set_err(LPP_E_VALUE, "accum_tagged: tags must share dst's alignment modulo 16");
  return accum_impl(dst, tags, dst_len, start, delta, n, scale, stamp, mode, stream);
}

static int accum_impl(float* dst, int32_t* tags, size_t dst_len, size_t start,
                      const float* delta, size_t n, float scale, int32_t stamp, int mode,
                      void* stream) {
  if (start > dst_len || n > dst_len - start)
    return set_err(LPP_E_INDEX, "update range out of bounds");
  if (n == 0) return LPP_OK;
  if (!dst || !delta) return set_err(LPP_E_VALUE, "accum: null buffer");
  if (mode != LPP_MODE_PLAIN && mode != LPP_MODE_RED)
    return set_err(LPP_E_VALUE, "accum: mode must be PLAIN or RED");
  float* d = dst + start;
  int* t = tags ? tags + start : nullptr;
  if (((uintptr_t)d ^ (uintptr_t)delta) & 15u) {
    // mismatched alignment: scalar path (treat everything as head)
    k_accum<<<grid_for((n + 3) / 4, current_sms()), kThreads, 0, (cudaStream_t)stream>>>(
        d, delta, n, n, 0, scale, mode, t, stamp);
  } else {
    size_t head = head_elems(d, n);
    size_t nvec = (n - head) / 4;
    k_accum<<<grid_for(nvec, current_sms()), kThreads, 0, (cudaStream_t)stream>>>(
        d, delta, n, head, nvec, scale, mode, t, stamp);
  }
  LAUNCH_CHECK("accum");
  return LPP_OK;
}

// ---------------------------------------------------------------------------
// K3: snapshot (replica refresh)

__global__ void __launch_bounds__(kThreads)
    k_snapshot(const float* src, float* __restrict__ out, size_t n, size_t head, size_t nvec) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float* sb = src + head;
  float4* ob = reinterpret_cast<float4*>(out + head);
  for (size_t i0 = tid; i0 < nvec; i0 += stride * kUnroll) {
    float4 r[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) r[u] = ld_cg4(sb + 4 * i);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) ob[i] = r[u];
    }
  }
  if (blockIdx.x == 0) {
    size_t tail0 = head + 4 * nvec;
    size_t nscalar = head + (n - tail0);
    for (size_t k = threadIdx.x; k < nscalar; k += blockDim.x) {
      size_t e = k < head ? k : tail0 + (k - head);
      out[e] = ld_cg(src + e);
    }
  }
}

extern "C" int lpp_snapshot(const float* src, float* out, size_t n, void* stream) {
  if (n == 0) return LPP_OK;
  if (!src || !out) return set_err(LPP_E_VALUE, "snapshot: null buffer");
  size_t head, nvec;
  if (((uintptr_t)src ^ (uintptr_t)out) & 15u) {
    head = n;
    nvec = 0;
  } else {
    head = head_elems(src, n);
    nvec = (n - head) / 4;
  }
  k_snapshot<<<grid_for(nvec ? nvec : 1, current_sms()), kThreads, 0, (cudaStream_t)stream>>>(
      src, out, n, head, nvec);
  LAUNCH_CHECK("snapshot");
  return LPP_OK;
}

// K5: tagged snapshot (tags first, fence, then values) + optional min tag,
// and the sampled-tag gather (snapshot_tagged_f64 / gather_i64).

__global__ void __launch_bounds__(kThreads)
    k_snapshot_tagged(const float* src, const int* tags, float* __restrict__ out,
                      int* __restrict__ out_tags, size_t n, size_t head, size_t nvec,
                      int* min_tag) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  int local_min = INT_MAX;
  for (size_t i0 = tid; i0 < nvec; i0 += stride * kUnroll) {
    int4 t[kUnroll];
    float4 r[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) t[u] = ld_tag4(tags + head + 4 * i);
    }
    fence_ar_sys();  // tags may come from peer GPUs' owners (.sys stores)
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) r[u] = ld_cg4(src + head + 4 * i);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
        if (out) reinterpret_cast<float4*>(out + head)[i] = r[u];
        if (out_tags) reinterpret_cast<int4*>(out_tags + head)[i] = t[u];
        local_min = min(local_min, min(min(t[u].x, t[u].y), min(t[u].z, t[u].w)));
      }
    }
  }
  if (blockIdx.x == 0) {
    size_t tail0 = head + 4 * nvec;
    size_t nscalar = head + (n - tail0);
    for (size_t k = threadIdx.x; k < nscalar; k += blockDim.x) {
      size_t e = k < head ? k : tail0 + (k - head);
      int tv = ld_tag(tags + e);
      fence_ar_sys();  // tags may come from peer GPUs' owners (.sys stores)
      float v = ld_cg(src + e);
      if (out) out[e] = v;
      if (out_tags) out_tags[e] = tv;
      local_min = min(local_min, tv);
    }
  }
  if (min_tag) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local_min = min(local_min, __shfl_xor_sync(0xffffffffu, local_min, o));
    if ((threadIdx.x & 31) == 0 && local_min != INT_MAX) atomicMin(min_tag, local_min);
  }
}

extern "C" int lpp_snapshot_tagged(const float* src, const int32_t* tags, float* out,
                                   int32_t* out_tags, size_t n, int32_t* min_tag_out,
                                   void* stream) {
  if (n == 0) return LPP_OK;
  if (!src || !tags) return set_err(LPP_E_VALUE, "snapshot_tagged: null src or tags");
  uintptr_t a = (uintptr_t)src;
  bool aligned = !(((a ^ (uintptr_t)tags) & 15u) || (out && ((a ^ (uintptr_t)out) & 15u)) ||
                   (out_tags && ((a ^ (uintptr_t)out_tags) & 15u)));
  size_t head = aligned ? head_elems(src, n) : n;
  size_t nvec = aligned ? (n - head) / 4 : 0;
  k_snapshot_tagged<<<grid_for(nvec ? nvec : 1, current_sms()), kThreads, 0,
                      (cudaStream_t)stream>>>(src, tags, out, out_tags, n, head, nvec,
                                              min_tag_out);
  LAUNCH_CHECK("snapshot_tagged");
  return LPP_OK;
}

__global__ void k_gather_tags(const int* tags, const int64_t* __restrict__ idx, size_t k,
                              int* __restrict__ out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = ld_tag(tags + idx[i]);
}

extern "C" int lpp_gather_tags(const int32_t* tags, const int64_t* idx, size_t k, int32_t* out,
                               void* stream) {
  if (k == 0) return LPP_OK;
  if (!tags || !idx || !out) return set_err(LPP_E_VALUE, "gather_tags: null buffer");
  unsigned grid = (unsigned)((k + kThreads - 1) / kThreads);
  k_gather_tags<<<grid, kThreads, 0, (cudaStream_t)stream>>>(tags, idx, k, out);
  LAUNCH_CHECK("gather_tags");
  return LPP_OK;
}

// ---------------------------------------------------------------------------
// K4: owner-computes averaging over a shard of Q arenas

struct ArenaTable {
  float* p[LPP_MAX_WORKERS];
  int* tag[LPP_MAX_WORKERS];   // K5: per-worker write tags (all null: untagged)
  int stamp[LPP_MAX_WORKERS];  // each worker's update-order stamp for this round
  int tagged;
};

// Q and TAGGED are compile-time so each instantiation keeps exactly the
// 2*Q float4 registers it needs (a runtime Q sized for LPP_MAX_WORKERS spilled
// occupancy to 1 CTA/SM).
template <int MODE, int Q, bool TAGGED>
__global__ void __launch_bounds__(kThreads)
    k_average(ArenaTable t, size_t lo, size_t n, size_t head, size_t nvec,
              float* __restrict__ mean_out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float fq = (float)Q;
  constexpr int U = 2;  // 2 x Q independent 16-byte loads in flight
  for (size_t i0 = tid; i0 < nvec; i0 += stride * U) {
    float4 v[U][Q];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
          v[u][q] = ld_cg4(t.p[q] + lo + head + 4 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
        float4 s = v[u][0];
#pragma unroll
        for (int q = 1; q < LPP_MAX_WORKERS; ++q) {
          if (q < Q) {
            s.x = __fadd_rn(s.x, v[u][q].x);
            s.y = __fadd_rn(s.y, v[u][q].y);
            s.z = __fadd_rn(s.z, v[u][q].z);
            s.w = __fadd_rn(s.w, v[u][q].w);
          }
        }
        float4 mean;
        mean.x = __fdiv_rn(s.x, fq);
        mean.y = __fdiv_rn(s.y, fq);
        mean.z = __fdiv_rn(s.z, fq);
        mean.w = __fdiv_rn(s.w, fq);
#pragma unroll
        for (int q = 0; q < LPP_MAX_WORKERS; ++q) {
          if (q < Q) {
            float4 c;
            c.x = __fsub_rn(mean.x, v[u][q].x);
            c.y = __fsub_rn(mean.y, v[u][q].y);
            c.z = __fsub_rn(mean.z, v[u][q].z);
            c.w = __fsub_rn(mean.w, v[u][q].w);
            float* dst = t.p[q] + lo + head + 4 * i;
            if (MODE == LPP_MODE_PLAIN) {
              float4 o;
              o.x = __fadd_rn(v[u][q].x, c.x);
              o.y = __fadd_rn(v[u][q].y, c.y);
              o.z = __fadd_rn(v[u][q].z, c.z);
              o.w = __fadd_rn(v[u][q].w, c.w);
              __stcg(reinterpret_cast<float4*>(dst), o);
            } else {
              red_add_v4(dst, c);
            }
          }
        }
        if (mean_out) reinterpret_cast<float4*>(mean_out + head)[i] = mean;
      }
    }
    if (TAGGED) {
      fence_ar_sys();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        size_t i = i0 + (size_t)u * stride;
        if (i < nvec) {
#pragma unroll
          for (int q = 0; q < LPP_MAX_WORKERS; ++q)
            if (q < Q) st_tag4_sys(t.tag[q] + lo + head + 4 * i, t.stamp[q]);
        }
      }
    }
  }
  if (blockIdx.x == 0) {
    size_t tail0 = head + 4 * nvec;
    size_t nscalar = head + (n - tail0);
    for (size_t k = threadIdx.x; k < nscalar; k += blockDim.x) {
      size_t e = k < head ? k : tail0 + (k - head);
      float vv[Q];
#pragma unroll
      for (int q = 0; q < LPP_MAX_WORKERS; ++q)
        if (q < Q) vv[q] = ld_cg(t.p[q] + lo + e);
      float s = vv[0];
#pragma unroll
      for (int q = 1; q < LPP_MAX_WORKERS; ++q)
        if (q < Q) s = __fadd_rn(s, vv[q]);
      float mean = __fdiv_rn(s, fq);
#pragma unroll
      for (int q = 0; q < LPP_MAX_WORKERS; ++q) {
        if (q < Q) {
          float c = __fsub_rn(mean, vv[q]);
          if (MODE == LPP_MODE_PLAIN)
            __stcg(t.p[q] + lo + e, __fadd_rn(vv[q], c));
          else
            red_add_f32(t.p[q] + lo + e, c);
        }
      }
      if (mean_out) mean_out[e] = mean;
      if (TAGGED) {
        fence_ar_sys();
#pragma unroll
        for (int q = 0; q < LPP_MAX_WORKERS; ++q)
          if (q < Q) st_tag_sys(t.tag[q] + lo + e, t.stamp[q]);
      }
    }
  }
}

// K4 mode BULK (untagged): the round staged through shared memory by the
// bulk-copy (TMA) engine.  Per tile one thread issues Q bulk loads (one per
// arena — peer arenas are read over NVLink by the copy engine, not by LSU
// loads) completing on an mbarrier; the CTA forms the fixed-order mean and
// overwrites each staged tile with its correction mean - v_q in place; one
// thread then hands the Q tiles to cp.reduce.async.bulk .add.f32 (the
// correction lands as element-wise atomic adds, exactly like K4's red.add).
// kAvgStages - 1 tiles' loads are in flight while a tile is reduced.
constexpr int kAvgTileV = 512;   // float4 per arena per tile (8 KB)
constexpr int kAvgStages = 2;   // 4 KB x 3 stages and 2 KB x 4 measured 1-8 % slower

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes,
                                          uint64_t* bar) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          d),
      "l"(gmem), "r"(bytes), "r"(b)
      : "memory");
}

template <int Q>
__global__ void __launch_bounds__(kThreads)
    k_average_bulk(ArenaTable t, size_t lo, size_t n, size_t head, size_t nvec,
                   float* __restrict__ mean_out) {
  extern __shared__ __align__(128) float4 s_avg[];   // [kAvgStages][Q][kAvgTileV]
  __shared__ __align__(8) uint64_t bars[kAvgStages];
  const float fq = (float)Q;
  const size_t ntiles = (nvec + kAvgTileV - 1) / kAvgTileV;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAvgStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t tile, int stage) {
    const size_t base = tile * kAvgTileV;
    const int cnt = (int)((nvec - base) < (size_t)kAvgTileV ? (nvec - base) : kAvgTileV);
    mbar_expect_tx(&bars[stage], (uint32_t)(Q * cnt * 16));
    for (int q = 0; q < Q; ++q)
      bulk_load(s_avg + ((size_t)stage * Q + q) * kAvgTileV, t.p[q] + lo + head + 4 * base,
                (uint32_t)(cnt * 16), &bars[stage]);
  };
  uint32_t phase[kAvgStages] = {};
  size_t tile = blockIdx.x;
  // prologue: the first kAvgStages - 1 tiles' loads in flight
  if (threadIdx.x == 0)
    for (int k = 0; k < kAvgStages - 1; ++k) {
      size_t tk = tile + (size_t)k * gridDim.x;
      if (tk < ntiles) issue(tk, k);
    }
  int stage = 0;
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    const size_t ahead = tile + (size_t)(kAvgStages - 1) * gridDim.x;
    const int astage = (stage + kAvgStages - 1) % kAvgStages;
    if (threadIdx.x == 0 && ahead < ntiles) {
      // astage is the stage the previous iteration just handed to the bulk
      // reductions (the most recent group): they must have read it first
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(ahead, astage);
    }
    mbar_wait(&bars[stage], phase[stage]);
    phase[stage] ^= 1;
    const size_t base = tile * kAvgTileV;
    const int cnt = (int)((nvec - base) < (size_t)kAvgTileV ? (nvec - base) : kAvgTileV);
    float4* buf = s_avg + (size_t)stage * Q * kAvgTileV;
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      float4 v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) v[q] = buf[q * kAvgTileV + j];
      float4 sum = v[0];
#pragma unroll
      for (int q = 1; q < Q; ++q) {
        sum.x = __fadd_rn(sum.x, v[q].x);
        sum.y = __fadd_rn(sum.y, v[q].y);
        sum.z = __fadd_rn(sum.z, v[q].z);
        sum.w = __fadd_rn(sum.w, v[q].w);
      }
      float4 mean;
      mean.x = __fdiv_rn(sum.x, fq);
      mean.y = __fdiv_rn(sum.y, fq);
      mean.z = __fdiv_rn(sum.z, fq);
      mean.w = __fdiv_rn(sum.w, fq);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        float4 c;
        c.x = __fsub_rn(mean.x, v[q].x);
        c.y = __fsub_rn(mean.y, v[q].y);
        c.z = __fsub_rn(mean.z, v[q].z);
        c.w = __fsub_rn(mean.w, v[q].w);
        buf[q * kAvgTileV + j] = c;
      }
      if (mean_out) reinterpret_cast<float4*>(mean_out + head)[base + j] = mean;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 0; q < Q; ++q) {
        uint32_t saddr = (uint32_t)__cvta_generic_to_shared(buf + q * kAvgTileV);
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                t.p[q] + lo + head + 4 * base),
            "r"(saddr), "r"(cnt * 16)
            : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    stage = (stage + 1) % kAvgStages;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // scalar head / tail (first block), as the LSU variant
  if (blockIdx.x == 0) {
    size_t tail0 = head + 4 * nvec;
    size_t nscalar = head + (n - tail0);
    for (size_t k = threadIdx.x; k < nscalar; k += blockDim.x) {
      size_t e = k < head ? k : tail0 + (k - head);
      float vv[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) vv[q] = ld_cg(t.p[q] + lo + e);
      float sm = vv[0];
#pragma unroll
      for (int q = 1; q < Q; ++q) sm = __fadd_rn(sm, vv[q]);
      float mean = __fdiv_rn(sm, fq);
#pragma unroll
      for (int q = 0; q < Q; ++q) red_add_f32(t.p[q] + lo + e, __fsub_rn(mean, vv[q]));
      if (mean_out) mean_out[e] = mean;
    }
  }
}

template <int Q>
static void launch_average_bulk_q(cudaStream_t st, const ArenaTable& t, size_t lo, size_t n,
                                  size_t head, size_t nvec, float* mean_out) {
  size_t smem = (size_t)kAvgStages * Q * kAvgTileV * sizeof(float4);
  // the dynamic shared-memory opt-in is per device (workers of one process
  // may sit on several GPUs)
  static std::atomic<unsigned long long> done_mask{0};
  int dev = 0;
  cudaGetDevice(&dev);
  unsigned long long bit = 1ull << (dev & 63);
  if (!(done_mask.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(k_average_bulk<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    done_mask.fetch_or(bit, std::memory_order_acq_rel);
  }
  size_t ntiles = (nvec + kAvgTileV - 1) / kAvgTileV;
  int per_sm = (int)((200 * 1024) / (smem + 64));
  if (per_sm < 1) per_sm = 1;
  size_t cap = (size_t)current_sms() * (size_t)per_sm;
  unsigned grid = (unsigned)(ntiles < cap ? (ntiles ? ntiles : 1) : cap);
  k_average_bulk<Q><<<grid, kThreads, smem, st>>>(t, lo, n, head, nvec, mean_out);
}

static void launch_average_bulk(int Q, cudaStream_t st, const ArenaTable& t, size_t lo, size_t n,
                                size_t head, size_t nvec, float* mean_out) {
  switch (Q) {
    case 1: launch_average_bulk_q<1>(st, t, lo, n, head, nvec, mean_out); break;
    case 2: launch_average_bulk_q<2>(st, t, lo, n, head, nvec, mean_out); break;
    case 3: launch_average_bulk_q<3>(st, t, lo, n, head, nvec, mean_out); break;
    case 4: launch_average_bulk_q<4>(st, t, lo, n, head, nvec, mean_out); break;
    case 5: launch_average_bulk_q<5>(st, t, lo, n, head, nvec, mean_out); break;
    case 6: launch_average_bulk_q<6>(st, t, lo, n, head, nvec, mean_out); break;
    case 7: launch_average_bulk_q<7>(st, t, lo, n, head, nvec, mean_out); break;
    default: launch_average_bulk_q<8>(st, t, lo, n, head, nvec, mean_out); break;
  }
}

template <int MODE, int Q>
static void launch_average_q(bool tagged, unsigned grid, cudaStream_t st, const ArenaTable& t,
                             size_t lo, size_t n, size_t head, size_t nvec, float* mean_out) {
  if (tagged)
    k_average<MODE, Q, true><<<grid, kThreads, 0, st>>>(t, lo, n, head, nvec, mean_out);
  else
    k_average<MODE, Q, false><<<grid, kThreads, 0, st>>>(t, lo, n, head, nvec, mean_out);
}

template <int MODE>
static void launch_average_m(int Q, bool tagged, unsigned grid, cudaStream_t st,
                             const ArenaTable& t, size_t lo, size_t n, size_t head, size_t nvec,
                             float* mean_out) {
  switch (Q) {
    case 1: launch_average_q<MODE, 1>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
    case 2: launch_average_q<MODE, 2>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
    case 3: launch_average_q<MODE, 3>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
    case 4: launch_average_q<MODE, 4>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
    case 5: launch_average_q<MODE, 5>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
    case 6: launch_average_q<MODE, 6>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
    case 7: launch_average_q<MODE, 7>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
    default: launch_average_q<MODE, 8>(tagged, grid, st, t, lo, n, head, nvec, mean_out); break;
  }
}

static void launch_average(int mode, int Q, bool tagged, unsigned grid, cudaStream_t st,
                           const ArenaTable& t, size_t lo, size_t n, size_t head, size_t nvec,
                           float* mean_out) {
  if (mode == LPP_MODE_BULK && !tagged)
    launch_average_bulk(Q, st, t, lo, n, head, nvec, mean_out);
  else if (mode == LPP_MODE_PLAIN)
    launch_average_m<LPP_MODE_PLAIN>(Q, tagged, grid, st, t, lo, n, head, nvec, mean_out);
  else
    launch_average_m<LPP_MODE_RED>(Q, tagged, grid, st, t, lo, n, head, nvec, mean_out);
}

static int average_impl(float* const* arenas, int32_t* const* tags, const int32_t* stamps, int Q,
                        size_t lo, size_t hi, float* mean_out, int mode, void* stream);

extern "C" int lpp_average_shard(float* const* arenas, int Q, size_t lo, size_t hi,
                                 float* mean_out, int mode, void* stream) {
  return average_impl(arenas, nullptr, nullptr, Q, lo, hi, mean_out, mode, stream);
}

extern "C" int lpp_average_shard_tagged(float* const* arenas, int32_t* const* tags,
                                        const int32_t* stamps, int Q, size_t lo, size_t hi,
                                        float* mean_out, int mode, void* stream) {
  if (!tags || !stamps) return set_err(LPP_E_VALUE, "average_shard_tagged: null tags/stamps");
  return average_impl(arenas, tags, stamps, Q, lo, hi, mean_out, mode, stream);
}

static int average_impl(float* const* arenas, int32_t* const* tags, const int32_t* stamps, int Q,
                        size_t lo, size_t hi, float* mean_out, int mode, void* stream) {
  if (Q < 1 || Q > LPP_MAX_WORKERS)
    return set_err(LPP_E_VALUE, "average_shard: Q=%d outside [1, %d]", Q, LPP_MAX_WORKERS);
  if (hi < lo) return set_err(LPP_E_INDEX, "average_shard: hi < lo");
  if (!arenas) return set_err(LPP_E_VALUE, "average_shard: null arena table");
  if (mode != LPP_MODE_PLAIN && mode != LPP_MODE_RED && mode != LPP_MODE_BULK)
    return set_err(LPP_E_VALUE, "average_shard: mode must be PLAIN, RED or BULK");
  size_t n = hi - lo;
  if (n == 0) return LPP_OK;
  ArenaTable t;
  memset(&t, 0, sizeof(t));
  for (int q = 0; q < Q; ++q) {
    if (!arenas[q]) return set_err(LPP_E_VALUE, "average_shard: null arena %d", q);
    if (((uintptr_t)arenas[q] ^ (uintptr_t)arenas[0]) & 15u)
      return set_err(LPP_E_VALUE, "average_shard: arenas must share 16-byte alignment");
    t.p[q] = arenas[q];
    if (tags) {
      if (!tags[q]) return set_err(LPP_E_VALUE, "average_shard_tagged: null tags %d", q);
      if (((uintptr_t)tags[q] ^ (uintptr_t)arenas[0]) & 15u)
        return set_err(LPP_E_VALUE, "average_shard_tagged: tags must share the arenas' alignment");
      t.tag[q] = tags[q];
      t.stamp[q] = stamps[q];
    }
  }
  t.tagged = tags ? 1 : 0;
  if (mean_out && ((((uintptr_t)mean_out) ^ (uintptr_t)(arenas[0] + lo)) & 15u))
    return set_err(LPP_E_VALUE, "average_shard: mean_out alignment must match the shard");
  size_t head = head_elems(arenas[0] + lo, n);
  size_t nvec = (n - head) / 4;
  unsigned grid = grid_for(nvec ? nvec : 1, current_sms());
  launch_average(mode, Q, t.tagged != 0, grid, (cudaStream_t)stream, t, lo, n, head, nvec,
                 mean_out);
  LAUNCH_CHECK("average_shard");
  return LPP_OK;
}

// ---------------------------------------------------------------------------
// arenas + peer mapping

struct lpp_arena {
  float* ptr;
  size_t n;
  int device;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

extern "C" int lpp_arena_create(int device, size_t n_elems, lpp_arena_t* out) {
  if (!out) return set_err(LPP_E_VALUE, "arena_create: null out");
  *out = nullptr;
  DeviceGuard guard(device);
  float* p = nullptr;
  size_t bytes = (n_elems ? n_elems : 1) * sizeof(float);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess)
    return set_err(LPP_E_NOMEM, "arena_create: cudaMalloc(%zu) failed: %s", bytes,
                   cudaGetErrorString(e));
  e = cudaMemset(p, 0, bytes);
  if (e != cudaSuccess) {
    cudaFree(p);
    return set_err(LPP_E_CUDA, "arena_create: memset failed: %s", cudaGetErrorString(e));
  }
  lpp_arena* a = new lpp_arena{p, n_elems, device};
  *out = a;
  return LPP_OK;
}

extern "C" int lpp_arena_destroy(lpp_arena_t a) {
  if (!a) return LPP_OK;
  DeviceGuard guard(a->device);
  cudaError_t e = cudaFree(a->ptr);
  delete a;
  if (e != cudaSuccess)
    return set_err(LPP_E_CUDA, "arena_destroy: %s", cudaGetErrorString(e));
  return LPP_OK;
}

extern "C" float* lpp_arena_data(lpp_arena_t a) { return a ? a->ptr : nullptr; }
extern "C" size_t lpp_arena_size(lpp_arena_t a) { return a ? a->n : 0; }
extern "C" int lpp_arena_device(lpp_arena_t a) { return a ? a->device : -1; }

extern "C" int lpp_arena_export_ipc(lpp_arena_t a, void* handle_out) {
  if (!a || !handle_out) return set_err(LPP_E_VALUE, "export_ipc: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == LPP_IPC_HANDLE_BYTES, "ipc handle size");
  DeviceGuard guard(a->device);
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, a->ptr));
  memcpy(handle_out, &h, sizeof(h));
  return LPP_OK;
}

extern "C" int lpp_ipc_open(int device, const void* handle, float** ptr_out) {
  if (!handle || !ptr_out) return set_err(LPP_E_VALUE, "ipc_open: null argument");
  DeviceGuard guard(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr_out = (float*)p;
  return LPP_OK;
}

extern "C" int lpp_ipc_close(int device, float* ptr) {
  DeviceGuard guard(device);
  CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return LPP_OK;
}

extern "C" int lpp_can_access_peer(int device, int peer, int* out) {
  if (!out) return set_err(LPP_E_VALUE, "can_access_peer: null out");
  CUDA_TRY(cudaDeviceCanAccessPeer(out, device, peer));
  return LPP_OK;
}

extern "C" int lpp_enable_peer_access(int device, int peer) {
  if (device == peer) return LPP_OK;
  DeviceGuard guard(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return LPP_OK;
  }
  if (e != cudaSuccess)
    return set_err(LPP_E_CUDA, "enable_peer_access(%d -> %d): %s", device, peer,
                   cudaGetErrorString(e));
  return LPP_OK;
}

// ---------------------------------------------------------------------------
// utilities

extern "C" int lpp_host_gather_rows(void* dst, const void* src, size_t n_rows, size_t row_bytes,
                                    const int64_t* idx, size_t n_idx) {
  if (n_idx == 0 || row_bytes == 0) return LPP_OK;
  if (!dst || !src || !idx) return set_err(LPP_E_VALUE, "host_gather_rows: null pointer");
  for (size_t i = 0; i < n_idx; ++i)
    if (idx[i] < 0 || (size_t)idx[i] >= n_rows)
      return set_err(LPP_E_INDEX, "host_gather_rows: index %lld outside [0, %zu)",
                     (long long)idx[i], n_rows);
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  for (size_t i = 0; i < n_idx; ++i) memcpy(d + i * row_bytes, s + (size_t)idx[i] * row_bytes, row_bytes);
  return LPP_OK;
}

extern "C" int lpp_graph_launch(void* graph_exec, void* stream) {
  if (!graph_exec) return set_err(LPP_E_VALUE, "graph_launch: null graph");
  CUDA_TRY(cudaGraphLaunch((cudaGraphExec_t)graph_exec, (cudaStream_t)stream));
  return LPP_OK;
}

extern "C" int lpp_copy_async(void* dst, const void* src, size_t n_bytes, void* stream) {
  if (n_bytes == 0) return LPP_OK;
  if (!dst || !src) return set_err(LPP_E_VALUE, "copy_async: null pointer");
  CUDA_TRY(cudaMemcpyAsync(dst, src, n_bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return LPP_OK;
}

extern "C" int lpp_l2_flush(void* scratch, size_t n_bytes, void* stream) {
  if (!scratch) return set_err(LPP_E_VALUE, "l2_flush: null scratch");
  CUDA_TRY(cudaMemsetAsync(scratch, 0x5a, n_bytes, (cudaStream_t)stream));
  return LPP_OK;
}

extern "C" int lpp_sm_count(int device, int* out) {
  if (!out) return set_err(LPP_E_VALUE, "sm_count: null out");
  CUDA_TRY(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device));
  return LPP_OK;
}

// ---------------------------------------------------------------------------
// NVLS (NVLink SHARP) averaging: SURVEY §8f rank 1.
//
// The reference round is snapshot -> mean all-reduce -> add_assign(mean -
// snapshot) (engine.py:418-421).  On NVSwitch the all-reduce runs IN the
// switch: every worker stages its snapshot in a VMM buffer bound to one
// multicast object; the owner of shard o issues multimem.ld_reduce (SASS
// LDGMC) on the multicast address — the switch reads shard o from all Q
// GPUs and returns the sum — and multimem.st broadcasts the mean into every
// worker's mean buffer; each worker then adds (mean - snapshot) into its own
// arena locally.  Per GPU and direction the NVLink bytes are ~4d(1 + 1/Q)
// instead of the 2·4d(Q-1)/Q of the P2P owner-computes round.

#include <cuda.h>

// The driver API is resolved at run time through the runtime's entry-point
// query, so the library needs no link-time libcuda (it loads on CPU-only
// build hosts; every device entry point then reports the missing driver).
namespace drv {
#define LPP_DRV_FN(name, ret, args) \
  typedef ret(*name##_t) args;      \
  static name##_t name = nullptr;
LPP_DRV_FN(cuGetErrorString, CUresult, (CUresult, const char**))
LPP_DRV_FN(cuDeviceGet, CUresult, (CUdevice*, int))
LPP_DRV_FN(cuDeviceGetAttribute, CUresult, (int*, CUdevice_attribute, CUdevice))
LPP_DRV_FN(cuMulticastGetGranularity, CUresult,
           (size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags))
LPP_DRV_FN(cuMemGetAllocationGranularity, CUresult,
           (size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags))
LPP_DRV_FN(cuMemCreate, CUresult,
           (CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long))
LPP_DRV_FN(cuMemAddressReserve, CUresult,
           (CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long))
LPP_DRV_FN(cuMemAddressFree, CUresult, (CUdeviceptr, size_t))
LPP_DRV_FN(cuMemMap, CUresult,
           (CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long))
LPP_DRV_FN(cuMemUnmap, CUresult, (CUdeviceptr, size_t))
LPP_DRV_FN(cuMemSetAccess, CUresult, (CUdeviceptr, size_t, const CUmemAccessDesc*, size_t))
LPP_DRV_FN(cuMemsetD8, CUresult, (CUdeviceptr, unsigned char, size_t))
LPP_DRV_FN(cuMemRelease, CUresult, (CUmemGenericAllocationHandle))
LPP_DRV_FN(cuMulticastCreate, CUresult, (CUmemGenericAllocationHandle*, const CUmulticastObjectProp*))
LPP_DRV_FN(cuMulticastAddDevice, CUresult, (CUmemGenericAllocationHandle, CUdevice))
LPP_DRV_FN(cuMulticastBindMem, CUresult,
           (CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
            unsigned long long))
LPP_DRV_FN(cuMulticastUnbind, CUresult, (CUmemGenericAllocationHandle, CUdevice, size_t, size_t))
LPP_DRV_FN(cuMemExportToShareableHandle, CUresult,
           (void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long))
LPP_DRV_FN(cuMemImportFromShareableHandle, CUresult,
           (CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType))
LPP_DRV_FN(cuStreamWriteValue32, CUresult, (CUstream, CUdeviceptr, cuuint32_t, unsigned int))
#undef LPP_DRV_FN

template <typename T>
static bool load(T& fn, const char* name) {
  if (fn) return true;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  fn = reinterpret_cast<T>(p);
  return true;
}

static int init() {
  static std::atomic<int> state{0};  // 0 unknown, 1 ok, -1 failed
  int st = state.load();
  if (st) return st > 0 ? LPP_OK : set_err(LPP_E_CUDA, "CUDA driver entry points unavailable");
  bool ok = load(cuGetErrorString, "cuGetErrorString") && load(cuDeviceGet, "cuDeviceGet") &&
            load(cuDeviceGetAttribute, "cuDeviceGetAttribute") &&
            load(cuMulticastGetGranularity, "cuMulticastGetGranularity") &&
            load(cuMemGetAllocationGranularity, "cuMemGetAllocationGranularity") &&
            load(cuMemCreate, "cuMemCreate") && load(cuMemAddressReserve, "cuMemAddressReserve") &&
            load(cuMemAddressFree, "cuMemAddressFree") && load(cuMemMap, "cuMemMap") &&
            load(cuMemUnmap, "cuMemUnmap") && load(cuMemSetAccess, "cuMemSetAccess") &&
            load(cuMemsetD8, "cuMemsetD8") && load(cuMemRelease, "cuMemRelease") &&
            load(cuMulticastCreate, "cuMulticastCreate") &&
            load(cuMulticastAddDevice, "cuMulticastAddDevice") &&
            load(cuMulticastBindMem, "cuMulticastBindMem") &&
            load(cuMulticastUnbind, "cuMulticastUnbind") &&
            load(cuMemExportToShareableHandle, "cuMemExportToShareableHandle") &&
            load(cuMemImportFromShareableHandle, "cuMemImportFromShareableHandle");
  state.store(ok ? 1 : -1);
  return ok ? LPP_OK : set_err(LPP_E_CUDA, "CUDA driver entry points unavailable");
}
}  // namespace drv

// K5: an update's block stamp, written by the stream's front end once the
// apply before it on the stream has completed, after a system-wide memory
// barrier (CU_STREAM_WRITE_VALUE_DEFAULT): every element reduction of the
// update is visible before the stamp.  The last write wins, as the
// reference's per-element tags (the CAS that lands last stamps last,
// _atomics.c:346-392).  A stream memory operation, not a kernel: the step's
// only launch of ours stays the fused apply.
extern "C" int lpp_publish_stamp(int32_t* stamps, int block_id, int32_t stamp, void* stream) {
  if (!stamps || block_id < 0) return set_err(LPP_E_VALUE, "publish_stamp: bad stamps / block");
  // resolved once, thread-safely (function-local static initialisation)
  static const bool have = drv::load(drv::cuStreamWriteValue32, "cuStreamWriteValue32") &&
                           drv::load(drv::cuGetErrorString, "cuGetErrorString");
  if (!have) return set_err(LPP_E_CUDA, "publish_stamp: cuStreamWriteValue32 unavailable");
  CUresult r = drv::cuStreamWriteValue32((CUstream)stream, (CUdeviceptr)(stamps + block_id),
                                         (cuuint32_t)stamp, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) {
    const char* e = nullptr;
    drv::cuGetErrorString(r, &e);
    return set_err(LPP_E_CUDA, "publish_stamp: cuStreamWriteValue32 failed: %s", e ? e : "?");
  }
  return LPP_OK;
}

#define CU_TRY(expr)                                                        \
  do {                                                                      \
    CUresult r_ = (drv::expr);                                              \
    if (r_ != CUDA_SUCCESS) {                                               \
      const char* s_ = nullptr;                                             \
      drv::cuGetErrorString(r_, &s_);                                       \
      return set_err(LPP_E_CUDA, "%s failed: %s", #expr, s_ ? s_ : "?");    \
    }                                                                       \
  } while (0)
#define DRV_INIT()                   \
  do {                               \
    int rc_ = drv::init();           \
    if (rc_) return rc_;             \
  } while (0)

struct lpp_vmm {
  CUmemGenericAllocationHandle h;
  CUdeviceptr ptr;
  size_t size;
  int device;
};

struct lpp_mc {
  CUmemGenericAllocationHandle h;
  size_t size;
  CUdeviceptr ptr;  // mapped multicast VA (0 until lpp_mc_map)
  int mapped_device;
  int bound_device;
  size_t bound_offset, bound_size;
};

static CUmemAllocationProp vmm_prop(int device) {
  CUmemAllocationProp p;
  memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

static int ensure_ctx(int device) {
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaFree(0));  // make the primary context current for the driver API
  return LPP_OK;
}

extern "C" int lpp_mc_supported(int device, int* out) {
  if (!out) return set_err(LPP_E_VALUE, "mc_supported: null out");
  DRV_INIT();
  CUDA_TRY(cudaFree(0));
  CUdevice dev;
  CU_TRY(cuDeviceGet(&dev, device));
  CU_TRY(cuDeviceGetAttribute(out, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  return LPP_OK;
}

extern "C" int lpp_mc_granularity(int device, int num_devices, size_t* out) {
  if (!out) return set_err(LPP_E_VALUE, "mc_granularity: null out");
  DRV_INIT();
  CUDA_TRY(cudaFree(0));
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)num_devices;
  mp.size = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g1 = 0, g2 = 0;
  CU_TRY(cuMulticastGetGranularity(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap = vmm_prop(device);
  CU_TRY(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  *out = g1 > g2 ? g1 : g2;
  return LPP_OK;
}

extern "C" int lpp_vmm_create(int device, size_t bytes, lpp_vmm_t* out) {
  if (!out) return set_err(LPP_E_VALUE, "vmm_create: null out");
  *out = nullptr;
  DeviceGuard guard(device);
  int rc = ensure_ctx(device);
  if (rc) return rc;
  size_t gran = 0;
  rc = lpp_mc_granularity(device, 1, &gran);
  if (rc) return rc;
  size_t size = ((bytes ? bytes : 1) + gran - 1) / gran * gran;
  CUmemAllocationProp prop = vmm_prop(device);
  lpp_vmm* v = new lpp_vmm{0, 0, size, device};
  CUresult r = drv::cuMemCreate(&v->h, size, &prop, 0);
  if (r != CUDA_SUCCESS) {
    delete v;
    return set_err(LPP_E_NOMEM, "vmm_create: cuMemCreate(%zu) failed (%d)", size, (int)r);
  }
  CU_TRY(cuMemAddressReserve(&v->ptr, size, gran, 0, 0));
  CU_TRY(cuMemMap(v->ptr, size, 0, v->h, 0));
  CUmemAccessDesc ad;
  memset(&ad, 0, sizeof(ad));
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = device;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU_TRY(cuMemSetAccess(v->ptr, size, &ad, 1));
  CU_TRY(cuMemsetD8(v->ptr, 0, size));
  *out = v;
  return LPP_OK;
}

extern "C" float* lpp_vmm_ptr(lpp_vmm_t v) { return v ? (float*)v->ptr : nullptr; }
extern "C" size_t lpp_vmm_size(lpp_vmm_t v) { return v ? v->size : 0; }

extern "C" int lpp_vmm_destroy(lpp_vmm_t v) {
  if (!v) return LPP_OK;
  DeviceGuard guard(v->device);
  CU_TRY(cuMemUnmap(v->ptr, v->size));
  CU_TRY(cuMemAddressFree(v->ptr, v->size));
  CU_TRY(cuMemRelease(v->h));
  delete v;
  return LPP_OK;
}

extern "C" int lpp_mc_create(int num_devices, size_t bytes, lpp_mc_t* out) {
  if (!out || num_devices < 1) return set_err(LPP_E_VALUE, "mc_create: bad arguments");
  DRV_INIT();
  CUDA_TRY(cudaFree(0));
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)num_devices;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  lpp_mc* m = new lpp_mc{0, bytes, 0, -1, -1, 0, 0};
  CUresult r = drv::cuMulticastCreate(&m->h, &mp);
  if (r != CUDA_SUCCESS) {
    delete m;
    const char* s = nullptr;
    drv::cuGetErrorString(r, &s);
    return set_err(LPP_E_CUDA, "cuMulticastCreate(%d devices, %zu B) failed: %s", num_devices,
                   bytes, s ? s : "?");
  }
  *out = m;
  return LPP_OK;
}

extern "C" int lpp_mc_export_fd(lpp_mc_t m, int* fd_out) {
  if (!m || !fd_out) return set_err(LPP_E_VALUE, "mc_export_fd: null argument");
  CU_TRY(cuMemExportToShareableHandle(fd_out, m->h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  return LPP_OK;
}

extern "C" int lpp_mc_import_fd(int fd, size_t bytes, lpp_mc_t* out) {
  if (!out) return set_err(LPP_E_VALUE, "mc_import_fd: null out");
  DRV_INIT();
  CUDA_TRY(cudaFree(0));
  lpp_mc* m = new lpp_mc{0, bytes, 0, -1, -1, 0, 0};
  CUresult r = drv::cuMemImportFromShareableHandle(&m->h, (void*)(uintptr_t)fd,
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) {
    delete m;
    return set_err(LPP_E_CUDA, "mc_import_fd failed (%d)", (int)r);
  }
  *out = m;
  return LPP_OK;
}

extern "C" int lpp_mc_add_device(lpp_mc_t m, int device) {
  if (!m) return set_err(LPP_E_VALUE, "mc_add_device: null mc");
  int rc = ensure_ctx(device);
  if (rc) return rc;
  CUdevice dev;
  CU_TRY(cuDeviceGet(&dev, device));
  CU_TRY(cuMulticastAddDevice(m->h, dev));
  return LPP_OK;
}

extern "C" int lpp_mc_bind(lpp_mc_t m, lpp_vmm_t mem, size_t mc_offset) {
  if (!m || !mem) return set_err(LPP_E_VALUE, "mc_bind: null argument");
  if (mc_offset + mem->size > m->size) return set_err(LPP_E_INDEX, "mc_bind: range outside object");
  DeviceGuard guard(mem->device);
  CU_TRY(cuMulticastBindMem(m->h, mc_offset, mem->h, 0, mem->size, 0));
  m->bound_device = mem->device;
  m->bound_offset = mc_offset;
  m->bound_size = mem->size;
  return LPP_OK;
}

extern "C" int lpp_mc_map(lpp_mc_t m, int device, float** ptr_out) {
  if (!m || !ptr_out) return set_err(LPP_E_VALUE, "mc_map: null argument");
  DeviceGuard guard(device);
  size_t gran = 0;
  int rc = lpp_mc_granularity(device, 1, &gran);
  if (rc) return rc;
  CU_TRY(cuMemAddressReserve(&m->ptr, m->size, gran, 0, 0));
  CU_TRY(cuMemMap(m->ptr, m->size, 0, m->h, 0));
  CUmemAccessDesc ad;
  memset(&ad, 0, sizeof(ad));
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = device;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU_TRY(cuMemSetAccess(m->ptr, m->size, &ad, 1));
  m->mapped_device = device;
  *ptr_out = (float*)m->ptr;
  return LPP_OK;
}

extern "C" int lpp_mc_destroy(lpp_mc_t m) {
  if (!m) return LPP_OK;
  if (m->ptr) {
    DeviceGuard guard(m->mapped_device);
    CU_TRY(cuMemUnmap(m->ptr, m->size));
    CU_TRY(cuMemAddressFree(m->ptr, m->size));
  }
  if (m->bound_device >= 0) {
    CUdevice dev;
    CU_TRY(cuDeviceGet(&dev, m->bound_device));
    CU_TRY(cuMulticastUnbind(m->h, dev, m->bound_offset, m->bound_size));
  }
  CU_TRY(cuMemRelease(m->h));
  delete m;
  return LPP_OK;
}

// owner: mean of shard [lo, hi) reduced in the switch, broadcast to all
__global__ void __launch_bounds__(kThreads)
    k_nvls_mean(const float* mc_stage, float* mc_mean, size_t lo, size_t n, size_t nvec, int Q) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float fq = (float)Q;
  for (size_t i0 = tid; i0 < nvec; i0 += stride * kUnroll) {
    float4 s[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(s[u].x), "=f"(s[u].y), "=f"(s[u].z), "=f"(s[u].w)
                     : "l"(mc_stage + lo + 4 * i)
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
        float4 m;
        m.x = __fdiv_rn(s[u].x, fq);
        m.y = __fdiv_rn(s[u].y, fq);
        m.z = __fdiv_rn(s[u].z, fq);
        m.w = __fdiv_rn(s[u].w, fq);
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(
                         mc_mean + lo + 4 * i),
                     "f"(m.x), "f"(m.y), "f"(m.z), "f"(m.w)
                     : "memory");
      }
    }
  }
  if (blockIdx.x == 0) {
    for (size_t e = 4 * nvec + threadIdx.x; e < n; e += blockDim.x) {
      float sum;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];"
                   : "=f"(sum)
                   : "l"(mc_stage + lo + e)
                   : "memory");
      asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc_mean + lo + e),
                   "f"(__fdiv_rn(sum, fq))
                   : "memory");
    }
  }
}

extern "C" int lpp_nvls_mean_shard(const float* mc_stage, float* mc_mean, size_t lo, size_t hi,
                                   int Q, void* stream) {
  if (!mc_stage || !mc_mean) return set_err(LPP_E_VALUE, "nvls_mean_shard: null pointer");
  if (hi < lo) return set_err(LPP_E_INDEX, "nvls_mean_shard: hi < lo");
  if (lo & 3u) return set_err(LPP_E_VALUE, "nvls_mean_shard: shard start must be a multiple of 4");
  if (Q < 1) return set_err(LPP_E_VALUE, "nvls_mean_shard: Q < 1");
  size_t n = hi - lo;
  if (n == 0) return LPP_OK;
  size_t nvec = n / 4;
  k_nvls_mean<<<grid_for(nvec ? nvec : 1, current_sms()), kThreads, 0, (cudaStream_t)stream>>>(
      mc_stage, mc_mean, lo, n, nvec, Q);
  LAUNCH_CHECK("nvls_mean_shard");
  return LPP_OK;
}

// local: x[e] += mean[e] - stage[e] (element-atomic), then the round's tag
__global__ void __launch_bounds__(kThreads)
    k_nvls_apply(float* x, const float* __restrict__ stage, const float* __restrict__ mean,
                 size_t n, size_t nvec, int* tags, int stamp) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (size_t i = tid; i < nvec; i += stride) {
    float4 s = __ldcg(reinterpret_cast<const float4*>(stage) + i);
    float4 m = __ldcg(reinterpret_cast<const float4*>(mean) + i);
    float4 c;
    c.x = __fsub_rn(m.x, s.x);
    c.y = __fsub_rn(m.y, s.y);
    c.z = __fsub_rn(m.z, s.z);
    c.w = __fsub_rn(m.w, s.w);
    red_add_v4(x + 4 * i, c);
    if (tags) {
      fence_ar_gpu();
      st_tag4(tags + 4 * i, stamp);
    }
  }
  if (blockIdx.x == 0) {
    for (size_t e = 4 * nvec + threadIdx.x; e < n; e += blockDim.x) {
      red_add_f32(x + e, __fsub_rn(ld_cg(mean + e), ld_cg(stage + e)));
      if (tags) {
        fence_ar_gpu();
        st_tag(tags + e, stamp);
      }
    }
  }
}

extern "C" int lpp_nvls_apply(float* x, const float* stage, const float* mean, size_t n,
                              int32_t* tags, int32_t stamp, void* stream) {
  if (n == 0) return LPP_OK;
  if (!x || !stage || !mean) return set_err(LPP_E_VALUE, "nvls_apply: null pointer");
  if ((((uintptr_t)x) | ((uintptr_t)stage) | ((uintptr_t)mean) | (tags ? (uintptr_t)tags : 0)) &
      15u)
    return set_err(LPP_E_VALUE, "nvls_apply: buffers must be 16-byte aligned");
  size_t nvec = n / 4;
  k_nvls_apply<<<grid_for(nvec ? nvec : 1, current_sms()), kThreads, 0, (cudaStream_t)stream>>>(
      x, stage, mean, n, nvec, tags, stamp);
  LAUNCH_CHECK("nvls_apply");
  return LPP_OK;
}
