// libblasx_cuda.so — the B200 tile engine behind include/blasx_cuda.h.
// Per device: one arena reservation, n compute streams + H2D / D2H / P2P copy streams,
// an event pool, a mapped-pinned singular flag.  See include/blasx_cuda.h for the seam
// each entry point replaces in the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/blasx_cuda.h"
#include <unordered_map>

#include "bx_gemm_dmma.cuh"
#include "bx_sgemm_tc.cuh"
#include "bx_trsm.cuh"

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CUDA_TRY(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      return set_err(BX_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " (" +     \
                                   std::to_string((int)e_) + ")");                           \
  } while (0)

constexpr int kMaxCompute = 16;
constexpr int kEvShift = 20;

// Per-device event pool.  Lookups (every wait/record/query) are lock-free: events live in
// fixed chunks published before `count`, so the per-GPU threads of concurrent mode never
// serialise on a global lock; only creation and release take the pool's own mutex.
struct EventPool {
  static constexpr int kChunk = 4096, kChunks = (1 << kEvShift) / kChunk;
  std::mutex mu;
  std::atomic<cudaEvent_t*> chunk[kChunks] = {};
  std::atomic<int> count{0};
  std::vector<uint8_t> timing;  // guarded by mu
  std::vector<uint8_t> in_use;  // guarded by mu: a double release would hand one event to two owners
  std::vector<int> free_sync, free_timing;
  ~EventPool() {
    for (auto& c : chunk) delete[] c.load();
  }
  bool lookup(int idx, cudaEvent_t* e) const {
    if (idx < 0 || idx >= count.load(std::memory_order_acquire)) return false;
    *e = chunk[idx / kChunk].load(std::memory_order_acquire)[idx % kChunk];
    return true;
  }
  bool release(int idx) {  // caller holds mu
    if (!in_use[idx]) return false;
    in_use[idx] = 0;
    (timing[idx] ? free_timing : free_sync).push_back(idx);
    return true;
  }
};

struct Device {
  int cuda_id = -1;
  int sms = 0;
  int ncomp = 0;
  cudaStream_t comp[kMaxCompute] = {};
  cudaStream_t h2d = nullptr, d2h = nullptr, p2p = nullptr;
  char* arena = nullptr;
  uint64_t arena_bytes = 0;
  int* flag_host = nullptr;  // mapped pinned
  int* flag_dev = nullptr;
  std::unique_ptr<EventPool> pool;  // id -> event (lock-free lookup)
  std::vector<const void*> attr_set;  // kernels whose smem attribute is set on this device
  bool ready = false;
};

std::mutex g_mu;
std::vector<Device> g_devs;  // index = logical device (order given to bx_init)
std::map<const void*, uint64_t> g_registered;

Device* dev_of(int d) {
  if (d < 0 || d >= (int)g_devs.size() || !g_devs[d].ready) return nullptr;
  return &g_devs[d];
}

cudaStream_t lane_stream(Device* D, int lane) {
  if (lane == BX_LANE_H2D) return D->h2d;
  if (lane == BX_LANE_D2H) return D->d2h;
  if (lane == BX_LANE_P2P) return D->p2p;
  if (lane >= 0 && lane < D->ncomp) return D->comp[lane];
  return nullptr;
}

int ev_get(int d, bool timing, cudaEvent_t* ev, int* id) {
  EventPool& P = *g_devs[d].pool;
  Device* D = &g_devs[d];
  std::lock_guard<std::mutex> lk(P.mu);
  auto& fl = timing ? P.free_timing : P.free_sync;
  int idx;
  if (!fl.empty()) {
    idx = fl.back();
    fl.pop_back();
    P.in_use[idx] = 1;
    P.lookup(idx, ev);
  } else {
    idx = P.count.load(std::memory_order_relaxed);
    if (idx >= (1 << kEvShift)) return set_err(BX_ENOMEM, "event pool exhausted");
    // events belong to the device current at creation: create on this slot's device
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != D->cuda_id) cudaSetDevice(D->cuda_id);
    cudaEvent_t e;
    cudaError_t err = cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
    if (cur != D->cuda_id && cur >= 0) cudaSetDevice(cur);
    if (err != cudaSuccess) return set_err(BX_ECUDA, std::string("cudaEventCreate: ") + cudaGetErrorString(err));
    cudaEvent_t* c = P.chunk[idx / EventPool::kChunk].load(std::memory_order_relaxed);
    if (!c) {
      c = new cudaEvent_t[EventPool::kChunk]();
      P.chunk[idx / EventPool::kChunk].store(c, std::memory_order_release);
    }
    c[idx % EventPool::kChunk] = e;
    P.timing.push_back(timing ? 1 : 0);
    P.in_use.push_back(1);
    P.count.store(idx + 1, std::memory_order_release);
    *ev = e;
  }
  *id = (d << kEvShift) | idx;
  return BX_OK;
}

bool ev_lookup(int id, cudaEvent_t* ev, int* d_out = nullptr) {
  if (id < 0) return false;
  int d = id >> kEvShift, idx = id & ((1 << kEvShift) - 1);
  if (d >= (int)g_devs.size() || !g_devs[d].pool) return false;
  if (!g_devs[d].pool->lookup(idx, ev)) return false;
  if (d_out) *d_out = d;
  return true;
}

int wait_all(cudaStream_t s, int n, const int* wait) {
  for (int i = 0; i < n; ++i) {
    cudaEvent_t e;
    if (!ev_lookup(wait[i], &e)) return set_err(BX_EINVAL, "bad wait event id " + std::to_string(wait[i]));
    CUDA_TRY(cudaStreamWaitEvent(s, e, 0));
  }
  return BX_OK;
}

int finish(int d, cudaStream_t s, int* ev_out) {
  if (!ev_out) return BX_OK;
  cudaEvent_t e;
  int id;
  int rc = ev_get(d, false, &e, &id);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(e, s));
  *ev_out = id;
  return BX_OK;
}

// ---- kernel launchers (raw pointers) ---------------------------------------------------

int current_dev_slot() {
  int id = -1;
  cudaGetDevice(&id);
  for (size_t i = 0; i < g_devs.size(); ++i)
    if (g_devs[i].ready && g_devs[i].cuda_id == id) return (int)i;
  return -1;
}

// cudaFuncSetAttribute is per device: remember which kernels were configured where.
bool need_attr(const void* kernel) {
  int d = current_dev_slot();
  if (d < 0) return true;
  auto& v = g_devs[d].attr_set;
  for (const void* k : v)
    if (k == kernel) return false;
  v.push_back(kernel);
  return true;
}

int g_gemm_variant = 0;  // tuning knob (bx_set_gemm_variant); 0 = default
int g_gemm_group = 8;    // raster group (m-tiles) of the FP64 task GEMM grid
int g_trsm_rhs = 32;     // right-hand sides per CTA of the TRSM panel kernel (8/16/32/64)
int g_trsm_leaf = 256;   // triangle order solved by a leaf kernel; larger ones recurse

template <class Cfg, bool TA, bool TB>
int launch_gemm_cfg(const bx::GemmTask& t, cudaStream_t s) {
  if (need_attr((const void*)bx::gemm_task_kernel<Cfg, TA, TB>)) {
    CUDA_TRY(cudaFuncSetAttribute(bx::gemm_task_kernel<Cfg, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Cfg::SMEM_BYTES));
  }
  int tiles = ((t.h + Cfg::BM - 1) / Cfg::BM) * ((t.w + Cfg::BN - 1) / Cfg::BN);
  bx::gemm_task_kernel<Cfg, TA, TB><<<tiles, Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(t);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return BX_OK;
}

template <class Cfg, bool TA, bool TB, bool KM>
int launch_gemm_ws_km(const bx::GemmTask& t, cudaStream_t s) {
  if (need_attr((const void*)bx::gemm_task_mb_kernel<Cfg, TA, TB, KM>)) {
    CUDA_TRY(cudaFuncSetAttribute(bx::gemm_task_mb_kernel<Cfg, TA, TB, KM>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
  }
  int tiles = ((t.h + Cfg::BM - 1) / Cfg::BM) * ((t.w + Cfg::BN - 1) / Cfg::BN);
  bx::gemm_task_mb_kernel<Cfg, TA, TB, KM><<<tiles, Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(t);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return BX_OK;
}

template <class Cfg, bool TA, bool TB>
int launch_gemm_ws(const bx::GemmTask& t, cudaStream_t s) {
  for (int i = 0; i < t.nsteps; ++i)
    if (t.steps[i].kmode != bx::KM_NONE) return launch_gemm_ws_km<Cfg, TA, TB, true>(t, s);
  return launch_gemm_ws_km<Cfg, TA, TB, false>(t, s);
}

template <bool TA, bool TB>
int launch_gemm_t(const bx::GemmTask& t, cudaStream_t s) {
  switch (g_gemm_variant) {
    case 1: return launch_gemm_cfg<bx::CfgWide, TA, TB>(t, s);
    case 2: return launch_gemm_cfg<bx::CfgDeep, TA, TB>(t, s);
    case 3: return launch_gemm_ws<bx::CfgMb2, TA, TB>(t, s);
    case 5: return launch_gemm_ws<bx::CfgMbPair, TA, TB>(t, s);
    case 6: return launch_gemm_ws<bx::CfgMbK32, TA, TB>(t, s);
    case 7: return launch_gemm_ws<bx::CfgMbS0, TA, TB>(t, s);
    case 9: return launch_gemm_ws<bx::CfgMb, TA, TB>(t, s);      // 8 warps of 64x32
    case 10: return launch_gemm_ws<bx::CfgMb16S0, TA, TB>(t, s);
    case 11: return launch_gemm_ws<bx::CfgMb16S2, TA, TB>(t, s);
    case 12: return launch_gemm_ws<bx::CfgMb16K32, TA, TB>(t, s);
    case 13: return launch_gemm_ws<bx::CfgMb16x64, TA, TB>(t, s);
    case 99: return launch_gemm_ws<bx::CfgMbNoLoad, TA, TB>(t, s);
    default: return launch_gemm_ws<bx::CfgMb16, TA, TB>(t, s);   // 16 warps of 32x32
  }
}

int launch_gemm(int ta, int tb, const bx::GemmTask& t, cudaStream_t s) {
  if (t.h <= 0 || t.w <= 0) return BX_OK;
  if (ta) return tb ? launch_gemm_t<true, true>(t, s) : launch_gemm_t<true, false>(t, s);
  return tb ? launch_gemm_t<false, true>(t, s) : launch_gemm_t<false, false>(t, s);
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// ---- TMA tensor maps (driver entry point fetched at run time: no -lcuda) --------------

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled g_encode = nullptr;

struct MapKey {
  uint64_t ptr, rows, cols, ld;
  uint32_t box0, box1, swz;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box0 == o.box0 && box1 == o.box1 &&
           swz == o.swz;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<uint64_t>()(k.ptr ^ (k.rows * 0x9E3779B97F4A7C15ull) ^ (k.cols << 20) ^ (k.ld << 40) ^
                                 ((uint64_t)k.box0 << 8) ^ ((uint64_t)k.box1 << 16) ^ ((uint64_t)k.swz << 4));
  }
};
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// 2-d fp32 column-major matrix (rows contiguous, leading dimension ld elements) -> tensor
// map with a {box0 (rows), box1 (cols)} box, 128-B swizzle, zero fill out of bounds.
int tensor_map_2d(const void* base, bool f64, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box0,
                  uint32_t box1, CUtensorMapSwizzle swz, CUtensorMap* out);
int tensor_map_f32(const float* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box0, uint32_t box1,
                   CUtensorMapSwizzle swz, CUtensorMap* out) {
  return tensor_map_2d(base, false, rows, cols, ld, box0, box1, swz, out);
}
int tensor_map_2d(const void* base, bool f64, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box0,
                  uint32_t box1, CUtensorMapSwizzle swz, CUtensorMap* out) {
  MapKey key{(uint64_t)base, rows, cols, ld, box0, box1, (uint32_t)swz | (f64 ? 0x100u : 0u)};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) { *out = it->second; return BX_OK; }
  }
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return set_err(BX_ECUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = (PFN_encodeTiled)fn;
  }
  cuuint64_t dims[2] = {rows, cols};
  cuuint64_t strides[1] = {ld * (f64 ? 8 : 4)};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  CUresult r = g_encode(&m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base,
                        dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(BX_EINVAL, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_maps.size() > 65536) g_maps.clear();
  g_maps[key] = m;
  *out = m;
  return BX_OK;
}

// MN-major fp32 operand (rows contiguous, rows % 32 == 0) as a 3-d tensor {32, cols, rows/32}
// with strides {ld, 32} elements, so ONE box {32, box_k, groups} stages `groups` 32-wide
// MN groups 4 KB apart — the layout the UMMA MN-major descriptor expects (LBO = 4 KB).
int tensor_map_f32_mn3d(const float* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_k,
                        uint32_t groups, CUtensorMap* out) {
  MapKey key{(uint64_t)base, rows, cols, ld, box_k, groups | 0x10000u, 0xF3u};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) { *out = it->second; return BX_OK; }
  }
  if (!g_encode) {
    CUtensorMap dummy;
    int rc = tensor_map_f32(base, rows, cols, ld, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, &dummy);
    if (rc) return rc;
  }
  cuuint64_t dims[3] = {32, cols, rows / 32};
  cuuint64_t strides[2] = {ld * 4, 128};
  cuuint32_t box[3] = {32, box_k, groups};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(BX_EINVAL, "cuTensorMapEncodeTiled (3-d) failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_maps.size() > 65536) g_maps.clear();
  g_maps[key] = m;
  *out = m;
  return BX_OK;
}

int g_sgemm_variant = 3;   // 0: 1-SM 128x256 tile, 1: 2-SM pair 256x256 tile,
                           // 2: persistent 2-SM with double-buffered TMEM accumulators
                           // (static round robin), 3: the same with cluster launch control
                           // (default: 98 % tensor pipe, profiles/sgemm_clc_r02.txt)
int g_sm_pairs = 74;       // clusters of the persistent SGEMM (one per TPC of a B200)
int g_sgemm_group = 0;     // persistent SGEMM raster group (m-tiles); 0 = kernel default
int g_sgemm_mn3d = 1;      // MN-major operands by one 3-d TMA box when the extent allows
int g_sgemm_debug = 0;     // diagnostic ablation bits (SgemmTask::dbg)

// fp32 task GEMM on tcgen05 (TF32 inputs, fp32 accumulation in TMEM)
int g_sgemm_precise = 0;   // 1: 3xTF32 split products (~fp32 accuracy, a third of the rate)

int sgemm_tf32(cudaStream_t s, int ta, int tb, int h, int w, int nsteps, const float* const* a, const int* lda,
               const float* const* b, const int* ldb, const int* depth, float alpha, float beta, float* c, int ldc);

// precise mode: per step, split op(A_s) and op(B_s) storage into TF32 hi/lo copies (stream-
// ordered scratch) and accumulate hi*hi + hi*lo + lo*hi with the TF32 kernels
int sgemm_precise(cudaStream_t s, int ta, int tb, int h, int w, int nsteps, const float* const* a, const int* lda,
                  const float* const* b, const int* ldb, const int* depth, float alpha, float beta, float* c,
                  int ldc) {
  for (int i = 0; i < nsteps; ++i) {
    const int d = depth[i];
    const int ar = ta ? d : h, ac = ta ? h : d;       // stored extents of A_s
    const int br = tb ? w : d, bc = tb ? d : w;       // stored extents of B_s
    const int lda4 = (ar + 3) & ~3, ldb4 = (br + 3) & ~3;
    const size_t abytes = (size_t)lda4 * ac * 4, bbytes = (size_t)ldb4 * bc * 4;
    void* buf = nullptr;
    CUDA_TRY(cudaMallocAsync(&buf, 2 * abytes + 2 * bbytes + 64, s));
    float* ahi = (float*)buf;
    float* alo = (float*)((char*)buf + abytes);
    float* bhi = (float*)((char*)buf + 2 * abytes);
    float* blo = (float*)((char*)buf + 2 * abytes + bbytes);
    dim3 blk(32, 8);
    bx::tf32_split_kernel<<<dim3((ar + 31) / 32, (ac + 7) / 8), blk, 0, s>>>(a[i], lda[i], ar, ac, ahi, alo, lda4);
    bx::tf32_split_kernel<<<dim3((br + 31) / 32, (bc + 7) / 8), blk, 0, s>>>(b[i], ldb[i], br, bc, bhi, blo, ldb4);
    g_launches += 2;
    CUDA_TRY(cudaGetLastError());
    const float* ap[3] = {ahi, ahi, alo};
    const float* bp[3] = {bhi, blo, bhi};
    int la[3] = {lda4, lda4, lda4}, lb[3] = {ldb4, ldb4, ldb4}, dd[3] = {d, d, d};
    // one 3-step launch: hi*hi + hi*lo + lo*hi (C read once, beta only on the first step)
    int rc = sgemm_tf32(s, ta, tb, h, w, 3, ap, la, bp, lb, dd, alpha, i == 0 ? beta : 1.0f, c, ldc);
    CUDA_TRY(cudaFreeAsync(buf, s));
    if (rc) return rc;
  }
  return BX_OK;
}

int sgemm_raw(cudaStream_t s, int ta, int tb, int h, int w, int nsteps, const float* const* a, const int* lda,
              const float* const* b, const int* ldb, const int* depth, float alpha, float beta, float* c, int ldc) {
  if (h <= 0 || w <= 0) return BX_OK;
  if (ldc < h) return set_err(BX_EINVAL, "sgemm: ldc < h");
  if (g_sgemm_precise && nsteps > 0)
    return sgemm_precise(s, ta, tb, h, w, nsteps, a, lda, b, ldb, depth, alpha, beta, c, ldc);
  return sgemm_tf32(s, ta, tb, h, w, nsteps, a, lda, b, ldb, depth, alpha, beta, c, ldc);
}

// fp32 task GEMM on tcgen05.mma.kind::tf32 (the kernels above)
int sgemm_tf32(cudaStream_t s, int ta, int tb, int h, int w, int nsteps, const float* const* a, const int* lda,
               const float* const* b, const int* ldb, const int* depth, float alpha, float beta, float* c, int ldc) {
  for (int s0 = 0; s0 < (nsteps > 0 ? nsteps : 1); s0 += bx::S_MAX_STEPS) {
    bx::SgemmTask t;
    memset(&t, 0, sizeof(t));
    int n = nsteps - s0 < bx::S_MAX_STEPS ? nsteps - s0 : bx::S_MAX_STEPS;
    if (n < 0) n = 0;
    t.c = c; t.ldc = ldc; t.h = h; t.w = w; t.nsteps = n; t.ta = ta; t.tb = tb;
    t.alpha = alpha;
    t.beta = (s0 == 0) ? beta : 1.0f;
    t.mn_lbo = 4096;   // MN-major: 32-wide MN groups (one TMA box) 4 KB apart
    t.mn_sbo = 512;    //           4-row k groups of the 128B_BASE32B atom
    t.dbg = g_sgemm_debug;
    t.group_m = g_sgemm_group;
    t.a3d = g_sgemm_mn3d && !ta && (h % 32) == 0;
    t.b3d = g_sgemm_mn3d && tb && (w % 32) == 0;
    for (int i = 0; i < n; ++i) {
      const int j = s0 + i, d = depth[j];
      if ((lda[j] & 3) || (ldb[j] & 3) || !aligned16(a[j]) || !aligned16(b[j]))
        return set_err(BX_EINVAL, "sgemm: operands must be 16-byte aligned with leading dimensions multiple of 4");
      t.steps[i].d = d;
      int rc;
      // A: untransposed M x K (MN-major boxes 32x32), transposed K x M (K-major box 32 x 128)
      const CUtensorMapSwizzle MN = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, KM = CU_TENSOR_MAP_SWIZZLE_128B;
      const uint32_t a_groups = g_sgemm_variant >= 1 ? 4u : (uint32_t)(bx::S_BM / 32);
      const uint32_t b_groups = g_sgemm_variant >= 1 ? 4u : (uint32_t)(bx::S_BN / 32);
      if (!ta && t.a3d) rc = tensor_map_f32_mn3d(a[j], h, d, lda[j], 32, a_groups, &t.steps[i].map_a);
      else if (!ta) rc = tensor_map_f32(a[j], h, d, lda[j], 32, 32, MN, &t.steps[i].map_a);
      else rc = tensor_map_f32(a[j], d, h, lda[j], bx::S_BK, bx::S_BM, KM, &t.steps[i].map_a);
      if (rc) return rc;
      // B: untransposed K x N (K-major box 32 x BN per CTA), transposed N x K (MN boxes 32x32)
      const uint32_t bn_box = g_sgemm_variant >= 1 ? 128u : (uint32_t)bx::S_BN;
      if (!tb) rc = tensor_map_f32(b[j], d, w, ldb[j], bx::S_BK, bn_box, KM, &t.steps[i].map_b);
      else if (t.b3d) rc = tensor_map_f32_mn3d(b[j], w, d, ldb[j], 32, b_groups, &t.steps[i].map_b);
      else rc = tensor_map_f32(b[j], w, d, ldb[j], 32, 32, MN, &t.steps[i].map_b);
      if (rc) return rc;
    }
    if (g_sgemm_variant == 2) {
      void (*k3)(bx::SgemmTask) = ta ? (tb ? bx::sgemm_tc2p_kernel<1, 1> : bx::sgemm_tc2p_kernel<1, 0>)
                                     : (tb ? bx::sgemm_tc2p_kernel<0, 1> : bx::sgemm_tc2p_kernel<0, 0>);
      if (need_attr((const void*)k3)) {
        CUDA_TRY(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, bx::P_SMEM_BYTES));
      }
      const int pair_tiles = ((h + bx::P_BM - 1) / bx::P_BM) * ((w + bx::P_BN - 1) / bx::P_BN);
      const int clusters = pair_tiles < g_sm_pairs ? pair_tiles : g_sm_pairs;
      k3<<<2 * clusters, bx::P_THREADS, bx::P_SMEM_BYTES, s>>>(t);
      g_launches++;
      CUDA_TRY(cudaGetLastError());
      if (nsteps <= 0) break;
      continue;
    }
    if (g_sgemm_variant == 3) {
      void (*k4)(bx::SgemmTask) = ta ? (tb ? bx::sgemm_tc2c_kernel<1, 1> : bx::sgemm_tc2c_kernel<1, 0>)
                                     : (tb ? bx::sgemm_tc2c_kernel<0, 1> : bx::sgemm_tc2c_kernel<0, 0>);
      if (need_attr((const void*)k4)) {
        CUDA_TRY(cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, bx::P_SMEM_BYTES));
      }
      int pairs = ((h + bx::P_BM - 1) / bx::P_BM) * ((w + bx::P_BN - 1) / bx::P_BN);
      k4<<<2 * pairs, bx::C_THREADS, bx::P_SMEM_BYTES, s>>>(t);
      g_launches++;
      CUDA_TRY(cudaGetLastError());
      if (nsteps <= 0) break;
      continue;
    }
    if (g_sgemm_variant == 1) {
      void (*k2)(bx::SgemmTask) = ta ? (tb ? bx::sgemm_tc2_kernel<1, 1> : bx::sgemm_tc2_kernel<1, 0>)
                                     : (tb ? bx::sgemm_tc2_kernel<0, 1> : bx::sgemm_tc2_kernel<0, 0>);
      if (need_attr((const void*)k2)) {
        CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, bx::P_SMEM_BYTES));
      }
      int pairs = ((h + bx::P_BM - 1) / bx::P_BM) * ((w + bx::P_BN - 1) / bx::P_BN);
      k2<<<2 * pairs, bx::P_THREADS, bx::P_SMEM_BYTES, s>>>(t);
      g_launches++;
      CUDA_TRY(cudaGetLastError());
      if (nsteps <= 0) break;
      continue;
    }
    int tiles = ((h + bx::S_BM - 1) / bx::S_BM) * ((w + bx::S_BN - 1) / bx::S_BN);
    void (*kern)(bx::SgemmTask) = ta ? (tb ? bx::sgemm_tc_kernel<1, 1> : bx::sgemm_tc_kernel<1, 0>)
                                     : (tb ? bx::sgemm_tc_kernel<0, 1> : bx::sgemm_tc_kernel<0, 0>);
    if (need_attr((const void*)kern)) {
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bx::S_SMEM_BYTES));
    }
    kern<<<tiles, bx::S_THREADS, bx::S_SMEM_BYTES, s>>>(t);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    if (nsteps <= 0) break;
  }
  return BX_OK;
}

// General gemm over raw pointers, splitting step lists longer than G_MAX_STEPS into
// several launches (later launches accumulate with beta = 1).
// FP64 task GEMM fed by TMA (bx::gemm_task_tma_kernel): tensor maps per step operand,
// cached by (pointer, extents, ld); steps beyond T_MAX_STEPS go to further launches.
int gemm_tma(cudaStream_t s, int ta, int tb, int tri, int h, int w, int nsteps, const double* const* a,
             const int* lda, const double* const* b, const int* ldb, const int* depth, double alpha,
             double beta, double* c, int ldc) {
  const CUtensorMapSwizzle SW = CU_TENSOR_MAP_SWIZZLE_128B;
  for (int s0 = 0; s0 < nsteps; s0 += bx::T_MAX_STEPS) {
    bx::GemmTmaTask t;
    memset(&t, 0, sizeof(t));
    t.c = c; t.ldc = ldc; t.h = h; t.w = w; t.tri = tri; t.group_m = g_gemm_group;
    t.alpha = alpha;
    t.beta = (s0 == 0) ? beta : 1.0;
    const int n = nsteps - s0 < bx::T_MAX_STEPS ? nsteps - s0 : bx::T_MAX_STEPS;
    t.nsteps = n;
    for (int i = 0; i < n; ++i) {
      const int j = s0 + i, d = depth[j];
      t.steps[i].d = d;
      int rc = ta ? tensor_map_2d(a[j], true, d, h, lda[j], bx::T_BK, bx::T_BM, SW, &t.steps[i].ma)
                  : tensor_map_2d(a[j], true, h, d, lda[j], 16, bx::T_BK, SW, &t.steps[i].ma);
      if (rc) return rc;
      rc = tb ? tensor_map_2d(b[j], true, w, d, ldb[j], 16, bx::T_BK, SW, &t.steps[i].mb)
              : tensor_map_2d(b[j], true, d, w, ldb[j], bx::T_BK, bx::T_BN, SW, &t.steps[i].mb);
      if (rc) return rc;
    }
    void (*k)(bx::GemmTmaTask) = ta ? (tb ? bx::gemm_task_tma_kernel<true, true> : bx::gemm_task_tma_kernel<true, false>)
                                    : (tb ? bx::gemm_task_tma_kernel<false, true> : bx::gemm_task_tma_kernel<false, false>);
    if (need_attr((const void*)k)) {
      CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bx::T_SMEM_BYTES));
    }
    const int tiles = ((h + bx::T_BM - 1) / bx::T_BM) * ((w + bx::T_BN - 1) / bx::T_BN);
    k<<<tiles, bx::T_THREADS_G, bx::T_SMEM_BYTES, s>>>(t);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
  }
  return BX_OK;
}

int gemm_raw(cudaStream_t s, int ta, int tb, int tri, int h, int w, int nsteps, const double* const* a,
             const int* lda, const double* const* b, const int* ldb, const int* depth, double alpha,
             double beta, double* c, int ldc, const int* kmode = nullptr) {
  if (h < 0 || w < 0 || nsteps < 0) return set_err(BX_EINVAL, "gemm: negative extent");
  if (ldc < (h > 1 ? h : 1)) return set_err(BX_EINVAL, "gemm: ldc < h");
  for (int i = 0; i < nsteps; ++i) {
    if (depth[i] < 0) return set_err(BX_EINVAL, "gemm: negative depth");
    int need_a = ta ? depth[i] : h, need_b = tb ? w : depth[i];
    if (lda[i] < (need_a > 1 ? need_a : 1) || ldb[i] < (need_b > 1 ? need_b : 1))
      return set_err(BX_EINVAL, "gemm: leading dimension too small");
    if ((lda[i] & 1) || (ldb[i] & 1) || !aligned16(a[i]) || !aligned16(b[i]))
      return set_err(BX_EINVAL, "gemm: operands must be 16-byte aligned with even leading dimensions");
  }
  if (nsteps == 0) {
    // C = beta*C (beta==0 -> zero) — expressed as a zero-depth task
    bx::GemmTask t{};
    t.c = c; t.ldc = ldc; t.h = h; t.w = w; t.nsteps = 0; t.tri = tri; t.group_m = g_gemm_group;
    t.alpha = alpha; t.beta = beta;
    return launch_gemm(ta, tb, t, s);
  }
  if (g_gemm_variant == 8) return gemm_tma(s, ta, tb, tri, h, w, nsteps, a, lda, b, ldb, depth, alpha, beta, c, ldc);
  for (int s0 = 0; s0 < nsteps; s0 += bx::G_MAX_STEPS) {
    bx::GemmTask t{};
    t.c = c; t.ldc = ldc; t.h = h; t.w = w; t.tri = tri; t.group_m = g_gemm_group;
    t.alpha = alpha;
    t.beta = (s0 == 0) ? beta : 1.0;
    int n = nsteps - s0 < bx::G_MAX_STEPS ? nsteps - s0 : bx::G_MAX_STEPS;
    t.nsteps = n;
    for (int i = 0; i < n; ++i) {
      t.steps[i].a = a[s0 + i]; t.steps[i].b = b[s0 + i];
      t.steps[i].lda = lda[s0 + i]; t.steps[i].ldb = ldb[s0 + i]; t.steps[i].d = depth[s0 + i];
      t.steps[i].kmode = kmode ? kmode[s0 + i] : bx::KM_NONE;
    }
    int rc = launch_gemm(ta, tb, t, s);
    if (rc) return rc;
  }
  return BX_OK;
}

int scale_raw(cudaStream_t s, double* b, int ld, int h, int w, double alpha) {
  dim3 blk(32, 8), grd((h + 31) / 32, (w + 7) / 8);
  bx::scale_kernel<<<grd, blk, 0, s>>>(b, ld, h, w, alpha);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return BX_OK;
}

template <int NR>
int launch_panel(cudaStream_t s, const bx::TrsmArgs& t) {
  constexpr int YP = bx::PanelCfg<NR>::YP;
  size_t smem = (size_t)t.n * YP * sizeof(double);
  if (smem > 200 * 1024) return set_err(BX_EINVAL, "trsm panel: triangle too large for this RHS width");
  if (need_attr((const void*)bx::trsm_panel_kernel<NR>)) {
    CUDA_TRY(cudaFuncSetAttribute(bx::trsm_panel_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
  }
  int grid = (t.nrhs + NR - 1) / NR;
  bx::trsm_panel_kernel<NR><<<grid, bx::T_THREADS, smem, s>>>(t);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return BX_OK;
}

int trsm_leaf(cudaStream_t s, int right, int eff_upper, int trans, int unit, int h, int w, double alpha,
              const double* a, int lda, double* b, int ldb, int* flag) {
  bx::TrsmArgs t{};
  t.a = a; t.b = b; t.lda = lda; t.ldb = ldb;
  t.n = right ? w : h;
  t.nrhs = right ? h : w;
  t.swap = (trans != 0) != (right != 0);
  t.rev = right ? !eff_upper : eff_upper;
  t.right = right; t.unit = unit; t.alpha = alpha; t.flag = flag;
  if (t.n == 0 || t.nrhs == 0) return BX_OK;
  if (t.n <= bx::LEAF_N) {
    int per_cta = bx::LEAF_RHS * bx::LEAF_WARPS;
    bx::trsm_leaf_kernel<<<(t.nrhs + per_cta - 1) / per_cta, bx::LEAF_WARPS * 32, 0, s>>>(t);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return BX_OK;
  }
  // the widest panel not above the knob whose Y block fits in shared memory
  int nr = g_trsm_rhs;
  while (nr > 8 && (size_t)t.n * (nr + 4) * sizeof(double) > 200 * 1024) nr /= 2;
  switch (nr) {
    case 8: { int rc = launch_panel<8>(s, t); if (rc) return rc; break; }
    case 32: { int rc = launch_panel<32>(s, t); if (rc) return rc; break; }
    case 64: { int rc = launch_panel<64>(s, t); if (rc) return rc; break; }
    default: { int rc = launch_panel<16>(s, t); if (rc) return rc; break; }
  }
  return BX_OK;
}

// Recursive blocked solve in physical coordinates (E = op(A) is eff_upper/lower); leaves of
// order <= leaf_max run the panel kernel, the off-diagonal updates run the DMMA task GEMM.
int trsm_rec(cudaStream_t s, int right, int eff_upper, int trans, int unit, int h, int w, double alpha,
             const double* a, int lda, double* b, int ldb, int* flag, int leaf_max) {
  int n = right ? w : h;
  if (n <= leaf_max) return trsm_leaf(s, right, eff_upper, trans, unit, h, w, alpha, a, lda, b, ldb, flag);
  if (alpha != 1.0) {
    int rc = scale_raw(s, b, ldb, h, w, alpha);
    if (rc) return rc;
    alpha = 1.0;
  }
  // split on a multiple of the leaf order so every leaf is full except the last
  int n1 = ((n / 2) + leaf_max - 1) / leaf_max * leaf_max, n2 = n - n1;
  if (n1 >= n) n1 = n - leaf_max;
  // E block (r0, c0, rows, cols) -> A pointer + transpose flag
  auto eblk = [&](int r0, int c0) -> const double* {
    return trans ? a + (size_t)r0 * lda + c0 : a + (size_t)c0 * lda + r0;
  };
  const double* e11 = eblk(0, 0);
  const double* e22 = eblk(n1, n1);
  int rc;
  if (!right) {
    double* b1 = b;
    double* b2 = b + n1;
    if (!eff_upper) {
      if ((rc = trsm_rec(s, 0, 0, trans, unit, n1, w, 1.0, e11, lda, b1, ldb, flag, leaf_max))) return rc;
      const double* e21 = eblk(n1, 0);
      int d = n1;
      if ((rc = gemm_raw(s, trans, 0, 0, n2, w, 1, &e21, &lda, (const double* const*)&b1, &ldb, &d, -1.0, 1.0, b2, ldb))) return rc;
      return trsm_rec(s, 0, 0, trans, unit, n2, w, 1.0, e22, lda, b2, ldb, flag, leaf_max);
    }
    if ((rc = trsm_rec(s, 0, 1, trans, unit, n2, w, 1.0, e22, lda, b2, ldb, flag, leaf_max))) return rc;
    const double* e12 = eblk(0, n1);
    int d = n2;
    if ((rc = gemm_raw(s, trans, 0, 0, n1, w, 1, &e12, &lda, (const double* const*)&b2, &ldb, &d, -1.0, 1.0, b1, ldb))) return rc;
    return trsm_rec(s, 0, 1, trans, unit, n1, w, 1.0, e11, lda, b1, ldb, flag, leaf_max);
  }
  double* b1 = b;
  double* b2 = b + (size_t)n1 * ldb;
  if (eff_upper) {
    if ((rc = trsm_rec(s, 1, 1, trans, unit, h, n1, 1.0, e11, lda, b1, ldb, flag, leaf_max))) return rc;
    const double* e12 = eblk(0, n1);
    int d = n1;
    if ((rc = gemm_raw(s, 0, trans, 0, h, n2, 1, (const double* const*)&b1, &ldb, &e12, &lda, &d, -1.0, 1.0, b2, ldb))) return rc;
    return trsm_rec(s, 1, 1, trans, unit, h, n2, 1.0, e22, lda, b2, ldb, flag, leaf_max);
  }
  if ((rc = trsm_rec(s, 1, 0, trans, unit, h, n2, 1.0, e22, lda, b2, ldb, flag, leaf_max))) return rc;
  const double* e21 = eblk(n1, 0);
  int d = n2;
  if ((rc = gemm_raw(s, 0, trans, 0, h, n1, 1, (const double* const*)&b2, &ldb, &e21, &lda, &d, -1.0, 1.0, b1, ldb))) return rc;
  return trsm_rec(s, 1, 0, trans, unit, h, n1, 1.0, e11, lda, b1, ldb, flag, leaf_max);
}

__global__ void identity_kernel(double* __restrict__ p, int ld, int n) {
  const int r = blockIdx.x * 32 + threadIdx.x, c = blockIdx.y * 8 + threadIdx.y;
  if (r < n && c < n) p[(size_t)c * ld + r] = (r == c) ? 1.0 : 0.0;
}

__global__ void fill_uniform_f32_kernel(float* p, uint64_t n, uint64_t seed) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = (float)((double)(z >> 40) * (2.0 / 16777216.0) - 1.0);
  }
}

__global__ void fill_uniform_kernel(double* p, uint64_t n, uint64_t seed) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

__global__ void dmma_probe_kernel(double* out, int iters) {
  double acc[8][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) bx::dmma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

}  // namespace

extern "C" {

int bx_version(void) { return 1; }

int bx_last_error(char* buf, int len) {
  if (buf && len > 0) {
    std::strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return BX_OK;
}

int bx_launch_count(uint64_t* n) {
  *n = g_launches.load();
  return BX_OK;
}

int bx_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) { *n = 0; return set_err(BX_ECUDA, cudaGetErrorString(e)); }
  *n = c;
  return BX_OK;
}

int bx_device_info(int dev, char* name, int name_len, int* sms, uint64_t* total_bytes, uint64_t* free_bytes) {
  cudaDeviceProp p;
  CUDA_TRY(cudaGetDeviceProperties(&p, dev));
  if (name && name_len > 0) { std::strncpy(name, p.name, name_len - 1); name[name_len - 1] = 0; }
  if (sms) *sms = p.multiProcessorCount;
  CUDA_TRY(cudaSetDevice(dev));
  size_t fr = 0, tot = 0;
  CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  if (total_bytes) *total_bytes = tot;
  if (free_bytes) *free_bytes = fr;
  return BX_OK;
}

int bx_mem_info(int dev, uint64_t* free_bytes, uint64_t* total_bytes) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  size_t fr = 0, tot = 0;
  CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  *free_bytes = fr;
  *total_bytes = tot;
  return BX_OK;
}

int bx_init(int ndev, const int* device_ids, const uint64_t* arena_bytes, int n_compute) {
  if (ndev <= 0 || n_compute <= 0 || n_compute > kMaxCompute) return set_err(BX_EINVAL, "bx_init: bad ndev/n_compute");
  int count = 0;
  CUDA_TRY(cudaGetDeviceCount(&count));
  if ((int)g_devs.size() < ndev) g_devs.resize(ndev);
  for (int d = 0; d < ndev; ++d) {
    Device& D = g_devs[d];
    int id = device_ids[d];
    if (id < 0 || id >= count) return set_err(BX_EINVAL, "bx_init: no such CUDA device " + std::to_string(id));
    if (D.ready && D.cuda_id != id) return set_err(BX_EINVAL, "bx_init: device slot remapped");
    CUDA_TRY(cudaSetDevice(id));
    if (!D.ready) {
      D.cuda_id = id;
      if (!D.pool) D.pool.reset(new EventPool());
      CUDA_TRY(cudaDeviceGetAttribute(&D.sms, cudaDevAttrMultiProcessorCount, id));
      CUDA_TRY(cudaHostAlloc((void**)&D.flag_host, sizeof(int), cudaHostAllocMapped));
      *D.flag_host = 0;
      CUDA_TRY(cudaHostGetDevicePointer((void**)&D.flag_dev, D.flag_host, 0));
      CUDA_TRY(cudaStreamCreateWithFlags(&D.h2d, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamCreateWithFlags(&D.d2h, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamCreateWithFlags(&D.p2p, cudaStreamNonBlocking));
      D.ready = true;
    }
    for (int s = D.ncomp; s < n_compute; ++s) CUDA_TRY(cudaStreamCreateWithFlags(&D.comp[s], cudaStreamNonBlocking));
    if (n_compute > D.ncomp) D.ncomp = n_compute;
    uint64_t want = arena_bytes ? arena_bytes[d] : 0;
    if (want > D.arena_bytes) {
      if (D.arena) { CUDA_TRY(cudaDeviceSynchronize()); CUDA_TRY(cudaFree(D.arena)); D.arena = nullptr; D.arena_bytes = 0; }
      cudaError_t e = cudaMalloc((void**)&D.arena, want);
      if (e != cudaSuccess) {
        D.arena = nullptr;
        cudaGetLastError();
        return set_err(BX_ENOMEM, "arena cudaMalloc of " + std::to_string(want) + " bytes failed: " + cudaGetErrorString(e));
      }
      D.arena_bytes = want;
    }
  }
  for (int a = 0; a < ndev; ++a)
    for (int b = 0; b < ndev; ++b) {
      if (a == b || g_devs[a].cuda_id == g_devs[b].cuda_id) continue;   // same GPU: no peer link
      int can = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&can, g_devs[a].cuda_id, g_devs[b].cuda_id));
      if (!can) continue;
      CUDA_TRY(cudaSetDevice(g_devs[a].cuda_id));
      cudaError_t e = cudaDeviceEnablePeerAccess(g_devs[b].cuda_id, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return set_err(BX_ECUDA, cudaGetErrorString(e));
      cudaGetLastError();
    }
  return BX_OK;
}

int bx_shutdown(void) {
  for (auto& D : g_devs) {
    if (!D.ready) continue;
    cudaSetDevice(D.cuda_id);
    cudaDeviceSynchronize();
    if (D.pool) {
      cudaEvent_t e;
      for (int i = 0, n = D.pool->count.load(); i < n; ++i)
        if (D.pool->lookup(i, &e)) cudaEventDestroy(e);
    }
    for (int s = 0; s < D.ncomp; ++s) cudaStreamDestroy(D.comp[s]);
    cudaStreamDestroy(D.h2d); cudaStreamDestroy(D.d2h); cudaStreamDestroy(D.p2p);
    if (D.arena) cudaFree(D.arena);
    if (D.flag_host) cudaFreeHost(D.flag_host);
  }
  g_devs.clear();
  return BX_OK;
}

int bx_arena_base(int dev, uint64_t* base) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  *base = (uint64_t)D->arena;
  return BX_OK;
}

int bx_peer_enabled(int a, int b, int* en) {
  Device *A = dev_of(a), *B = dev_of(b);
  if (!A || !B) return set_err(BX_EINVAL, "bad device");
  int can = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can, A->cuda_id, B->cuda_id));
  *en = can;
  return BX_OK;
}

int bx_host_register(void* ptr, uint64_t bytes) {
  if (!ptr || !bytes) return set_err(BX_EINVAL, "register: null");
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_registered.count(ptr)) return BX_OK;
  }
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) { cudaGetLastError(); return BX_OK; }
  if (e != cudaSuccess) { cudaGetLastError(); return set_err(BX_ECUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e)); }
  std::lock_guard<std::mutex> lk(g_mu);
  g_registered[ptr] = bytes;
  return BX_OK;
}

int bx_host_unregister(void* ptr) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_registered.erase(ptr)) return BX_OK;
  }
  CUDA_TRY(cudaHostUnregister(ptr));
  return BX_OK;
}

int bx_host_is_registered(const void* ptr, int* yes) {
  std::lock_guard<std::mutex> lk(g_mu);
  *yes = 0;
  auto it = g_registered.upper_bound(ptr);
  if (it != g_registered.begin()) {
    --it;
    if ((const char*)ptr < (const char*)it->first + it->second) *yes = 1;
  }
  return BX_OK;
}

int bx_h2d_tile(int dev, uint64_t dst_off, int dst_ld, const void* src, int64_t src_ld, int h, int w, int eb,
                int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  if (h <= 0 || w <= 0 || dst_ld < h || src_ld < h) return set_err(BX_EINVAL, "h2d: bad extents");
  if (dst_off + (uint64_t)dst_ld * w * eb > D->arena_bytes) return set_err(BX_EINVAL, "h2d: outside arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(D->h2d, n_wait, wait);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpy2DAsync(D->arena + dst_off, (size_t)dst_ld * eb, src, (size_t)src_ld * eb, (size_t)h * eb, w,
                             cudaMemcpyHostToDevice, D->h2d));
  return finish(dev, D->h2d, ev_out);
}

int bx_d2h_tile(int dev, uint64_t src_off, int src_ld, void* dst, int64_t dst_ld, int h, int w, int eb, int n_wait,
                const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  if (h <= 0 || w <= 0 || src_ld < h || dst_ld < h) return set_err(BX_EINVAL, "d2h: bad extents");
  if (src_off + (uint64_t)src_ld * w * eb > D->arena_bytes) return set_err(BX_EINVAL, "d2h: outside arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(D->d2h, n_wait, wait);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)dst_ld * eb, D->arena + src_off, (size_t)src_ld * eb, (size_t)h * eb, w,
                             cudaMemcpyDeviceToHost, D->d2h));
  return finish(dev, D->d2h, ev_out);
}

int bx_p2p_tile(int dst_dev, uint64_t dst_off, int src_dev, uint64_t src_off, uint64_t bytes, int n_wait,
                const int* wait, int* ev_out) {
  Device *D = dev_of(dst_dev), *S = dev_of(src_dev);
  if (!D || !S) return set_err(BX_EINVAL, "bad device");
  if (dst_off + bytes > D->arena_bytes || src_off + bytes > S->arena_bytes) return set_err(BX_EINVAL, "p2p: outside arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(D->p2p, n_wait, wait);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyPeerAsync(D->arena + dst_off, D->cuda_id, S->arena + src_off, S->cuda_id, bytes, D->p2p));
  return finish(dst_dev, D->p2p, ev_out);
}

// A launch group's tile fetches in one call (the runtime's resident issue path): each row
// {kind | eb << 8, dst_off, dst_ld, src, src_ld | src_off, h | bytes, w, wait_ev} is a
// 2-d H2D tile copy (kind 0: src = pinned host address, src_ld elements, h x w of eb
// bytes) or a peer copy (kind 1: src = device slot, src_off, bytes), optionally after a
// wait event (-1: none; e.g. the source tile's own arrival on the peer).  One event per
// lane used is recorded after the batch: the lanes are in-order, so that event marks the
// arrival of every tile the batch put on it.
int bx_copy_batch(int dev, int n, const int64_t* ops, int n_wait, const int* wait, int* ev_h2d, int* ev_p2p) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  if (n < 0) return set_err(BX_EINVAL, "copy batch: negative count");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  bool used_h2d = false, used_p2p = false;
  for (int i = 0; i < n; ++i) {
    const int64_t* r = ops + 8 * i;
    const int kind = (int)(r[0] & 0xff), eb = (int)(r[0] >> 8);
    const uint64_t dst_off = (uint64_t)r[1];
    const int64_t wait_ev = r[7];
    if (kind == 0) {
      const int dst_ld = (int)r[2], h = (int)r[5], w = (int)r[6];
      const int64_t src_ld = r[4];
      if (h <= 0 || w <= 0 || dst_ld < h || src_ld < h || (eb != 4 && eb != 8) || !r[3])
        return set_err(BX_EINVAL, "copy batch: bad h2d extents");
      if (dst_off + (uint64_t)dst_ld * w * eb > D->arena_bytes) return set_err(BX_EINVAL, "copy batch: h2d outside arena");
      if (!used_h2d && n_wait > 0) { int rc = wait_all(D->h2d, n_wait, wait); if (rc) return rc; }
      if (wait_ev >= 0) { int we = (int)wait_ev; int rc = wait_all(D->h2d, 1, &we); if (rc) return rc; }
      CUDA_TRY(cudaMemcpy2DAsync(D->arena + dst_off, (size_t)dst_ld * eb, (const void*)r[3], (size_t)src_ld * eb,
                                 (size_t)h * eb, w, cudaMemcpyHostToDevice, D->h2d));
      used_h2d = true;
    } else if (kind == 1) {
      Device* S = dev_of((int)r[3]);
      const uint64_t src_off = (uint64_t)r[4], bytes = (uint64_t)r[5];
      if (!S) return set_err(BX_EINVAL, "copy batch: bad peer slot");
      if (dst_off + bytes > D->arena_bytes || src_off + bytes > S->arena_bytes)
        return set_err(BX_EINVAL, "copy batch: p2p outside arena");
      if (!used_p2p && n_wait > 0) { int rc = wait_all(D->p2p, n_wait, wait); if (rc) return rc; }
      if (wait_ev >= 0) { int we = (int)wait_ev; int rc = wait_all(D->p2p, 1, &we); if (rc) return rc; }
      CUDA_TRY(cudaMemcpyPeerAsync(D->arena + dst_off, D->cuda_id, S->arena + src_off, S->cuda_id, bytes, D->p2p));
      used_p2p = true;
    } else {
      return set_err(BX_EINVAL, "copy batch: unknown op kind");
    }
  }
  if (ev_h2d) *ev_h2d = -1;
  if (ev_p2p) *ev_p2p = -1;
  if (used_h2d) { int rc = finish(dev, D->h2d, ev_h2d); if (rc) return rc; }
  if (used_p2p) { int rc = finish(dev, D->p2p, ev_p2p); if (rc) return rc; }
  return BX_OK;
}

static int gemm_task_k(int dev, int stream, int ta, int tb, int tri, int h, int w, int nsteps, const uint64_t* a_off,
                       const int* lda, const uint64_t* b_off, const int* ldb, const int* depth, const int* kmode,
                       double alpha, double beta, uint64_t c_off, int ldc, int n_wait, const int* wait, int* ev_out);

int bx_gemm_task(int dev, int stream, int ta, int tb, int tri, int h, int w, int nsteps, const uint64_t* a_off,
                 const int* lda, const uint64_t* b_off, const int* ldb, const int* depth, double alpha, double beta,
                 uint64_t c_off, int ldc, int n_wait, const int* wait, int* ev_out) {
  return gemm_task_k(dev, stream, ta, tb, tri, h, w, nsteps, a_off, lda, b_off, ldb, depth, nullptr, alpha, beta,
                     c_off, ldc, n_wait, wait, ev_out);
}

static int gemm_task_k(int dev, int stream, int ta, int tb, int tri, int h, int w, int nsteps, const uint64_t* a_off,
                       const int* lda, const uint64_t* b_off, const int* ldb, const int* depth, const int* kmode,
                       double alpha, double beta, uint64_t c_off, int ldc, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  if (tri < 0 || tri > 2 || (tri && h != w)) return set_err(BX_EINVAL, "gemm: triangle mode needs a square tile");
  if (nsteps > 4096) return set_err(BX_EINVAL, "gemm: too many steps");
  std::vector<const double*> ap(nsteps > 0 ? nsteps : 1), bp(nsteps > 0 ? nsteps : 1);
  for (int i = 0; i < nsteps; ++i) {
    if (a_off[i] >= D->arena_bytes || b_off[i] >= D->arena_bytes) return set_err(BX_EINVAL, "gemm: operand outside arena");
    ap[i] = (const double*)(D->arena + a_off[i]);
    bp[i] = (const double*)(D->arena + b_off[i]);
  }
  if (c_off + (uint64_t)ldc * w * 8 > D->arena_bytes) return set_err(BX_EINVAL, "gemm: C outside arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  rc = gemm_raw(s, ta, tb, tri, h, w, nsteps, ap.data(), lda, bp.data(), ldb, depth, alpha, beta, (double*)(D->arena + c_off), ldc,
                kmode);
  if (rc) return rc;
  return finish(dev, s, ev_out);
}

int bx_sgemm_task(int dev, int stream, int ta, int tb, int h, int w, int nsteps, const uint64_t* a_off,
                  const int* lda, const uint64_t* b_off, const int* ldb, const int* depth, float alpha, float beta,
                  uint64_t c_off, int ldc, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  if (nsteps < 0 || nsteps > 4096) return set_err(BX_EINVAL, "sgemm: bad step count");
  std::vector<const float*> ap(nsteps > 0 ? nsteps : 1), bp(nsteps > 0 ? nsteps : 1);
  for (int i = 0; i < nsteps; ++i) {
    if (a_off[i] >= D->arena_bytes || b_off[i] >= D->arena_bytes) return set_err(BX_EINVAL, "sgemm: operand outside arena");
    ap[i] = (const float*)(D->arena + a_off[i]);
    bp[i] = (const float*)(D->arena + b_off[i]);
  }
  if (c_off + (uint64_t)ldc * w * 4 > D->arena_bytes) return set_err(BX_EINVAL, "sgemm: C outside arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  rc = sgemm_raw(s, ta, tb, h, w, nsteps, ap.data(), lda, bp.data(), ldb, depth, alpha, beta, (float*)(D->arena + c_off), ldc);
  if (rc) return rc;
  return finish(dev, s, ev_out);
}

int bx_gemm_task_packed(int dev, int stream, int f32, int ta, int tb, int tri, int h, int w, int nsteps,
                        const int64_t* steps, double alpha, double beta, uint64_t c_off, int ldc, int n_wait,
                        const int* wait, int* ev_out) {
  if (nsteps < 0 || nsteps > 4096) return set_err(BX_EINVAL, "gemm: bad step count");
  std::vector<uint64_t> ao(nsteps > 0 ? nsteps : 1), bo(nsteps > 0 ? nsteps : 1);
  std::vector<int> la(nsteps > 0 ? nsteps : 1), lb(nsteps > 0 ? nsteps : 1), dp(nsteps > 0 ? nsteps : 1);
  std::vector<int> km(nsteps > 0 ? nsteps : 1);
  for (int i = 0; i < nsteps; ++i) {
    const int64_t* r = steps + 6 * i;
    if (r[0] < 0 || r[2] < 0) return set_err(BX_EINVAL, "gemm: negative operand offset");
    if (r[5] < bx::KM_NONE || r[5] > bx::KM_B_LOWER) return set_err(BX_EINVAL, "gemm: bad triangular-operand mode");
    ao[i] = (uint64_t)r[0]; la[i] = (int)r[1]; bo[i] = (uint64_t)r[2]; lb[i] = (int)r[3]; dp[i] = (int)r[4];
    km[i] = (int)r[5];
  }
  if (f32) {
    if (tri) return set_err(BX_EINVAL, "sgemm: no triangle mode");
    return bx_sgemm_task(dev, stream, ta, tb, h, w, nsteps, ao.data(), la.data(), bo.data(), lb.data(), dp.data(),
                         (float)alpha, (float)beta, c_off, ldc, n_wait, wait, ev_out);
  }
  return gemm_task_k(dev, stream, ta, tb, tri, h, w, nsteps, ao.data(), la.data(), bo.data(), lb.data(), dp.data(),
                     km.data(), alpha, beta, c_off, ldc, n_wait, wait, ev_out);
}

int bx_sgemm_device(int dev, int stream, int ta, int tb, int m, int n, int k, float alpha, uint64_t a, int lda,
                    uint64_t b, int ldb, float beta, uint64_t c, int ldc) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  const float* ap = (const float*)a;
  const float* bp = (const float*)b;
  return sgemm_raw(s, ta, tb, m, n, 1, &ap, &lda, &bp, &ldb, &k, alpha, beta, (float*)c, ldc);
}

int bx_trsm_tile(int dev, int stream, int side_right, int upper, int trans, int unit, int h, int w, double alpha,
                 uint64_t a_off, int lda, uint64_t b_off, int ldb, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  int n = side_right ? w : h;
  if (lda < n || ldb < h || (lda & 1) || (ldb & 1)) return set_err(BX_EINVAL, "trsm: bad leading dimension");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  int eff_upper = (upper != 0) != (trans != 0);
  rc = trsm_rec(s, side_right, eff_upper, trans, unit, h, w, alpha, (const double*)(D->arena + a_off), lda,
                (double*)(D->arena + b_off), ldb, D->flag_dev, g_trsm_leaf);
  if (rc) return rc;
  return finish(dev, s, ev_out);
}

// Inverse of a diagonal tile's triangle for the inverse-based TRSM diagonal step:
// inv(E), E = op(tri(A)) of order n, by the substitution solve E Z = I (the same kernels
// and division rule as bx_trsm_tile, so an exact zero on a non-unit diagonal raises the
// singular flag).  Z has exact zeros outside E's triangle.
int bx_trsm_inverse(int dev, int stream, int upper, int trans, int unit, int n, uint64_t a_off, int lda,
                    uint64_t inv_off, int ldi, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  if (n <= 0 || lda < n || ldi < n || (lda & 1) || (ldi & 1)) return set_err(BX_EINVAL, "trsm inverse: bad extents");
  if (inv_off + (uint64_t)ldi * n * 8 > D->arena_bytes || a_off + (uint64_t)lda * (n - 1) * 8 + 8 * n > D->arena_bytes)
    return set_err(BX_EINVAL, "trsm inverse: outside arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  double* z = (double*)(D->arena + inv_off);
  dim3 blk(32, 8), grd((n + 31) / 32, (n + 7) / 8);
  identity_kernel<<<grd, blk, 0, s>>>(z, ldi, n);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  const int eff_upper = (upper != 0) != (trans != 0);
  rc = trsm_rec(s, 0, eff_upper, trans, unit, n, n, 1.0, (const double*)(D->arena + a_off), lda, z, ldi, D->flag_dev,
                g_trsm_leaf);
  if (rc) return rc;
  return finish(dev, s, ev_out);
}

// The TRSM diagonal step with a precomputed inverse: X = alpha inv(E) B (left) or
// X = alpha B inv(E) (right) into a separate tile x, on the FP64 task GEMM with the
// triangular-operand k-range (each CTA reads only where inv(E) can be non-zero).
int bx_trsm_apply(int dev, int stream, int side_right, int eff_upper, int h, int w, double alpha, uint64_t inv_off,
                  int ldi, uint64_t b_off, int ldb, uint64_t x_off, int ldx, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  const int n = side_right ? w : h;
  if (h <= 0 || w <= 0 || ldi < n || ldb < h || ldx < h) return set_err(BX_EINVAL, "trsm apply: bad extents");
  if (x_off + (uint64_t)ldx * w * 8 > D->arena_bytes || b_off + (uint64_t)ldb * w * 8 > D->arena_bytes ||
      inv_off + (uint64_t)ldi * n * 8 > D->arena_bytes)
    return set_err(BX_EINVAL, "trsm apply: outside arena");
  if (x_off == b_off) return set_err(BX_EINVAL, "trsm apply: the result must not alias B");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  const double* inv = (const double*)(D->arena + inv_off);
  const double* bp = (const double*)(D->arena + b_off);
  double* x = (double*)(D->arena + x_off);
  if (!side_right) {
    const int km = eff_upper ? bx::KM_A_UPPER : bx::KM_A_LOWER;
    rc = gemm_raw(s, 0, 0, 0, h, w, 1, &inv, &ldi, &bp, &ldb, &n, alpha, 0.0, x, ldx, &km);
  } else {
    const int km = eff_upper ? bx::KM_B_UPPER : bx::KM_B_LOWER;
    rc = gemm_raw(s, 0, 0, 0, h, w, 1, &bp, &ldb, &inv, &ldi, &n, alpha, 0.0, x, ldx, &km);
  }
  if (rc) return rc;
  return finish(dev, s, ev_out);
}

int bx_materialize(int dev, int stream, int mode_sym, int upper, int trans, int unit, int n, uint64_t a_off, int lda,
                   uint64_t dst_off, int ldd, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  if (n <= 0 || lda < n || ldd < n) return set_err(BX_EINVAL, "materialize: bad extents");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  dim3 blk(32, 8), grd((n + 31) / 32, (n + 7) / 8);
  bx::materialize_kernel<<<grd, blk, 0, s>>>((const double*)(D->arena + a_off), lda, (double*)(D->arena + dst_off), ldd,
                                            n, mode_sym, upper, trans, unit);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return finish(dev, s, ev_out);
}

// dst (h x w) += beta * src: the deferred beta*C0 term of a task whose first GEMM launch
// ran with beta = 0 (the C0 tile's host copy is then off the task's critical path).
// One warp per 32 rows x 8 columns; both tiles column-major in the arena.
int bx_axpy_tile(int dev, int stream, int elem_bytes, int h, int w, double beta, uint64_t src_off, int src_ld,
                 uint64_t dst_off, int dst_ld, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  if (h < 0 || w < 0 || src_ld < h || dst_ld < h || (elem_bytes != 8 && elem_bytes != 4))
    return set_err(BX_EINVAL, "axpy: bad extents");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  if (h > 0 && w > 0) {
    dim3 blk(32, 8), grd((h + 31) / 32, (w + 7) / 8);
    if (elem_bytes == 8)
      bx::axpy_tile_kernel<double><<<grd, blk, 0, s>>>((double*)(D->arena + dst_off), dst_ld,
                                                   (const double*)(D->arena + src_off), src_ld, h, w, beta);
    else
      bx::axpy_tile_kernel<float><<<grd, blk, 0, s>>>((float*)(D->arena + dst_off), dst_ld,
                                                  (const float*)(D->arena + src_off), src_ld, h, w, (float)beta);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
  }
  return finish(dev, s, ev_out);
}

int bx_singular_flag(int dev, int reset, int* flag) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  *flag = *(volatile int*)D->flag_host;
  if (reset) *(volatile int*)D->flag_host = 0;
  return BX_OK;
}

int bx_event_record(int dev, int stream, int timing, int* ev_out) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s) return set_err(BX_EINVAL, "bad stream");
  cudaEvent_t e;
  int id;
  int rc = ev_get(dev, timing != 0, &e, &id);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  CUDA_TRY(cudaEventRecord(e, s));
  *ev_out = id;
  return BX_OK;
}

int bx_event_query(int ev) {
  cudaEvent_t e;
  if (!ev_lookup(ev, &e)) return set_err(BX_EINVAL, "bad event");
  cudaError_t r = cudaEventQuery(e);
  if (r == cudaSuccess) return 0;
  if (r == cudaErrorNotReady) { cudaGetLastError(); return 1; }
  return set_err(BX_ECUDA, std::string("event: ") + cudaGetErrorString(r));
}

int bx_event_sync(int ev) {
  cudaEvent_t e;
  if (!ev_lookup(ev, &e)) return set_err(BX_EINVAL, "bad event");
  CUDA_TRY(cudaEventSynchronize(e));
  return BX_OK;
}

int bx_event_wait_any(int n, const int* evs, int* index, int spin_us) {
  if (n <= 0) return set_err(BX_EINVAL, "wait_any: empty");
  std::vector<cudaEvent_t> es(n);
  for (int i = 0; i < n; ++i)
    if (!ev_lookup(evs[i], &es[i])) return set_err(BX_EINVAL, "bad event");
  auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    for (int i = 0; i < n; ++i) {
      cudaError_t r = cudaEventQuery(es[i]);
      if (r == cudaSuccess) { *index = i; return BX_OK; }
      if (r != cudaErrorNotReady) return set_err(BX_ECUDA, cudaGetErrorString(r));
    }
    cudaGetLastError();
    if (spin_us >= 0) {
      auto us = std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count();
      if (us >= spin_us) { *index = -1; return BX_OK; }
    }
    std::this_thread::yield();
  }
}

int bx_event_elapsed(int ev0, int ev1, float* ms) {
  cudaEvent_t a, b;
  if (!ev_lookup(ev0, &a) || !ev_lookup(ev1, &b)) return set_err(BX_EINVAL, "bad event");
  CUDA_TRY(cudaEventElapsedTime(ms, a, b));
  return BX_OK;
}

int bx_event_release(int ev) {
  if (ev < 0) return BX_OK;
  int d = ev >> kEvShift, idx = ev & ((1 << kEvShift) - 1);
  if (d >= (int)g_devs.size() || !g_devs[d].pool) return set_err(BX_EINVAL, "bad event");
  EventPool& P = *g_devs[d].pool;
  std::lock_guard<std::mutex> lk(P.mu);
  if (idx >= P.count.load()) return set_err(BX_EINVAL, "bad event");
  if (!P.release(idx)) return set_err(BX_EINVAL, "event " + std::to_string(ev) + " released twice");
  return BX_OK;
}

int bx_event_release_many(int n, const int* evs) {
  for (int i = 0; i < n; ++i) {
    const int ev = evs[i];
    if (ev < 0) continue;
    const int d = ev >> kEvShift, idx = ev & ((1 << kEvShift) - 1);
    if (d >= (int)g_devs.size() || !g_devs[d].pool) return set_err(BX_EINVAL, "bad event");
    EventPool& P = *g_devs[d].pool;
    std::lock_guard<std::mutex> lk(P.mu);
    if (idx >= P.count.load()) return set_err(BX_EINVAL, "bad event");
    if (!P.release(idx)) return set_err(BX_EINVAL, "event " + std::to_string(ev) + " released twice");
  }
  return BX_OK;
}

int bx_stream_wait(int dev, int stream, int ev) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s) return set_err(BX_EINVAL, "bad stream");
  cudaEvent_t e;
  if (!ev_lookup(ev, &e)) return set_err(BX_EINVAL, "bad event");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  CUDA_TRY(cudaStreamWaitEvent(s, e, 0));
  return BX_OK;
}

int bx_device_sync(int dev) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  CUDA_TRY(cudaDeviceSynchronize());
  return BX_OK;
}

int bx_dev_alloc(int dev, uint64_t bytes, uint64_t* ptr) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) { cudaGetLastError(); return set_err(BX_ENOMEM, cudaGetErrorString(e)); }
  *ptr = (uint64_t)p;
  return BX_OK;
}

int bx_dev_free(int dev, uint64_t ptr) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  CUDA_TRY(cudaFree((void*)ptr));
  return BX_OK;
}

int bx_dev_fill_uniform(int dev, uint64_t ptr, uint64_t n, uint64_t seed, int stream) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s) return set_err(BX_EINVAL, "bad stream");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  fill_uniform_kernel<<<D->sms * 8, 256, 0, s>>>((double*)ptr, n, seed);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return BX_OK;
}

int bx_dev_fill_uniform_f32(int dev, uint64_t ptr, uint64_t n, uint64_t seed, int stream) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s) return set_err(BX_EINVAL, "bad stream");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  fill_uniform_f32_kernel<<<D->sms * 8, 256, 0, s>>>((float*)ptr, n, seed);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return BX_OK;
}

int bx_dev_copy_h2d(int dev, uint64_t dst, const void* src, uint64_t bytes) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  CUDA_TRY(cudaMemcpy((void*)dst, src, bytes, cudaMemcpyHostToDevice));
  return BX_OK;
}

int bx_dev_copy_d2h(int dev, void* dst, uint64_t src, uint64_t bytes) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  CUDA_TRY(cudaMemcpy(dst, (const void*)src, bytes, cudaMemcpyDeviceToHost));
  return BX_OK;
}

int bx_dgemm_device(int dev, int stream, int ta, int tb, int m, int n, int k, double alpha, uint64_t a, int lda,
                    uint64_t b, int ldb, double beta, uint64_t c, int ldc) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, stream);
  if (!s || stream < 0) return set_err(BX_EINVAL, "bad compute stream");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  const double* ap = (const double*)a;
  const double* bp = (const double*)b;
  return gemm_raw(s, ta, tb, 0, m, n, 1, &ap, &lda, &bp, &ldb, &k, alpha, beta, (double*)c, ldc);
}

int bx_set_gemm_group(int g) {
  if (g < 1 || g > 64) return set_err(BX_EINVAL, "gemm raster group must be in [1, 64]");
  g_gemm_group = g;
  return BX_OK;
}

int bx_set_gemm_variant(int v) {
  g_gemm_variant = v;
  return BX_OK;
}

int bx_set_sgemm_variant(int v) {
  if (v < 0 || v > 3) return set_err(BX_EINVAL, "sgemm variant must be 0, 1, 2 or 3");
  g_sgemm_variant = v;
  return BX_OK;
}

int bx_set_sgemm_precise(int on) {
  g_sgemm_precise = on != 0;
  return BX_OK;
}

int bx_set_sgemm_mn3d(int on) {
  g_sgemm_mn3d = on != 0;
  return BX_OK;
}

int bx_set_sgemm_debug(int bits) {
  // bits 0..7: ablation switches; bits 8..15: persistent-kernel raster group (tuning)
  g_sgemm_debug = bits & 0xFF;
  g_sgemm_group = (bits >> 8) & 0xFF;
  return BX_OK;
}

int bx_set_trsm_rhs(int nr) {
  if (nr != 8 && nr != 16 && nr != 32 && nr != 64)
    return set_err(BX_EINVAL, "trsm panel RHS width must be 8, 16, 32 or 64");
  g_trsm_rhs = nr;
  return BX_OK;
}

int bx_set_trsm_leaf(int n) {
  if (n < 32 || n > bx::T_NMAX) return set_err(BX_EINVAL, "trsm leaf must be in [32, 2048]");
  g_trsm_leaf = n;
  return BX_OK;
}

int bx_fp64_peak_probe(int dev, int iters, double* tflops) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  double* out;
  CUDA_TRY(cudaMalloc(&out, 4096));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  cudaStream_t s = D->comp[0];
  dmma_probe_kernel<<<D->sms * 2, 256, 0, s>>>(out, iters);
  g_launches++;
  CUDA_TRY(cudaEventRecord(e0, s));
  dmma_probe_kernel<<<D->sms * 2, 256, 0, s>>>(out, iters);
  g_launches++;
  CUDA_TRY(cudaEventRecord(e1, s));
  CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  *tflops = (double)D->sms * 2 * 8 * (double)iters * 8 * 512.0 / ms / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return BX_OK;
}

// ---- one process per GPU: IPC arenas, device-visible flags, host atomics ---------------

int bx_ipc_arena_handle(int dev, void* handle64, uint64_t* arena_bytes) {
  Device* D = dev_of(dev);
  if (!D || !D->arena) return set_err(BX_EINVAL, "ipc handle: no arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, D->arena));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle64, &h, sizeof(h));
  *arena_bytes = D->arena_bytes;
  return BX_OK;
}

int bx_ipc_open(int dev, const void* handle64, uint64_t* base) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *base = (uint64_t)p;
  return BX_OK;
}

int bx_ipc_close(int dev, uint64_t base) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  CUDA_TRY(cudaIpcCloseMemHandle((void*)base));
  return BX_OK;
}

int bx_host_register_mapped(void* ptr, uint64_t bytes, uint64_t* dev_ptr) {
  if (!ptr || !bytes) return set_err(BX_EINVAL, "register: null");
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e == cudaErrorHostMemoryAlreadyRegistered) cudaGetLastError();
  else if (e != cudaSuccess) { cudaGetLastError(); return set_err(BX_ECUDA, std::string("cudaHostRegister(mapped): ") + cudaGetErrorString(e)); }
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_registered[ptr] = bytes;
  }
  void* d = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(&d, ptr, 0));
  *dev_ptr = (uint64_t)d;
  return BX_OK;
}

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitValue32 g_wait32 = nullptr;
PFN_writeValue32 g_write32 = nullptr;

int stream_ops_init() {
  if (g_wait32 && g_write32) return BX_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return set_err(BX_ECUDA, "cuStreamWaitValue32 unavailable");
  g_wait32 = (PFN_waitValue32)fn;
  fn = nullptr;
  CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return set_err(BX_ECUDA, "cuStreamWriteValue32 unavailable");
  g_write32 = (PFN_writeValue32)fn;
  return BX_OK;
}

int bx_copy_remote(int dst_dev, uint64_t dst_off, uint64_t src_ptr, uint64_t bytes, uint64_t flag_dptr,
                   uint32_t flag_min, int n_wait, const int* wait, int* ev_out) {
  Device* D = dev_of(dst_dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  if (!src_ptr || dst_off + bytes > D->arena_bytes) return set_err(BX_EINVAL, "copy_remote: outside arena");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = wait_all(D->p2p, n_wait, wait);
  if (rc) return rc;
  if (flag_dptr) {
    rc = stream_ops_init();
    if (rc) return rc;
    CUresult r = g_wait32((CUstream)D->p2p, (CUdeviceptr)flag_dptr, flag_min, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return set_err(BX_ECUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
  }
  CUDA_TRY(cudaMemcpyAsync(D->arena + dst_off, (const void*)src_ptr, bytes, cudaMemcpyDeviceToDevice, D->p2p));
  return finish(dst_dev, D->p2p, ev_out);
}

int bx_write_flag(int dev, int lane, uint64_t flag_dptr, uint32_t value, int n_wait, const int* wait) {
  Device* D = dev_of(dev);
  if (!D) return set_err(BX_EINVAL, "bad device");
  cudaStream_t s = lane_stream(D, lane);
  if (!s || !flag_dptr) return set_err(BX_EINVAL, "write_flag: bad lane / flag");
  CUDA_TRY(cudaSetDevice(D->cuda_id));
  int rc = stream_ops_init();
  if (rc) return rc;
  rc = wait_all(s, n_wait, wait);
  if (rc) return rc;
  CUresult r = g_write32((CUstream)s, (CUdeviceptr)flag_dptr, value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return set_err(BX_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
  return BX_OK;
}

int bx_atomic_add(int64_t* p, int64_t v, int64_t* old) {
  if (!p || ((uintptr_t)p & 7)) return set_err(BX_EINVAL, "atomic_add: misaligned");
  *old = __atomic_fetch_add(p, v, __ATOMIC_SEQ_CST);
  return BX_OK;
}

int bx_atomic_cas(int64_t* p, int64_t expected, int64_t desired, int64_t* old) {
  if (!p || ((uintptr_t)p & 7)) return set_err(BX_EINVAL, "atomic_cas: misaligned");
  int64_t e = expected;
  __atomic_compare_exchange_n(p, &e, desired, false, __ATOMIC_SEQ_CST, __ATOMIC_SEQ_CST);
  *old = e;
  return BX_OK;
}

// ---- resident issue engine ------------------------------------------------------------
// One routine call's input tiles in a per-GPU region of each arena (resident arenas hold
// every input tile, so nothing is ever evicted).  The Python runtime keeps the scheduling
// policy (stations, Eq. 3, stealing) and hands a launch's operands over as tile ids; the
// translation (L1 hit / L2 copy from the lowest-id peer holding the tile / H2D from the
// pinned host operand, the reference's policy, scheduler.py:426-461 + cache.py:97-113),
// the copies and the launch are one C call.  The tile table (offsets, arrival events,
// holder masks) is exported to Python as plain arrays for Eq. 3 and the metrics.

struct IcTile {
  uint64_t host;
  int64_t host_ld;
  int h, w, esz, ld;
  uint64_t bytes;
};

struct IcCall {
  int ndev = 0, ntiles = 0, l2 = 1;
  std::vector<int> slot, group;
  std::vector<IcTile> tiles;
  std::vector<int64_t> off;       // [d * ntiles + t]: arena offset, -1 = not on GPU d
  std::vector<int32_t> ev;        // arrival event (shared by a copy batch), -1 = landed
  std::vector<uint32_t> holders;  // [t]: bit d set once GPU d holds (or is fetching) t
  std::vector<uint64_t> cur, end; // per-GPU bump allocator inside its region
  std::vector<int64_t> met;       // [d * 8 + k]: h2d bytes, d2d-in bytes, host fetches,
                                  // L2 hits, d2d-out bytes, tile references served
  std::vector<int> owned;         // arrival events, released by bx_ic_destroy
  std::vector<uint32_t> stamp;    // per-tile dedupe marks for one resolve
  uint32_t epoch = 0;
  std::mutex mu;
};

std::mutex g_ic_mu;
std::vector<std::unique_ptr<IcCall>> g_ic;

IcCall* ic_of(int id) {
  std::lock_guard<std::mutex> lk(g_ic_mu);
  if (id < 0 || id >= (int)g_ic.size()) return nullptr;
  return g_ic[id].get();
}

// Make every tile of `tids` present on GPU d (caller holds C.mu): missing tiles are
// allocated in d's region and fetched — over L2 from the lowest-id peer of d's group that
// holds the tile (the copy waits on that holder's arrival event), else from the host —
// with one arrival event per copy lane for the whole batch.  Appends the distinct
// arrival events the caller's launch must wait on to `waits`.
int ic_resolve(IcCall& C, int d, int n, const int32_t* tids, std::vector<int>& waits) {
  Device* D = dev_of(C.slot[d]);
  if (!D) return set_err(BX_EINVAL, "ic: bad device");
  const int nt = C.ntiles;
  if (++C.epoch == 0) { std::fill(C.stamp.begin(), C.stamp.end(), 0u); C.epoch = 1; }
  std::vector<int> new_h, new_p;
  bool set_dev = false;
  for (int i = 0; i < n; ++i) {
    const int t = tids[i];
    if (t < 0 || t >= nt) return set_err(BX_EINVAL, "ic: tile id out of range");
    if (C.stamp[t] == C.epoch) continue;
    C.stamp[t] = C.epoch;
    const size_t idx = (size_t)d * nt + t;
    int64_t* m = &C.met[(size_t)d * 8];
    if (C.off[idx] >= 0) {
      const int e = C.ev[idx];
      if (e >= 0) {
        cudaEvent_t ce;
        if (ev_lookup(e, &ce) && cudaEventQuery(ce) == cudaSuccess) C.ev[idx] = -1;
        else if (std::find(waits.begin(), waits.end(), e) == waits.end()) waits.push_back(e);
      }
      continue;
    }
    const IcTile& T = C.tiles[t];
    const uint64_t o = (C.cur[d] + 255) & ~(uint64_t)255;
    if (o + T.bytes > C.end[d]) return set_err(BX_ENOMEM, "ic: resident region exhausted");
    C.cur[d] = o + T.bytes;
    C.off[idx] = (int64_t)o;
    if (!set_dev) { CUDA_TRY(cudaSetDevice(D->cuda_id)); set_dev = true; }
    int src = -1;
    if (C.l2) {
      const uint32_t h = C.holders[t];
      for (int e = 0; e < C.ndev; ++e)
        if (e != d && ((h >> e) & 1u) && C.group[e] == C.group[d]) { src = e; break; }
    }
    const uint64_t payload = (uint64_t)T.h * T.w * T.esz;
    if (src >= 0) {
      const size_t sidx = (size_t)src * nt + t;
      Device* S = dev_of(C.slot[src]);
      if (!S) return set_err(BX_EINVAL, "ic: bad peer device");
      if (C.ev[sidx] >= 0) { int we = C.ev[sidx]; int rc = wait_all(D->p2p, 1, &we); if (rc) return rc; }
      CUDA_TRY(cudaMemcpyPeerAsync(D->arena + o, D->cuda_id, S->arena + C.off[sidx], S->cuda_id, T.bytes, D->p2p));
      new_p.push_back(t);
      m[1] += (int64_t)payload;
      m[3] += 1;
      C.met[(size_t)src * 8 + 4] += (int64_t)payload;
    } else {
      CUDA_TRY(cudaMemcpy2DAsync(D->arena + o, (size_t)T.ld * T.esz, (const void*)T.host,
                                 (size_t)T.host_ld * T.esz, (size_t)T.h * T.esz, T.w,
                                 cudaMemcpyHostToDevice, D->h2d));
      new_h.push_back(t);
      m[0] += (int64_t)payload;
      m[2] += 1;
    }
    C.holders[t] |= 1u << d;
  }
  for (int lane = 0; lane < 2; ++lane) {
    std::vector<int>& lst = lane == 0 ? new_h : new_p;
    if (lst.empty()) continue;
    int e = -1;
    int rc = finish(C.slot[d], lane == 0 ? D->h2d : D->p2p, &e);
    if (rc) return rc;
    C.owned.push_back(e);
    for (int t : lst) C.ev[(size_t)d * nt + t] = e;
    waits.push_back(e);
  }
  return BX_OK;
}

int bx_ic_create(int ndev, const int* slots, const int* groups, int ntiles, const int64_t* tiles,
                 const uint64_t* region_off, const uint64_t* region_bytes, int l2, int* id) {
  if (ndev <= 0 || ndev > 32 || ntiles < 0) return set_err(BX_EINVAL, "ic: bad sizes");
  std::unique_ptr<IcCall> C(new IcCall());
  C->ndev = ndev;
  C->ntiles = ntiles;
  C->l2 = l2;
  C->slot.assign(slots, slots + ndev);
  C->group.assign(groups, groups + ndev);
  C->tiles.resize(ntiles);
  for (int t = 0; t < ntiles; ++t) {
    const int64_t* r = tiles + 6 * t;   // host address, host ld, h, w, element bytes, device ld
    IcTile& T = C->tiles[t];
    T.host = (uint64_t)r[0]; T.host_ld = r[1]; T.h = (int)r[2]; T.w = (int)r[3]; T.esz = (int)r[4];
    T.ld = (int)r[5];
    if (!T.host || T.h <= 0 || T.w <= 0 || T.ld < T.h || T.host_ld < T.h || (T.esz != 4 && T.esz != 8))
      return set_err(BX_EINVAL, "ic: bad tile descriptor " + std::to_string(t));
    T.bytes = (uint64_t)T.ld * T.w * T.esz;
  }
  for (int d = 0; d < ndev; ++d) {
    Device* D = dev_of(slots[d]);
    if (!D) return set_err(BX_EINVAL, "ic: bad device slot");
    if (region_off[d] + region_bytes[d] > D->arena_bytes) return set_err(BX_EINVAL, "ic: region outside arena");
  }
  C->off.assign((size_t)ndev * ntiles, -1);
  C->ev.assign((size_t)ndev * ntiles, -1);
  C->holders.assign(ntiles, 0u);
  C->cur.assign(region_off, region_off + ndev);
  C->end.resize(ndev);
  for (int d = 0; d < ndev; ++d) C->end[d] = region_off[d] + region_bytes[d];
  C->met.assign((size_t)ndev * 8, 0);
  C->stamp.assign(ntiles, 0u);
  std::lock_guard<std::mutex> lk(g_ic_mu);
  for (int i = 0; i < (int)g_ic.size(); ++i)
    if (!g_ic[i]) { g_ic[i] = std::move(C); *id = i; return BX_OK; }
  g_ic.push_back(std::move(C));
  *id = (int)g_ic.size() - 1;
  return BX_OK;
}

int bx_ic_destroy(int id) {
  std::unique_ptr<IcCall> C;
  {
    std::lock_guard<std::mutex> lk(g_ic_mu);
    if (id < 0 || id >= (int)g_ic.size() || !g_ic[id]) return set_err(BX_EINVAL, "ic: bad id");
    C = std::move(g_ic[id]);
  }
  if (!C->owned.empty()) return bx_event_release_many((int)C->owned.size(), C->owned.data());
  return BX_OK;
}

int bx_ic_state(int id, int64_t** off, int32_t** ev, uint32_t** holders, int64_t** metrics) {
  IcCall* C = ic_of(id);
  if (!C) return set_err(BX_EINVAL, "ic: bad id");
  *off = C->off.data();
  *ev = C->ev.data();
  *holders = C->holders.data();
  *metrics = C->met.data();
  return BX_OK;
}

int bx_ic_resolve(int id, int d, int n, const int32_t* tids, int64_t* off_out, int32_t* ld_out, int* n_wait,
                  int* wait_out, int wait_cap) {
  IcCall* C = ic_of(id);
  if (!C || d < 0 || d >= C->ndev) return set_err(BX_EINVAL, "ic: bad id/device");
  std::lock_guard<std::mutex> lk(C->mu);
  std::vector<int> waits;
  int rc = ic_resolve(*C, d, n, tids, waits);
  if (rc) return rc;
  if ((int)waits.size() > wait_cap) return set_err(BX_EINVAL, "ic: wait buffer too small");
  for (int i = 0; i < n; ++i) {
    off_out[i] = C->off[(size_t)d * C->ntiles + tids[i]];
    ld_out[i] = C->tiles[tids[i]].ld;
  }
  for (size_t i = 0; i < waits.size(); ++i) wait_out[i] = waits[i];
  *n_wait = (int)waits.size();
  C->met[(size_t)d * 8 + 5] += n;
  return BX_OK;
}

// One task GEMM launch whose operands are tile ids: steps = nsteps rows of
// {a, b, depth, kmode}; an operand id < 0 names raw[-id - 1] = (arena offset, ld) (scratch
// tiles).  The launch waits on `wait` plus the arrival events of its tiles.
int bx_ic_gemm(int id, int d, int stream, int f32, int ta, int tb, int tri, int h, int w, int nsteps,
               const int32_t* steps, const int64_t* raw, int nraw, double alpha, double beta, uint64_t c_off,
               int ldc, int n_wait, const int* wait, int* ev_out) {
  IcCall* C = ic_of(id);
  if (!C || d < 0 || d >= C->ndev) return set_err(BX_EINVAL, "ic: bad id/device");
  if (nsteps < 0 || nsteps > 4096) return set_err(BX_EINVAL, "ic gemm: bad step count");
  std::vector<int> waits(wait, wait + n_wait);
  std::vector<int32_t> tids;
  tids.reserve(2 * nsteps);
  for (int i = 0; i < 2 * nsteps; ++i) {
    const int32_t v = steps[4 * (i / 2) + (i & 1)];
    if (v >= 0) tids.push_back(v);
    else if (-v - 1 >= nraw) return set_err(BX_EINVAL, "ic gemm: raw operand out of range");
  }
  std::vector<uint64_t> ao(nsteps > 0 ? nsteps : 1), bo(nsteps > 0 ? nsteps : 1);
  std::vector<int> la(nsteps > 0 ? nsteps : 1), lb(nsteps > 0 ? nsteps : 1), dp(nsteps > 0 ? nsteps : 1),
      km(nsteps > 0 ? nsteps : 1);
  {
    std::lock_guard<std::mutex> lk(C->mu);
    int rc = ic_resolve(*C, d, (int)tids.size(), tids.data(), waits);
    if (rc) return rc;
    C->met[(size_t)d * 8 + 5] += (int64_t)tids.size();
    const int nt = C->ntiles;
    for (int i = 0; i < nsteps; ++i) {
      const int32_t* r = steps + 4 * i;
      for (int o = 0; o < 2; ++o) {
        uint64_t off;
        int ld;
        if (r[o] >= 0) {
          off = (uint64_t)C->off[(size_t)d * nt + r[o]];
          ld = C->tiles[r[o]].ld;
        } else {
          off = (uint64_t)raw[2 * (-r[o] - 1)];
          ld = (int)raw[2 * (-r[o] - 1) + 1];
        }
        (o ? bo : ao)[i] = off;
        (o ? lb : la)[i] = ld;
      }
      dp[i] = r[2];
      km[i] = r[3];
      if (km[i] < bx::KM_NONE || km[i] > bx::KM_B_LOWER) return set_err(BX_EINVAL, "ic gemm: bad kmode");
    }
  }
  if (f32) {
    if (tri) return set_err(BX_EINVAL, "sgemm: no triangle mode");
    return bx_sgemm_task(C->slot[d], stream, ta, tb, h, w, nsteps, ao.data(), la.data(), bo.data(), lb.data(),
                         dp.data(), (float)alpha, (float)beta, c_off, ldc, (int)waits.size(), waits.data(), ev_out);
  }
  return gemm_task_k(C->slot[d], stream, ta, tb, tri, h, w, nsteps, ao.data(), la.data(), bo.data(), lb.data(),
                     dp.data(), km.data(), alpha, beta, c_off, ldc, (int)waits.size(), waits.data(), ev_out);
}

}  // extern "C"
