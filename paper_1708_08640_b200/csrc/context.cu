// context.cu -- C ABI (include/cmtf_b200.h) of the B200 S^3CMTF path:
// device-resident DataBundle and model, the epoch driver (run_epoch /
// train), evaluation, per-entry probes.  Host logic mirrors the reference
// trainer (/root/reference/proj/core/src/trainer.cpp) and is native C++;
// every O(nnz) step runs on the device.
#include <cub/device/device_radix_sort.cuh>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is resolved at run time (nccl_api)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "../../include/cmtf_b200.h"
#include "common.cuh"
#include "generic.cuh"
#include "hog3.cuh"
#include "hog3v2.cuh"
#include "hog4.cuh"
#include "hog4tm.cuh"
#include "hog3tm.cuh"
#include "eval3tm.cuh"
#include "stateless64.cuh"

#include "host_rng.hpp"

using namespace cmtfb;

namespace {

// NCCL is resolved on first use (dlopen), never at load time: the process's
// NCCL is whichever libnccl.so.2 is already mapped (PyTorch's bundled copy
// when torch is imported first), else the CMTF_NCCL_LIB path, else the
// system library.  Linking it would map the system NCCL at import and break
// a later `import torch` that needs a newer NCCL.
struct NcclApi {
  bool tried = false;
  std::string error;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  // point-to-point and broadcast (DSGD row-block rotation, consolidation)
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    if (const char* p = std::getenv("CMTF_NCCL_LIB")) h = dlopen(p, RTLD_NOW);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW);
  if (!h) {
    api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
  api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
  api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
  api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
  api.getErrorString =
      reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
  api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
  api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
  api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
  api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
  api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
  if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.allReduce ||
      !api.getErrorString || !api.send || !api.recv || !api.broadcast || !api.groupStart ||
      !api.groupEnd) {
    api.error = "libnccl.so.2 lacks a required symbol";
    api.getUniqueId = nullptr;
  }
  return api;
}


thread_local std::string g_last_error;

struct DevMatrix {
  int mode = 0;
  uint32_t rows = 0, cols = 0;
  uint64_t nnz = 0;
  double weight = 1.0;
  uint32_t* rec = nullptr;   // sorted by row, 3 words
  uint32_t* pos = nullptr;   // entry id -> sorted position
  uint32_t* count = nullptr; // per col
  float* vreg = nullptr;     // lambda_m * lambda / count
  float* V = nullptr;        // cols x JP
};

}  // namespace

constexpr int kUpChunks = 16;                 // upload copy/pack chunks (at most)
constexpr uint64_t kUpChunkMin = 1ull << 20;  // entries per chunk (at least)

struct cmtf_gpu_ctx {
  cmtf_gpu_config cfg{};
  std::vector<uint32_t> ranks;
  int order = 0;
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;

  // bundle
  std::vector<uint32_t> dims;
  uint64_t nnz = 0;
  int sort_mode = 0;
  uint32_t* rec = nullptr;  // sorted tensor records, (order+1) words
  uint32_t* pos = nullptr;  // training id -> sorted position
  uint32_t* count[kMaxOrder] = {};
  float* reg[kMaxOrder] = {};
  std::vector<DevMatrix> mats;
  std::vector<DevMatrix> spare;  // parked by clear_matrices

  // model
  float* U[kMaxOrder] = {};
  float* G = nullptr;
  bool have_model = false;

  // state (TrainState, include/cmtf/trainer.hpp:49-56)
  int32_t epoch = 0;
  double eta = 0.0;
  std::vector<uint64_t> schedule;  // serial mode only
  uint64_t* d_sched = nullptr;
  uint64_t d_sched_cap = 0;

  // upload scratch (grow-only)
  uint32_t* s_idx = nullptr;
  uint64_t s_idx_cap = 0;
  double* s_vals = nullptr;
  uint64_t s_vals_cap = 0;
  uint32_t* s_rec = nullptr;
  uint64_t s_rec_cap = 0;
  uint32_t* s_keys = nullptr;
  uint64_t s_keys_cap = 0;
  uint32_t* s_ids = nullptr;
  uint64_t s_ids_cap = 0;
  uint64_t rec_cap = 0, pos_cap = 0;
  // per-epoch reshuffle: double buffers, and the affine map (posA, posB)
  // from pos[] to the current physical position of an entry
  uint32_t* rec_alt = nullptr;
  uint64_t rec_alt_cap = 0;
  uint64_t posA = 1, posB = 0;
  // pos_affine: pos[] still holds the upload's placement (pa e + pb) mod n
  bool pos_affine = false;
  uint64_t up_pa = 1, up_pb = 0;
  uint4* mrec_alt = nullptr;
  uint64_t mrec_alt_cap = 0;
  // hog3tm: per record {lambda/count_1(i1), lambda/count_2(i2),
  // lambda/count_3(i3), 0}, stored beside rec in the same order (a streamed
  // 16-byte read instead of three random 4-byte lookups per entry: each of
  // those costs a full L2 fill once the count arrays miss L2), permuted with
  // rec by the per-epoch reshuffle
  float4* rrec = nullptr;
  float4* rrec_alt = nullptr;
  uint64_t rrec_cap = 0, rrec_alt_cap = 0;
  bool rrec_valid = false;
  // virtual visiting order (hog3tm, vt_on): the records stay in place and
  // every epoch's order is the segment table d_vtab; blk_B x blk_B strata
  // (blk_B = 1: one segment, no re-layout), blk_n / blk_off = stratum sizes
  // and offsets by stratum id.  pos_ids: pos[] is stale and is rebuilt from
  // the entry ids in rrec[].w.
  uint32_t blk_B = 0;
  bool vt_on = false, pos_ids = false;
  std::vector<uint64_t> blk_n, blk_off;
  uint32_t* blk_hist = nullptr;  // [2][kMaxBlk^2]: stratum sizes, offsets
  uint32_t* part_cnt = nullptr;  // [chunk][stratum] counts -> run starts
  uint64_t part_cnt_cap = 0;
  uint4* d_vtab = nullptr;
  std::vector<uint4> h_vtab;
  // the next epoch's gathers run on a side stream, overlapping the current
  // sweep (they only read rec / mrec and write the spare buffers)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_side_start = nullptr, ev_side_done = nullptr;
  int64_t pend_t_epoch = -1, pend_m_epoch = -1;  // epoch whose order sits in *_alt
  uint64_t pend_ta = 1, pend_tb = 0;

  // scratch
  double* d_partial = nullptr;
  double* d_partial2 = nullptr;  // reduce_partials' second level
  uint64_t partial2_cap = 0;
  uint64_t partial_cap = 0;
  unsigned long long* d_first = nullptr;

  // duplicate-index check scratch (grow-only)
  unsigned long long* dup_keys = nullptr;  // [2][cap]
  uint64_t dup_keys_cap = 0;
  uint32_t* dup_ids = nullptr;  // [2][cap]
  uint64_t dup_ids_cap = 0;
  uint8_t* dup_tmp = nullptr;
  uint64_t dup_tmp_cap = 0;

  // device-side hot-row selection scratch
  unsigned long long* hs_keys = nullptr;  // [2][cap]
  uint64_t hs_keys_cap = 0;
  uint8_t* hs_tmp = nullptr;
  uint64_t hs_tmp_cap = 0;
  uint32_t* hs_cnt = nullptr;  // [1 + 16]: candidate count, per-array H

  // v2 sweep state (built lazily after a bundle change)
  bool v2_dirty = true;
  uint4* mrec = nullptr;  // merged matrix records {row, col, bits(y), m}, random order
  uint64_t mnnz = 0, mrec_cap = 0;
  uint4* s_m4 = nullptr;
  uint64_t s_m4_cap = 0;
  struct HotHost {
    int32_t* slot = nullptr;
    uint32_t* row_of = nullptr;
    uint64_t slot_cap = 0, row_cap = 0;
    uint32_t H = 0;
    float* base = nullptr;
    uint64_t base_cap = 0;
    uint32_t off = 0, stat_off = 0;
  };
  HotHost hot[kMaxOrder];
  HotHost hotV[kMaxMats];
  int v2_blocks = 0;
  int v2_nw = 8;
  int v2_e = 2;
  size_t v2_smem = 0;
  uint32_t tm_stage_off = 0;  // hog3tm bulk row-step staging (floats; 0 = REDs)
  bool schedule_given = false;  // cmtf_gpu_set_schedule: replay it next serial epoch
  // debug_count_visits: per tensor record / merged matrix record visit counts
  // of the current epoch (indexed by record position)
  uint32_t* visits = nullptr;
  uint32_t* mvisits = nullptr;
  uint64_t visits_cap = 0, mvisits_cap = 0;
  int64_t visits_epoch = -1;
  bool visits_ok = true;  // every sweep of this epoch ran a counting kernel

  // DSGD: replicated parameters, global sizes, communicator
  uint64_t nnz_global = 0;  // 0 = local nnz
  int world = 1;
  uint32_t shared_modes = 0, shared_mats = 0;
  std::vector<uint64_t> mat_base;  // offset of matrix m in the merged stream
  float* baseU[kMaxOrder] = {};
  float* baseV[kMaxMats] = {};
  float* baseG = nullptr;
  float* sync_buf = nullptr;
  uint64_t sync_cap = 0;
  ncclComm_t comm = nullptr;

  // timing
  cudaEvent_t ev[6] = {};
  cudaEvent_t uev[8] = {};
  cudaEvent_t cev[16] = {};  // upload chunk copies (kUpChunks)
  double last_ms[4] = {0, 0, 0, 0};
  int32_t last_launches = 0;
  int kernel_which = 0;
  float* probe = nullptr;       // kernel probe outputs (cmtf_gpu_kernel_probe)
  float* probe_core = nullptr;
  // test / experiment switches, read once when the context is created
  struct Env {
    bool v4_tc = true;     // CMTF_V4_TC=0: order-4 CUDA-core sweep
    bool v4_tm = true;     // CMTF_V4_TM=0: order-4 opt on hog4 (mma.sync) instead of hog4tm (tcgen05)
    bool v3_tm = true;     // CMTF_V3_TM=0: order-3 opt on hog3v2 instead of hog3tm
    int v2_shape = 0;      // CMTF_V2_SHAPE: 1 = "8x1", 2 = "8x2"
    bool hot_host = false; // CMTF_HOT_HOST: host hot-row selection
    bool hot_check = false;// CMTF_HOT_CHECK: compare device vs host selection
    bool tm_red = false;   // CMTF_TM_RED=1: hog3tm cold-row steps as REDs (no bulk staging)
    int tm_strided = 0;    // CMTF_TM_STRIDED=1: hog3tm lanes take strided records
    int tm_blocks = -1;    // CMTF_TM_BLOCKS=B: blocked order with B x B strata (0/1 off, -1 auto)
    int tm_seq = 1;        // CMTF_TM_SEQ=0: random stratum sequence (1: mode-1-block-major)
    int tm_pfl2 = -1;      // CMTF_TM_PFL2=0/1: hog3tm L2 prefetch of the next entry's rows (-1 auto)
    bool tm_vorder = true; // CMTF_TM_VORDER=0: hog3tm reshuffles its records physically
    int tm_bulk = -1;      // CMTF_TM_BULK=mask: modes whose cold-row steps are bulk reductions (-1 auto)
    int tm_gather_ca = -1; // CMTF_TM_GATHER_CA=0/1: order-3 row gathers through L1 (-1: when the tables exceed L2)
    bool tm_galt = true;   // CMTF_TM_GALT=0: both warpgroups convert every core refresh
    bool rrec_late = true; // CMTF_RREC_LATE=0: hog3tm's rrec built before the blocked re-layout
    int up_chunks = 16;    // CMTF_UP_CHUNKS=n: upload copy/pack chunks (1..16)
    bool eval_stream3 = true; // CMTF_EVAL_STREAM3=0: eval3tm reads the unblocked mode's rows with plain loads
    bool eval_tm = true;   // CMTF_EVAL_TM=0: order-3 eval on eval3_kernel (CUDA cores) instead of eval3tm
  } env;
  int hog_threads_used = 0;

  uint32_t J(int n) const { return ranks[n]; }
  uint32_t JP(int n) const { return (uint32_t)round_up4((int)ranks[n]); }
  uint64_t core_size() const {
    uint64_t s = 1;
    for (auto j : ranks) s *= j;
    return s;
  }
};

namespace {

int set_err(cmtf_gpu_ctx* ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  if (ctx) ctx->err = buf;
  return code;
}

#define CU(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return set_err(ctx, CMTF_ECUDA, "CUDA error %s at %s:%d: %s",           \
                     cudaGetErrorName(e_), __FILE__, __LINE__,                \
                     cudaGetErrorString(e_));                                 \
  } while (0)

#define TRY(expr)             \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != CMTF_OK) return rc_; \
  } while (0)

// splitmix-mixed mt19937_64 streams: host_rng.hpp (src/rng.cpp:8-26).

template <typename T>
int dalloc(cmtf_gpu_ctx* ctx, T** p, size_t n) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  if (n == 0) n = 1;
  CU(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
  return CMTF_OK;
}
// Grow-only device buffer (re-uploads of a same-sized bundle reuse it).
template <typename T>
int ensure(cmtf_gpu_ctx* ctx, T** p, uint64_t* cap, uint64_t n) {
  if (*p && *cap >= n) return CMTF_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  CU(cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(T)));
  *cap = n;
  return CMTF_OK;
}

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// ---------------- preprocessing kernels ----------------
// 32-bit avalanche hash (murmur3 finaliser) keyed by the seed: sorting by it
// gives a seeded random permutation of the entries.
__device__ __forceinline__ uint32_t mix32(uint32_t x, uint32_t seed) {
  x ^= seed * 0x9e3779b9u;
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}

// Count with one atomic per distinct index per warp: Zipf heads would
// otherwise serialise millions of same-address atomics in L2.
__device__ __forceinline__ void count_aggregated(uint32_t* count, uint32_t i, bool valid) {
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, valid ? i : 0xffffffffu);
  if (valid && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(count + i, __popc(peers));
}

// Records [e_lo, e_hi) of the upload: validation, counts, packing.
// perm_n > 0: the record goes straight to its place in the affine entry
// order, p = (pa * e + pb) mod perm_n (pos[e] = p), instead of position e.
__global__ void pack_tensor_kernel(const uint32_t* idx, const double* vals, uint64_t e_lo,
                                   uint64_t e_hi, int order, ModeTables mt,
                                   int sort_mode, uint32_t seed, uint32_t* rec,
                                   uint32_t* keys, uint32_t* ids,
                                   unsigned long long* bad, uint64_t perm_n = 0,
                                   uint64_t pa = 1, uint64_t pb = 0, uint32_t* pos = nullptr) {
  for (uint64_t e = e_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < e_hi;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = perm_n ? (uint64_t)(((unsigned __int128)pa * e + pb) % perm_n) : e;
    if (perm_n) pos[e] = (uint32_t)p;
    if (order == 3) {  // one 16-byte record store
      uint4 r;
      uint32_t* ri = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const uint32_t i = idx[e * 3 + n];
        const bool ok = i < mt.dims[n];
        if (!ok) atomicMin(&bad[0], (unsigned long long)e);
        count_aggregated(const_cast<uint32_t*>(mt.count[n]), i, ok);
        ri[n] = i;
      }
      const double v = vals[e];
      if (!isfinite(v)) atomicMin(&bad[1], (unsigned long long)e);
      r.w = __float_as_uint((float)v);
      reinterpret_cast<uint4*>(rec)[p] = r;
    } else {
      for (int n = 0; n < order; ++n) {
        const uint32_t i = idx[e * order + n];
        const bool ok = i < mt.dims[n];
        if (!ok) atomicMin(&bad[0], (unsigned long long)e);
        count_aggregated(const_cast<uint32_t*>(mt.count[n]), i, ok);
        rec[p * (order + 1) + n] = i;
      }
      const double v = vals[e];
      if (!isfinite(v)) atomicMin(&bad[1], (unsigned long long)e);
      rec[p * (order + 1) + order] = __float_as_uint((float)v);
    }
    if (keys) {  // sorted order only
      keys[e] = sort_mode >= 0 ? idx[e * order + sort_mode] : mix32((uint32_t)e, seed);
      ids[e] = (uint32_t)e;
    }
  }
}

// Seeded affine bijection p -> (a*p + b) mod n with gcd(a, n) = 1: a random
// entry order without a sort (the reference reshuffles its schedule,
// src/trainer.cpp:122-128; a fixed pseudo-random order is used here).
__global__ void scatter_affine_kernel(const uint32_t* src, uint64_t n, int words,
                                      uint64_t a, uint64_t b, uint32_t* dst, uint32_t* pos) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = (uint64_t)(((unsigned __int128)a * e + b) % n);
    for (int w = 0; w < words; ++w) dst[p * words + w] = src[e * words + w];
    pos[e] = (uint32_t)p;
  }
}

__global__ void gather_records_kernel(const uint32_t* src, const uint32_t* ids,
                                      uint64_t n, int words, uint32_t* dst,
                                      uint32_t* pos) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[s];
    for (int w = 0; w < words; ++w) dst[s * words + w] = src[(uint64_t)id * words + w];
    pos[id] = (uint32_t)s;
  }
}

// Per-epoch reshuffle (the reference reshuffles its schedule every epoch,
// src/trainer.cpp:122-128): the records move in groups of kShuffleGroup
// consecutive ones (the storage order is already a random permutation, so a
// group is a random set; 8 x 16 B = one 128-B line keeps the gather at
// streaming efficiency): dst group g = src group (a*g + b) mod ng.  Records
// past ng * kShuffleGroup stay in place.  Each warp walks runs of 32 records
// (32 / kShuffleGroup groups), a lane's source group advancing by
// step = (32 / kShuffleGroup) * a mod ng.
constexpr int kShuffleGroup = 8;
constexpr int kReshuffleRun = 64;
template <int WORDS>
__global__ void reshuffle_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                 uint64_t n, uint64_t a, uint64_t b, uint64_t step) {
  const int lane = threadIdx.x & 31;
  const uint64_t ng = n / kShuffleGroup, body = ng * kShuffleGroup;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t run = 32ull * kReshuffleRun;
  for (uint64_t base = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * run;
       base < n; base += warps * run) {
    uint64_t i = base + lane;
    uint64_t g = i / kShuffleGroup;
    uint64_t pg = g < ng ? (uint64_t)(((unsigned __int128)a * g + b) % ng) : 0;
    for (int r = 0; r < kReshuffleRun && i < n; ++r, i += 32) {
      const uint64_t q = i < body ? pg * kShuffleGroup + (i % kShuffleGroup) : i;
      if (WORDS == 4) {  // evict-first: L2 stays with the epoch kernel's factor rows
        __stcs(reinterpret_cast<uint4*>(dst) + i, __ldcs(reinterpret_cast<const uint4*>(src) + q));
      } else {
#pragma unroll
        for (int w = 0; w < WORDS; ++w) dst[i * WORDS + w] = __ldg(src + q * WORDS + w);
      }
      pg += step;
      if (pg >= ng) pg -= ng;
    }
  }
}

// pos[i] <- current position: group (A * group + B) mod ng, same offset
__global__ void remap_pos_kernel(uint32_t* pos, uint64_t count, uint64_t n, uint64_t A,
                                 uint64_t B) {
  const uint64_t ng = n / kShuffleGroup, body = ng * kShuffleGroup;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = pos[i];
    if (p < body)
      pos[i] = (uint32_t)((((unsigned __int128)A * (p / kShuffleGroup) + B) % ng) *
                              kShuffleGroup + p % kShuffleGroup);
  }
}

// ---- Virtual visiting order and the L2-blocked layout (hog3tm) ----
// The tcgen05 epoch never moves its records between epochs: each epoch's
// random order is a table of segments the kernel maps virtual positions
// through (vphys, hog3tm.cuh) -- the reference reshuffles its whole schedule
// every epoch, src/trainer.cpp:122-128.  With factor tables beyond L2 the
// records are first laid out stratum-major: stratum s = (mode-1 block b1,
// mode-2 block b2), s = b1 * B + b2, blocks = B equal row ranges; the lanes
// take strided records, so the whole grid sweeps one stratum at a time and
// the two active row blocks (2/B of U1 and U2) stay in L2 while it lasts.
// Each epoch draws a random stratum sequence and a group-affine map per
// stratum.  rrec[p].w carries the entry id of record p (pos[] is rebuilt
// from it after the re-layout).
constexpr int kMaxBlk = 64;

// block of row i: floor(i * B / d), by a float estimate and an exact
// correction (a 64-bit division is a ~100-instruction routine)
__device__ __forceinline__ uint32_t block_of(uint32_t i, uint32_t B, uint64_t d, float scale) {
  uint32_t q = (uint32_t)((float)i * scale);
  if (q >= B) q = B - 1;
  const uint64_t x = (uint64_t)i * B;
  if ((uint64_t)q * d > x) --q;
  else if ((uint64_t)(q + 1) * d <= x) ++q;
  return q;
}
__device__ __forceinline__ uint32_t stratum_of(uint32_t i1, uint32_t i2, uint32_t B, uint64_t d0,
                                               uint64_t d1) {
  return block_of(i1, B, d0, (float)B / (float)d0) * B + block_of(i2, B, d1, (float)B / (float)d1);
}

// Partition of the records by stratum (chunks of kPartChunk
// records): counts per (chunk, stratum), an exclusive scan per stratum
// across the chunks, then each chunk writes its records, in position order,
// to consecutive places of each stratum's run.  Reads stream; writes form
// runs that fill whole lines in L2.
// (chunk size grows with the stratum count so the count table stays small)
inline uint32_t part_chunk(uint32_t S) { return 8192u * std::max(1u, S / 64u); }
__global__ void part_hist_kernel(const uint4* rec, uint64_t n, uint32_t B, uint64_t d0,
                                 uint64_t d1, uint32_t* cnt, uint32_t* total,
                                 uint32_t kPartChunk) {
  __shared__ uint32_t h[kMaxBlk * kMaxBlk];
  const uint32_t S = B * B;
  const uint64_t nch = (n + kPartChunk - 1) / kPartChunk;
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    for (uint32_t s = threadIdx.x; s < S; s += blockDim.x) h[s] = 0;
    __syncthreads();
    const uint64_t p1 = min(n, (c + 1) * (uint64_t)kPartChunk);
    for (uint64_t p = c * (uint64_t)kPartChunk + threadIdx.x; p < p1; p += blockDim.x) {
      const uint4 r = __ldcs(rec + p);
      atomicAdd(h + stratum_of(r.x, r.y, B, d0, d1), 1u);
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < S; s += blockDim.x) {
      if (cnt) cnt[c * S + s] = h[s];
      if (h[s]) atomicAdd(total + s, h[s]);
    }
    __syncthreads();
  }
}

// one warp per stratum: cnt[c][s] <- off[s] + sum of cnt[c'][s], c' < c
__global__ void part_scan_kernel(uint32_t* cnt, uint64_t nch, uint32_t S, const uint32_t* off) {
  const uint32_t s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  uint32_t run = off[s];
  for (uint64_t c0 = 0; c0 < nch; c0 += 32) {
    const uint64_t c = c0 + lane;
    const uint32_t v = c < nch ? cnt[c * S + s] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (c < nch) cnt[c * S + s] = run + x - v;
    run += __shfl_sync(0xffffffffu, x, 31);
  }
}

// rrec[pos[e]].w = e (pos exact)
__global__ void rrec_ids_kernel(const uint32_t* pos, uint64_t n, float4* rrec) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint32_t*>(rrec + pos[e])[3] = (uint32_t)e;
}

__global__ void pos_from_ids_kernel(const float4* rrec, uint64_t n, uint32_t* pos) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x)
    pos[__float_as_uint(__ldg(&rrec[p].w))] = (uint32_t)p;
}

// Entry id of record position q in closed form while pos[] is still the
// upload's affine placement p0 = (pa e + pb) mod n followed by the composed
// group map (posA, posB) of the per-epoch reshuffles: no scatter pass.
struct IdMap {
  uint64_t n, ng, iA, B, ia, pb;
  uint64_t m_n, m_ng;  // floor((2^64 - 1) / n), / ng: Barrett reduction instead of 64-bit divisions
  int closed;
};
// x mod d with m = floor((2^64 - 1) / d): the quotient estimate is at most one short
__device__ __forceinline__ uint64_t mod_magic(uint64_t x, uint64_t d, uint64_t m) {
  uint64_t r = x - __umul64hi(x, m) * d;
  if (r >= d) r -= d;
  return r;
}
__device__ __forceinline__ uint32_t entry_of(const IdMap& m, uint64_t q) {
  uint64_t p0 = q;
  if (q < m.ng * kShuffleGroup) {
    uint64_t g = q / kShuffleGroup + m.ng - m.B;  // B < ng
    if (g >= m.ng) g -= m.ng;
    p0 = mod_magic(m.iA * g, m.ng, m.m_ng) * kShuffleGroup + q % kShuffleGroup;
  }
  uint64_t t = p0 + m.n - m.pb;  // pb < n
  if (t >= m.n) t -= m.n;
  return (uint32_t)mod_magic(m.ia * t, m.n, m.m_n);
}

// One block per chunk at a time: a record's place = the next free place of
// its stratum's run for the chunk (shared-memory counters seeded with the
// run starts; the order inside a run is the order the atomics land in --
// the input is a random permutation already and the layout is kept for the
// whole training, so stability buys nothing).
__global__ void __launch_bounds__(256) part_scatter_kernel(
    const uint4* __restrict__ rec, const uint4* __restrict__ rrec, uint64_t n, uint32_t B,
    uint64_t d0, uint64_t d1, const uint32_t* __restrict__ base, uint4* __restrict__ rec_out,
    uint4* __restrict__ rrec_out, const IdMap m, uint32_t kPartChunk) {
  __shared__ uint32_t run[kMaxBlk * kMaxBlk];
  const uint32_t S = B * B;
  const uint64_t nch = (n + kPartChunk - 1) / kPartChunk;
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    for (uint32_t s = threadIdx.x; s < S; s += 256) run[s] = base[c * S + s];
    __syncthreads();
    const uint64_t p1 = min(n, (c + 1) * (uint64_t)kPartChunk);
    for (uint64_t p = c * (uint64_t)kPartChunk + threadIdx.x; p < p1; p += 256) {
      const uint4 r = __ldcs(rec + p);
      uint4 q = __ldcs(rrec + p);
      const uint32_t d = atomicAdd(run + stratum_of(r.x, r.y, B, d0, d1), 1u);
      if (m.closed) q.w = entry_of(m, p);
      rec_out[d] = r;
      rrec_out[d] = q;
    }
    __syncthreads();
  }
}

// Partition pass with coalesced writes.  Scattering record by record (the
// kernel above) issues two 16-byte writes per record to ~S different runs:
// 2.6e10 scattered writes/s is the memory system's ceiling for them (75 ms
// per 9e8 records).  Here a block sorts a tile of kTile records by key in
// shared memory (at most 64 keys), claims a piece of every key's global run
// with one atomic per key, and writes each piece as consecutive 16-byte
// stores.  With more than 64 strata the partition takes two passes: by
// mode-1 block (PASS 1), then -- over that output, tile by tile inside every
// mode-1 block's run (RunTab) -- by mode-2 block (PASS 2).  PASS 0: one pass
// over <= 64 strata.  The order inside a stratum is whatever the atomics
// give (the input is a random permutation; the layout then stays).
constexpr int kTile = 1024;
struct RunTab {  // PASS 2: the mode-1 blocks' runs and their tile counts (prefix sums)
  uint32_t off[kMaxBlk + 1];
  uint32_t tpre[kMaxBlk + 1];
};
template <int PASS>
__global__ void __launch_bounds__(256) part_tile_kernel(
    const uint4* __restrict__ rec, const uint4* __restrict__ rrec, uint64_t n, uint32_t B,
    uint64_t d0, uint64_t d1, uint32_t* __restrict__ cursor, uint4* __restrict__ rec_out,
    uint4* __restrict__ rrec_out, const IdMap m, const RunTab rt) {
  __shared__ uint4 srec[kTile];
  __shared__ uint4 srr[kTile];
  __shared__ uint8_t skey[kTile];
  __shared__ uint32_t hist[64], start[64], gbase[64];
  const float sc0 = (float)B / (float)d0, sc1 = (float)B / (float)d1;
  const uint64_t ntile = PASS == 2 ? rt.tpre[B] : (n + kTile - 1) / kTile;
  for (uint64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    uint64_t p0 = tile * kTile;
    uint32_t cnt = (uint32_t)min((uint64_t)kTile, n - p0);
    uint32_t run = 0;  // PASS 2: the mode-1 block this tile lies in
    if (PASS == 2) {
      while (tile >= rt.tpre[run + 1]) ++run;
      p0 = rt.off[run] + (tile - rt.tpre[run]) * kTile;
      cnt = (uint32_t)min((uint64_t)kTile, rt.off[run + 1] - p0);
    }
    if (threadIdx.x < 64) hist[threadIdx.x] = 0;
    __syncthreads();
    uint4 r[kTile / 256], q[kTile / 256];
    uint32_t key[kTile / 256], rank[kTile / 256];
#pragma unroll
    for (int j = 0; j < kTile / 256; ++j) {
      const uint32_t t = threadIdx.x + 256 * j;
      if (t < cnt) {
        r[j] = __ldcs(rec + p0 + t);
        q[j] = rrec ? __ldcs(rrec + p0 + t) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int j = 0; j < kTile / 256; ++j) {
      const uint32_t t = threadIdx.x + 256 * j;
      if (t < cnt) {
        if (PASS == 1) key[j] = block_of(r[j].x, B, d0, sc0);
        else {
          const uint32_t b2 = block_of(r[j].y, B, d1, sc1);
          key[j] = PASS == 0 ? block_of(r[j].x, B, d0, sc0) * B + b2 : b2;
        }
        if (PASS != 2 && m.closed) q[j].w = entry_of(m, p0 + t);
        rank[j] = atomicAdd(hist + key[j], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 64 counts, one global claim per key
      const uint32_t h0 = hist[threadIdx.x], h1 = hist[threadIdx.x + 32];
      uint32_t x0 = h0, x1 = h1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, d);
        const uint32_t y1 = __shfl_up_sync(0xffffffffu, x1, d);
        if ((int)threadIdx.x >= d) {
          x0 += y0;
          x1 += y1;
        }
      }
      const uint32_t tot0 = __shfl_sync(0xffffffffu, x0, 31);
      start[threadIdx.x] = x0 - h0;
      start[threadIdx.x + 32] = tot0 + x1 - h1;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const uint32_t k = threadIdx.x + 32 * half, h = half ? h1 : h0;
        const uint32_t gi = PASS == 2 ? run * B + k : k;
        gbase[k] = h ? atomicAdd(cursor + gi, h) : 0u;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kTile / 256; ++j) {
      const uint32_t t = threadIdx.x + 256 * j;
      if (t < cnt) {
        const uint32_t slot = start[key[j]] + rank[j];
        srec[slot] = r[j];
        srr[slot] = q[j];
        skey[slot] = (uint8_t)key[j];
      }
    }
    __syncthreads();
    for (uint32_t slot = threadIdx.x; slot < cnt; slot += 256) {
      const uint32_t k = skey[slot];
      const uint32_t d = gbase[k] + (slot - start[k]);
      rec_out[d] = srec[slot];
      rrec_out[d] = srr[slot];
    }
    __syncthreads();
  }
}

__global__ void reg_kernel(const uint32_t* count, uint32_t n, float lambda,
                           float* reg) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x)
    reg[i] = count[i] ? lambda / (float)count[i] : 0.f;
}

// rrec[p] = the three regulariser coefficients of record p (order 3)
// (keep_w: the fourth word holds the entry id of a blocked layout; kept)
__global__ void build_rrec_kernel(const uint4* rec, uint64_t n, const float* r0, const float* r1,
                                  const float* r2, float4* out, int keep_w) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 r = rec[p];
    out[p] = make_float4(__ldg(r0 + r.x), __ldg(r1 + r.y), __ldg(r2 + r.z),
                         keep_w ? out[p].w : 0.f);
  }
}

constexpr uint32_t kPackHistCols = 8192;
// Entries [e_lo, e_hi) of a matrix upload; perm_n > 0: each record goes
// straight to its place p = (pa * e + pb) mod perm_n of the entry order.
__global__ void pack_matrix_kernel(const uint32_t* idx, const double* vals,
                                   uint64_t e_lo, uint64_t nnz, uint32_t rows, uint32_t cols,
                                   int shuffled, uint32_t seed, uint32_t* rec,
                                   uint32_t* keys, uint32_t* ids, uint32_t* count,
                                   unsigned long long* bad, uint64_t perm_n = 0,
                                   uint64_t pa = 1, uint64_t pb = 0, uint32_t* pos = nullptr) {
  // few columns (e.g. a 200-column side matrix): per-block shared-memory
  // histogram, one global atomic per (block, column) -- two million entries on
  // 200 column counters otherwise serialise in L2
  extern __shared__ uint32_t hist[];
  const bool small = cols <= kPackHistCols;
  if (small) {
    for (uint32_t c = threadIdx.x; c < cols; c += blockDim.x) hist[c] = 0;
    __syncthreads();
  }
  for (uint64_t e = e_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = idx[2 * e], j = idx[2 * e + 1];
    const bool ok = i < rows && j < cols;
    if (!ok) atomicMin(&bad[0], (unsigned long long)e);
    if (small) {
      if (ok) atomicAdd(hist + j, 1u);
    } else {
      count_aggregated(count, j, ok);
    }
    const double v = vals[e];
    if (!isfinite(v)) atomicMin(&bad[1], (unsigned long long)e);
    const uint64_t p = perm_n ? (uint64_t)(((unsigned __int128)pa * e + pb) % perm_n) : e;
    if (perm_n) pos[e] = (uint32_t)p;
    rec[3 * p] = i;
    rec[3 * p + 1] = j;
    rec[3 * p + 2] = __float_as_uint((float)v);
    if (keys) {
      keys[e] = shuffled ? mix32((uint32_t)e, seed) : i;
      ids[e] = (uint32_t)e;
    }
  }
  if (small) {
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < cols; c += blockDim.x)
      if (hist[c]) atomicAdd(count + c, hist[c]);
  }
}

int normalize_pos(cmtf_gpu_ctx* ctx);  // reshuffle machinery, below
uint32_t blocks_wanted(const cmtf_gpu_ctx* ctx);
bool tables_beyond_l2(const cmtf_gpu_ctx* ctx);
int vt_setup(cmtf_gpu_ctx* ctx, uint32_t B, bool rrec_in = true);
bool vt_wanted(const cmtf_gpu_ctx* ctx);
int vt_table(cmtf_gpu_ctx* ctx, uint64_t epoch);
bool tensor_shuffles(const cmtf_gpu_ctx* ctx);
int take_matrix_order(cmtf_gpu_ctx* ctx);
int prefetch_orders(cmtf_gpu_ctx* ctx, bool tensor, bool matrices);
void drain_side(cmtf_gpu_ctx* ctx);

uint64_t gcd64(uint64_t x, uint64_t y) {
  while (y) {
    const uint64_t t = x % y;
    x = y;
    y = t;
  }
  return x;
}

// multiplier ~ n / golden ratio, coprime with n; offset from the seed
void affine_params(uint64_t n, uint64_t seed, uint64_t* a, uint64_t* b) {
  uint64_t m = (uint64_t)((double)n * 0.6180339887498949) | 1ull;
  if (m >= n) m = n > 1 ? n - 1 : 1;
  while (m > 1 && gcd64(m, n) != 1) --m;
  *a = m ? m : 1;
  uint64_t s = seed * 0x9e3779b97f4a7c15ULL + 0x632be59bd9b4e019ULL;
  s ^= s >> 29;
  *b = n ? s % n : 0;
}

// A fresh affine visiting order for (seed, epoch, stream): multiplier drawn
// uniformly among the units mod n, offset uniform.
void epoch_affine(uint64_t n, uint64_t seed, uint64_t epoch, uint64_t stream, uint64_t* a,
                  uint64_t* b) {
  *a = 1;
  *b = 0;
  if (n < 3) return;
  auto mix = [](uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  };
  const uint64_t s = mix(mix(mix(seed) ^ epoch) ^ (stream * 0x632be59bd9b4e019ULL));
  uint64_t m = 1 + mix(s) % (n - 1);
  while (gcd64(m, n) != 1) m = m + 1 < n ? m + 1 : 1;
  *a = m;
  *b = mix(s + 1) % n;
}

unsigned grid_for(uint64_t n, unsigned bt = 256) {
  uint64_t g = (n + bt - 1) / bt;
  if (g > 148ull * 32) g = 148ull * 32;
  if (g == 0) g = 1;
  return (unsigned)g;
}

// Sort 32-bit keys with 32-bit ids (stable LSD radix sort).
int sort_ids(cmtf_gpu_ctx* ctx, uint32_t* keys, uint32_t* ids, uint64_t n,
             uint32_t max_key, uint32_t** sorted_ids_out) {
  uint32_t *keys_out = nullptr, *ids_out = nullptr;
  TRY(dalloc(ctx, &keys_out, n));
  TRY(dalloc(ctx, &ids_out, n));
  int end_bit = 1;
  while (end_bit < 32 && (1ull << end_bit) <= max_key) ++end_bit;
  size_t temp = 0;
  CU(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys, keys_out, ids, ids_out,
                                     (int64_t)n, 0, end_bit, ctx->stream));
  void* d_temp = nullptr;
  CU(cudaMalloc(&d_temp, temp ? temp : 1));
  CU(cub::DeviceRadixSort::SortPairs(d_temp, temp, keys, keys_out, ids, ids_out,
                                     (int64_t)n, 0, end_bit, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_temp);
  cudaFree(keys_out);
  *sorted_ids_out = ids_out;
  return CMTF_OK;
}

uint64_t nnz_all_of(const cmtf_gpu_ctx* ctx) {
  return ctx->nnz_global ? ctx->nnz_global : ctx->nnz;
}

ModeTables mode_tables(const cmtf_gpu_ctx* ctx) {
  ModeTables mt{};
  for (int n = 0; n < ctx->order; ++n) {
    mt.U[n] = ctx->U[n];
    mt.reg[n] = ctx->reg[n];
    mt.count[n] = ctx->count[n];
    mt.J[n] = ctx->J(n);
    mt.JP[n] = ctx->JP(n);
    mt.dims[n] = n < (int)ctx->dims.size() ? ctx->dims[n] : 0;
  }
  return mt;
}

CoreShape core_shape(const cmtf_gpu_ctx* ctx) {
  CoreShape cs{};
  cs.order = ctx->order;
  uint32_t off = 0;
  for (int n = 0; n < ctx->order; ++n) {
    cs.J[n] = ctx->ranks[n];
    cs.off[n] = off;
    off += ctx->ranks[n];
  }
  cs.off[ctx->order] = off;
  cs.size = (uint32_t)ctx->core_size();
  cs.cp = ctx->cfg.core_structure == 1;
  cs.dstep = 0;
  for (int n = ctx->order - 1, st = 1; n >= 0; --n) {
    cs.dstep += (uint32_t)st;
    st *= (int)ctx->ranks[n];
  }
  return cs;
}

int ensure_partials(cmtf_gpu_ctx* ctx, uint64_t n) {
  if (n <= ctx->partial_cap) return CMTF_OK;
  TRY(dalloc(ctx, &ctx->d_partial, n));
  ctx->partial_cap = n;
  return CMTF_OK;
}

// blocked_sum's pairwise combine over block partials (src/eval.cpp:46-48) on
// the device: the reference's tree -- element i takes element
// i + width at every width = 1, 2, 4, ... -- evaluated chunk by chunk (a
// 1024-aligned chunk's subtree is closed under the pairing, so the chunk
// results combine by the same rule one level up).  Missing partners are
// zeros (x + 0 = x), so the result is bit-identical to the host loop.
__global__ void __launch_bounds__(512) pairwise_chunk_kernel(const double* in, uint64_t n,
                                                              double* out) {
  __shared__ double s[1024];
  const uint64_t base = (uint64_t)blockIdx.x * 1024;
  for (int i = threadIdx.x; i < 1024; i += 512) s[i] = base + i < n ? in[base + i] : 0.0;
  __syncthreads();
  for (int w = 1; w < 1024; w *= 2) {
    const int i = threadIdx.x * 2 * w;
    if (i + w < 1024) s[i] += s[i + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

// Sum of d_partial[0, n) by the pairwise tree; only the result crosses PCIe.
int reduce_partials(cmtf_gpu_ctx* ctx, uint64_t n, double* out) {
  const uint64_t n1 = (n + 1023) / 1024;
  if (n1 + 1 > ctx->partial2_cap) {
    TRY(dalloc(ctx, &ctx->d_partial2, n1 + 1));
    ctx->partial2_cap = n1 + 1;
  }
  const double* src = ctx->d_partial;
  double* dst = ctx->d_partial2;
  double* other = ctx->d_partial;  // level >= 2 results go back into the front of d_partial
  uint64_t m = n;
  do {
    const uint64_t nb = (m + 1023) / 1024;
    pairwise_chunk_kernel<<<(unsigned)nb, 512, 0, ctx->stream>>>(src, m, dst);
    CU(cudaGetLastError());
    src = dst;
    std::swap(dst, other);
    m = nb;
  } while (m > 1);
  CU(cudaMemcpyAsync(out, src, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return CMTF_OK;
}

bool fast3_supported(const cmtf_gpu_ctx* ctx, int* J) {
  if (ctx->order != 3 || ctx->cfg.force_generic) return false;
  if (ctx->ranks[0] != ctx->ranks[1] || ctx->ranks[1] != ctx->ranks[2]) return false;
  const int j = (int)ctx->ranks[0];
  if (j != 2 && j != 4 && j != 5 && j != 8 && j != 10 && j != 16 && j != 20) return false;
  *J = j;
  return true;
}

template <int J, bool OPT, int CM>
int launch_hog3_t(cmtf_gpu_ctx* ctx, const Hog3Args& args, int threads) {
  constexpr int BT = J >= 16 ? 128 : 256;
  auto kern = hog3_kernel<J, J, J, OPT, CM, BT>;
  const size_t smem = Hog3Layout<J, J, J>::template B<BT>::bytes();
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BT, smem));
  if (per_sm < 1) per_sm = 1;
  int blocks = ctx->num_sms * per_sm;
  if (threads > 0) blocks = std::max(1, threads / BT);
  else {
    // auto: keep at least ~64 entries per worker (staleness)
    const uint64_t cap = std::max<uint64_t>(1, args.nnz / (64ull * BT));
    blocks = (int)std::min<uint64_t>((uint64_t)blocks, cap);
  }
  ctx->hog_threads_used = blocks * BT;
  kern<<<blocks, BT, smem, ctx->stream>>>(args);
  CU(cudaGetLastError());
  return CMTF_OK;
}

template <int J>
int launch_hog3_j(cmtf_gpu_ctx* ctx, const Hog3Args& args, bool opt, int cm,
                  int threads) {
  if (opt) {
    if (cm == 0) return launch_hog3_t<J, true, 0>(ctx, args, threads);
    if (cm == 1) return launch_hog3_t<J, true, 1>(ctx, args, threads);
    return launch_hog3_t<J, true, 2>(ctx, args, threads);
  }
  if (cm == 0) return launch_hog3_t<J, false, 0>(ctx, args, threads);
  if (cm == 1) return launch_hog3_t<J, false, 1>(ctx, args, threads);
  return launch_hog3_t<J, false, 2>(ctx, args, threads);
}

int launch_hog3(cmtf_gpu_ctx* ctx, int J, const Hog3Args& args, bool opt,
                int cm, int threads) {
  switch (J) {
    case 2: return launch_hog3_j<2>(ctx, args, opt, cm, threads);
    case 4: return launch_hog3_j<4>(ctx, args, opt, cm, threads);
    case 5: return launch_hog3_j<5>(ctx, args, opt, cm, threads);
    case 8: return launch_hog3_j<8>(ctx, args, opt, cm, threads);
    case 10: return launch_hog3_j<10>(ctx, args, opt, cm, threads);
    case 16: return launch_hog3_j<16>(ctx, args, opt, cm, threads);
    case 20: return launch_hog3_j<20>(ctx, args, opt, cm, threads);
  }
  return set_err(ctx, CMTF_EUNSUPPORTED, "no specialised kernel for J=%d", J);
}

template <int J>
int launch_eval3_t(cmtf_gpu_ctx* ctx, const uint32_t* rec, uint64_t nnz,
                   double* partial) {
  if constexpr (J == 4 || J == 5 || J == 8 || J == 10) {
    if (ctx->env.eval_tm) {  // the contraction on tcgen05 (eval3tm.cuh)
      const uint64_t nblk = (nnz + kEvalBlock - 1) / kEvalBlock;
      const uint64_t cap = (uint64_t)ctx->num_sms * CMTF_EVAL_TM_OCC;
      const unsigned grid = (unsigned)(nblk < cap ? nblk : cap);
      eval3tm_kernel<J><<<grid, 128, 0, ctx->stream>>>(reinterpret_cast<const uint4*>(rec), nnz,
                                                       ctx->U[0], ctx->U[1], ctx->U[2], ctx->G,
                                                       partial, nblk,
                                                       rec == ctx->rec && ctx->vt_on && ctx->env.eval_stream3 ? 1 : 0);
      CU(cudaGetLastError());
      return CMTF_OK;
    }
  }
  constexpr int J3P = round_up4(J);
  const size_t smem = sizeof(float) * (size_t)(J * J * J3P + 4 * round_up4(J) * 256);
  auto kern = eval3_kernel<J, J, J>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  const unsigned nb = (unsigned)((nnz + kEvalBlock - 1) / kEvalBlock);
  kern<<<nb, 256, smem, ctx->stream>>>(reinterpret_cast<const uint4*>(rec), nnz,
                                       ctx->U[0], ctx->U[1], ctx->U[2], ctx->G,
                                       partial);
  CU(cudaGetLastError());
  return CMTF_OK;
}

// Tensor SSE over a record array (sorted or not) -> deterministic double.
int tensor_sse(cmtf_gpu_ctx* ctx, const uint32_t* rec, uint64_t nnz,
               double* out) {
  if (nnz == 0) {
    *out = 0.0;
    return CMTF_OK;
  }
  const uint64_t nb = (nnz + kEvalBlock - 1) / kEvalBlock;
  TRY(ensure_partials(ctx, nb));
  int J = 0;
  if (ctx->order == 4 && ctx->ranks[0] == 8 && ctx->ranks[1] == 8 && ctx->ranks[2] == 8 &&
      ctx->ranks[3] == 8 && !ctx->cfg.force_generic) {
    if (ctx->env.eval_tm) {  // the contraction on tcgen05 (eval3tm.cuh)
      CU(cudaFuncSetAttribute(eval4tm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kEval4tmSmem));
      const uint64_t cap = (uint64_t)ctx->num_sms * CMTF_EVAL_TM_OCC;
      eval4tm_kernel<<<(unsigned)std::min<uint64_t>(nb, cap), 128, kEval4tmSmem, ctx->stream>>>(
          rec, nnz, ctx->U[0], ctx->U[1], ctx->U[2], ctx->U[3], ctx->G, ctx->d_partial, nb);
    } else {
      const size_t smem = sizeof(float) * 8 * 8 * 8 * 8;
      eval4_kernel<<<(unsigned)nb, 256, smem, ctx->stream>>>(rec, nnz, ctx->U[0], ctx->U[1],
                                                             ctx->U[2], ctx->U[3], ctx->G,
                                                             ctx->d_partial);
    }
    CU(cudaGetLastError());
  } else if (fast3_supported(ctx, &J)) {
    switch (J) {
      case 2: TRY(launch_eval3_t<2>(ctx, rec, nnz, ctx->d_partial)); break;
      case 4: TRY(launch_eval3_t<4>(ctx, rec, nnz, ctx->d_partial)); break;
      case 5: TRY(launch_eval3_t<5>(ctx, rec, nnz, ctx->d_partial)); break;
      case 8: TRY(launch_eval3_t<8>(ctx, rec, nnz, ctx->d_partial)); break;
      case 10: TRY(launch_eval3_t<10>(ctx, rec, nnz, ctx->d_partial)); break;
      case 16: TRY(launch_eval3_t<16>(ctx, rec, nnz, ctx->d_partial)); break;
      case 20: TRY(launch_eval3_t<20>(ctx, rec, nnz, ctx->d_partial)); break;
    }
  } else {
    const CoreShape cs = core_shape(ctx);
    const int bt = 256;
    const size_t smem = sizeof(float) * (cs.size + (bt / 32) * cs.off[cs.order]);
    CU(cudaFuncSetAttribute(eval_generic_kernel,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    eval_generic_kernel<<<(unsigned)nb, bt, smem, ctx->stream>>>(
        cs, ctx->G, rec, nnz, mode_tables(ctx), ctx->d_partial);
    CU(cudaGetLastError());
  }
  return reduce_partials(ctx, nb, out);
}

int matrix_sse(cmtf_gpu_ctx* ctx, const DevMatrix& m, double* out) {
  if (m.nnz == 0) {
    *out = 0.0;
    return CMTF_OK;
  }
  const uint64_t nb = (m.nnz + kEvalBlock - 1) / kEvalBlock;
  TRY(ensure_partials(ctx, nb));
  eval_matrix_kernel<<<(unsigned)nb, 256, 0, ctx->stream>>>(
      m.rec, m.nnz, ctx->U[m.mode], m.V, ctx->J(m.mode), ctx->JP(m.mode),
      ctx->d_partial);
  CU(cudaGetLastError());
  return reduce_partials(ctx, nb, out);
}

int row_norms(cmtf_gpu_ctx* ctx, const float* F, uint32_t rows, uint32_t J,
              uint32_t JP, const uint32_t* count, double* out) {
  const unsigned nb = std::min<unsigned>(grid_for(rows), 1024);
  TRY(ensure_partials(ctx, nb));
  row_norms_kernel<<<nb, 256, 0, ctx->stream>>>(F, rows, J, JP, count,
                                                ctx->d_partial);
  CU(cudaGetLastError());
  std::vector<double> h(nb);
  CU(cudaMemcpyAsync(h.data(), ctx->d_partial, nb * sizeof(double),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (double v : h) s += v;
  *out = s;
  return CMTF_OK;
}

int require_bundle(cmtf_gpu_ctx* ctx) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (!ctx->rec) return set_err(ctx, CMTF_EVALIDATION, "no training tensor set");
  if (!ctx->have_model)
    return set_err(ctx, CMTF_EVALIDATION, "no model (call cmtf_gpu_make_state)");
  return CMTF_OK;
}

// find_non_finite (src/trainer.cpp:239-263) on the device.
int scan_nonfinite(cmtf_gpu_ctx* ctx, std::string* offender) {
  const int narr = 1 + ctx->order + (int)ctx->mats.size();
  CU(cudaMemsetAsync(ctx->d_first, 0xff, sizeof(unsigned long long) * narr,
                     ctx->stream));
  const uint64_t core = ctx->core_size();
  nonfinite_kernel<<<grid_for(core), 256, 0, ctx->stream>>>(
      ctx->G, 1, (uint32_t)core, (uint32_t)core, ctx->d_first);
  for (int n = 0; n < ctx->order; ++n)
    nonfinite_kernel<<<grid_for((uint64_t)ctx->dims[n] * ctx->JP(n)), 256, 0,
                       ctx->stream>>>(ctx->U[n], ctx->dims[n], ctx->J(n),
                                      ctx->JP(n), ctx->d_first + 1 + n);
  for (size_t m = 0; m < ctx->mats.size(); ++m) {
    const auto& M = ctx->mats[m];
    nonfinite_kernel<<<grid_for((uint64_t)M.cols * ctx->JP(M.mode)), 256, 0,
                       ctx->stream>>>(M.V, M.cols, ctx->J(M.mode),
                                      ctx->JP(M.mode),
                                      ctx->d_first + 1 + ctx->order + m);
  }
  CU(cudaGetLastError());
  ctx->last_launches += narr;
  std::vector<unsigned long long> h(narr);
  CU(cudaMemcpyAsync(h.data(), ctx->d_first, sizeof(unsigned long long) * narr,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  offender->clear();
  const unsigned long long none = ~0ull;
  if (h[0] != none) {
    *offender = "core element " + std::to_string(h[0] + 1);
    return CMTF_OK;
  }
  for (int n = 0; n < ctx->order; ++n)
    if (h[1 + n] != none) {
      const uint64_t cols = ctx->J(n);
      *offender = "factor " + std::to_string(n + 1) + ", row " +
                  std::to_string(h[1 + n] / cols + 1) + ", column " +
                  std::to_string(h[1 + n] % cols + 1);
      return CMTF_OK;
    }
  for (size_t m = 0; m < ctx->mats.size(); ++m) {
    const auto v = h[1 + ctx->order + m];
    if (v != none) {
      const uint64_t cols = ctx->J(ctx->mats[m].mode);
      *offender = "coupled factor " + std::to_string(m + 1) + ", row " +
                  std::to_string(v / cols + 1) + ", column " +
                  std::to_string(v % cols + 1);
      return CMTF_OK;
    }
  }
  return CMTF_OK;
}

int matrix_sweep(cmtf_gpu_ctx* ctx, const DevMatrix& M0, float eta, uint64_t lo, uint64_t hi,
                 uint32_t* visits = nullptr) {
  DevMatrix M = M0;
  if (hi > M0.nnz) hi = M0.nnz;
  if (hi <= lo) return CMTF_OK;
  M.rec = M0.rec + 3 * lo;
  M.nnz = hi - lo;
  const int JP = (int)ctx->JP(M.mode);
  const int bt = 256;
  uint64_t threads = std::min<uint64_t>((uint64_t)ctx->num_sms * 2048,
                                        std::max<uint64_t>(bt, M.nnz / 16));
  if (ctx->cfg.hog_threads > 0) threads = (uint64_t)ctx->cfg.hog_threads;
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, threads / bt);
  const float w = (float)M.weight;
  float* U = ctx->U[M.mode];
#define MS_CASE(JPV)                                                           \
  case JPV:                                                                   \
    matrix_sweep_kernel<JPV><<<blocks, bt, 0, ctx->stream>>>(                   \
        M.rec, M.nnz, U, M.V, M.vreg, w, eta, ctx->cfg.nonnegative,           \
        visits ? visits + lo : nullptr);                                      \
    break;
  switch (JP) {
    MS_CASE(4) MS_CASE(8) MS_CASE(12) MS_CASE(16) MS_CASE(20) MS_CASE(24)
    MS_CASE(28) MS_CASE(32) MS_CASE(36) MS_CASE(40) MS_CASE(44) MS_CASE(48)
    MS_CASE(52) MS_CASE(56) MS_CASE(60) MS_CASE(64)
    default:
      return set_err(ctx, CMTF_EUNSUPPORTED, "matrix rank %d unsupported",
                     (int)ctx->J(M.mode));
  }
#undef MS_CASE
  CU(cudaGetLastError());
  return CMTF_OK;
}

// ---------------------------------------------------------------------
// v2 epoch kernel (order 3, equal ranks): preparation and launch
// ---------------------------------------------------------------------
constexpr int kV2Warps = 8;  // default; 12 when registers and shared memory allow

// order 4, opt kernel: the sweep's core contractions on the tensor cores
// (CMTF_V4_TC=0 selects the CUDA-core sweep, for comparison)
bool v4_tc(const cmtf_gpu_ctx* ctx) {
  if (ctx->cfg.kernel != CMTF_KERNEL_OPT) return false;
  return ctx->env.v4_tc;
}
// order 4, opt kernel on tcgen05 (hog4tm)
bool v4_tm(const cmtf_gpu_ctx* ctx) {
  return ctx->cfg.kernel == CMTF_KERNEL_OPT && ctx->env.v4_tc && ctx->env.v4_tm;
}

bool v2_supported(const cmtf_gpu_ctx* ctx, int* J) {
  if (ctx->cfg.kernel_version == 1) return false;
  if (!fast3_supported(ctx, J)) return false;
  return *J == 4 || *J == 5 || *J == 8 || *J == 10;
}

// order 3, opt kernel: the sweep's core contractions and the core gradient
// on the tcgen05 tensor cores with tensor-memory accumulators (hog3tm).
// CMTF_V3_TM=0 selects the CUDA-core hog3v2.
bool v3_tm(const cmtf_gpu_ctx* ctx) {
  if (ctx->order != 3 || ctx->cfg.kernel != CMTF_KERNEL_OPT) return false;
  int J = 0;
  if (!v2_supported(ctx, &J)) return false;
  return ctx->env.v3_tm;
}

__global__ void merge_matrix_kernel(const uint32_t* rec, uint64_t n, uint32_t m, uint64_t base,
                                    uint4* out) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x)
    out[base + e] = make_uint4(rec[3 * e], rec[3 * e + 1], rec[3 * e + 2], m);
}

__global__ void gather_uint4_kernel(const uint4* src, const uint32_t* ids, uint64_t n,
                                    uint4* dst) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n;
       s += (uint64_t)gridDim.x * blockDim.x)
    dst[s] = src[ids[s]];
}

template <int J, int NW, int E>
size_t v2_fixed_bytes() {
  return sizeof(float) * (size_t)V2Layout<J, true, NW, E>::FIXED_FLOATS;
}

// (warps per block, entries per lane) of the v2 sweep
struct V2Shape {
  int nw, e;
};

V2Shape v2_shape(const cmtf_gpu_ctx* ctx, int J) {
  // 8 warps x 2 entries per lane; one entry per lane for J <= 5, whose tiny
  // sweep leaves the row gathers exposed (config 5 at rank 5: 22.2 vs 24.1
  // ms/epoch; 4 entries per lane: 26.7 ms)
  V2Shape s{8, J <= 5 ? 1 : 2};
  if (ctx->env.v2_shape == 1) s = {8, 1};  // experiments
  if (ctx->env.v2_shape == 2) s = {8, 2};
  return s;
}

size_t v2_fixed_bytes_rt(int J, V2Shape sh) {
#define FB(JV)                                                                  \
  case JV:                                                                      \
    return sh.e == 1 ? v2_fixed_bytes<JV, 8, 1>() : v2_fixed_bytes<JV, 8, 2>();
  switch (J) {
    FB(4) FB(5) FB(8) FB(10)
  }
#undef FB
  return 0;
}

// ---------------------------------------------------------------------
// Device-side hot-row selection (the host path below is the reference for
// it): candidates are rows with count >= thr, ordered by count descending,
// then array (modes, then matrices), then row -- the order of the host's
// stable sort -- via one 64-bit radix key ((~count) << 32 | arr << 28 | row).
// ---------------------------------------------------------------------
struct HotArrays {
  const uint32_t* count[16];
  uint32_t n[16];
  int32_t* slot[16];
  uint32_t* row_of[16];
  uint32_t start[16];
  int narr;
};

__global__ void hot_cand_kernel(HotArrays h, uint64_t thr, unsigned long long* keys,
                                uint32_t* ncand, bool write) {
  const int arr = blockIdx.y;
  if (arr >= h.narr) return;
  const uint32_t* c = h.count[arr];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < h.n[arr];
       i += gridDim.x * blockDim.x) {
    const uint32_t v = c[i];
    if (v >= thr) {
      const uint32_t q = atomicAdd(ncand, 1u);
      if (write)
        keys[q] = ((unsigned long long)(0xffffffffu - v) << 32) |
                  ((unsigned long long)arr << 28) | i;
    }
  }
}

__global__ void hot_count_kernel(const unsigned long long* keys, uint64_t take, uint32_t* H,
                                 unsigned long long* keys2) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < take;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t arr = (uint32_t)(keys[q] >> 28) & 15u;
    atomicAdd(H + arr, 1u);
    keys2[q] = ((unsigned long long)arr << 32) | q;  // group by array, keep rank order
  }
}

__global__ void hot_assign_kernel(const unsigned long long* keys, const unsigned long long* keys2,
                                  uint64_t take, HotArrays h) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < take;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t arr = (uint32_t)(keys2[x] >> 32);
    const uint32_t q = (uint32_t)keys2[x];
    const uint32_t row = (uint32_t)keys[q] & ((1u << 28) - 1u);
    const uint32_t slot = (uint32_t)x - h.start[arr];
    h.row_of[arr][slot] = row;
    h.slot[arr][row] = (int32_t)slot;
  }
}

// hog3tm: flag records whose U / V row is hot (kMrecHotU / kMrecHotV)
struct MatHotSlots {
  const int32_t* su[kV2MaxMats];
  const int32_t* sv[kV2MaxMats];
};
__global__ void mrec_hot_flags_kernel(uint4* mrec, uint64_t n, MatHotSlots f) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint4 r = mrec[e];
    const uint32_t m = r.w & kMrecMat;
    uint32_t w = m;
    if (f.su[m] && f.su[m][r.x] >= 0) w |= kMrecHotU;
    if (f.sv[m] && f.sv[m][r.y] >= 0) w |= kMrecHotV;
    r.w = w;
    mrec[e] = r;
  }
}

// Build the merged random-order matrix records and the hot-row replicas.
int prepare_v2(cmtf_gpu_ctx* ctx, int J) {
  static const bool ptime = std::getenv("CMTF_PREP_TIMING") != nullptr;
  auto pt0 = std::chrono::steady_clock::now();
  auto ptick = [&](const char* what) {
    if (!ptime) return;
    cudaStreamSynchronize(ctx->stream);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "prepare_v2 %-12s %.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - pt0).count());
    pt0 = t;
  };
  drain_side(ctx);  // mrec is rebuilt below
  ptick("drain");
  const uint32_t JP = (uint32_t)round_up4(J);
  const bool four = ctx->order == 4;  // hog4: 8 warps, one entry per lane
  // grid: one block of kV2Warps warps per SM unless the caller caps workers
  const bool tm3 = !four && v3_tm(ctx);
  const V2Shape sh = four || tm3 ? V2Shape{8, 1} : v2_shape(ctx, J);
  const int NW = sh.nw;
  ctx->v2_nw = NW;
  ctx->v2_e = sh.e;
  int blocks = ctx->num_sms;
  if (ctx->cfg.hog_threads > 0) blocks = std::max(1, ctx->cfg.hog_threads / (NW * 32));
  else {
    // auto: at least ~112 entries per worker slot per epoch (at most ~1/112
    // of the data in flight; 1/1024 for order 4, whose 8^4 core and four
    // factor rows per entry make stale reads costlier: measured on
    // synth.config4_small), so small problems stay close to sequential SGD
    // while large ones fill every SM
    const uint64_t per_slot = four ? 1024 : 112;
    // hog3tm sweeps 256 entries per block per iteration like hog3v2 at E = 1,
    // but it keeps hog3v2's block count (E = 2): more blocks means more
    // replicas of every hot row and more, smaller, core pushes -- measured on
    // config 2 at 10% scale: 31 blocks +0.78% RMSE vs the reference, 15
    // blocks +0.40% (hog3v2: +0.34%)
    const uint64_t e_rule = tm3 ? 2 : (uint64_t)sh.e;
    const uint64_t cap = std::max<uint64_t>(1, ctx->nnz / (per_slot * NW * 32 * e_rule));
    blocks = (int)std::min<uint64_t>((uint64_t)blocks, cap);
  }
  ctx->v2_blocks = blocks;
  const double W = (double)blocks * NW * 32 * sh.e;  // entries in flight

  // merged matrix records (random order, seeded affine permutation)
  ctx->mnnz = 0;
  for (auto& M : ctx->mats) ctx->mnnz += M.nnz;
  if (ctx->mnnz) {
    TRY(ensure(ctx, &ctx->s_m4, &ctx->s_m4_cap, ctx->mnnz));
    TRY(ensure(ctx, &ctx->mrec, &ctx->mrec_cap, ctx->mnnz));
    TRY(ensure(ctx, &ctx->s_ids, &ctx->s_ids_cap, ctx->mnnz));
    uint64_t base = 0;
    ctx->mat_base.assign(ctx->mats.size() + 1, 0);
    for (size_t m = 0; m < ctx->mats.size(); ++m) {
      const auto& M = ctx->mats[m];
      ctx->mat_base[m] = base;
      if (M.nnz)
        merge_matrix_kernel<<<grid_for(M.nnz), 256, 0, ctx->stream>>>(M.rec, M.nnz,
                                                                      (uint32_t)m, base,
                                                                      ctx->s_m4);
      base += M.nnz;
    }
    ctx->mat_base[ctx->mats.size()] = base;
    uint64_t pa = 1, pb = 0;  // caller order keeps the concatenation
    if (ctx->cfg.order_policy != 2) affine_params(ctx->mnnz, ctx->cfg.seed + 1, &pa, &pb);
    scatter_affine_kernel<<<grid_for(ctx->mnnz), 256, 0, ctx->stream>>>(
        reinterpret_cast<const uint32_t*>(ctx->s_m4), ctx->mnnz, 4, pa, pb,
        reinterpret_cast<uint32_t*>(ctx->mrec), ctx->s_ids);
    CU(cudaGetLastError());
  }

  ptick("merge");
  // hot rows: expected concurrent updates count * W / nnz >= tau, by count,
  // within the shared-memory budget left after the fixed layout
  float tau = ctx->cfg.hot_tau == 0.f ? 0.5f : ctx->cfg.hot_tau;
  size_t fixed = four ? (v4_tm(ctx) ? (size_t)TM4Layout::FIXED_BYTES
                                    : sizeof(float) *
                                          (size_t)(v4_tc(ctx) ? V4Layout<8, 8, true>::FIXED_FLOATS
                                                              : V4Layout<8, 8>::FIXED_FLOATS))
                      : v2_fixed_bytes_rt(J, sh);
  if (tm3) {
    switch (J) {
      case 4: fixed = (size_t)TMLayout<4>::FIXED_BYTES; break;
      case 5: fixed = (size_t)TMLayout<5>::FIXED_BYTES; break;
      case 8: fixed = (size_t)TMLayout<8>::FIXED_BYTES; break;
      case 10: fixed = (size_t)TMLayout<10>::FIXED_BYTES; break;
    }
  }
  const size_t limit = 227 * 1024 - 2048;  // room for a co-resident gather block
  const size_t budget_floats = fixed < limit ? (limit - fixed) / sizeof(float) : 0;
  const uint64_t thr = tau > 0 ? (uint64_t)std::ceil(tau * (double)ctx->nnz / W) : ~0ull;
  const size_t per_row = JP + 3;
  const size_t slack = 4 * (ctx->order + ctx->mats.size());  // alignment padding
  const uint64_t max_take = budget_floats > slack ? (budget_floats - slack) / per_row : 0;
  uint32_t off = (uint32_t)(fixed / sizeof(float));
  // per-array replica layout and device tables for H hot rows
  auto place = [&](cmtf_gpu_ctx::HotHost& h, uint32_t H, uint32_t nrows) -> int {
    h.H = H;
    if (!h.H) return CMTF_OK;
    TRY(ensure(ctx, &h.slot, &h.slot_cap, nrows));
    TRY(ensure(ctx, &h.row_of, &h.row_cap, h.H));
    const uint64_t need = (uint64_t)blocks * h.H * JP;
    if (h.base_cap < need) {
      TRY(dalloc(ctx, &h.base, need));
      h.base_cap = need;
    }
    h.off = off;  // float4-aligned (off and H*JP are multiples of 4)
    off += h.H * JP;
    h.stat_off = off;
    off += (3 * h.H + 3) & ~3u;
    return CMTF_OK;
  };
  bool device_sel = !ctx->env.hot_host && ctx->order + ctx->mats.size() <= 16 &&
                    ctx->order <= 8;
  for (int n = 0; n < ctx->order; ++n) device_sel = device_sel && ctx->dims[n] < (1u << 28);
  for (auto& M : ctx->mats) device_sel = device_sel && M.cols < (1u << 28);
  if (device_sel) {
    HotArrays ha{};
    ha.narr = 16;
    for (int n = 0; n < ctx->order; ++n) {
      ha.count[n] = ctx->count[n];
      ha.n[n] = tau > 0 ? ctx->dims[n] : 0;
    }
    for (size_t m = 0; m < ctx->mats.size(); ++m) {
      ha.count[8 + m] = ctx->mats[m].count;
      ha.n[8 + m] = tau > 0 ? ctx->mats[m].cols : 0;
    }
    if (!ctx->hs_cnt) TRY(dalloc(ctx, &ctx->hs_cnt, 17));
    uint32_t hcnt[17] = {0};
    CU(cudaMemsetAsync(ctx->hs_cnt, 0, 17 * sizeof(uint32_t), ctx->stream));
    const uint64_t th = std::max<uint64_t>(thr, 1);
    hot_cand_kernel<<<dim3(64, 16), 256, 0, ctx->stream>>>(ha, th, nullptr, ctx->hs_cnt, false);
    CU(cudaMemcpyAsync(hcnt, ctx->hs_cnt, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    const uint64_t ncand = hcnt[0];
    const uint64_t take = std::min<uint64_t>(ncand, max_take);
    uint32_t H[16] = {0};
    if (take) {
      // [0, n): candidates, then (array, rank) keys; [n, 2n): sorted
      // candidates; [2n, 3n): sorted (array, rank) keys
      TRY(ensure(ctx, &ctx->hs_keys, &ctx->hs_keys_cap, 3 * ncand));
      unsigned long long* k_in = ctx->hs_keys;
      unsigned long long* k_out = ctx->hs_keys + ncand;
      CU(cudaMemsetAsync(ctx->hs_cnt, 0, 17 * sizeof(uint32_t), ctx->stream));
      hot_cand_kernel<<<dim3(64, 16), 256, 0, ctx->stream>>>(ha, th, k_in, ctx->hs_cnt, true);
      size_t tb = 0;
      CU(cub::DeviceRadixSort::SortKeys(nullptr, tb, k_in, k_out, (int)ncand, 0, 64,
                                        ctx->stream));
      TRY(ensure(ctx, &ctx->hs_tmp, &ctx->hs_tmp_cap, tb));
      CU(cub::DeviceRadixSort::SortKeys(ctx->hs_tmp, tb, k_in, k_out, (int)ncand, 0, 64,
                                        ctx->stream));
      // k_out = sorted candidates; k_in is reused for the (array, rank) keys
      hot_count_kernel<<<grid_for(take), 256, 0, ctx->stream>>>(k_out, take, ctx->hs_cnt + 1,
                                                                k_in);
      CU(cudaMemcpyAsync(H, ctx->hs_cnt + 1, 16 * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                         ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    }
    uint32_t start = 0;
    for (int n = 0; n < ctx->order; ++n) {
      TRY(place(ctx->hot[n], H[n], ctx->dims[n]));
      ha.slot[n] = ctx->hot[n].slot;
      ha.row_of[n] = ctx->hot[n].row_of;
      ha.start[n] = start;
      start += H[n];
      if (H[n]) CU(cudaMemsetAsync(ctx->hot[n].slot, 0xff, ctx->dims[n] * sizeof(int32_t),
                                   ctx->stream));
    }
    for (int n = ctx->order; n < 8; ++n) ha.start[n] = start;
    for (size_t m = 0; m < ctx->mats.size(); ++m) {
      TRY(place(ctx->hotV[m], H[8 + m], ctx->mats[m].cols));
      ha.slot[8 + m] = ctx->hotV[m].slot;
      ha.row_of[8 + m] = ctx->hotV[m].row_of;
      ha.start[8 + m] = start;
      start += H[8 + m];
      if (H[8 + m]) CU(cudaMemsetAsync(ctx->hotV[m].slot, 0xff, ctx->mats[m].cols * sizeof(int32_t),
                                       ctx->stream));
    }
    if (take) {
      size_t tb = 0;
      unsigned long long* k2_in = ctx->hs_keys;
      unsigned long long* k_sorted = ctx->hs_keys + ncand;
      unsigned long long* k2_out = ctx->hs_keys + 2 * ncand;
      CU(cub::DeviceRadixSort::SortKeys(nullptr, tb, k2_in, k2_out, (int)take, 0, 36,
                                        ctx->stream));
      TRY(ensure(ctx, &ctx->hs_tmp, &ctx->hs_tmp_cap, tb));
      CU(cub::DeviceRadixSort::SortKeys(ctx->hs_tmp, tb, k2_in, k2_out, (int)take, 0, 36,
                                        ctx->stream));
      hot_assign_kernel<<<grid_for(take), 256, 0, ctx->stream>>>(k_sorted, k2_out, take, ha);
      CU(cudaGetLastError());
    }
    if (ctx->env.hot_check) {
      CU(cudaStreamSynchronize(ctx->stream));
      // test hook: the host's stable-sort selection must give the same rows
      // in the same slots
      struct C2 { uint32_t count; int arr; uint32_t row; };
      std::vector<C2> cand;
      std::vector<std::vector<uint32_t>> cnt(16);
      for (int a = 0; a < 16; ++a) {
        if (!ha.n[a]) continue;
        cnt[a].resize(ha.n[a]);
        CU(cudaMemcpy(cnt[a].data(), ha.count[a], ha.n[a] * sizeof(uint32_t),
                      cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < ha.n[a]; ++i)
          if (cnt[a][i] >= th) cand.push_back({cnt[a][i], a, i});
      }
      std::stable_sort(cand.begin(), cand.end(),
                       [](const C2& x, const C2& y) { return x.count > y.count; });
      std::vector<std::vector<uint32_t>> want(16);
      for (uint64_t q = 0; q < std::min<uint64_t>(cand.size(), max_take); ++q)
        want[cand[q].arr].push_back(cand[q].row);
      for (int a = 0; a < 16; ++a) {
        if (want[a].size() != H[a])
          return set_err(ctx, CMTF_ECUDA, "hot check: array %d has %u rows, host %zu", a, H[a],
                         want[a].size());
        if (!H[a]) continue;
        std::vector<uint32_t> got(H[a]);
        std::vector<int32_t> sl(ha.n[a]);
        CU(cudaMemcpy(got.data(), ha.row_of[a], H[a] * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(sl.data(), ha.slot[a], ha.n[a] * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (uint32_t q = 0; q < H[a]; ++q)
          if (got[q] != want[a][q] || sl[want[a][q]] != (int32_t)q)
            return set_err(ctx, CMTF_ECUDA, "hot check: array %d slot %u differs", a, q);
        uint64_t nhot = 0;
        for (int32_t v : sl) nhot += v >= 0;
        if (nhot != H[a]) return set_err(ctx, CMTF_ECUDA, "hot check: array %d stray slots", a);
      }
    }
  } else {
    struct Cand {
      uint32_t count;
      int arr;  // 0..N-1 modes, 100+m matrices
      uint32_t row;
    };
    std::vector<Cand> cand;
    std::vector<std::vector<uint32_t>> hcounts(ctx->order), vcounts(ctx->mats.size());
    for (int n = 0; n < ctx->order; ++n) {
      hcounts[n].resize(ctx->dims[n]);
      CU(cudaMemcpy(hcounts[n].data(), ctx->count[n], ctx->dims[n] * sizeof(uint32_t),
                    cudaMemcpyDeviceToHost));
      if (tau > 0)
        for (uint32_t i = 0; i < ctx->dims[n]; ++i)
          if (hcounts[n][i] >= std::max<uint64_t>(thr, 1)) cand.push_back({hcounts[n][i], n, i});
    }
    for (size_t m = 0; m < ctx->mats.size(); ++m) {
      const auto& M = ctx->mats[m];
      vcounts[m].resize(M.cols);
      CU(cudaMemcpy(vcounts[m].data(), M.count, M.cols * sizeof(uint32_t),
                    cudaMemcpyDeviceToHost));
      // a V row's updates are spread over the same iterations as the tensor's
      if (tau > 0)
        for (uint32_t j = 0; j < M.cols; ++j)
          if (vcounts[m][j] >= std::max<uint64_t>(thr, 1))
            cand.push_back({vcounts[m][j], 100 + (int)m, j});
    }
    ptick("counts+cand");
    std::stable_sort(cand.begin(), cand.end(),
                     [](const Cand& x, const Cand& y) { return x.count > y.count; });
    size_t take = std::min<size_t>(cand.size(), max_take);
    std::vector<std::vector<uint32_t>> rows_of(ctx->order), vrows_of(ctx->mats.size());
    for (size_t q = 0; q < take; ++q) {
      if (cand[q].arr < 100) rows_of[cand[q].arr].push_back(cand[q].row);
      else vrows_of[cand[q].arr - 100].push_back(cand[q].row);
    }
    auto build = [&](cmtf_gpu_ctx::HotHost& h, const std::vector<uint32_t>& rows,
                     uint32_t nrows) -> int {
      h.H = (uint32_t)rows.size();
      if (!h.H) return CMTF_OK;
      std::vector<int32_t> slot(nrows, -1);
      for (uint32_t s = 0; s < h.H; ++s) slot[rows[s]] = (int32_t)s;
      TRY(ensure(ctx, &h.slot, &h.slot_cap, nrows));
      TRY(ensure(ctx, &h.row_of, &h.row_cap, h.H));
      CU(cudaMemcpy(h.slot, slot.data(), nrows * sizeof(int32_t), cudaMemcpyHostToDevice));
      CU(cudaMemcpy(h.row_of, rows.data(), h.H * sizeof(uint32_t), cudaMemcpyHostToDevice));
      const uint64_t need = (uint64_t)blocks * h.H * JP;
      if (h.base_cap < need) {
        TRY(dalloc(ctx, &h.base, need));
        h.base_cap = need;
      }
      h.off = off;  // float4-aligned (off and H*JP are multiples of 4)
      off += h.H * JP;
      h.stat_off = off;
      off += (3 * h.H + 3) & ~3u;
      return CMTF_OK;
    };
    CU(cudaStreamSynchronize(ctx->stream));  // the previous sweep may still read the slots
    for (int n = 0; n < ctx->order; ++n) TRY(build(ctx->hot[n], rows_of[n], ctx->dims[n]));
    for (size_t m = 0; m < ctx->mats.size(); ++m)
      TRY(build(ctx->hotV[m], vrows_of[m], ctx->mats[m].cols));
  }
  ptick("build");
  if (tm3 && ctx->mnnz && CMTF_TM_MPF) {
    MatHotSlots f{};
    for (size_t m = 0; m < ctx->mats.size(); ++m) {
      const int mode = ctx->mats[m].mode;
      f.su[m] = ctx->hot[mode].H ? ctx->hot[mode].slot : nullptr;
      f.sv[m] = ctx->hotV[m].H ? ctx->hotV[m].slot : nullptr;
    }
    mrec_hot_flags_kernel<<<grid_for(ctx->mnnz), 256, 0, ctx->stream>>>(ctx->mrec, ctx->mnnz, f);
    CU(cudaGetLastError());
  }
  // hog3tm: per-thread staging rows for the bulk asynchronous row steps
  // (3 rows x JP floats per thread) when they fit beside the hot replicas
  // Not with the L2-blocked order: its mode-1/2 rows are L2-resident and
  // REDs on them are cheap, while each bulk reduction costs the issuing warp
  // a 32-lane uniform-operand loop (config 5 @1e9: 244 -> 213 ms/epoch with
  // REDs; config 3 unchanged).  CMTF_TM_BULK overrides.
  ctx->tm_stage_off = 0;
  const bool want_bulk = ctx->env.tm_bulk > 0 || (ctx->env.tm_bulk < 0 && !vt_wanted(ctx));
  if (tm3 && !ctx->cfg.nonnegative && !ctx->env.tm_red && want_bulk) {
    const uint32_t so = (off + 3) & ~3u;
    const size_t need = (size_t)(so + 256 * 3 * JP) * sizeof(float);
    if (need <= limit) {
      ctx->tm_stage_off = so;
      off = so + 256 * 3 * JP;
    }
  }
  ctx->v2_smem = (size_t)off * sizeof(float);
  // hog3tm allocates all 512 TMEM columns: keep it at one block per SM
  if (tm3) ctx->v2_smem = std::max<size_t>(ctx->v2_smem, 116 * 1024);
  ctx->v2_dirty = false;
  return CMTF_OK;
}

template <int J, bool OPT, int NW, int E>
int launch_v2_nw(cmtf_gpu_ctx* ctx, const Hog3v2Args& args) {
  auto kern = hog3v2_kernel<J, OPT, NW, E>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)ctx->v2_smem));
  kern<<<ctx->v2_blocks, NW * 32, ctx->v2_smem, ctx->stream>>>(args);
  CU(cudaGetLastError());
  return CMTF_OK;
}

template <int J, bool OPT>
int launch_v2_t(cmtf_gpu_ctx* ctx, const Hog3v2Args& args) {
  if (ctx->v2_e == 1) return launch_v2_nw<J, OPT, 8, 1>(ctx, args);
  return launch_v2_nw<J, OPT, 8, 2>(ctx, args);
}


template <int J>
int launch_v3tm(cmtf_gpu_ctx* ctx, const Hog3v2Args& args) {
  auto kern = hog3tm_kernel<J>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)ctx->v2_smem));
  kern<<<ctx->v2_blocks, 8 * 32, ctx->v2_smem, ctx->stream>>>(args);
  CU(cudaGetLastError());
  return CMTF_OK;
}

// Fill the sweep arguments shared by hog3v2 and hog4 for tensor records
// [t_lo, t_hi) and matrix records [m_lo[m], m_hi[m]) (NULL ranges = every
// matrix entry).  Returns false when there is nothing to sweep.
template <int NM, class Args>
bool fill_sweep_args(cmtf_gpu_ctx* ctx, Args& a, float eta, uint64_t t_lo, uint64_t t_hi,
                     const uint64_t* m_lo, const uint64_t* m_hi) {
  a.nnz = t_hi - t_lo;
  a.mrec = ctx->mrec;
  a.n_mat = (int)ctx->mats.size();
  if (m_lo && m_hi) {
    a.n_mr = (int)ctx->mats.size();
    a.mnnz = 0;
    for (size_t m = 0; m < ctx->mats.size(); ++m) {
      a.mr_lo[m] = ctx->mat_base[m] + m_lo[m];
      a.mr_n[m] = m_hi[m] - m_lo[m];
      a.mnnz += a.mr_n[m];
    }
  } else {
    a.n_mr = 1;
    a.mr_lo[0] = 0;
    a.mr_n[0] = ctx->mnnz;
    a.mnnz = ctx->mnnz;
  }
  if (a.nnz == 0 && a.mnnz == 0) return false;
  // hot-row merge window: 16 iterations (hog3tm: 32 -- its 256-entry
  // iterations are half as long; config 2 full scale -6% epoch time, RMSE
  // unchanged, 10% scale +0.51% vs +0.37%)
  const int F = ctx->cfg.flush_every > 0 ? ctx->cfg.flush_every : (v3_tm(ctx) ? 32 : 16);
  const double W = (double)ctx->v2_blocks * ctx->v2_nw * 32;
  // entries processed GPU-wide between two flushes of one warp: W * F * E
  // (an epoch shorter than one window: every row gets at most its count)
  const double win = std::min(W * F * ctx->v2_e, (double)std::max<uint64_t>(1, ctx->nnz));
  const float nhat_scale = (float)(win / (double)std::max<uint64_t>(1, ctx->nnz));
  auto hd = [&](const cmtf_gpu_ctx::HotHost& h, const uint32_t* count, bool shared) {
    HotDesc d{};
    d.slot = h.H ? h.slot : nullptr;
    d.row_of = h.row_of;
    d.count = count;
    d.H = h.H;
    d.off = h.off;
    d.stat_off = h.stat_off;
    d.base = h.base;
    // replicated parameters are updated by `world` ranks at once
    d.nhat_scale = nhat_scale * (shared ? (float)ctx->world : 1.f);
    return d;
  };
  for (int n = 0; n < NM; ++n) {
    a.U[n] = ctx->U[n];
    a.reg[n] = ctx->reg[n];
    a.hot[n] = hd(ctx->hot[n], ctx->count[n], (ctx->shared_modes >> n) & 1u);
  }
  for (size_t m = 0; m < ctx->mats.size(); ++m) {
    const auto& M = ctx->mats[m];
    a.mats[m].mode = M.mode;
    a.mats[m].V = M.V;
    a.mats[m].vreg = M.vreg;
    a.mats[m].weight = (float)M.weight;
    a.mats[m].hotV = hd(ctx->hotV[m], M.count, (ctx->shared_mats >> m) & 1u);
  }
  a.G = ctx->G;
  a.eta = eta;
  const uint64_t nnz_all = ctx->nnz_global ? ctx->nnz_global : ctx->nnz;
  a.core_reg = (float)(ctx->cfg.lambda_reg / (double)nnz_all);
  a.kappa = ctx->cfg.kappa > 0.f ? ctx->cfg.kappa : 0.5f;
  a.kappa_core = ctx->cfg.kappa_core > 0.f ? ctx->cfg.kappa_core : 2.0f;
  // core pushes: every iteration, or -- hog3tm with long sweeps (>= 2048
  // iterations per lane and epoch: configs 3 and 5) -- every second one: the
  // push (TMEM read-out, coalesced REDs, refresh of the shared core copies)
  // is 13% of an iteration; config 5 @1e9 195 -> 187 ms/epoch with the same
  // RMSE after 8 epochs (0.10042), config 5 @1e8 0.32399 vs 0.32407.  Short
  // sweeps keep every iteration (config 2: RMSE +0.2% otherwise).
  const bool long_sweep = ctx->order == 3 && v3_tm(ctx) && W > 0 &&
                          (double)ctx->nnz / W >= 2048.0;
  // hog4tm's push is a block-wide step (two block barriers, a 4096-element
  // refresh of the fp16 core copies): every 8th iteration on long sweeps,
  // scaled down to every iteration below 1024 iterations per lane
  int fg4 = 1;
  if (ctx->order == 4 && v4_tm(ctx) && W > 0)
    fg4 = (int)std::min(8.0, std::max(1.0, std::floor((double)ctx->nnz / W / 512.0)));
  const int FG = ctx->cfg.core_flush_every > 0 ? ctx->cfg.core_flush_every
                                               : (ctx->order == 4 ? fg4 : (long_sweep ? 2 : 1));
  a.nhat_core = (float)(W * FG * ctx->v2_e * ctx->world);
  a.flush_every = F;
  a.core_every = FG;
  a.nonneg = ctx->cfg.nonnegative;
  a.probe = ctx->probe;
  a.probe_core = ctx->probe_core;
  a.visits = ctx->cfg.debug_count_visits ? ctx->visits + t_lo : nullptr;
  a.mvisits = ctx->cfg.debug_count_visits ? ctx->mvisits : nullptr;
  ctx->hog_threads_used = (int)W;
  return true;
}

// One v2 sweep (order 3) over a tensor range and matrix ranges.
int v2_sweep(cmtf_gpu_ctx* ctx, int J, float eta, uint64_t t_lo, uint64_t t_hi,
             const uint64_t* m_lo, const uint64_t* m_hi) {
  if (ctx->v2_dirty) TRY(prepare_v2(ctx, J));
  const bool mshuf = ctx->cfg.order_policy == 1 && !(m_lo && m_hi);
  if (mshuf) TRY(take_matrix_order(ctx));
  Hog3v2Args a{};
  if (!fill_sweep_args<3>(ctx, a, eta, t_lo, t_hi, m_lo, m_hi)) return CMTF_OK;
  const bool whole = t_lo == 0 && t_hi == ctx->nnz && !(m_lo && m_hi);
  const bool relayout = !ctx->vt_on && whole && vt_wanted(ctx);
  // rrec: the regulariser coefficients beside the records, built from this
  // epoch's record order (no gather of the next order is pending here; from
  // now on the reshuffle keeps rrec aligned with rec); a blocked layout keeps
  // its entry ids in the fourth word.  When the blocked layout is about to be
  // made from a fresh upload (ids in closed form), the coefficients are
  // looked up AFTER the partition: two of the three lookups per record then
  // fall into the stratum's row blocks (L2) instead of three 40 MB tables,
  // and the partition's first pass does not read rrec at all.
  const bool rrec_late = v3_tm(ctx) && !ctx->rrec_valid && relayout && ctx->pos_affine &&
                         !ctx->pos_ids && ctx->env.rrec_late;
  auto build_rrec = [&](int keep_w) -> int {
    TRY(ensure(ctx, &ctx->rrec, &ctx->rrec_cap, ctx->nnz));
    build_rrec_kernel<<<grid_for(ctx->nnz), 256, 0, ctx->stream>>>(
        reinterpret_cast<const uint4*>(ctx->rec), ctx->nnz, ctx->reg[0], ctx->reg[1],
        ctx->reg[2], ctx->rrec, keep_w);
    CU(cudaGetLastError());
    ctx->rrec_valid = true;
    ctx->last_launches += 1;
    return CMTF_OK;
  };
  if (v3_tm(ctx) && !ctx->rrec_valid && !rrec_late) TRY(build_rrec(ctx->vt_on ? 1 : 0));
  if (relayout) {
    if (rrec_late) TRY(ensure(ctx, &ctx->rrec, &ctx->rrec_cap, ctx->nnz));
    TRY(vt_setup(ctx, blocks_wanted(ctx), /*rrec_in=*/!rrec_late));
    if (rrec_late) TRY(build_rrec(1));
    TRY(vt_table(ctx, (uint64_t)ctx->epoch));
  }
  a.rec = reinterpret_cast<const uint4*>(ctx->rec) + t_lo;  // after a re-layout
  // row gathers through L1 where the factor tables miss L2 (hog3tm, hog3v2: cp_async16_sel)
  a.gather_ca = ctx->env.tm_gather_ca >= 0 ? ctx->env.tm_gather_ca : (tables_beyond_l2(ctx) ? 1 : 0);
  TRY(prefetch_orders(ctx, mshuf && t_lo == 0 && t_hi == ctx->nnz, mshuf));
  ctx->kernel_which = 3;
  const bool opt = ctx->cfg.kernel == CMTF_KERNEL_OPT;
  if (v3_tm(ctx)) {
    a.rrec = ctx->rrec + t_lo;
    a.stage_off = ctx->tm_stage_off;
    a.bulk_mask = ctx->env.tm_bulk >= 0 ? ctx->env.tm_bulk : 7;
    a.g_alt = ctx->env.tm_galt ? 1 : 0;
    a.vtab = ctx->vt_on && whole ? ctx->d_vtab : nullptr;
    a.strided = ctx->env.tm_strided || (a.vtab && ctx->blk_B > 1);
    a.pf_l2 = ctx->env.tm_pfl2 > 0 ? 1 : 0;  // measured +10% epoch time on config 5: off
    ctx->kernel_which = 5;
    switch (J) {
      case 4: return launch_v3tm<4>(ctx, a);
      case 5: return launch_v3tm<5>(ctx, a);
      case 8: return launch_v3tm<8>(ctx, a);
      case 10: return launch_v3tm<10>(ctx, a);
    }
  }
#define V2_CASE(JV)                                                            \
  case JV:                                                                     \
    return opt ? launch_v2_t<JV, true>(ctx, a) : launch_v2_t<JV, false>(ctx, a);
  switch (J) {
    V2_CASE(4) V2_CASE(5) V2_CASE(8) V2_CASE(10)
  }
#undef V2_CASE
  return set_err(ctx, CMTF_EUNSUPPORTED, "no v2 kernel for J=%d", J);
}

// order 4, all ranks 8 (BASELINE configs[3])
bool v4_supported(const cmtf_gpu_ctx* ctx) {
  if (ctx->order != 4 || ctx->cfg.force_generic || ctx->cfg.kernel_version == 1) return false;
  for (int n = 0; n < 4; ++n)
    if (ctx->ranks[n] != 8) return false;
  return ctx->mats.size() <= (size_t)kV2MaxMats;
}

template <int MODE>
int launch_v4(cmtf_gpu_ctx* ctx, const Hog4Args& args) {
  auto kern = hog4_kernel<8, MODE, 8>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)ctx->v2_smem));
  kern<<<ctx->v2_blocks, 8 * 32, ctx->v2_smem, ctx->stream>>>(args);
  CU(cudaGetLastError());
  return CMTF_OK;
}

int v4_sweep(cmtf_gpu_ctx* ctx, float eta, uint64_t t_lo, uint64_t t_hi, const uint64_t* m_lo,
             const uint64_t* m_hi) {
  if (ctx->v2_dirty) TRY(prepare_v2(ctx, 8));
  const bool mshuf = ctx->cfg.order_policy == 1 && !(m_lo && m_hi);
  if (mshuf) TRY(take_matrix_order(ctx));
  Hog4Args a{};
  a.rec = ctx->rec + t_lo * 5;
  if (!fill_sweep_args<4>(ctx, a, eta, t_lo, t_hi, m_lo, m_hi)) return CMTF_OK;
  TRY(prefetch_orders(ctx, mshuf && t_lo == 0 && t_hi == ctx->nnz, mshuf));
  ctx->kernel_which = 2;
  if (ctx->cfg.kernel != CMTF_KERNEL_OPT) return launch_v4<0>(ctx, a);
  if (v4_tm(ctx)) {
    ctx->kernel_which = 6;
    CU(cudaFuncSetAttribute(hog4tm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ctx->v2_smem));
    hog4tm_kernel<<<ctx->v2_blocks, 256, ctx->v2_smem, ctx->stream>>>(a);
    CU(cudaGetLastError());
    return CMTF_OK;
  }
  return v4_tc(ctx) ? launch_v4<2>(ctx, a) : launch_v4<1>(ctx, a);
}

int hogwild_tensor_sweep(cmtf_gpu_ctx* ctx, float eta, uint64_t t_lo, uint64_t t_hi) {
  const bool opt = ctx->cfg.kernel == CMTF_KERNEL_OPT;
  int J = 0;
  if (t_hi <= t_lo) return CMTF_OK;
  if (fast3_supported(ctx, &J)) {
    Hog3Args a{};
    a.rec = reinterpret_cast<const uint4*>(ctx->rec) + t_lo;
    a.nnz = t_hi - t_lo;
    for (int n = 0; n < 3; ++n) {
      a.U[n] = ctx->U[n];
      a.reg[n] = ctx->reg[n];
    }
    a.G = ctx->G;
    a.eta = eta;
    a.eta_core = eta;
    a.core_reg = (float)(ctx->cfg.lambda_reg / (double)nnz_all_of(ctx));
    a.nonneg = ctx->cfg.nonnegative;
    a.visits = ctx->cfg.debug_count_visits ? ctx->visits + t_lo : nullptr;
    ctx->kernel_which = 1;
    return launch_hog3(ctx, J, a, opt, ctx->cfg.order_policy == 1 ? 0 : ctx->sort_mode,
                       ctx->cfg.hog_threads);
  }
  ctx->kernel_which = 0;
  HogArgs a{};
  a.cs = core_shape(ctx);
  a.G = ctx->G;
  a.rec = ctx->rec + t_lo * (ctx->order + 1);
  a.nnz = t_hi - t_lo;
  a.mt = mode_tables(ctx);
  a.eta = eta;
  a.core_reg = (float)(ctx->cfg.lambda_reg / (double)nnz_all_of(ctx));
  a.nonneg = ctx->cfg.nonnegative;
  a.visits = ctx->cfg.debug_count_visits ? ctx->visits + t_lo : nullptr;
  const int bt = 256;
  const size_t smem =
      sizeof(float) * (2 * a.cs.size + (bt / 32) * 2 * a.cs.off[a.cs.order]);
  auto kern = opt ? hogwild_generic_kernel<true> : hogwild_generic_kernel<false>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, bt, smem));
  if (per_sm < 1) per_sm = 1;
  int blocks = ctx->num_sms * per_sm;
  if (ctx->cfg.hog_threads > 0) blocks = std::max(1, ctx->cfg.hog_threads / 32 / (bt / 32));
  else {
    const uint64_t cap = std::max<uint64_t>(1, a.nnz / (1024ull * (bt / 32)));
    blocks = (int)std::min<uint64_t>((uint64_t)blocks, cap);
  }
  ctx->hog_threads_used = blocks * (bt / 32);
  kern<<<blocks, bt, smem, ctx->stream>>>(a);
  CU(cudaGetLastError());
  return CMTF_OK;
}


int serial_epoch(cmtf_gpu_ctx* ctx, float eta) {
  // build_schedule / shuffle_schedule (src/trainer.cpp:114-128), applied to
  // the persisted schedule so shuffles accumulate across epochs.
  uint64_t total = ctx->nnz;
  for (auto& m : ctx->mats) total += m.nnz;
  if (ctx->schedule.size() != total) {
    ctx->schedule.resize(total);
    for (uint64_t i = 0; i < total; ++i) ctx->schedule[i] = i;
  }
  if (ctx->schedule_given) {
    ctx->schedule_given = false;  // the caller's order for this epoch, as given
  } else {
    auto rng = make_rng(ctx->cfg.seed, 0x02, (uint64_t)ctx->epoch);
    for (uint64_t i = total; i > 1; --i)
      std::swap(ctx->schedule[i - 1], ctx->schedule[bounded(rng, i)]);
  }
  if (ctx->d_sched_cap < total) {
    TRY(dalloc(ctx, &ctx->d_sched, total));
    ctx->d_sched_cap = total;
  }
  CU(cudaMemcpyAsync(ctx->d_sched, ctx->schedule.data(), total * sizeof(uint64_t),
                     cudaMemcpyHostToDevice, ctx->stream));
  TRY(normalize_pos(ctx));
  SerialArgs a{};
  a.cs = core_shape(ctx);
  a.G = ctx->G;
  a.rec = ctx->rec;
  a.pos = ctx->pos;
  a.mt = mode_tables(ctx);
  a.nnz = ctx->nnz;
  a.n_mat = (int)ctx->mats.size();
  a.mat_base[0] = ctx->nnz;
  for (size_t m = 0; m < ctx->mats.size(); ++m) {
    const auto& M = ctx->mats[m];
    a.mats[m] = MatDev{M.mode, M.rows, M.cols, M.nnz, M.rec, M.pos,
                       M.V, M.vreg, M.count, (float)M.weight};
    a.mat_base[m + 1] = a.mat_base[m] + M.nnz;
  }
  a.sched = ctx->d_sched;
  a.n_sched = total;
  a.eta = eta;
  a.eta_core = eta;  // P = 1: core step eta (src/trainer.cpp:211-219)
  a.core_reg = (float)(ctx->cfg.lambda_reg / (double)nnz_all_of(ctx));
  a.nonneg = ctx->cfg.nonnegative;
  const int bt = 256;
  const size_t smem = sizeof(float) * (a.cs.size + 2 * a.cs.off[a.cs.order] + 32);
  auto kern = ctx->cfg.kernel == CMTF_KERNEL_OPT ? serial_epoch_kernel<true>
                                                  : serial_epoch_kernel<false>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  kern<<<1, bt, smem, ctx->stream>>>(a);
  CU(cudaGetLastError());
  ctx->kernel_which = 0;
  ctx->hog_threads_used = 1;
  return CMTF_OK;
}

int validate_config(const cmtf_gpu_config* c) {
  if (!c) return set_err(nullptr, CMTF_EVALIDATION, "null config");
  if (c->order < 2 || c->order > kMaxOrder)
    return set_err(nullptr, CMTF_EVALIDATION,
                   "tensor order must be between 2 and %d on the device", kMaxOrder);
  if (!c->ranks) return set_err(nullptr, CMTF_EVALIDATION, "null ranks");
  uint64_t size = 1;
  for (int n = 0; n < c->order; ++n) {
    if (c->ranks[n] == 0)
      return set_err(nullptr, CMTF_EVALIDATION, "ranks must be positive");
    if (c->ranks[n] > (uint32_t)kMaxRank)
      return set_err(nullptr, CMTF_EUNSUPPORTED, "rank %u exceeds device limit %d",
                     c->ranks[n], kMaxRank);
    size *= c->ranks[n];
  }
  if (size > (uint64_t)kMaxCore)
    return set_err(nullptr, CMTF_EUNSUPPORTED,
                   "core of %llu elements exceeds device limit %d",
                   (unsigned long long)size, kMaxCore);
  if (c->core_structure != 0 && c->core_structure != 1)
    return set_err(nullptr, CMTF_EVALIDATION, "unknown core structure %d", c->core_structure);
  // validate_config (src/trainer.cpp:69-72)
  if (c->core_structure == 1)
    for (int n = 1; n < c->order; ++n)
      if (c->ranks[n] != c->ranks[0])
        return set_err(nullptr, CMTF_EVALIDATION, "CP mode requires equal ranks on every mode");
  // src/trainer.cpp:79-91
  if (!(c->eta0 >= 0)) return set_err(nullptr, CMTF_EVALIDATION, "eta0 must be nonnegative");
  if (!(c->mu >= 0)) return set_err(nullptr, CMTF_EVALIDATION, "mu must be nonnegative");
  if (!(c->lambda_reg >= 0))
    return set_err(nullptr, CMTF_EVALIDATION, "lambda_reg must be nonnegative");
  if (c->workers < 1) return set_err(nullptr, CMTF_EVALIDATION, "workers must be >= 1");
  if (c->max_epochs < 0)
    return set_err(nullptr, CMTF_EVALIDATION, "max_epochs must be nonnegative");
  if (!(c->rel_tol >= 0)) return set_err(nullptr, CMTF_EVALIDATION, "rel_tol must be nonnegative");
  if (!(c->init_scale > 0))
    return set_err(nullptr, CMTF_EVALIDATION, "init_scale must be positive");
  if (c->kernel != CMTF_KERNEL_NAIVE && c->kernel != CMTF_KERNEL_OPT)
    return set_err(nullptr, CMTF_EVALIDATION, "unknown kernel %d", c->kernel);
  if (c->exec_mode != CMTF_EXEC_HOGWILD && c->exec_mode != CMTF_EXEC_SERIAL)
    return set_err(nullptr, CMTF_EVALIDATION, "unknown exec mode %d", c->exec_mode);
  return CMTF_OK;
}

}  // namespace

// ======================================================================
// C ABI
// ======================================================================
extern "C" {

void cmtf_gpu_config_default(cmtf_gpu_config* c) {
  std::memset(c, 0, sizeof *c);
  c->eta0 = 1e-3;
  c->mu = 0.1;
  c->lambda_reg = 0.1;
  c->workers = 1;
  c->max_epochs = 100;
  c->rel_tol = 1e-4;
  c->seed = 0;
  c->kernel = CMTF_KERNEL_OPT;
  c->init_scale = 1.0;
  c->exec_mode = CMTF_EXEC_HOGWILD;
  c->sort_mode = -1;
  c->order_policy = 1;
}

const char* cmtf_gpu_last_error(void) { return g_last_error.c_str(); }
const char* cmtf_gpu_ctx_error(const cmtf_gpu_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}
int32_t cmtf_gpu_abi_version(void) { return 2; }

int cmtf_gpu_create(const cmtf_gpu_config* cfg, cmtf_gpu_ctx** out) {
  cmtf_gpu_ctx* ctx = nullptr;
  if (!out) return set_err(nullptr, CMTF_EVALIDATION, "null output pointer");
  *out = nullptr;
  TRY(validate_config(cfg));
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_err(nullptr, CMTF_ECUDA, "no CUDA device available (%s)",
                   cudaGetErrorString(e));
  if (cfg->device < 0 || cfg->device >= ndev)
    return set_err(nullptr, CMTF_EVALIDATION, "device %d out of range", cfg->device);
  ctx = new cmtf_gpu_ctx();
  ctx->cfg = *cfg;
  // CP cores run on the generic kernels (dense storage, superdiagonal steps)
  if (cfg->core_structure == 1) ctx->cfg.force_generic = 1;
  ctx->order = cfg->order;
  ctx->ranks.assign(cfg->ranks, cfg->ranks + cfg->order);
  ctx->cfg.ranks = ctx->ranks.data();
  ctx->device = cfg->device;
  ctx->eta = cfg->eta0;
  {
    auto off = [](const char* name) {
      const char* v = std::getenv(name);
      return v && v[0] == '0';
    };
    ctx->env.v4_tc = !off("CMTF_V4_TC");
    ctx->env.v4_tm = !off("CMTF_V4_TM");
    ctx->env.v3_tm = !off("CMTF_V3_TM");
    if (const char* v = std::getenv("CMTF_V2_SHAPE"))
      ctx->env.v2_shape = std::string(v) == "8x1" ? 1 : std::string(v) == "8x2" ? 2 : 0;
    ctx->env.hot_host = std::getenv("CMTF_HOT_HOST") != nullptr;
    ctx->env.hot_check = std::getenv("CMTF_HOT_CHECK") != nullptr;
    {
      const char* v = std::getenv("CMTF_TM_RED");
      ctx->env.tm_red = v && v[0] == '1';
      const char* w = std::getenv("CMTF_TM_STRIDED");
      ctx->env.tm_strided = w && w[0] == '1';
      ctx->env.tm_vorder = !off("CMTF_TM_VORDER");
      ctx->env.eval_tm = !off("CMTF_EVAL_TM");
      ctx->env.eval_stream3 = !off("CMTF_EVAL_STREAM3");
      ctx->env.rrec_late = !off("CMTF_RREC_LATE");
      if (const char* v = std::getenv("CMTF_UP_CHUNKS"))
        ctx->env.up_chunks = std::min(kUpChunks, std::max(1, std::atoi(v)));
      if (const char* h = std::getenv("CMTF_TM_SEQ")) ctx->env.tm_seq = atoi(h);
      if (const char* h = std::getenv("CMTF_TM_PFL2")) ctx->env.tm_pfl2 = atoi(h) ? 1 : 0;
      if (const char* b = std::getenv("CMTF_TM_BLOCKS"))
        ctx->env.tm_blocks = std::max(0, std::min(kMaxBlk, atoi(b)));
      if (const char* b = std::getenv("CMTF_TM_BULK")) ctx->env.tm_bulk = atoi(b) & 7;
      ctx->env.tm_galt = !off("CMTF_TM_GALT");
      if (const char* h = std::getenv("CMTF_TM_GATHER_CA")) ctx->env.tm_gather_ca = atoi(h) ? 1 : 0;
    }
  }
  auto cleanup = [&](int rc) {
    delete ctx;
    return rc;
  };
  if (cudaSetDevice(ctx->device) != cudaSuccess)
    return cleanup(set_err(nullptr, CMTF_ECUDA, "cudaSetDevice failed"));
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  // L2 fill granularity for misses: the epoch's row gathers and regulariser
  // lookups are random 16-48 byte accesses, so a wider fill only adds DRAM
  // traffic (CMTF_L2_FETCH overrides; 0 keeps the driver default)
  {
    int g = 32;
    if (const char* v = std::getenv("CMTF_L2_FETCH")) g = std::atoi(v);
    if (g > 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)g);
    cudaGetLastError();
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(set_err(nullptr, CMTF_ECUDA, "stream creation failed"));
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  for (auto& ev : ctx->uev) cudaEventCreate(&ev);
  for (auto& ev : ctx->cev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(set_err(nullptr, CMTF_ECUDA, "stream creation failed"));
  cudaEventCreateWithFlags(&ctx->ev_side_start, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_side_done, cudaEventDisableTiming);
  if (cudaMalloc(&ctx->d_first, sizeof(unsigned long long) * (1 + kMaxOrder + kMaxMats)) !=
      cudaSuccess)
    return cleanup(set_err(nullptr, CMTF_ECUDA, "allocation failed"));
  *out = ctx;
  return CMTF_OK;
}

int cmtf_gpu_destroy(cmtf_gpu_ctx* ctx) {
  if (!ctx) return CMTF_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->side) cudaStreamSynchronize(ctx->side);
  dfree(ctx->rec);
  dfree(ctx->pos);
  dfree(ctx->rec_alt);
  dfree(ctx->mrec_alt);
  dfree(ctx->rrec);
  dfree(ctx->rrec_alt);
  dfree(ctx->blk_hist);
  dfree(ctx->d_vtab);
  dfree(ctx->part_cnt);
  dfree(ctx->visits);
  dfree(ctx->mvisits);
  dfree(ctx->s_idx);
  dfree(ctx->s_vals);
  dfree(ctx->s_rec);
  dfree(ctx->s_keys);
  dfree(ctx->s_ids);
  dfree(ctx->hs_keys);
  dfree(ctx->hs_tmp);
  dfree(ctx->hs_cnt);
  dfree(ctx->dup_keys);
  dfree(ctx->dup_ids);
  dfree(ctx->dup_tmp);
  for (int n = 0; n < kMaxOrder; ++n) {
    dfree(ctx->count[n]);
    dfree(ctx->reg[n]);
    dfree(ctx->U[n]);
  }
  for (auto& m : ctx->mats) {
    dfree(m.rec);
    dfree(m.pos);
    dfree(m.count);
    dfree(m.vreg);
    dfree(m.V);
  }
  for (auto& m : ctx->spare) {
    dfree(m.V);
    dfree(m.rec);
    dfree(m.pos);
    dfree(m.count);
    dfree(m.vreg);
  }
  dfree(ctx->mrec);
  dfree(ctx->s_m4);
  for (auto& b : ctx->baseU) dfree(b);
  for (auto& b : ctx->baseV) dfree(b);
  dfree(ctx->baseG);
  dfree(ctx->sync_buf);
  if (ctx->comm) nccl_api().commDestroy(ctx->comm);
  for (auto& h : ctx->hot) { dfree(h.slot); dfree(h.row_of); dfree(h.base); }
  for (auto& h : ctx->hotV) { dfree(h.slot); dfree(h.row_of); dfree(h.base); }
  dfree(ctx->G);
  dfree(ctx->d_sched);
  dfree(ctx->d_partial);
  dfree(ctx->d_partial2);
  dfree(ctx->d_first);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : ctx->uev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : ctx->cev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_side_start) cudaEventDestroy(ctx->ev_side_start);
  if (ctx->ev_side_done) cudaEventDestroy(ctx->ev_side_done);
  delete ctx;
  return CMTF_OK;
}

// ---------------------------------------------------------------------
// Duplicate coordinates (check_entries, src/sparse_data.cpp:44-63): the
// reference rejects a bundle whose tensor or matrix repeats an index tuple,
// reporting the lexicographically smallest one.  Device version: a mixed-radix
// key per entry in a device hash set when the dims fit 64 bits; otherwise a
// stable LSD radix sort of the entry ids by the full tuple and a scan of
// neighbours.
// ---------------------------------------------------------------------
struct DupKey {
  uint32_t dims[kMaxOrder];
  int order;
  int exact;
};

__global__ void iota_u32_kernel(uint32_t* ids, uint64_t n) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x)
    ids[e] = (uint32_t)e;
}

// keys[i] = mode-n index of entry ids[i] (one LSD pass of the tuple sort)
__global__ void mode_key_kernel(const uint32_t* idx, uint64_t nnz, int order, int n,
                                const uint32_t* ids, uint32_t* keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = idx[(uint64_t)ids[i] * order + n];
}

// first i with tuple(ids[i]) == tuple(ids[i-1]) (keys: optional pre-filter)
__global__ void dup_scan_kernel(const uint32_t* idx, uint64_t nnz, int order,
                                const unsigned long long* keys, const uint32_t* ids,
                                unsigned long long* first) {
  for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (keys && keys[i] != keys[i - 1]) continue;
    const uint32_t* a = idx + (uint64_t)ids[i] * order;
    const uint32_t* b = idx + (uint64_t)ids[i - 1] * order;
    bool same = true;
    for (int n = 0; n < order; ++n) same = same && a[n] == b[n];
    if (same) atomicMin(first, (unsigned long long)i);
  }
}

// Exact keys: open-addressing set on the device (load factor <= 1/2); a
// thread whose CAS finds its own key has a duplicate; the smallest duplicated
// key (= the lexicographically smallest tuple) wins an atomicMin.
__global__ void dup_hash_kernel(const uint32_t* idx, uint64_t nnz, DupKey k,
                                unsigned long long* table, uint64_t cap_mask,
                                unsigned long long* first_key) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0;
    for (int n = 0; n < k.order; ++n) key = key * k.dims[n] + idx[e * k.order + n];
    unsigned long long h = key * 0x9e3779b97f4a7c15ull;
    h ^= h >> 29;
    for (uint64_t s = h & cap_mask;; s = (s + 1) & cap_mask) {
      const unsigned long long prev = atomicCAS(table + s, ~0ull, key);
      if (prev == ~0ull) break;
      if (prev == key) {
        atomicMin(first_key, key);
        break;
      }
    }
  }
}

// The duplicate check of an upload, chunk by chunk as the chunks land (it
// overlaps the rest of the host-to-device copy).  Exact mixed-radix keys
// when the index space fits 64 bits (a repeated key is a duplicate; the
// smallest wins an atomicMin, = the lexicographically smallest tuple);
// otherwise 64-bit hashes of the tuples: equal tuples always collide, so no
// collision proves there is no duplicate, and a collision (a duplicate or a
// hash collision) sends the upload to the exact LSD-sort check.
__global__ void dup_insert_kernel(const uint32_t* idx, uint64_t e_lo, uint64_t e_hi, DupKey k,
                                  unsigned long long* table, uint64_t cap_mask,
                                  unsigned long long* first_key) {
  for (uint64_t e = e_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < e_hi;
       e += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0;
    if (k.exact) {
      for (int n = 0; n < k.order; ++n) key = key * k.dims[n] + idx[e * k.order + n];
    } else {
      key = 0x243f6a8885a308d3ull;
      for (int n = 0; n < k.order; ++n) {
        key ^= idx[e * k.order + n] + 0x9e3779b97f4a7c15ull + (key << 6) + (key >> 2);
        key *= 0xbf58476d1ce4e5b9ull;
        key ^= key >> 31;
      }
      if (key == ~0ull) key = 0;  // the empty-slot marker
    }
    unsigned long long h = key * 0x9e3779b97f4a7c15ull;
    h ^= h >> 29;
    for (uint64_t s = h & cap_mask;; s = (s + 1) & cap_mask) {
      const unsigned long long prev = atomicCAS(table + s, ~0ull, key);
      if (prev == ~0ull) break;
      if (prev == key) {
        atomicMin(first_key, k.exact ? key : 0ull);
        break;
      }
    }
  }
}

// check_entries' first failure (src/sparse_data.cpp:29-41) from the device
// validation's first bad entries: bad[0] = first index out of range, bad[1] =
// first non-finite value.  The reference scans entries in order and checks an
// entry's indices before its value; the offending tuple is read back from the
// device staging copy (the caller's idx may be a device pointer).
int entry_error(cmtf_gpu_ctx* ctx, const char* what, const uint32_t* d_idx, int order,
                const uint32_t* dims, const unsigned long long* bad) {
  if (bad[0] != ~0ull && bad[0] <= bad[1]) {
    std::vector<uint32_t> tup(order);
    CU(cudaMemcpy(tup.data(), d_idx + bad[0] * (uint64_t)order, order * sizeof(uint32_t),
                  cudaMemcpyDeviceToHost));
    for (int n = 0; n < order; ++n)
      if (tup[n] >= dims[n])
        return set_err(ctx, CMTF_EVALIDATION, "%s index out of range: mode %d index %u > size %u",
                       what, n + 1, tup[n] + 1, dims[n]);
  }
  return set_err(ctx, CMTF_EVALIDATION, "%s value is not finite", what);
}

// An upload source that already lives on this context's device is read in
// place (no staging copy); host (pageable or pinned) and other devices' memory
// goes through the chunked staging copy.
bool on_device(const cmtf_gpu_ctx* ctx, const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice && at.device == ctx->device;
}

// CMTF_PREP_TIMING: phase times of an upload (synchronising at each tick)
struct PhaseTimer {
  const char* what;
  cmtf_gpu_ctx* ctx;
  bool on;
  std::chrono::steady_clock::time_point t0;
  PhaseTimer(const char* w, cmtf_gpu_ctx* c)
      : what(w), ctx(c), on(std::getenv("CMTF_PREP_TIMING") != nullptr),
        t0(std::chrono::steady_clock::now()) {}
  void tick(const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(ctx->side);
    cudaStreamSynchronize(ctx->stream);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "%s %-14s %.3f ms\n", what, phase,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};


// The upload staging (up to ~45 bytes per entry: 45 GB at 1e9 entries) is
// released after every upload instead of living with the context (keeping it
// while memory is plentiful was measured: no gain beyond the noise of the
// host-to-device copies, scripts/ab_upload.py).
void release_staging(cmtf_gpu_ctx* ctx) {
  cudaStreamSynchronize(ctx->side);
  cudaStreamSynchronize(ctx->stream);
  dfree(ctx->s_idx);
  dfree(ctx->s_vals);
  dfree(ctx->s_rec);
  dfree(ctx->s_keys);
  dfree(ctx->s_ids);
  ctx->s_idx_cap = ctx->s_vals_cap = ctx->s_rec_cap = ctx->s_keys_cap = ctx->s_ids_cap = 0;
}

// 0: no duplicate; else writes the duplicated tuple (0-based) to *tuple.
int find_duplicate_impl(cmtf_gpu_ctx* ctx, const uint32_t* d_idx, uint64_t nnz, int order,
                        const uint32_t* dims, std::vector<uint32_t>* tuple, bool* found) {
  *found = false;
  if (nnz < 2) return CMTF_OK;
  DupKey k{};
  k.order = order;
  double bits = 0;
  for (int n = 0; n < order; ++n) {
    k.dims[n] = dims[n];
    bits += std::log2((double)std::max<uint32_t>(dims[n], 1));
  }
  k.exact = bits < 63.5;
  if (k.exact) {
    uint64_t cap = 1;
    while (cap < 2 * nnz) cap <<= 1;
    TRY(ensure(ctx, &ctx->dup_keys, &ctx->dup_keys_cap, cap));
    unsigned long long* first = ctx->d_first;  // [0] is free after validation
    CU(cudaMemsetAsync(ctx->dup_keys, 0xff, cap * sizeof(unsigned long long), ctx->stream));
    CU(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), ctx->stream));
    dup_hash_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(d_idx, nnz, k, ctx->dup_keys,
                                                            cap - 1, first);
    unsigned long long f = ~0ull;
    CU(cudaMemcpyAsync(&f, first, sizeof f, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (f != ~0ull) {  // decode the mixed-radix key
      tuple->assign(order, 0u);
      for (int n = order - 1; n >= 0; --n) {
        (*tuple)[n] = (uint32_t)(f % dims[n]);
        f /= dims[n];
      }
      *found = true;
    }
    return CMTF_OK;
  }
  // beyond 64 bits: stable LSD radix sort of the entry ids by the full tuple
  // (one 32-bit pass per mode, last mode first), so equal tuples are adjacent
  // and the first equal neighbour pair is the lexicographically smallest
  // duplicate, exactly the reference's sort + scan
  TRY(ensure(ctx, &ctx->dup_keys, &ctx->dup_keys_cap, nnz));  // 2 x u32 keys
  TRY(ensure(ctx, &ctx->dup_ids, &ctx->dup_ids_cap, 2 * nnz));
  uint32_t* keys = reinterpret_cast<uint32_t*>(ctx->dup_keys);
  uint32_t* keys2 = keys + nnz;
  uint32_t *ids = ctx->dup_ids, *ids2 = ctx->dup_ids + nnz;
  unsigned long long* first = ctx->d_first;  // [0] is free after validation
  iota_u32_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(ids, nnz);
  size_t tb = 0;
  CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, ids, ids2, nnz, 0, 32,
                                     ctx->stream));
  TRY(ensure(ctx, &ctx->dup_tmp, &ctx->dup_tmp_cap, tb));
  for (int n = order - 1; n >= 0; --n) {
    mode_key_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(d_idx, nnz, order, n, ids, keys);
    const int end_bit = std::max(1, (int)std::ceil(std::log2((double)dims[n] + 1.0)));
    CU(cub::DeviceRadixSort::SortPairs(ctx->dup_tmp, tb, keys, keys2, ids, ids2, nnz, 0,
                                       std::min(32, end_bit), ctx->stream));
    std::swap(ids, ids2);
  }
  CU(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), ctx->stream));
  dup_scan_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(d_idx, nnz, order, nullptr, ids, first);
  CU(cudaGetLastError());
  unsigned long long f = ~0ull;
  CU(cudaMemcpyAsync(&f, first, sizeof f, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (f != ~0ull) {
    uint32_t id = 0;
    CU(cudaMemcpy(&id, ids + f, sizeof id, cudaMemcpyDeviceToHost));
    tuple->resize(order);
    CU(cudaMemcpy(tuple->data(), d_idx + (uint64_t)id * order, order * sizeof(uint32_t),
                  cudaMemcpyDeviceToHost));
    *found = true;
  }
  return CMTF_OK;
}

// The check's scratch (up to 16 B per entry: 16 GB at 1e9 entries) is
// released as soon as the check is done instead of living with the context.
int find_duplicate(cmtf_gpu_ctx* ctx, const uint32_t* d_idx, uint64_t nnz, int order,
                   const uint32_t* dims, std::vector<uint32_t>* tuple, bool* found) {
  const int rc = find_duplicate_impl(ctx, d_idx, nnz, order, dims, tuple, found);
  cudaStreamSynchronize(ctx->stream);
  dfree(ctx->dup_keys);
  dfree(ctx->dup_ids);
  dfree(ctx->dup_tmp);
  ctx->dup_keys_cap = ctx->dup_ids_cap = ctx->dup_tmp_cap = 0;
  return rc;
}

std::string dup_message(const char* what, const std::vector<uint32_t>& t) {
  std::string msg = std::string("duplicate ") + what + " index (";
  for (size_t n = 0; n < t.size(); ++n) msg += (n ? " " : "") + std::to_string(t[n] + 1);
  return msg + ")";
}

// check_entries' range and finiteness pass (src/sparse_data.cpp:29-41):
// first entry with an index out of range / a non-finite value
__global__ void check_entries_kernel(const uint32_t* idx, const double* vals, uint64_t nnz,
                                     DupKey k, unsigned long long* bad) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x) {
    for (int n = 0; n < k.order; ++n)
      if (idx[e * k.order + n] >= k.dims[n]) atomicMin(&bad[0], (unsigned long long)e);
    if (!isfinite(vals[e])) atomicMin(&bad[1], (unsigned long long)e);
  }
}

int cmtf_gpu_check_entries(int32_t device, int32_t order, const uint32_t* dims,
                           const uint32_t* idx, const double* vals, uint64_t nnz,
                           int32_t is_matrix) {
  const char* what = is_matrix ? "matrix" : "tensor";
  if (!dims || order < 1 || order > kMaxOrder)
    return set_err(nullptr, CMTF_EVALIDATION, "invalid arguments");
  if (order < 2 && !is_matrix)
    return set_err(nullptr, CMTF_EVALIDATION, "tensor order must be at least 2");
  for (int n = 0; n < order; ++n)
    if (dims[n] == 0) return set_err(nullptr, CMTF_EVALIDATION, "mode sizes must be positive");
  if (nnz == 0) return CMTF_OK;
  cmtf_gpu_config cfg;
  cmtf_gpu_config_default(&cfg);
  std::vector<uint32_t> ones(order, 1u);
  cfg.order = order;
  cfg.ranks = ones.data();
  cfg.device = device;
  cmtf_gpu_ctx* ctx = nullptr;
  TRY(cmtf_gpu_create(&cfg, &ctx));
  auto run = [&]() -> int {
    uint32_t* d_idx = nullptr;
    double* d_vals = nullptr;
    if (on_device(ctx, idx) || on_device(ctx, vals)) CU(cudaDeviceSynchronize());
    TRY(dalloc(ctx, &d_idx, nnz * (uint64_t)order));
    TRY(dalloc(ctx, &d_vals, nnz));
    auto cleanup = [&](int rc) {
      dfree(d_idx);
      dfree(d_vals);
      return rc;
    };
    if (cudaMemcpyAsync(d_idx, idx, nnz * order * sizeof(uint32_t), cudaMemcpyDefault,
                        ctx->stream) != cudaSuccess ||
        cudaMemcpyAsync(d_vals, vals, nnz * sizeof(double), cudaMemcpyDefault, ctx->stream) !=
            cudaSuccess)
      return cleanup(set_err(ctx, CMTF_ECUDA, "copy of the entries failed"));
    DupKey k{};
    k.order = order;
    for (int n = 0; n < order; ++n) k.dims[n] = dims[n];
    cudaMemsetAsync(ctx->d_first, 0xff, 2 * sizeof(unsigned long long), ctx->stream);
    check_entries_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(d_idx, d_vals, nnz, k,
                                                                 ctx->d_first);
    unsigned long long bad[2];
    if (cudaMemcpyAsync(bad, ctx->d_first, sizeof bad, cudaMemcpyDeviceToHost, ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return cleanup(set_err(ctx, CMTF_ECUDA, "entry check failed"));
    if (bad[0] != ~0ull || bad[1] != ~0ull)
      return cleanup(entry_error(ctx, what, d_idx, order, dims, bad));
    std::vector<uint32_t> tup;
    bool dup = false;
    const int rc = find_duplicate(ctx, d_idx, nnz, order, dims, &tup, &dup);
    if (rc) return cleanup(rc);
    if (dup) return cleanup(set_err(ctx, CMTF_EVALIDATION, "%s", dup_message(what, tup).c_str()));
    return cleanup(CMTF_OK);
  };
  const int rc = run();
  const std::string msg = ctx->err;
  cmtf_gpu_destroy(ctx);
  if (rc) g_last_error = msg;
  return rc;
}

int cmtf_gpu_set_tensor(cmtf_gpu_ctx* ctx, const uint32_t* dims,
                        const uint32_t* idx, const double* vals, uint64_t nnz) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  CU(cudaSetDevice(ctx->device));
  const int N = ctx->order;
  if (nnz == 0) return set_err(ctx, CMTF_EVALIDATION, "training tensor has no entries");
  if (nnz >= 0xffffffffull)
    return set_err(ctx, CMTF_EUNSUPPORTED, "nnz >= 2^32 per device; shard the tensor");
  for (int n = 0; n < N; ++n) {
    if (dims[n] == 0) return set_err(ctx, CMTF_EVALIDATION, "mode sizes must be positive");
    // validate_config: rank <= dim unless nonnegative (src/trainer.cpp:70-76)
    if (!ctx->cfg.nonnegative && ctx->ranks[n] > dims[n])
      return set_err(ctx, CMTF_EVALIDATION,
                     "rank of mode %d exceeds its size; orthogonalization needs J_n <= I_n",
                     n + 1);
  }
  const bool same_shape =
      ctx->dims.size() == (size_t)N && std::equal(ctx->dims.begin(), ctx->dims.end(), dims);
  drain_side(ctx);  // a pending reshuffle reads rec
  ctx->rrec_valid = false;
  ctx->vt_on = ctx->pos_ids = false;  // the upload lays records out anew
  ctx->dims.assign(dims, dims + N);
  ctx->nnz = nnz;
  ctx->v2_dirty = true;
  if (!same_shape) ctx->have_model = false;
  int sm = ctx->cfg.sort_mode;
  if (sm < 0 || sm >= N) {
    sm = 0;  // auto: the mode with the most rows (ties: lowest index)
    for (int n = 1; n < N; ++n)
      if (dims[n] > dims[sm]) sm = n;
  }
  ctx->sort_mode = sm;

  PhaseTimer pt("set_tensor", ctx);
  const bool in_place = on_device(ctx, idx) && on_device(ctx, vals);
  // device-resident inputs may still be written by work on the caller's
  // streams (the context's streams are non-blocking): wait for the device
  if (in_place) CU(cudaDeviceSynchronize());
  const bool sorted_order = ctx->cfg.order_policy == 0;  // sorted order needs keys + a gather
  if (!in_place) {
    TRY(ensure(ctx, &ctx->s_idx, &ctx->s_idx_cap, nnz * N));
    TRY(ensure(ctx, &ctx->s_vals, &ctx->s_vals_cap, nnz));
  }
  if (sorted_order) {
    TRY(ensure(ctx, &ctx->s_rec, &ctx->s_rec_cap, nnz * (N + 1)));
    TRY(ensure(ctx, &ctx->s_keys, &ctx->s_keys_cap, nnz));
    TRY(ensure(ctx, &ctx->s_ids, &ctx->s_ids_cap, nnz));
  }
  const uint32_t* d_idx = in_place ? idx : ctx->s_idx;
  const double* d_vals = in_place ? vals : ctx->s_vals;
  uint32_t *d_rec = ctx->s_rec, *d_keys = ctx->s_keys, *d_ids = ctx->s_ids;
  // Host (pageable or pinned) or another device's memory: the copies run in
  // chunks on the side stream; each chunk is packed on the main stream as
  // soon as it lands (H2D overlaps validation and packing).
  // the last chunk's pack + duplicate insert run after the copies end: many
  // chunks keep that tail short (4 chunks: 40 ms at 9e8 entries), a floor on
  // the chunk size keeps small uploads at one launch
  const int kChunks = ctx->env.up_chunks;
  const uint64_t chunk = std::max<uint64_t>((nnz + kChunks - 1) / kChunks, kUpChunkMin);
  for (int k = 0; k < kChunks; ++k) {
    const uint64_t c0 = k * chunk, c1 = std::min<uint64_t>(nnz, c0 + chunk);
    if (c0 >= c1) break;
    if (!in_place) {
      CU(cudaMemcpyAsync(ctx->s_idx + c0 * N, idx + c0 * N, (c1 - c0) * N * sizeof(uint32_t),
                         cudaMemcpyDefault, ctx->side));
      CU(cudaMemcpyAsync(ctx->s_vals + c0, vals + c0, (c1 - c0) * sizeof(double),
                         cudaMemcpyDefault, ctx->side));
    }
    CU(cudaEventRecord(ctx->cev[k], ctx->side));
  }
  for (int n = 0; n < N; ++n) {
    if (!same_shape || !ctx->count[n]) {
      TRY(dalloc(ctx, &ctx->count[n], dims[n]));
      TRY(dalloc(ctx, &ctx->reg[n], dims[n]));
    }
    CU(cudaMemsetAsync(ctx->count[n], 0, dims[n] * sizeof(uint32_t), ctx->stream));
  }
  CU(cudaMemsetAsync(ctx->d_first, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
  ModeTables mt = mode_tables(ctx);
  const bool shuffled = ctx->cfg.order_policy == 1;
  const bool need_keys = ctx->cfg.order_policy == 0;  // sorted order needs the sort keys
  // random and caller orders: each record is packed straight into its place
  // in the entry order (no separate scatter pass)
  const bool direct = ctx->cfg.order_policy != 0;
  uint64_t pa = 1, pb = 0;
  if (shuffled) affine_params(nnz, ctx->cfg.seed, &pa, &pb);
  if (direct) {
    TRY(ensure(ctx, &ctx->rec, &ctx->rec_cap, nnz * (N + 1)));
    TRY(ensure(ctx, &ctx->pos, &ctx->pos_cap, nnz));
  }
  ctx->pos_affine = direct;
  ctx->up_pa = pa;
  ctx->up_pb = pb;
  // duplicate-check table (load factor <= 1/2), filled chunk by chunk
  DupKey dk{};
  dk.order = N;
  {
    double bits = 0;
    for (int n = 0; n < N; ++n) {
      dk.dims[n] = dims[n];
      bits += std::log2((double)std::max<uint32_t>(dims[n], 1));
    }
    dk.exact = bits < 63.5;
  }
  uint64_t dcap = 1;
  while (dcap < 2 * nnz) dcap <<= 1;
  TRY(ensure(ctx, &ctx->dup_keys, &ctx->dup_keys_cap, dcap));
  CU(cudaMemsetAsync(ctx->dup_keys, 0xff, dcap * sizeof(unsigned long long), ctx->stream));
  CU(cudaMemsetAsync(ctx->d_first + 2, 0xff, sizeof(unsigned long long), ctx->stream));
  for (int k = 0; k < kChunks; ++k) {
    const uint64_t c0 = k * chunk, c1 = std::min<uint64_t>(nnz, c0 + chunk);
    if (c0 >= c1) break;
    CU(cudaStreamWaitEvent(ctx->stream, ctx->cev[k], 0));
    pack_tensor_kernel<<<grid_for(c1 - c0), 256, 0, ctx->stream>>>(
        d_idx, d_vals, c0, c1, N, mt, shuffled ? -1 : sm, (uint32_t)ctx->cfg.seed + 0x5bd1e995u,
        direct ? ctx->rec : d_rec, need_keys ? d_keys : nullptr, d_ids, ctx->d_first,
        direct ? nnz : 0, pa, pb, ctx->pos);
    dup_insert_kernel<<<grid_for(c1 - c0), 256, 0, ctx->stream>>>(
        d_idx, c0, c1, dk, ctx->dup_keys, dcap - 1, ctx->d_first + 2);
  }
  CU(cudaGetLastError());
  unsigned long long bad[3];
  CU(cudaMemcpyAsync(bad, ctx->d_first, sizeof bad, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  dfree(ctx->dup_keys);
  ctx->dup_keys_cap = 0;
  pt.tick("h2d+pack+dup");
  if (bad[0] != ~0ull || bad[1] != ~0ull) {
    dfree(ctx->rec);
    ctx->rec_cap = 0;
    const int rc = entry_error(ctx, "tensor", d_idx, N, dims, bad);
    release_staging(ctx);
    return rc;
  }
  if (bad[2] != ~0ull) {  // a repeated key (exact) or hash (wide tuples)
    std::vector<uint32_t> tup;
    bool dup = false;
    int rc = CMTF_OK;
    if (dk.exact) {  // decode the smallest duplicated mixed-radix key
      unsigned long long f = bad[2];
      tup.assign(N, 0u);
      for (int n = N - 1; n >= 0; --n) {
        tup[n] = (uint32_t)(f % dims[n]);
        f /= dims[n];
      }
      dup = true;
    } else {  // exact check: the smallest duplicated tuple, or a hash collision
      rc = find_duplicate(ctx, d_idx, nnz, N, dims, &tup, &dup);
    }
    if (rc || dup) {
      dfree(ctx->rec);
      ctx->rec_cap = 0;
      release_staging(ctx);
      if (rc) return rc;
      return set_err(ctx, CMTF_EVALIDATION, "%s", dup_message("tensor", tup).c_str());
    }
  }
  pt.tick("duplicates");
  TRY(ensure(ctx, &ctx->rec, &ctx->rec_cap, nnz * (N + 1)));
  TRY(ensure(ctx, &ctx->pos, &ctx->pos_cap, nnz));
  ctx->posA = 1;
  ctx->posB = 0;
  uint32_t* sorted_ids = nullptr;
  if (!direct) {
    TRY(sort_ids(ctx, d_keys, d_ids, nnz, dims[sm], &sorted_ids));
    gather_records_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(
        d_rec, sorted_ids, nnz, N + 1, ctx->rec, ctx->pos);
  }
  CU(cudaGetLastError());
  for (int n = 0; n < N; ++n)
    reg_kernel<<<grid_for(dims[n]), 256, 0, ctx->stream>>>(
        ctx->count[n], dims[n], (float)ctx->cfg.lambda_reg, ctx->reg[n]);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(ctx->stream));
  if (sorted_ids) cudaFree(sorted_ids);
  release_staging(ctx);
  pt.tick("finish");
  // model buffers (allocated with the bundle's shapes; kept on re-upload of a
  // same-shaped bundle, as run_epoch(state, bundle) keeps the state's model)
  if (!same_shape || !ctx->G) {
    for (int n = 0; n < N; ++n)
      TRY(dalloc(ctx, &ctx->U[n], (uint64_t)dims[n] * ctx->JP(n)));
    TRY(dalloc(ctx, &ctx->G, ctx->core_size()));
    ctx->have_model = false;
  }
  return CMTF_OK;
}

int cmtf_gpu_clear_matrices(cmtf_gpu_ctx* ctx) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  for (auto& v : ctx->spare) {
    dfree(v.V);
    dfree(v.rec);
    dfree(v.pos);
    dfree(v.count);
    dfree(v.vreg);
  }
  ctx->spare.clear();
  // every buffer (and the coupled factor) is kept for a same-shaped re-add
  for (auto& m : ctx->mats) ctx->spare.push_back(m);
  ctx->mats.clear();
  return CMTF_OK;
}

int cmtf_gpu_add_matrix(cmtf_gpu_ctx* ctx, int32_t mode0, uint32_t rows,
                        uint32_t cols, const uint32_t* idx, const double* vals,
                        uint64_t nnz, double weight) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (ctx->dims.empty())
    return set_err(ctx, CMTF_EVALIDATION, "set the tensor before adding matrices");
  CU(cudaSetDevice(ctx->device));
  // CoupledMatrix ctor + make_bundle checks (src/sparse_data.cpp:230-240,364-375)
  if (mode0 < 0 || mode0 >= ctx->order)
    return set_err(ctx, CMTF_EVALIDATION, "coupled mode out of range");
  if (!(weight > 0)) return set_err(ctx, CMTF_EVALIDATION, "lambda_m must be positive");
  if (rows != ctx->dims[mode0])
    return set_err(ctx, CMTF_EVALIDATION,
                   "coupled matrix row space does not match mode %d", mode0 + 1);
  if (cols == 0) return set_err(ctx, CMTF_EVALIDATION, "mode sizes must be positive");
  if ((int)ctx->mats.size() >= kMaxMats)
    return set_err(ctx, CMTF_EUNSUPPORTED, "at most %d coupled matrices", kMaxMats);
  if (nnz >= 0xffffffffull)
    return set_err(ctx, CMTF_EUNSUPPORTED, "matrix nnz >= 2^32 per device");
  DevMatrix M;
  const size_t slot = ctx->mats.size();
  DevMatrix* sp = slot < ctx->spare.size() ? &ctx->spare[slot] : nullptr;
  const bool reuse = sp && sp->V && sp->mode == mode0 && sp->cols == cols && sp->nnz >= nnz;
  if (reuse) {
    M = *sp;  // buffers and the coupled factor of the state
    *sp = DevMatrix();
  } else {
    TRY(dalloc(ctx, &M.count, cols));
    TRY(dalloc(ctx, &M.vreg, cols));
    TRY(dalloc(ctx, &M.V, (uint64_t)cols * ctx->JP(mode0)));
    TRY(dalloc(ctx, &M.rec, nnz * 3));
    TRY(dalloc(ctx, &M.pos, nnz));
    ctx->have_model = false;
  }
  M.mode = mode0;
  M.rows = rows;
  M.cols = cols;
  M.nnz = nnz;
  M.weight = weight;
  CU(cudaMemsetAsync(M.count, 0, cols * sizeof(uint32_t), ctx->stream));
  if (nnz > 0) {
    const bool in_place = on_device(ctx, idx) && on_device(ctx, vals);
    if (in_place) CU(cudaDeviceSynchronize());  // see cmtf_gpu_set_tensor
    if (!in_place) {
      TRY(ensure(ctx, &ctx->s_idx, &ctx->s_idx_cap, nnz * 2));
      TRY(ensure(ctx, &ctx->s_vals, &ctx->s_vals_cap, nnz));
    }
    if (ctx->cfg.order_policy == 0) {
      TRY(ensure(ctx, &ctx->s_rec, &ctx->s_rec_cap, nnz * 3));
      TRY(ensure(ctx, &ctx->s_keys, &ctx->s_keys_cap, nnz));
      TRY(ensure(ctx, &ctx->s_ids, &ctx->s_ids_cap, nnz));
    }
    const uint32_t* d_idx = in_place ? idx : ctx->s_idx;
    const double* d_vals = in_place ? vals : ctx->s_vals;
    uint32_t *d_rec = ctx->s_rec, *d_keys = ctx->s_keys, *d_ids = ctx->s_ids;
    // chunked H2D on the side stream, each chunk packed as it lands; random
    // and caller orders pack straight into the entry order (no scatter pass)
    const int shuffled = ctx->cfg.order_policy == 1;
    const bool direct = ctx->cfg.order_policy != 0;
    uint64_t pa = 1, pb = 0;
    if (shuffled) affine_params(nnz, ctx->cfg.seed + 7 + ctx->mats.size(), &pa, &pb);
    const int kChunks = ctx->env.up_chunks;
    const uint64_t chunk = std::max<uint64_t>((nnz + kChunks - 1) / kChunks, kUpChunkMin);
    CU(cudaEventRecord(ctx->ev_side_start, ctx->stream));  // count memset, staging reuse
    CU(cudaStreamWaitEvent(ctx->side, ctx->ev_side_start, 0));
    for (int k = 0; k < kChunks; ++k) {
      const uint64_t c0 = k * chunk, c1 = std::min<uint64_t>(nnz, c0 + chunk);
      if (c0 >= c1) break;
      if (!in_place) {
        CU(cudaMemcpyAsync(ctx->s_idx + 2 * c0, idx + 2 * c0, (c1 - c0) * 2 * sizeof(uint32_t),
                           cudaMemcpyDefault, ctx->side));
        CU(cudaMemcpyAsync(ctx->s_vals + c0, vals + c0, (c1 - c0) * sizeof(double),
                           cudaMemcpyDefault, ctx->side));
      }
      CU(cudaEventRecord(ctx->cev[k], ctx->side));
    }
    CU(cudaMemsetAsync(ctx->d_first, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
    for (int k = 0; k < kChunks; ++k) {
      const uint64_t c0 = k * chunk, c1 = std::min<uint64_t>(nnz, c0 + chunk);
      if (c0 >= c1) break;
      CU(cudaStreamWaitEvent(ctx->stream, ctx->cev[k], 0));
      pack_matrix_kernel<<<grid_for(c1 - c0), 256,
                           cols <= kPackHistCols ? cols * sizeof(uint32_t) : 0, ctx->stream>>>(
          d_idx, d_vals, c0, c1, rows, cols, shuffled,
          (uint32_t)ctx->cfg.seed + 0x27d4eb2fu + (uint32_t)ctx->mats.size(),
          direct ? M.rec : d_rec, direct ? nullptr : d_keys, d_ids, M.count, ctx->d_first,
          direct ? nnz : 0, pa, pb, M.pos);
    }
    CU(cudaGetLastError());
    unsigned long long bad[2];
    CU(cudaMemcpyAsync(bad, ctx->d_first, sizeof bad, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (bad[0] != ~0ull || bad[1] != ~0ull) {
      dfree(M.count);
      dfree(M.vreg);
      dfree(M.V);
      dfree(M.rec);
      dfree(M.pos);
      const uint32_t mdims[2] = {rows, cols};
      const int rc = entry_error(ctx, "matrix", d_idx, 2, mdims, bad);
      release_staging(ctx);
      return rc;
    }
    {
      std::vector<uint32_t> tup;
      bool dup = false;
      const uint32_t mdims[2] = {rows, cols};
      const int rc = find_duplicate(ctx, d_idx, nnz, 2, mdims, &tup, &dup);
      if (rc || dup) {
        dfree(M.count);
        dfree(M.vreg);
        dfree(M.V);
        dfree(M.rec);
        dfree(M.pos);
        release_staging(ctx);
        if (rc) return rc;
        return set_err(ctx, CMTF_EVALIDATION, "%s", dup_message("matrix", tup).c_str());
      }
    }
    uint32_t* sorted_ids = nullptr;
    if (!direct) {
      TRY(sort_ids(ctx, d_keys, d_ids, nnz, rows, &sorted_ids));
      gather_records_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(
          d_rec, sorted_ids, nnz, 3, M.rec, M.pos);
    }
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
    if (sorted_ids) cudaFree(sorted_ids);
    release_staging(ctx);
  }
  reg_kernel<<<grid_for(cols), 256, 0, ctx->stream>>>(
      M.count, cols, (float)(weight * ctx->cfg.lambda_reg), M.vreg);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->mats.push_back(M);
  ctx->v2_dirty = true;
  return CMTF_OK;
}

}  // extern "C"

namespace {
// The core as the caller sees it (CoreTensor::stored(), include/cmtf/tucker.hpp):
// dense, or for a CP core its ranks[0] superdiagonal values; on the device
// it is always dense (off-diagonal zeros).
uint64_t stored_core_size(const cmtf_gpu_ctx* ctx) {
  return ctx->cfg.core_structure == 1 ? ctx->ranks[0] : ctx->core_size();
}
uint64_t cp_step(const cmtf_gpu_ctx* ctx) {
  uint64_t step = 0, st = 1;
  for (int n = ctx->order - 1; n >= 0; --n) {
    step += st;
    st *= ctx->ranks[n];
  }
  return step;
}
std::vector<float> dense_core(const cmtf_gpu_ctx* ctx, const double* stored) {
  std::vector<float> c(ctx->core_size(), 0.f);
  if (ctx->cfg.core_structure == 1) {
    const uint64_t step = cp_step(ctx);
    for (uint32_t k = 0; k < ctx->ranks[0]; ++k) c[k * step] = (float)stored[k];
  } else {
    for (size_t d = 0; d < c.size(); ++d) c[d] = (float)stored[d];
  }
  return c;
}
void stored_core(const cmtf_gpu_ctx* ctx, const std::vector<float>& dense, double* out) {
  if (ctx->cfg.core_structure == 1) {
    const uint64_t step = cp_step(ctx);
    for (uint32_t k = 0; k < ctx->ranks[0]; ++k) out[k] = dense[k * step];
  } else {
    for (size_t d = 0; d < dense.size(); ++d) out[d] = dense[d];
  }
}
}  // namespace

extern "C" {

// random_model (src/trainer.cpp:30-58) with make_rng(seed, Init)
// (src/trainer.cpp:100); uploaded as f32 with zeroed row padding.  The core
// draws cover its stored values (a CP core: ranks[0] of them).
int cmtf_gpu_make_state(cmtf_gpu_ctx* ctx) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (!ctx->rec) return set_err(ctx, CMTF_EVALIDATION, "no training tensor set");
  CU(cudaSetDevice(ctx->device));
  auto rng = make_rng(ctx->cfg.seed, 0x01, 0);
  const double scale = ctx->cfg.init_scale;
  std::vector<double> drawn(stored_core_size(ctx));
  for (auto& g : drawn) g = (double)(float)(0.0 + (scale - 0.0) * uniform01(rng));
  const std::vector<float> core = dense_core(ctx, drawn.data());
  CU(cudaMemcpyAsync(ctx->G, core.data(), core.size() * sizeof(float),
                     cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  auto draw = [&](float* dst, uint32_t rows, uint32_t J, uint32_t JP) -> int {
    const double hi = scale / std::sqrt((double)J);
    std::vector<float> h((uint64_t)rows * JP, 0.f);
    for (uint64_t i = 0; i < rows; ++i)
      for (uint32_t k = 0; k < J; ++k)
        h[i * JP + k] = (float)(0.0 + (hi - 0.0) * uniform01(rng));
    CU(cudaMemcpy(dst, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
    return CMTF_OK;
  };
  for (int n = 0; n < ctx->order; ++n)
    TRY(draw(ctx->U[n], ctx->dims[n], ctx->J(n), ctx->JP(n)));
  for (auto& M : ctx->mats) TRY(draw(M.V, M.cols, ctx->J(M.mode), ctx->JP(M.mode)));
  ctx->have_model = true;
  ctx->epoch = 0;
  ctx->eta = ctx->cfg.eta0;
  ctx->schedule.clear();
  return CMTF_OK;
}

int cmtf_gpu_set_model(cmtf_gpu_ctx* ctx, const double* core,
                       const double* const* factors, const double* const* couplings) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (!ctx->rec) return set_err(ctx, CMTF_EVALIDATION, "no training tensor set");
  CU(cudaSetDevice(ctx->device));
  // the context streams are non-blocking: no kernel may still read the model
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaStreamSynchronize(ctx->side));
  const std::vector<float> c = dense_core(ctx, core);
  CU(cudaMemcpy(ctx->G, c.data(), c.size() * sizeof(float), cudaMemcpyHostToDevice));
  auto put = [&](float* dst, const double* src, uint32_t rows, uint32_t J,
                 uint32_t JP) -> int {
    std::vector<float> h((uint64_t)rows * JP, 0.f);
    for (uint64_t i = 0; i < rows; ++i)
      for (uint32_t k = 0; k < J; ++k) h[i * JP + k] = (float)src[i * J + k];
    CU(cudaMemcpy(dst, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
    return CMTF_OK;
  };
  for (int n = 0; n < ctx->order; ++n)
    TRY(put(ctx->U[n], factors[n], ctx->dims[n], ctx->J(n), ctx->JP(n)));
  for (size_t m = 0; m < ctx->mats.size(); ++m)
    TRY(put(ctx->mats[m].V, couplings[m], ctx->mats[m].cols, ctx->J(ctx->mats[m].mode),
            ctx->JP(ctx->mats[m].mode)));
  ctx->have_model = true;
  return CMTF_OK;
}

int cmtf_gpu_get_model(cmtf_gpu_ctx* ctx, double* core, double* const* factors,
                       double* const* couplings) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize(ctx->stream));
  if (core) {
    std::vector<float> c(ctx->core_size());
    CU(cudaMemcpy(c.data(), ctx->G, c.size() * sizeof(float), cudaMemcpyDeviceToHost));
    stored_core(ctx, c, core);
  }
  auto get = [&](double* dst, const float* src, uint32_t rows, uint32_t J,
                 uint32_t JP) -> int {
    std::vector<float> h((uint64_t)rows * JP);
    CU(cudaMemcpy(h.data(), src, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < rows; ++i)
      for (uint32_t k = 0; k < J; ++k) dst[i * J + k] = h[i * JP + k];
    return CMTF_OK;
  };
  if (factors)
    for (int n = 0; n < ctx->order; ++n)
      TRY(get(factors[n], ctx->U[n], ctx->dims[n], ctx->J(n), ctx->JP(n)));
  if (couplings)
    for (size_t m = 0; m < ctx->mats.size(); ++m)
      TRY(get(couplings[m], ctx->mats[m].V, ctx->mats[m].cols,
              ctx->J(ctx->mats[m].mode), ctx->JP(ctx->mats[m].mode)));
  return CMTF_OK;
}

int cmtf_gpu_get_state(cmtf_gpu_ctx* ctx, int32_t* epoch, double* eta) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (epoch) *epoch = ctx->epoch;
  if (eta) *eta = ctx->eta;
  return CMTF_OK;
}

int cmtf_gpu_set_state(cmtf_gpu_ctx* ctx, int32_t epoch, double eta) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  ctx->epoch = epoch;
  ctx->eta = eta;
  return CMTF_OK;
}

}  // extern "C"

namespace {

uint64_t mulmod(uint64_t x, uint64_t y, uint64_t n) {
  return (uint64_t)(((unsigned __int128)x * y) % n);
}
uint64_t inv_mod(uint64_t a, uint64_t n) {  // gcd(a, n) = 1
  __int128 t = 0, nt = 1, r = (__int128)n, nr = (__int128)(a % n);
  while (nr != 0) {
    const __int128 q = r / nr, tt = t - q * nt, rr = r - q * nr;
    t = nt; nt = tt; r = nr; nr = rr;
  }
  if (t < 0) t += n;
  return (uint64_t)t;
}

template <int WORDS>
void launch_reshuffle(const uint32_t* src, uint32_t* dst, uint64_t n, uint64_t a, uint64_t b,
                      cudaStream_t st) {
  const uint64_t ng = n / kShuffleGroup;
  const uint64_t per_block = 8ull * 32 * kReshuffleRun;  // 8 warps
  uint64_t blocks = (n + per_block - 1) / per_block;
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  reshuffle_kernel<WORDS><<<(unsigned)std::max<uint64_t>(1, blocks), 256, 0, st>>>(
      src, dst, n, a, b, mulmod(a, (32 / kShuffleGroup) % ng, ng));
}

int launch_tensor_gather(cmtf_gpu_ctx* ctx, uint64_t epoch, cudaStream_t st, uint64_t* a,
                         uint64_t* b) {
  const uint64_t n = ctx->nnz, ng = n / kShuffleGroup;
  epoch_affine(ng, ctx->cfg.seed, epoch, 1, a, b);
  switch (ctx->order + 1) {
    case 4: launch_reshuffle<4>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 5: launch_reshuffle<5>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 3: launch_reshuffle<3>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 6: launch_reshuffle<6>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 7: launch_reshuffle<7>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 8: launch_reshuffle<8>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 9: launch_reshuffle<9>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 10: launch_reshuffle<10>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 11: launch_reshuffle<11>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 12: launch_reshuffle<12>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 13: launch_reshuffle<13>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 14: launch_reshuffle<14>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 15: launch_reshuffle<15>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 16: launch_reshuffle<16>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    case 17: launch_reshuffle<17>(ctx->rec, ctx->rec_alt, n, *a, *b, st); break;
    default: return set_err(ctx, CMTF_EUNSUPPORTED, "order %d", ctx->order);
  }
  if (ctx->rrec_valid) {
    TRY(ensure(ctx, &ctx->rrec_alt, &ctx->rrec_alt_cap, n));
    launch_reshuffle<4>(reinterpret_cast<const uint32_t*>(ctx->rrec),
                        reinterpret_cast<uint32_t*>(ctx->rrec_alt), n, *a, *b, st);
  }
  CU(cudaGetLastError());
  return CMTF_OK;
}

void launch_matrix_gather(cmtf_gpu_ctx* ctx, uint64_t epoch, cudaStream_t st) {
  uint64_t a = 1, b = 0;
  epoch_affine(ctx->mnnz / kShuffleGroup, ctx->cfg.seed, epoch, 2, &a, &b);
  launch_reshuffle<4>(reinterpret_cast<const uint32_t*>(ctx->mrec),
                      reinterpret_cast<uint32_t*>(ctx->mrec_alt), ctx->mnnz, a, b, st);
}

// Drop pending next-epoch gathers (before buffers change or are reallocated).
void drain_side(cmtf_gpu_ctx* ctx) {
  if (ctx->side) cudaStreamSynchronize(ctx->side);
  ctx->pend_t_epoch = ctx->pend_m_epoch = -1;
}

bool tensor_shuffles(const cmtf_gpu_ctx* ctx) { return ctx->nnz / kShuffleGroup >= 3; }
bool matrix_shuffles(const cmtf_gpu_ctx* ctx) {
  return ctx->mrec && ctx->mnnz / kShuffleGroup >= 3;
}

// This epoch's random visiting order of the training records (random order
// policy, whole-epoch sweeps): the gather prefetched during the previous
// epoch if there is one, else a gather now; then swap buffers.  pos[] stays
// valid through the group map (posA, posB).
int take_tensor_order(cmtf_gpu_ctx* ctx) {
  if (ctx->vt_on) return vt_table(ctx, (uint64_t)ctx->epoch);  // records stay in place
  if (vt_wanted(ctx)) return CMTF_OK;  // the sweep lays them out and draws the order
  if (!tensor_shuffles(ctx)) return CMTF_OK;
  const uint64_t ng = ctx->nnz / kShuffleGroup;
  uint64_t a = 1, b = 0;
  if (ctx->pend_t_epoch == ctx->epoch) {
    CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side_done, 0));
    a = ctx->pend_ta;
    b = ctx->pend_tb;
    ctx->pend_t_epoch = -1;
  } else {
    drain_side(ctx);
    TRY(ensure(ctx, &ctx->rec_alt, &ctx->rec_alt_cap, ctx->nnz * (ctx->order + 1)));
    TRY(launch_tensor_gather(ctx, (uint64_t)ctx->epoch, ctx->stream, &a, &b));
    ctx->last_launches += 1;
  }
  std::swap(ctx->rec, ctx->rec_alt);
  std::swap(ctx->rec_cap, ctx->rec_alt_cap);
  if (ctx->rrec_valid) {  // permuted by the same gather
    std::swap(ctx->rrec, ctx->rrec_alt);
    std::swap(ctx->rrec_cap, ctx->rrec_alt_cap);
  }
  // the group at old position G moves to a^-1 (G - b)
  const uint64_t ai = inv_mod(a, ng);
  ctx->posA = mulmod(ai, ctx->posA, ng);
  ctx->posB = mulmod(ai, (ctx->posB + ng - b) % ng, ng);
  return CMTF_OK;
}

int take_matrix_order(cmtf_gpu_ctx* ctx) {
  if (!matrix_shuffles(ctx)) return CMTF_OK;
  if (ctx->pend_m_epoch == ctx->epoch) {
    CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side_done, 0));
    ctx->pend_m_epoch = -1;
  } else {
    drain_side(ctx);
    TRY(ensure(ctx, &ctx->mrec_alt, &ctx->mrec_alt_cap, ctx->mnnz));
    launch_matrix_gather(ctx, (uint64_t)ctx->epoch, ctx->stream);
    CU(cudaGetLastError());
    ctx->last_launches += 1;
  }
  std::swap(ctx->mrec, ctx->mrec_alt);
  std::swap(ctx->mrec_cap, ctx->mrec_alt_cap);
  return CMTF_OK;
}

// Start the next epoch's gathers on the side stream; call right before the
// sweep launch (the spare buffers were last read before this point).
int prefetch_orders(cmtf_gpu_ctx* ctx, bool tensor, bool matrices) {
  tensor = tensor && tensor_shuffles(ctx) && !ctx->vt_on;
  matrices = matrices && matrix_shuffles(ctx);
  if (!tensor && !matrices) return CMTF_OK;
  const uint64_t next = (uint64_t)ctx->epoch + 1;
  if (tensor) TRY(ensure(ctx, &ctx->rec_alt, &ctx->rec_alt_cap, ctx->nnz * (ctx->order + 1)));
  if (matrices) TRY(ensure(ctx, &ctx->mrec_alt, &ctx->mrec_alt_cap, ctx->mnnz));
  CU(cudaEventRecord(ctx->ev_side_start, ctx->stream));
  CU(cudaStreamWaitEvent(ctx->side, ctx->ev_side_start, 0));
  if (tensor) {
    TRY(launch_tensor_gather(ctx, next, ctx->side, &ctx->pend_ta, &ctx->pend_tb));
    ctx->pend_t_epoch = (int64_t)next;
  }
  if (matrices) {
    launch_matrix_gather(ctx, next, ctx->side);
    CU(cudaGetLastError());
    ctx->pend_m_epoch = (int64_t)next;
  }
  CU(cudaEventRecord(ctx->ev_side_done, ctx->side));
  ctx->last_launches += (tensor ? 1 : 0) + (matrices ? 1 : 0);
  return CMTF_OK;
}

// Make pos[] exact again (serial replay and probes index records by pos).
int normalize_pos(cmtf_gpu_ctx* ctx) {
  if (ctx->pos_ids) {
    pos_from_ids_kernel<<<grid_for(ctx->nnz), 256, 0, ctx->stream>>>(ctx->rrec, ctx->nnz,
                                                                     ctx->pos);
    CU(cudaGetLastError());
    ctx->pos_ids = false;
    return CMTF_OK;
  }
  if (ctx->posA == 1 && ctx->posB == 0) return CMTF_OK;
  remap_pos_kernel<<<grid_for(ctx->nnz), 256, 0, ctx->stream>>>(ctx->pos, ctx->nnz, ctx->nnz,
                                                                 ctx->posA, ctx->posB);
  CU(cudaGetLastError());
  ctx->pos_affine = false;
  ctx->posA = 1;
  ctx->posB = 0;
  return CMTF_OK;
}

// Blocked order wanted for this context (0 = no): hog3tm (order 3, random
// order, whole sweeps) when the three factor tables exceed L2 -- then every
// entry's three row gathers miss L2 and fill 128-B lines from DRAM (config 5:
// 2.4 TB/s of random line traffic, the measured ceiling); blocking keeps
// mode 1 and 2's active blocks L2-resident (config 5 @1e9: -12% epoch time,
// RMSE within 0.3%, scripts/blocked_order_exp.py).  B = 32 with a
// mode-1-block-major stratum sequence (the mode-1 block stays across B
// strata): ncu DRAM traffic at config 5 @1e9 769 GB unblocked, 621 GB at
// B = 8 random sequence, 528 GB at B = 32 block-major (201 -> 193 ms); the
// rows of a block are reused only while the lines streamed between two
// touches (~300 B per entry of the unblocked mode and the records) fit L2,
// which B = 8's 1.25M-row blocks do not.
uint32_t blocks_wanted(const cmtf_gpu_ctx* ctx);
// the tcgen05 epoch will run (or runs) the blocked virtual order
bool vt_wanted(const cmtf_gpu_ctx* ctx) {
  return v3_tm(ctx) && ctx->cfg.order_policy == 1 && ctx->env.tm_vorder &&
         tensor_shuffles(ctx) && blocks_wanted(ctx) > 1;
}

// the factor tables do not fit L2 together
bool tables_beyond_l2(const cmtf_gpu_ctx* ctx) {
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
  uint64_t bytes = 0;
  for (int n = 0; n < ctx->order; ++n) bytes += (uint64_t)ctx->dims[n] * ctx->JP(n) * sizeof(float);
  return bytes > (uint64_t)l2;
}

uint32_t blocks_wanted(const cmtf_gpu_ctx* ctx) {
  if (ctx->order != 3 || ctx->cfg.order_policy != 1 || ctx->nnz / kShuffleGroup < 3) return 0;
  if (ctx->env.tm_blocks >= 0) return (uint32_t)ctx->env.tm_blocks;
  if (!tables_beyond_l2(ctx) || ctx->nnz < (1ull << 22)) return 0;
  return 32;
}

// Switch to the virtual order with B x B strata: lay the records (and
// rrec, ids in .w) out stratum-major -- a stable radix sort of the positions
// by stratum keeps the random order inside a stratum -- and rebuild pos[]
// from the ids.  The layout then stays until the next upload.
int vt_setup(cmtf_gpu_ctx* ctx, uint32_t B, bool rrec_in_valid) {
  const uint64_t n = ctx->nnz;
  PhaseTimer pt("vt_setup", ctx);
  drain_side(ctx);
  IdMap im{};
  im.closed = ctx->pos_affine && !ctx->pos_ids;
  if (im.closed) {
    im.n = n;
    im.ng = n / kShuffleGroup;
    im.iA = inv_mod(ctx->posA, im.ng);
    im.B = ctx->posB;
    im.ia = inv_mod(ctx->up_pa, n);
    im.pb = ctx->up_pb;
    im.m_n = ~0ull / n;
    im.m_ng = ~0ull / im.ng;
  } else {  // pos[] exact, then each record's id scattered into rrec
    TRY(normalize_pos(ctx));
    rrec_ids_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(ctx->pos, n, ctx->rrec);
    CU(cudaGetLastError());
  }
  const uint32_t S = B * B;
  const uint32_t kPartChunk = part_chunk(S);
  const uint64_t nch = (n + kPartChunk - 1) / kPartChunk;
  constexpr uint32_t kS = kMaxBlk * kMaxBlk;
  // blk_hist: [0] stratum sizes, [1] stratum cursors (run starts), [2] mode-1 block cursors
  if (!ctx->blk_hist) TRY(dalloc(ctx, &ctx->blk_hist, 3 * kS));
  CU(cudaMemsetAsync(ctx->blk_hist, 0, kS * sizeof(uint32_t), ctx->stream));
  const unsigned pg = (unsigned)std::min<uint64_t>(nch, 148ull * 8);
  part_hist_kernel<<<pg, 256, 0, ctx->stream>>>(reinterpret_cast<const uint4*>(ctx->rec), n, B,
                                                ctx->dims[0], ctx->dims[1], nullptr,
                                                ctx->blk_hist, kPartChunk);
  CU(cudaGetLastError());
  std::vector<uint32_t> hist(S), off(S, 0), off1(B, 0);
  CU(cudaMemcpyAsync(hist.data(), ctx->blk_hist, S * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  for (uint32_t s = 1; s < S; ++s) off[s] = off[s - 1] + hist[s - 1];
  for (uint32_t b = 0; b < B; ++b) off1[b] = off[b * B];
  CU(cudaMemcpyAsync(ctx->blk_hist + kS, off.data(), S * sizeof(uint32_t), cudaMemcpyHostToDevice,
                     ctx->stream));
  CU(cudaMemcpyAsync(ctx->blk_hist + 2 * kS, off1.data(), B * sizeof(uint32_t),
                     cudaMemcpyHostToDevice, ctx->stream));
  pt.tick("count");
  TRY(ensure(ctx, &ctx->rec_alt, &ctx->rec_alt_cap, n * 4));
  TRY(ensure(ctx, &ctx->rrec_alt, &ctx->rrec_alt_cap, n));
  const unsigned tg = (unsigned)std::min<uint64_t>((n + kTile - 1) / kTile, 148ull * 4);
  const uint4* rec_in = reinterpret_cast<const uint4*>(ctx->rec);
  // rrec not built yet (closed-form ids): the first pass writes {0, 0, 0, id}
  const uint4* rrec_in = rrec_in_valid ? reinterpret_cast<const uint4*>(ctx->rrec) : nullptr;
  uint4* rec_o = reinterpret_cast<uint4*>(ctx->rec_alt);
  uint4* rrec_o = reinterpret_cast<uint4*>(ctx->rrec_alt);
  if (S <= 64) {  // one pass; the result is in the alternate buffers
    part_tile_kernel<0><<<tg, 256, 0, ctx->stream>>>(rec_in, rrec_in, n, B, ctx->dims[0],
                                                     ctx->dims[1], ctx->blk_hist + kS, rec_o,
                                                     rrec_o, im, RunTab{});
    CU(cudaGetLastError());
    std::swap(ctx->rec, ctx->rec_alt);
    std::swap(ctx->rec_cap, ctx->rec_alt_cap);
    std::swap(ctx->rrec, ctx->rrec_alt);
    std::swap(ctx->rrec_cap, ctx->rrec_alt_cap);
  } else {  // by mode-1 block into the alternate buffers, then by mode-2 block back
    part_tile_kernel<1><<<tg, 256, 0, ctx->stream>>>(rec_in, rrec_in, n, B, ctx->dims[0],
                                                     ctx->dims[1], ctx->blk_hist + 2 * kS, rec_o,
                                                     rrec_o, im, RunTab{});
    CU(cudaGetLastError());
    RunTab rt{};
    for (uint32_t b = 0; b <= B; ++b) {
      rt.off[b] = b < B ? off1[b] : (uint32_t)n;
      if (b) rt.tpre[b] = rt.tpre[b - 1] + (rt.off[b] - rt.off[b - 1] + kTile - 1) / kTile;
    }
    part_tile_kernel<2><<<tg, 256, 0, ctx->stream>>>(
        rec_o, rrec_o, n, B, ctx->dims[0], ctx->dims[1], ctx->blk_hist + kS,
        reinterpret_cast<uint4*>(ctx->rec), reinterpret_cast<uint4*>(ctx->rrec), im, rt);
    CU(cudaGetLastError());
  }
  CU(cudaStreamSynchronize(ctx->stream));
  pt.tick("scatter");
  ctx->blk_B = B;
  ctx->blk_n.assign(hist.begin(), hist.end());
  ctx->blk_off.assign(B * B, 0);
  for (uint32_t s = 1; s < B * B; ++s) ctx->blk_off[s] = ctx->blk_off[s - 1] + ctx->blk_n[s - 1];
  ctx->vt_on = true;
  ctx->pos_ids = true;
  ctx->posA = 1;  // the group map no longer applies: pos[] comes from the ids
  ctx->posB = 0;
  ctx->pos_affine = false;
  ctx->last_launches += 4;
  return CMTF_OK;  // pos[] is rebuilt from the ids when something asks for it (normalize_pos)
}

// This epoch's segment table: a random stratum sequence (host draws from
// the epoch's stream) and a group-affine map per stratum.
int vt_table(cmtf_gpu_ctx* ctx, uint64_t epoch) {
  const uint32_t S = (uint32_t)ctx->blk_n.size();
  auto rng = make_rng(ctx->cfg.seed, 0x0B, epoch);
  std::vector<uint32_t> seq(S);
  for (uint32_t s = 0; s < S; ++s) seq[s] = s;
  if (ctx->env.tm_seq == 1) {
    // mode-1-block-major: a random order of the mode-1 blocks and, inside
    // each, a random order of the mode-2 blocks -- the mode-1 block stays
    // L2-resident across B consecutive strata
    const uint32_t B = ctx->blk_B;
    std::vector<uint32_t> o1(B), o2(B);
    for (uint32_t i = 0; i < B; ++i) o1[i] = i;
    for (uint32_t k = B; k > 1; --k) std::swap(o1[k - 1], o1[bounded(rng, k)]);
    for (uint32_t i = 0; i < B; ++i) {
      for (uint32_t j = 0; j < B; ++j) o2[j] = j;
      for (uint32_t k = B; k > 1; --k) std::swap(o2[k - 1], o2[bounded(rng, k)]);
      for (uint32_t j = 0; j < B; ++j) seq[i * B + j] = o1[i] * B + o2[j];
    }
  } else {
    for (uint32_t k = S; k > 1; --k) std::swap(seq[k - 1], seq[bounded(rng, k)]);
  }
  auto& h = ctx->h_vtab;
  h.clear();
  uint64_t v = 0;
  for (uint32_t k = 0; k < S; ++k) {
    const uint32_t s = seq[k];
    const uint64_t ns = ctx->blk_n[s], ng = ns / kShuffleGroup;
    if (ns == 0) continue;
    uint64_t a = 1, b = 0;
    if (ng >= 3) {
      a = 1 + bounded(rng, ng - 1);
      while (gcd64(a, ng) != 1) a = a + 1 < ng ? a + 1 : 1;
      b = bounded(rng, ng);
    }
    const uint64_t m = ng ? ~0ull / ng : 0;
    h.push_back(make_uint4((uint32_t)v, (uint32_t)ctx->blk_off[s],
                           (uint32_t)(ng * kShuffleGroup), (uint32_t)ng));
    h.push_back(make_uint4((uint32_t)a, (uint32_t)b, (uint32_t)m, (uint32_t)(m >> 32)));
    v += ns;
  }
  h.push_back(make_uint4(0xffffffffu, 0, 0, 0));
  h.push_back(make_uint4(0, 0, 0, 0));
  if (v != ctx->nnz)
    return set_err(ctx, CMTF_ECUDA, "visiting order covers %llu of %llu records",
                   (unsigned long long)v, (unsigned long long)ctx->nnz);
  if (!ctx->d_vtab) TRY(dalloc(ctx, &ctx->d_vtab, 2 * (kMaxBlk * kMaxBlk + 1)));
  CU(cudaMemcpyAsync(ctx->d_vtab, h.data(), h.size() * sizeof(uint4), cudaMemcpyHostToDevice,
                     ctx->stream));
  return CMTF_OK;
}

// One sweep (no epoch bookkeeping) over a tensor range and matrix ranges.
int sweep(cmtf_gpu_ctx* ctx, uint64_t t_lo, uint64_t t_hi, const uint64_t* m_lo,
          const uint64_t* m_hi) {
  const float eta = (float)ctx->eta;
  if (ctx->cfg.debug_count_visits && ctx->visits_epoch != ctx->epoch) {
    // a new epoch: fresh counts (the reference fills visit_counts per epoch)
    uint64_t mtot = 0;
    for (auto& M : ctx->mats) mtot += M.nnz;
    TRY(ensure(ctx, &ctx->visits, &ctx->visits_cap, std::max<uint64_t>(1, ctx->nnz)));
    TRY(ensure(ctx, &ctx->mvisits, &ctx->mvisits_cap, std::max<uint64_t>(1, mtot)));
    CU(cudaMemsetAsync(ctx->visits, 0, ctx->nnz * sizeof(uint32_t), ctx->stream));
    CU(cudaMemsetAsync(ctx->mvisits, 0, mtot * sizeof(uint32_t), ctx->stream));
    ctx->visits_epoch = ctx->epoch;
    ctx->visits_ok = ctx->cfg.exec_mode != CMTF_EXEC_SERIAL;
  }
  if (ctx->cfg.exec_mode == CMTF_EXEC_SERIAL) {
    TRY(serial_epoch(ctx, eta));
    ctx->last_launches += 1;
    CU(cudaEventRecord(ctx->ev[1], ctx->stream));
    CU(cudaEventRecord(ctx->ev[2], ctx->stream));
    return CMTF_OK;
  }
  const bool whole = t_lo == 0 && t_hi == ctx->nnz && !m_lo;
  if (ctx->cfg.order_policy == 1 && whole) TRY(take_tensor_order(ctx));
  int J = 0;
  if (v4_supported(ctx)) {
    TRY(v4_sweep(ctx, eta, t_lo, t_hi, m_lo, m_hi));  // + interleaved matrices
    ctx->last_launches += 1;
    CU(cudaEventRecord(ctx->ev[1], ctx->stream));
    CU(cudaEventRecord(ctx->ev[2], ctx->stream));
    return CMTF_OK;
  }
  if (v2_supported(ctx, &J)) {
    TRY(v2_sweep(ctx, J, eta, t_lo, t_hi, m_lo, m_hi));  // + interleaved matrices
    ctx->last_launches += 1;
    CU(cudaEventRecord(ctx->ev[1], ctx->stream));
    CU(cudaEventRecord(ctx->ev[2], ctx->stream));
    return CMTF_OK;
  }
  if (ctx->cfg.order_policy == 1 && whole) TRY(prefetch_orders(ctx, true, false));
  TRY(hogwild_tensor_sweep(ctx, eta, t_lo, t_hi));
  ctx->last_launches += 1;
  CU(cudaEventRecord(ctx->ev[1], ctx->stream));
  uint64_t vbase = 0;  // visit counts: the matrices' records concatenated
  for (size_t m = 0; m < ctx->mats.size(); ++m) {
    const auto& M = ctx->mats[m];
    const uint64_t lo = m_lo ? m_lo[m] : 0, hi = m_hi ? m_hi[m] : M.nnz;
    TRY(matrix_sweep(ctx, M, eta, lo, hi,
                     ctx->cfg.debug_count_visits ? ctx->mvisits + vbase : nullptr));
    vbase += M.nnz;
    ctx->last_launches += hi > lo ? 1 : 0;
  }
  CU(cudaEventRecord(ctx->ev[2], ctx->stream));
  return CMTF_OK;
}

// Tail of run_epoch (src/trainer.cpp:309-315): decay, divergence check.
int end_epoch(cmtf_gpu_ctx* ctx) {
  std::string offender;
  TRY(scan_nonfinite(ctx, &offender));
  CU(cudaEventRecord(ctx->ev[3], ctx->stream));
  CU(cudaEventSynchronize(ctx->ev[3]));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  ctx->last_ms[0] = ms;
  cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
  ctx->last_ms[1] = ms;
  cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
  ctx->last_ms[2] = ms;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]);
  ctx->last_ms[3] = ms;
  ctx->epoch += 1;
  ctx->eta = ctx->cfg.eta0 / (1.0 + ctx->cfg.mu * ctx->epoch);
  if (!offender.empty())
    return set_err(ctx, CMTF_EDIVERGENCE,
                   "non-finite parameter after epoch %d: %s; try a smaller initial "
                   "learning rate",
                   ctx->epoch, offender.c_str());
  return CMTF_OK;
}

}  // namespace

extern "C" {

int cmtf_gpu_run_epoch(cmtf_gpu_ctx* ctx) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  ctx->last_launches = 0;
  CU(cudaEventRecord(ctx->ev[0], ctx->stream));
  TRY(sweep(ctx, 0, ctx->nnz, nullptr, nullptr));
  return end_epoch(ctx);
}

int cmtf_gpu_sweep_range(cmtf_gpu_ctx* ctx, uint64_t t_lo, uint64_t t_hi, const uint64_t* m_lo,
                         const uint64_t* m_hi) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  if (t_hi > ctx->nnz || t_lo > t_hi)
    return set_err(ctx, CMTF_EVALIDATION, "tensor range out of bounds");
  if (m_lo && m_hi)
    for (size_t m = 0; m < ctx->mats.size(); ++m)
      if (m_hi[m] > ctx->mats[m].nnz || m_lo[m] > m_hi[m])
        return set_err(ctx, CMTF_EVALIDATION, "matrix range out of bounds");
  if (ctx->cfg.exec_mode == CMTF_EXEC_SERIAL)
    return set_err(ctx, CMTF_EUNSUPPORTED, "range sweeps are Hogwild-only");
  if (ctx->cfg.order_policy != 2 && m_lo)
    return set_err(ctx, CMTF_EVALIDATION, "matrix ranges need order_policy 2 (caller order)");
  CU(cudaEventRecord(ctx->ev[0], ctx->stream));
  return sweep(ctx, t_lo, t_hi, m_lo, m_hi);
}

int cmtf_gpu_end_epoch(cmtf_gpu_ctx* ctx) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  return end_epoch(ctx);
}

}  // extern "C"

// ---- DSGD support -------------------------------------------------------
namespace {

int snapshot_bases(cmtf_gpu_ctx* ctx) {
  auto snap = [&](float** base, const float* cur, uint64_t n) -> int {
    if (!*base) CU(cudaMalloc(reinterpret_cast<void**>(base), n * sizeof(float)));
    CU(cudaMemcpyAsync(*base, cur, n * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    return CMTF_OK;
  };
  for (int n = 0; n < ctx->order; ++n)
    TRY(snap(&ctx->baseU[n], ctx->U[n], (uint64_t)ctx->dims[n] * ctx->JP(n)));
  for (size_t m = 0; m < ctx->mats.size(); ++m)
    TRY(snap(&ctx->baseV[m], ctx->mats[m].V, (uint64_t)ctx->mats[m].cols * ctx->JP(ctx->mats[m].mode)));
  TRY(snap(&ctx->baseG, ctx->G, ctx->core_size()));
  CU(cudaStreamSynchronize(ctx->stream));
  return CMTF_OK;
}

}  // namespace

extern "C" {

int cmtf_gpu_set_shared(cmtf_gpu_ctx* ctx, int32_t world, uint32_t mode_mask, uint32_t mat_mask,
                        uint64_t nnz_global) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  if (world < 1) return set_err(ctx, CMTF_EVALIDATION, "world must be >= 1");
  ctx->world = world;
  ctx->shared_modes = mode_mask;
  ctx->shared_mats = mat_mask;
  ctx->nnz_global = nnz_global;
  ctx->v2_dirty = true;
  return snapshot_bases(ctx);
}

int cmtf_gpu_set_counts(cmtf_gpu_ctx* ctx, int32_t which, const uint32_t* counts, uint32_t n) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  CU(cudaSetDevice(ctx->device));
  uint32_t* dst = nullptr;
  float* reg = nullptr;
  float lam = (float)ctx->cfg.lambda_reg;
  if (which >= 0 && which < ctx->order) {
    if (n != ctx->dims[which]) return set_err(ctx, CMTF_EVALIDATION, "count length mismatch");
    dst = ctx->count[which];
    reg = ctx->reg[which];
  } else if (which >= 100 && which - 100 < (int)ctx->mats.size()) {
    auto& M = ctx->mats[which - 100];
    if (n != M.cols) return set_err(ctx, CMTF_EVALIDATION, "count length mismatch");
    dst = M.count;
    reg = M.vreg;
    lam = (float)(M.weight * ctx->cfg.lambda_reg);
  } else {
    return set_err(ctx, CMTF_EVALIDATION, "no such count array");
  }
  CU(cudaStreamSynchronize(ctx->stream));  // non-blocking stream: prior readers done
  CU(cudaMemcpy(dst, counts, n * sizeof(uint32_t), cudaMemcpyHostToDevice));
  drain_side(ctx);
  if (which < ctx->order) ctx->rrec_valid = false;
  reg_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(dst, n, lam, reg);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->v2_dirty = true;  // hot sets follow the counts
  return CMTF_OK;
}

}  // extern "C"

namespace {

__global__ void delta_kernel(const float* cur, const float* base, float* d, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = cur[i] - base[i];
}
__global__ void accum_delta_kernel(const float* cur, const float* base, float* d, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    d[i] += cur[i] - base[i];
}
__global__ void rebase_kernel(float* cur, float* base, const float* d, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = base[i] + d[i];
    cur[i] = v;
    base[i] = v;
  }
}

struct SyncArr {
  float* cur;
  float* base;
  uint64_t n;
};

std::vector<SyncArr> sync_arrays(cmtf_gpu_ctx* ctx, uint32_t mode_mask, uint32_t mat_mask,
                                 int core) {
  std::vector<SyncArr> v;
  for (int n = 0; n < ctx->order; ++n)
    if ((mode_mask >> n) & 1u)
      v.push_back({ctx->U[n], ctx->baseU[n], (uint64_t)ctx->dims[n] * ctx->JP(n)});
  for (size_t m = 0; m < ctx->mats.size(); ++m)
    if ((mat_mask >> m) & 1u)
      v.push_back({ctx->mats[m].V, ctx->baseV[m],
                   (uint64_t)ctx->mats[m].cols * ctx->JP(ctx->mats[m].mode)});
  if (core) v.push_back({ctx->G, ctx->baseG, ctx->core_size()});
  return v;
}

}  // namespace

extern "C" {

int cmtf_gpu_comm_unique_id(void* id_out) {
  NcclApi& N = nccl_api();
  if (!N.getUniqueId) return set_err(nullptr, CMTF_ENCCL, "%s", N.error.c_str());
  ncclUniqueId id;
  ncclResult_t r = N.getUniqueId(&id);
  if (r != ncclSuccess)
    return set_err(nullptr, CMTF_ENCCL, "ncclGetUniqueId: %s", N.getErrorString(r));
  std::memcpy(id_out, &id, sizeof id);
  return CMTF_OK;
}

int cmtf_gpu_comm_init(cmtf_gpu_ctx* ctx, int32_t nranks, int32_t rank, const void* unique_id) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  CU(cudaSetDevice(ctx->device));
  NcclApi& N = nccl_api();
  if (!N.getUniqueId) return set_err(ctx, CMTF_ENCCL, "%s", N.error.c_str());
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  if (ctx->comm) N.commDestroy(ctx->comm);
  ctx->comm = nullptr;
  ncclResult_t r = N.commInitRank(&ctx->comm, nranks, id, rank);
  if (r != ncclSuccess)
    return set_err(ctx, CMTF_ENCCL, "ncclCommInitRank: %s", N.getErrorString(r));
  return CMTF_OK;
}

int cmtf_gpu_sync(cmtf_gpu_ctx* ctx, uint32_t mode_mask, uint32_t mat_mask, int32_t core) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  if (!ctx->baseG) return set_err(ctx, CMTF_EVALIDATION, "call cmtf_gpu_set_shared first");
  auto arrs = sync_arrays(ctx, mode_mask, mat_mask, core);
  uint64_t total = 0;
  for (auto& s : arrs) total += s.n;
  TRY(ensure(ctx, &ctx->sync_buf, &ctx->sync_cap, total));
  uint64_t off = 0;
  for (auto& s : arrs) {
    delta_kernel<<<grid_for(s.n), 256, 0, ctx->stream>>>(s.cur, s.base, ctx->sync_buf + off, s.n);
    off += s.n;
  }
  CU(cudaGetLastError());
  if (ctx->comm && total) {
    NcclApi& N = nccl_api();
    ncclResult_t r = N.allReduce(ctx->sync_buf, ctx->sync_buf, total, ncclFloat, ncclSum,
                                 ctx->comm, ctx->stream);
    if (r != ncclSuccess)
      return set_err(ctx, CMTF_ENCCL, "ncclAllReduce: %s", N.getErrorString(r));
  }
  off = 0;
  for (auto& s : arrs) {
    rebase_kernel<<<grid_for(s.n), 256, 0, ctx->stream>>>(s.cur, s.base, ctx->sync_buf + off, s.n);
    off += s.n;
  }
  CU(cudaGetLastError());
  // no host wait: the next sweep is ordered after the reduction on the
  // context's stream
  return CMTF_OK;
}

namespace {
// rows [lo, hi) of factor `which` (mode n, or 100 + m for coupled factor m)
int rows_of(cmtf_gpu_ctx* ctx, int32_t which, uint32_t lo, uint32_t hi, float** p, uint64_t* n) {
  uint32_t rows = 0, JP = 0;
  float* base = nullptr;
  if (which >= 0 && which < ctx->order) {
    rows = ctx->dims[which];
    JP = ctx->JP(which);
    base = ctx->U[which];
  } else if (which >= 100 && which - 100 < (int)ctx->mats.size()) {
    const auto& M = ctx->mats[which - 100];
    rows = M.cols;
    JP = ctx->JP(M.mode);
    base = M.V;
  } else {
    return set_err(ctx, CMTF_EVALIDATION, "no such factor %d", which);
  }
  if (lo > hi || hi > rows) return set_err(ctx, CMTF_EVALIDATION, "row range out of bounds");
  *p = base + (uint64_t)lo * JP;
  *n = (uint64_t)(hi - lo) * JP;
  return CMTF_OK;
}
}  // namespace

int cmtf_gpu_exchange_rows(cmtf_gpu_ctx* ctx, int32_t which, uint32_t send_lo, uint32_t send_hi,
                           int32_t send_peer, uint32_t recv_lo, uint32_t recv_hi,
                           int32_t recv_peer) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  if (!ctx->comm) return set_err(ctx, CMTF_EVALIDATION, "no communicator (cmtf_gpu_comm_init)");
  float *sp = nullptr, *rp = nullptr;
  uint64_t sn = 0, rn = 0;
  TRY(rows_of(ctx, which, send_lo, send_hi, &sp, &sn));
  TRY(rows_of(ctx, which, recv_lo, recv_hi, &rp, &rn));
  NcclApi& N = nccl_api();
  ncclResult_t r = N.groupStart();
  if (r == ncclSuccess && sn) r = N.send(sp, sn, ncclFloat, send_peer, ctx->comm, ctx->stream);
  if (r == ncclSuccess && rn) r = N.recv(rp, rn, ncclFloat, recv_peer, ctx->comm, ctx->stream);
  const ncclResult_t r2 = N.groupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return set_err(ctx, CMTF_ENCCL, "ncclSend/ncclRecv: %s", N.getErrorString(r));
  return CMTF_OK;
}

int cmtf_gpu_exchange_rows_local(cmtf_gpu_ctx* src, cmtf_gpu_ctx* dst, int32_t which, uint32_t lo,
                                 uint32_t hi) {
  TRY(require_bundle(src));
  TRY(require_bundle(dst));
  cmtf_gpu_ctx* ctx = dst;
  if (src->device != dst->device) return set_err(dst, CMTF_EVALIDATION, "exchange_rows_local needs one device");
  CU(cudaSetDevice(dst->device));
  float *sp = nullptr, *dp = nullptr;
  uint64_t sn = 0, dn = 0;
  TRY(rows_of(src, which, lo, hi, &sp, &sn));
  TRY(rows_of(dst, which, lo, hi, &dp, &dn));
  if (sn != dn) return set_err(dst, CMTF_EVALIDATION, "row layouts differ");
  CU(cudaStreamSynchronize(src->stream));
  CU(cudaMemcpyAsync(dp, sp, sn * sizeof(float), cudaMemcpyDeviceToDevice, dst->stream));
  CU(cudaStreamSynchronize(dst->stream));
  return CMTF_OK;
}

int cmtf_gpu_broadcast_rows(cmtf_gpu_ctx* ctx, int32_t which, int32_t n_blocks,
                            const uint32_t* lo, const uint32_t* hi) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  if (!ctx->comm) return set_err(ctx, CMTF_EVALIDATION, "no communicator (cmtf_gpu_comm_init)");
  NcclApi& N = nccl_api();
  ncclResult_t r = N.groupStart();
  for (int b = 0; b < n_blocks && r == ncclSuccess; ++b) {
    float* p = nullptr;
    uint64_t n = 0;
    TRY(rows_of(ctx, which, lo[b], hi[b], &p, &n));
    if (n) r = N.broadcast(p, p, n, ncclFloat, b, ctx->comm, ctx->stream);
  }
  const ncclResult_t r2 = N.groupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return set_err(ctx, CMTF_ENCCL, "ncclBroadcast: %s", N.getErrorString(r));
  return CMTF_OK;
}

int cmtf_gpu_sync_local(cmtf_gpu_ctx* const* ctxs, int32_t n, uint32_t mode_mask,
                        uint32_t mat_mask, int32_t core) {
  cmtf_gpu_ctx* ctx = n > 0 ? ctxs[0] : nullptr;
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "no contexts");
  for (int i = 0; i < n; ++i) {
    TRY(require_bundle(ctxs[i]));
    if (ctxs[i]->device != ctx->device)
      return set_err(ctx, CMTF_EVALIDATION, "sync_local needs one device");
    if (!ctxs[i]->baseG) return set_err(ctx, CMTF_EVALIDATION, "call cmtf_gpu_set_shared first");
    CU(cudaStreamSynchronize(ctxs[i]->stream));
  }
  CU(cudaSetDevice(ctx->device));
  auto a0 = sync_arrays(ctx, mode_mask, mat_mask, core);
  uint64_t total = 0;
  for (auto& s : a0) total += s.n;
  TRY(ensure(ctx, &ctx->sync_buf, &ctx->sync_cap, total));
  CU(cudaMemsetAsync(ctx->sync_buf, 0, total * sizeof(float), ctx->stream));
  for (int i = 0; i < n; ++i) {
    auto ai = sync_arrays(ctxs[i], mode_mask, mat_mask, core);
    uint64_t off = 0;
    for (auto& s : ai) {
      accum_delta_kernel<<<grid_for(s.n), 256, 0, ctx->stream>>>(s.cur, s.base,
                                                                 ctx->sync_buf + off, s.n);
      off += s.n;
    }
  }
  for (int i = 0; i < n; ++i) {
    auto ai = sync_arrays(ctxs[i], mode_mask, mat_mask, core);
    uint64_t off = 0;
    for (auto& s : ai) {
      rebase_kernel<<<grid_for(s.n), 256, 0, ctx->stream>>>(s.cur, s.base, ctx->sync_buf + off,
                                                            s.n);
      off += s.n;
    }
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(ctx->stream));
  return CMTF_OK;
}

int cmtf_gpu_epoch_stats(cmtf_gpu_ctx* ctx, double lambda_reg, double* train_rmse,
                         double* objective) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  double sse = 0.0;
  TRY(tensor_sse(ctx, ctx->rec, ctx->nnz, &sse));
  std::vector<float> core(ctx->core_size());
  CU(cudaMemcpy(core.data(), ctx->G, core.size() * sizeof(float), cudaMemcpyDeviceToHost));
  double gn = 0.0;
  for (float g : core) gn += (double)g * g;
  double f_t = sse + lambda_reg * gn;
  for (int n = 0; n < ctx->order; ++n) {
    double rn = 0.0;
    TRY(row_norms(ctx, ctx->U[n], ctx->dims[n], ctx->J(n), ctx->JP(n), ctx->count[n], &rn));
    f_t += lambda_reg * rn;
  }
  double obj = 0.5 * f_t;
  for (auto& M : ctx->mats) {
    double f_m = 0.0, rn = 0.0;
    TRY(matrix_sse(ctx, M, &f_m));
    TRY(row_norms(ctx, M.V, M.cols, ctx->J(M.mode), ctx->JP(M.mode), M.count, &rn));
    f_m += lambda_reg * rn;
    obj += 0.5 * M.weight * f_m;
  }
  if (train_rmse) *train_rmse = std::sqrt(sse / (double)ctx->nnz);
  if (objective) *objective = obj;
  return CMTF_OK;
}

int cmtf_gpu_test_rmse(cmtf_gpu_ctx* ctx, const uint32_t* idx, const double* vals,
                       uint64_t nnz, double* rmse) {
  TRY(require_bundle(ctx));
  if (nnz == 0) return set_err(ctx, CMTF_EVALIDATION, "cannot evaluate an empty tensor");
  CU(cudaSetDevice(ctx->device));
  const int N = ctx->order;
  uint32_t* d_idx = nullptr;
  double* d_vals = nullptr;
  uint32_t *d_rec = nullptr, *d_keys = nullptr, *d_ids = nullptr;
  if (on_device(ctx, idx) || on_device(ctx, vals)) CU(cudaDeviceSynchronize());
  TRY(dalloc(ctx, &d_idx, nnz * N));
  TRY(dalloc(ctx, &d_vals, nnz));
  TRY(dalloc(ctx, &d_rec, nnz * (N + 1)));
  TRY(dalloc(ctx, &d_keys, nnz));
  TRY(dalloc(ctx, &d_ids, nnz));
  // cudaMemcpyDefault: host (pageable or pinned) or device source (UVA)
  CU(cudaMemcpyAsync(d_idx, idx, nnz * N * sizeof(uint32_t), cudaMemcpyDefault,
                     ctx->stream));
  CU(cudaMemcpyAsync(d_vals, vals, nnz * sizeof(double), cudaMemcpyDefault,
                     ctx->stream));
  // counts of a test tensor must not touch the training counts: use scratch
  std::vector<uint32_t*> scratch(N, nullptr);
  ModeTables mt = mode_tables(ctx);
  for (int n = 0; n < N; ++n) {
    TRY(dalloc(ctx, &scratch[n], ctx->dims[n]));
    CU(cudaMemsetAsync(scratch[n], 0, ctx->dims[n] * sizeof(uint32_t), ctx->stream));
    mt.count[n] = scratch[n];
  }
  CU(cudaMemsetAsync(ctx->d_first, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
  pack_tensor_kernel<<<grid_for(nnz), 256, 0, ctx->stream>>>(
      d_idx, d_vals, 0, nnz, N, mt, 0, 0u, d_rec, nullptr, nullptr, ctx->d_first);
  CU(cudaGetLastError());
  unsigned long long bad[2];
  CU(cudaMemcpyAsync(bad, ctx->d_first, sizeof bad, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  int rc = CMTF_OK;
  if (bad[0] != ~0ull) rc = set_err(ctx, CMTF_EVALIDATION, "test tensor index out of range");
  else if (bad[1] != ~0ull) rc = set_err(ctx, CMTF_EVALIDATION, "test tensor value is not finite");
  double sse = 0.0;
  if (rc == CMTF_OK) rc = tensor_sse(ctx, d_rec, nnz, &sse);
  cudaFree(d_idx);
  cudaFree(d_vals);
  cudaFree(d_rec);
  cudaFree(d_keys);
  cudaFree(d_ids);
  for (auto p : scratch) cudaFree(p);
  if (rc != CMTF_OK) return rc;
  *rmse = std::sqrt(sse / (double)nnz);
  return CMTF_OK;
}

int cmtf_gpu_matrix_rmse(cmtf_gpu_ctx* ctx, int32_t m, double* rmse) {
  TRY(require_bundle(ctx));
  if (m < 0 || m >= (int)ctx->mats.size())
    return set_err(ctx, CMTF_EVALIDATION, "no coupled factor for this matrix");
  if (ctx->mats[m].nnz == 0)
    return set_err(ctx, CMTF_EVALIDATION, "cannot evaluate an empty matrix");
  double sse = 0.0;
  TRY(matrix_sse(ctx, ctx->mats[m], &sse));
  *rmse = std::sqrt(sse / (double)ctx->mats[m].nnz);
  return CMTF_OK;
}

// ---------------------------------------------------------------------
// finalize_orthogonalize (src/tucker.cpp:226-283): every factor U_n = Q R
// with Q orthonormal and R upper triangular with a nonnegative diagonal (the
// reference's sign fix after Householder QR, :250-255) -- for a full-rank U_n
// that factorisation is unique, so it is computed here as CholeskyQR2 in f64
// on the device (Gram matrix -> Cholesky -> Q = U R^{-1}, twice); the core
// takes core x_n R (core_mode_product, :167-206) and every coupled factor of
// mode n becomes V R^T (:270-282).  Output only: the device training state is
// left as it is (the reference finalises the model train() returns).
// ---------------------------------------------------------------------
__global__ void rows_to_f64_kernel(const float* U, uint64_t rows, uint32_t J, uint32_t JP,
                                   double* X) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < rows * J;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = q / J;
    X[q] = (double)U[i * JP + (q - i * J)];
  }
}

// gram[a][b] += sum_i X[i][a] X[i][b]; the J*J pairs are strided over the
// block (any J up to kMaxRank with a fixed 256-thread block)
__global__ void gram_f64_kernel(const double* X, uint64_t rows, uint32_t J, double* gram) {
  for (uint32_t t = threadIdx.x; t < J * J; t += blockDim.x) {
    const uint32_t a = t / J, b = t - (t / J) * J;
    double acc = 0.0;
    for (uint64_t i = blockIdx.x; i < rows; i += gridDim.x) acc += X[i * J + a] * X[i * J + b];
    atomicAdd(gram + t, acc);
  }
}

// X <- X M (M: J x J row-major)
__global__ void right_mult_f64_kernel(double* X, uint64_t rows, uint32_t J, const double* M) {
  extern __shared__ double Ms[];
  for (uint32_t q = threadIdx.x; q < J * J; q += blockDim.x) Ms[q] = M[q];
  __syncthreads();
  double row[kMaxRank];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
       i += (uint64_t)gridDim.x * blockDim.x) {
    for (uint32_t k = 0; k < J; ++k) row[k] = X[i * J + k];
    for (uint32_t k = 0; k < J; ++k) {
      double acc = 0.0;
      for (uint32_t j = 0; j < J; ++j) acc += row[j] * Ms[j * J + k];
      X[i * J + k] = acc;
    }
  }
}

namespace {
// Upper R (row-major, J x J) with R^T R = A; false if A is not (numerically)
// positive definite: a pivot below 1e-13 of its diagonal means the factor's
// condition number is beyond what CholeskyQR2 resolves in f64 (~1e6.5), and
// the caller falls back to Householder QR.
bool cholesky_upper(const std::vector<double>& A, uint32_t J, std::vector<double>& R) {
  R.assign((size_t)J * J, 0.0);
  for (uint32_t k = 0; k < J; ++k) {
    double d = A[(size_t)k * J + k];
    const double diag = d;
    for (uint32_t i = 0; i < k; ++i) d -= R[(size_t)i * J + k] * R[(size_t)i * J + k];
    if (!(d > 1e-13 * diag)) return false;
    const double rkk = std::sqrt(d);
    R[(size_t)k * J + k] = rkk;
    for (uint32_t j = k + 1; j < J; ++j) {
      double v = A[(size_t)k * J + j];
      for (uint32_t i = 0; i < k; ++i) v -= R[(size_t)i * J + k] * R[(size_t)i * J + j];
      R[(size_t)k * J + j] = v / rkk;
    }
  }
  return true;
}

// Householder QR of X (rows x J, row-major, f64) in place: X <- Q (thin,
// rows x J) and R (J x J, upper), with the reference's sign fix (a negative
// R diagonal flips that row of R and column of Q, src/tucker.cpp:250-255).
// The host fallback of the device CholeskyQR2 for ill-conditioned or
// rank-deficient factors, where Eigen's HouseholderQR (the reference) still
// returns a factorisation.
void householder_qr(std::vector<double>& X, uint64_t rows, uint32_t J, std::vector<double>& R) {
  std::vector<std::vector<double>> V(J);
  std::vector<double> beta(J, 0.0);
  for (uint32_t k = 0; k < J; ++k) {
    double nrm = 0.0;
    for (uint64_t i = k; i < rows; ++i) nrm += X[i * J + k] * X[i * J + k];
    nrm = std::sqrt(nrm);
    std::vector<double>& v = V[k];
    v.assign(rows - k, 0.0);
    for (uint64_t i = k; i < rows; ++i) v[i - k] = X[i * J + k];
    const double x0 = v[0];
    const double alpha = x0 >= 0 ? -nrm : nrm;
    v[0] = x0 - alpha;
    double vv = 0.0;
    for (double q : v) vv += q * q;
    beta[k] = vv > 0.0 ? 2.0 / vv : 0.0;
    for (uint32_t j = k; j < J; ++j) {  // A[k:, j] -= beta v (v . A[k:, j])
      double dot = 0.0;
      for (uint64_t i = k; i < rows; ++i) dot += v[i - k] * X[i * J + j];
      dot *= beta[k];
      for (uint64_t i = k; i < rows; ++i) X[i * J + j] -= dot * v[i - k];
    }
  }
  R.assign((size_t)J * J, 0.0);
  for (uint32_t a = 0; a < J; ++a)
    for (uint32_t b = a; b < J; ++b) R[(size_t)a * J + b] = X[(uint64_t)a * J + b];
  // Q = H_0 ... H_{J-1} [I; 0]
  std::fill(X.begin(), X.end(), 0.0);
  for (uint32_t k = 0; k < J; ++k) X[(uint64_t)k * J + k] = 1.0;
  for (int k = (int)J - 1; k >= 0; --k) {
    const std::vector<double>& v = V[k];
    for (uint32_t j = 0; j < J; ++j) {
      double dot = 0.0;
      for (uint64_t i = k; i < rows; ++i) dot += v[i - k] * X[i * J + j];
      dot *= beta[k];
      for (uint64_t i = k; i < rows; ++i) X[i * J + j] -= dot * v[i - k];
    }
  }
  for (uint32_t k = 0; k < J; ++k)
    if (R[(size_t)k * J + k] < 0) {
      for (uint32_t b = 0; b < J; ++b) R[(size_t)k * J + b] = -R[(size_t)k * J + b];
      for (uint64_t i = 0; i < rows; ++i) X[i * J + k] = -X[i * J + k];
    }
}

// inverse of an upper-triangular R (row-major)
std::vector<double> upper_inverse(const std::vector<double>& R, uint32_t J) {
  std::vector<double> X((size_t)J * J, 0.0);
  for (uint32_t c = 0; c < J; ++c) {  // solve R x = e_c by back substitution
    for (int r = (int)J - 1; r >= 0; --r) {
      double v = (uint32_t)r == c ? 1.0 : 0.0;
      for (uint32_t k = r + 1; k < J; ++k) v -= R[(size_t)r * J + k] * X[(size_t)k * J + c];
      X[(size_t)r * J + c] = v / R[(size_t)r * J + r];
    }
  }
  return X;
}

std::vector<double> matmul(const std::vector<double>& A, const std::vector<double>& B, uint32_t J) {
  std::vector<double> C((size_t)J * J, 0.0);
  for (uint32_t i = 0; i < J; ++i)
    for (uint32_t k = 0; k < J; ++k)
      for (uint32_t j = 0; j < J; ++j) C[(size_t)i * J + j] += A[(size_t)i * J + k] * B[(size_t)k * J + j];
  return C;
}
}  // namespace

// apply_nonnegative_projection (src/trainer.cpp:348-387), on host f64 copies:
// clamp at 0, unit-norm factor columns, norms absorbed by the core slices and
// the coupled factors' columns.
int finalize_nonnegative(cmtf_gpu_ctx* ctx, double* core, double* const* factors,
                         double* const* couplings) {
  const int N = ctx->order;
  std::vector<double> G(ctx->core_size());
  std::vector<std::vector<double>> F(N), V(ctx->mats.size());
  std::vector<double*> fp(N), vp(ctx->mats.size());
  for (int n = 0; n < N; ++n) {
    F[n].resize((uint64_t)ctx->dims[n] * ctx->J(n));
    fp[n] = F[n].data();
  }
  for (size_t m = 0; m < ctx->mats.size(); ++m) {
    V[m].resize((uint64_t)ctx->mats[m].cols * ctx->J(ctx->mats[m].mode));
    vp[m] = V[m].data();
  }
  TRY(cmtf_gpu_get_model(ctx, G.data(), fp.data(), vp.empty() ? nullptr : vp.data()));
  const bool cp = ctx->cfg.core_structure == 1;
  if (cp) G.resize(ctx->ranks[0]);  // the stored superdiagonal (src/trainer.cpp:370-371)
  auto clamp = [](std::vector<double>& v) {
    for (double& x : v)
      if (x < 0) x = 0;
  };
  clamp(G);
  for (auto& f : F) clamp(f);
  for (auto& v : V) clamp(v);
  for (int n = 0; n < N; ++n) {
    const uint32_t J = ctx->J(n);
    uint64_t stride = 1;
    for (int m = N - 1; m > n; --m) stride *= ctx->J(m);
    for (uint32_t k = 0; k < J; ++k) {
      double nsq = 0.0;
      for (uint64_t i = 0; i < ctx->dims[n]; ++i) nsq += F[n][i * J + k] * F[n][i * J + k];
      if (nsq == 0.0) continue;  // absorbed as norm 1
      const double norm = std::sqrt(nsq);
      for (uint64_t i = 0; i < ctx->dims[n]; ++i) F[n][i * J + k] /= norm;
      if (cp) {
        G[k] *= norm;
      } else {
        const uint64_t block = stride * J;
        for (uint64_t base = 0; base < G.size(); base += block)
          for (uint64_t t = 0; t < stride; ++t) G[base + k * stride + t] *= norm;
      }
      for (size_t m = 0; m < ctx->mats.size(); ++m)
        if (ctx->mats[m].mode == n)
          for (uint64_t i = 0; i < ctx->mats[m].cols; ++i) V[m][i * J + k] *= norm;
    }
  }
  if (core) std::copy(G.begin(), G.end(), core);
  for (int n = 0; n < N; ++n)
    if (factors && factors[n]) std::copy(F[n].begin(), F[n].end(), factors[n]);
  for (size_t m = 0; m < ctx->mats.size(); ++m)
    if (couplings && couplings[m]) std::copy(V[m].begin(), V[m].end(), couplings[m]);
  return CMTF_OK;
}

int cmtf_gpu_finalize_model(cmtf_gpu_ctx* ctx, double* core, double* const* factors,
                            double* const* couplings) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize(ctx->stream));
  // train()'s tail (src/trainer.cpp:342-345)
  if (ctx->cfg.nonnegative) return finalize_nonnegative(ctx, core, factors, couplings);
  const int N = ctx->order;
  for (int n = 0; n < N; ++n)
    if (ctx->dims[n] < ctx->ranks[n])
      return set_err(ctx, CMTF_EVALIDATION,
                     "mode %d has fewer rows than its rank; cannot orthogonalize", n + 1);
  // the core in f64, row-major, last mode fastest (src/tucker.cpp:49-54)
  std::vector<float> cf(ctx->core_size());
  CU(cudaMemcpy(cf.data(), ctx->G, cf.size() * sizeof(float), cudaMemcpyDeviceToHost));
  std::vector<double> G(cf.begin(), cf.end());
  uint64_t maxrows = 0;
  for (int n = 0; n < N; ++n) maxrows = std::max<uint64_t>(maxrows, ctx->dims[n]);
  for (auto& M : ctx->mats) maxrows = std::max<uint64_t>(maxrows, M.cols);
  uint32_t maxJ = 0;
  for (int n = 0; n < N; ++n) maxJ = std::max(maxJ, ctx->J(n));
  double *X = nullptr, *dM = nullptr, *dgram = nullptr;
  CU(cudaMalloc(&X, maxrows * maxJ * sizeof(double)));
  CU(cudaMalloc(&dM, (size_t)maxJ * maxJ * sizeof(double)));
  CU(cudaMalloc(&dgram, (size_t)maxJ * maxJ * sizeof(double)));
  std::vector<std::vector<double>> R_by_mode(N);
  int rc = CMTF_OK;
  auto run = [&]() -> int {
    for (int n = 0; n < N; ++n) {
      const uint32_t J = ctx->J(n), JP = ctx->JP(n);
      const uint64_t rows = ctx->dims[n];
      rows_to_f64_kernel<<<grid_for(rows * J), 256, 0, ctx->stream>>>(ctx->U[n], rows, J, JP, X);
      CU(cudaGetLastError());
      std::vector<double> R((size_t)J * J, 0.0);
      for (uint32_t k = 0; k < J; ++k) R[(size_t)k * J + k] = 1.0;
      bool chol_ok = true;
      for (int pass = 0; pass < 2 && chol_ok; ++pass) {  // CholeskyQR2
        CU(cudaMemsetAsync(dgram, 0, (size_t)J * J * sizeof(double), ctx->stream));
        gram_f64_kernel<<<(unsigned)std::min<uint64_t>(rows, 4096), 256, 0, ctx->stream>>>(
            X, rows, J, dgram);
        CU(cudaGetLastError());
        std::vector<double> A((size_t)J * J), Rk;
        CU(cudaMemcpyAsync(A.data(), dgram, A.size() * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (!cholesky_upper(A, J, Rk)) {
          chol_ok = false;
          break;
        }
        const std::vector<double> Ri = upper_inverse(Rk, J);
        CU(cudaMemcpyAsync(dM, Ri.data(), Ri.size() * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        right_mult_f64_kernel<<<grid_for(rows), 128, (size_t)J * J * sizeof(double),
                                ctx->stream>>>(X, rows, J, dM);
        CU(cudaGetLastError());
        R = matmul(Rk, R, J);
        CU(cudaStreamSynchronize(ctx->stream));  // Ri lives on the host stack
      }
      if (!chol_ok) {
        // ill-conditioned or rank-deficient factor: Householder QR on the
        // host from the factor as trained (the reference's algorithm)
        rows_to_f64_kernel<<<grid_for(rows * J), 256, 0, ctx->stream>>>(ctx->U[n], rows, J, JP,
                                                                        X);
        CU(cudaGetLastError());
        std::vector<double> hX(rows * J);
        CU(cudaMemcpyAsync(hX.data(), X, hX.size() * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        householder_qr(hX, rows, J, R);
        CU(cudaMemcpyAsync(X, hX.data(), hX.size() * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
      }
      if (factors && factors[n]) {
        CU(cudaMemcpyAsync(factors[n], X, rows * J * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
      }
      // core <- core x_n R: new[.. j ..] = sum_i R[j][i] core[.. i ..]
      uint64_t stride = 1;
      for (int m = N - 1; m > n; --m) stride *= ctx->J(m);
      const uint64_t outer = G.size() / (stride * J);
      std::vector<double> H(G.size(), 0.0);
      for (uint64_t o = 0; o < outer; ++o)
        for (uint32_t j = 0; j < J; ++j)
          for (uint32_t i = 0; i < J; ++i) {
            const double r = R[(size_t)j * J + i];
            if (r == 0.0) continue;
            const double* src = G.data() + (o * J + i) * stride;
            double* dst = H.data() + (o * J + j) * stride;
            for (uint64_t s2 = 0; s2 < stride; ++s2) dst[s2] += r * src[s2];
          }
      G.swap(H);
      R_by_mode[n] = R;
    }
    // coupled factors: V <- V R^T
    for (size_t m = 0; m < ctx->mats.size(); ++m) {
      const auto& M = ctx->mats[m];
      const uint32_t J = ctx->J(M.mode), JP = ctx->JP(M.mode);
      if (!couplings || !couplings[m]) continue;
      std::vector<double> Rt((size_t)J * J);
      for (uint32_t a = 0; a < J; ++a)
        for (uint32_t b = 0; b < J; ++b) Rt[(size_t)a * J + b] = R_by_mode[M.mode][(size_t)b * J + a];
      rows_to_f64_kernel<<<grid_for((uint64_t)M.cols * J), 256, 0, ctx->stream>>>(M.V, M.cols, J,
                                                                                  JP, X);
      CU(cudaMemcpyAsync(dM, Rt.data(), Rt.size() * sizeof(double), cudaMemcpyHostToDevice,
                         ctx->stream));
      right_mult_f64_kernel<<<grid_for(M.cols), 128, (size_t)J * J * sizeof(double),
                              ctx->stream>>>(X, M.cols, J, dM);
      // (the context stream is non-blocking: copy on it, then wait)
      CU(cudaMemcpyAsync(couplings[m], X, (uint64_t)M.cols * J * sizeof(double),
                         cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    }
    if (core) std::copy(G.begin(), G.end(), core);
    return CMTF_OK;
  };
  rc = run();
  cudaFree(X);
  cudaFree(dM);
  cudaFree(dgram);
  return rc;
}

// train (src/trainer.cpp:318-346) minus the QR finalisation.
int cmtf_gpu_train(cmtf_gpu_ctx* ctx, double* log, int32_t log_capacity,
                   int32_t* n_log) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  TRY(cmtf_gpu_make_state(ctx));
  const auto start = std::chrono::steady_clock::now();
  double prev = std::numeric_limits<double>::quiet_NaN();
  int32_t nl = 0;
  if (n_log) *n_log = 0;
  for (int ep = 0; ep < ctx->cfg.max_epochs; ++ep) {
    TRY(cmtf_gpu_run_epoch(ctx));
    double rmse = 0, obj = 0;
    TRY(cmtf_gpu_epoch_stats(ctx, ctx->cfg.lambda_reg, &rmse, &obj));
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    if (log && nl < log_capacity) {
      log[4 * nl + 0] = ctx->epoch;
      log[4 * nl + 1] = rmse;
      log[4 * nl + 2] = obj;
      log[4 * nl + 3] = secs;
    }
    ++nl;
    if (n_log) *n_log = nl;
    if (std::isfinite(prev) && prev > 0 && std::abs(prev - rmse) / prev < ctx->cfg.rel_tol)
      break;
    prev = rmse;
  }
  return CMTF_OK;
}

int cmtf_gpu_entry_grads(cmtf_gpu_ctx* ctx, const uint64_t* ids, uint64_t n,
                         double* xhat, double* residual, double* grow, double* gcore) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  if (n == 0) return CMTF_OK;
  for (uint64_t e = 0; e < n; ++e)
    if (ids[e] >= ctx->nnz) return set_err(ctx, CMTF_EVALIDATION, "entry id out of range");
  const CoreShape cs = core_shape(ctx);
  const uint32_t sumJ = cs.off[cs.order];
  uint64_t* d_ids = nullptr;
  float *d_x = nullptr, *d_r = nullptr, *d_grow = nullptr, *d_gcore = nullptr;
  TRY(dalloc(ctx, &d_ids, n));
  TRY(dalloc(ctx, &d_x, n));
  TRY(dalloc(ctx, &d_r, n));
  TRY(dalloc(ctx, &d_grow, n * sumJ));
  if (gcore) TRY(dalloc(ctx, &d_gcore, n * cs.size));
  CU(cudaMemcpyAsync(d_ids, ids, n * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  TRY(normalize_pos(ctx));
  ProbeArgs a{};
  a.cs = cs;
  a.G = ctx->G;
  a.rec = ctx->rec;
  a.pos = ctx->pos;
  a.ids = d_ids;
  a.mt = mode_tables(ctx);
  a.n = n;
  a.core_reg = (float)(ctx->cfg.lambda_reg / (double)nnz_all_of(ctx));
  a.with_core = gcore != nullptr;
  a.xhat = d_x;
  a.resid = d_r;
  a.grow = d_grow;
  a.gcore = d_gcore;
  const int bt = 128;
  const size_t smem = sizeof(float) * (bt / 32) * 2 * sumJ;
  auto kern = ctx->cfg.kernel == CMTF_KERNEL_OPT ? probe_kernel<true> : probe_kernel<false>;
  kern<<<grid_for(n, bt / 32), bt, smem, ctx->stream>>>(a);
  CU(cudaGetLastError());
  std::vector<float> hx(n), hr(n), hg(n * sumJ), hc(gcore ? n * cs.size : 0);
  CU(cudaMemcpyAsync(hx.data(), d_x, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(hr.data(), d_r, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(hg.data(), d_grow, n * sumJ * sizeof(float), cudaMemcpyDeviceToHost,
                     ctx->stream));
  if (gcore)
    CU(cudaMemcpyAsync(hc.data(), d_gcore, hc.size() * sizeof(float),
                       cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_ids);
  cudaFree(d_x);
  cudaFree(d_r);
  cudaFree(d_grow);
  if (d_gcore) cudaFree(d_gcore);
  for (uint64_t e = 0; e < n; ++e) {
    if (xhat) xhat[e] = hx[e];
    if (residual) residual[e] = hr[e];
  }
  for (uint64_t q = 0; q < n * sumJ; ++q) grow[q] = hg[q];
  if (gcore)
    for (uint64_t q = 0; q < hc.size(); ++q) gcore[q] = hc[q];
  return CMTF_OK;
}

// The product epoch kernel's own per-entry arithmetic at the frozen device
// model: one hog3tm sweep with eta = 0 (every step and push is zero, so the
// model does not change) that records each tensor entry's x_hat, residual and
// row gradients (compute_gradient_opt, src/gradients.cpp:130-223) and the
// summed data term sum_e -r_e u1 (x) u2 (x) u3 of the core gradient, as the
// kernel computed them inside its tensor-core tiles.
int cmtf_gpu_kernel_probe(cmtf_gpu_ctx* ctx, double* xhat, double* residual, double* grow,
                          double* gcore_data) {
  TRY(require_bundle(ctx));
  CU(cudaSetDevice(ctx->device));
  int J = 0;
  if (ctx->cfg.exec_mode == CMTF_EXEC_SERIAL || ctx->order != 3 || !v2_supported(ctx, &J) ||
      !v3_tm(ctx))
    return set_err(ctx, CMTF_EUNSUPPORTED,
                   "kernel probe: the epoch does not run the order-3 tcgen05 kernel");
  const uint64_t nnz = ctx->nnz, rec_len = 2 + 3 * (uint64_t)J, csz = ctx->core_size();
  float *d_p = nullptr, *d_c = nullptr;
  TRY(dalloc(ctx, &d_p, nnz * rec_len));
  TRY(dalloc(ctx, &d_c, csz));
  int rc = CMTF_OK;
  auto run = [&]() -> int {
    CU(cudaMemsetAsync(d_c, 0, csz * sizeof(float), ctx->stream));
    TRY(normalize_pos(ctx));
    ctx->probe = d_p;
    ctx->probe_core = d_c;
    const int r = v2_sweep(ctx, J, 0.f, 0, nnz, nullptr, nullptr);
    ctx->probe = ctx->probe_core = nullptr;
    TRY(r);
    std::vector<float> hp(nnz * rec_len), hc(csz);
    std::vector<uint32_t> pos(nnz);
    CU(cudaMemcpyAsync(hp.data(), d_p, hp.size() * sizeof(float), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaMemcpyAsync(hc.data(), d_c, hc.size() * sizeof(float), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaMemcpyAsync(pos.data(), ctx->pos, nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (uint64_t k = 0; k < nnz; ++k) {
      const float* q = hp.data() + (uint64_t)pos[k] * rec_len;
      if (xhat) xhat[k] = q[0];
      if (residual) residual[k] = q[1];
      if (grow)
        for (uint64_t t = 0; t < 3 * (uint64_t)J; ++t) grow[k * 3 * J + t] = q[2 + t];
    }
    if (gcore_data)
      for (uint64_t t = 0; t < csz; ++t) gcore_data[t] = hc[t];
    return CMTF_OK;
  };
  rc = run();
  cudaFree(d_p);
  cudaFree(d_c);
  return rc;
}

int cmtf_gpu_compute_gradient(int32_t kernel, int32_t order, const uint32_t* ranks,
                              int32_t core_structure, const double* core, uint64_t n,
                              const double* x, const double* rows, const uint32_t* counts,
                              double lambda_reg, uint64_t nnz_total, int32_t with_core,
                              double* grow, double* gcore, double* residual,
                              double* intermediate, int32_t device) {
  if (order < 1 || order > kMaxOrder)
    return set_err(nullptr, CMTF_EVALIDATION, "kernel argument order mismatch");
  CoreShape cs{};
  cs.order = order;
  uint32_t off = 0;
  uint64_t size = 1;
  for (int q = 0; q < order; ++q) {
    if (ranks[q] == 0 || ranks[q] > (uint32_t)kMaxRank)
      return set_err(nullptr, CMTF_EVALIDATION, "bad rank");
    cs.J[q] = ranks[q];
    cs.off[q] = off;
    off += ranks[q];
    size *= ranks[q];
  }
  if (size > (uint64_t)kMaxCore)
    return set_err(nullptr, CMTF_EUNSUPPORTED, "core too large for the device kernels");
  cs.off[order] = off;
  cs.size = (uint32_t)size;
  const bool cp = core_structure == 1;
  if (cp)
    for (int q = 1; q < order; ++q)
      if (ranks[q] != ranks[0])
        return set_err(nullptr, CMTF_EVALIDATION, "CP mode requires equal ranks on every mode");
  cs.cp = cp;
  cs.dstep = 0;
  for (int q = order - 1, st = 1; q >= 0; --q) {
    cs.dstep += (uint32_t)st;
    st *= (int)ranks[q];
  }
  // a CP core is passed as its stored superdiagonal (ranks[0] values) and
  // returns its gradient and intermediate tensor the same way
  // (src/gradients.cpp:108-115,145-152)
  const uint64_t stored = cp ? ranks[0] : size;
  for (uint64_t e = 0; e < n * order; ++e)
    if (counts[e] == 0)
      return set_err(nullptr, CMTF_EVALIDATION, "mode counts must be >= 1");
  if (n == 0) return CMTF_OK;
  cmtf_gpu_ctx* ctx = nullptr;
  CU(cudaSetDevice(device));
  std::vector<double> hcore(size, 0.0);
  for (uint64_t q = 0; q < stored; ++q) hcore[cp ? q * cs.dstep : q] = core[q];
  double *d_core = nullptr, *d_rows = nullptr, *d_x = nullptr, *d_r = nullptr,
         *d_grow = nullptr, *d_gcore = nullptr, *d_inter = nullptr;
  uint32_t* d_counts = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_core);
    cudaFree(d_rows);
    cudaFree(d_x);
    cudaFree(d_r);
    cudaFree(d_grow);
    cudaFree(d_counts);
    if (d_gcore) cudaFree(d_gcore);
    if (d_inter) cudaFree(d_inter);
  };
  auto run = [&]() -> int {
    TRY(dalloc(ctx, &d_core, size));
    TRY(dalloc(ctx, &d_rows, n * off));
    TRY(dalloc(ctx, &d_x, n));
    TRY(dalloc(ctx, &d_r, n));
    TRY(dalloc(ctx, &d_grow, n * off));
    TRY(dalloc(ctx, &d_counts, n * order));
    if (with_core) TRY(dalloc(ctx, &d_gcore, n * size));
    if (intermediate && kernel == CMTF_KERNEL_OPT) TRY(dalloc(ctx, &d_inter, n * size));
    CU(cudaMemcpy(d_core, hcore.data(), size * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_rows, rows, n * off * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_x, x, n * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_counts, counts, n * order * sizeof(uint32_t), cudaMemcpyHostToDevice));
    Probe64Args a{};
    a.cs = cs;
    a.G = d_core;
    a.rows = d_rows;
    a.x = d_x;
    a.counts = d_counts;
    a.lambda = lambda_reg;
    a.n = n;
    a.core_reg = lambda_reg / (double)nnz_total;
    a.with_core = with_core;
    a.resid = d_r;
    a.grow = d_grow;
    a.gcore = d_gcore;
    a.inter = d_inter;
    const int bt = 128;
    const size_t smem = sizeof(double) * (bt / 32) * 3 * off;
    if (kernel == CMTF_KERNEL_OPT)
      probe64_kernel<true><<<grid_for(n, bt / 32), bt, smem>>>(a);
    else
      probe64_kernel<false><<<grid_for(n, bt / 32), bt, smem>>>(a);
    CU(cudaGetLastError());
    std::vector<double> hc(d_gcore ? n * size : 0), hs(d_inter ? n * size : 0);
    if (residual) CU(cudaMemcpy(residual, d_r, n * sizeof(double), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(grow, d_grow, n * off * sizeof(double), cudaMemcpyDeviceToHost));
    if (d_gcore)
      CU(cudaMemcpy(hc.data(), d_gcore, hc.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (d_inter)
      CU(cudaMemcpy(hs.data(), d_inter, hs.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (uint64_t e = 0; e < n; ++e)
      for (uint64_t q = 0; q < stored; ++q) {
        const uint64_t d = e * size + (cp ? q * cs.dstep : q);
        if (with_core && gcore) gcore[e * stored + q] = hc[d];
        if (intermediate && d_inter) intermediate[e * stored + q] = hs[d];
      }
    return CMTF_OK;
  };
  const int rc = run();
  cleanup();
  return rc;
}

int cmtf_gpu_matrix_entry_gradients(uint64_t n, uint32_t j, const double* y,
                                    const double* u, const double* v, double lambda_m,
                                    double lambda_reg, const uint32_t* col_count,
                                    double* du, double* dv, double* residual,
                                    int32_t device) {
  cmtf_gpu_ctx* ctx = nullptr;
  if (n == 0) return CMTF_OK;
  if (j == 0) return set_err(nullptr, CMTF_EVALIDATION, "coupled rows must have equal length");
  CU(cudaSetDevice(device));
  double *d_y = nullptr, *d_u = nullptr, *d_v = nullptr, *d_du = nullptr, *d_dv = nullptr,
         *d_r = nullptr;
  uint32_t* d_c = nullptr;
  auto run = [&]() -> int {
    TRY(dalloc(ctx, &d_y, n));
    TRY(dalloc(ctx, &d_u, n * j));
    TRY(dalloc(ctx, &d_v, n * j));
    TRY(dalloc(ctx, &d_du, n * j));
    TRY(dalloc(ctx, &d_dv, n * j));
    TRY(dalloc(ctx, &d_r, n));
    TRY(dalloc(ctx, &d_c, n));
    CU(cudaMemcpy(d_y, y, n * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_u, u, n * j * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_v, v, n * j * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_c, col_count, n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    matrix_probe64_kernel<<<grid_for(n), 256>>>(n, j, d_y, d_u, d_v, lambda_m, lambda_reg, d_c,
                                                d_du, d_dv, d_r);
    CU(cudaGetLastError());
    CU(cudaMemcpy(du, d_du, n * j * sizeof(double), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(dv, d_dv, n * j * sizeof(double), cudaMemcpyDeviceToHost));
    if (residual) CU(cudaMemcpy(residual, d_r, n * sizeof(double), cudaMemcpyDeviceToHost));
    return CMTF_OK;
  };
  const int rc = run();
  for (auto p : {d_y, d_u, d_v, d_du, d_dv, d_r}) cudaFree(p);
  cudaFree(d_c);
  return rc;
}

int cmtf_gpu_collapse(int32_t order, const uint32_t* ranks, int32_t core_structure,
                      const double* values, int32_t mode, double* out, int32_t device) {
  cmtf_gpu_ctx* ctx = nullptr;
  if (order < 1 || order > kMaxOrder || !ranks)
    return set_err(nullptr, CMTF_EVALIDATION, "invalid core shape");
  if (mode < 0 || mode >= order) return set_err(nullptr, CMTF_EVALIDATION, "collapse mode out of range");
  CoreShape cs{};
  cs.order = order;
  uint64_t size = 1;
  for (int q = 0; q < order; ++q) {
    cs.J[q] = ranks[q];
    size *= ranks[q];
  }
  if (core_structure == 1) {  // CP: element (k,...,k) is the only one with mode index k
    for (uint32_t k = 0; k < ranks[mode]; ++k) out[k] = values[k];
    return CMTF_OK;
  }
  if (size > (uint64_t)kMaxCore) return set_err(nullptr, CMTF_EUNSUPPORTED, "core too large");
  cs.size = (uint32_t)size;
  CU(cudaSetDevice(device));
  double *d_s = nullptr, *d_o = nullptr;
  auto run = [&]() -> int {
    TRY(dalloc(ctx, &d_s, size));
    TRY(dalloc(ctx, &d_o, ranks[mode]));
    CU(cudaMemcpy(d_s, values, size * sizeof(double), cudaMemcpyHostToDevice));
    collapse64_kernel<<<1, 64>>>(cs, d_s, mode, d_o);
    CU(cudaGetLastError());
    CU(cudaMemcpy(out, d_o, ranks[mode] * sizeof(double), cudaMemcpyDeviceToHost));
    return CMTF_OK;
  };
  const int rc = run();
  cudaFree(d_s);
  cudaFree(d_o);
  return rc;
}

int cmtf_gpu_visit_counts(cmtf_gpu_ctx* ctx, uint32_t* tensor_counts, uint32_t* matrix_counts) {
  TRY(require_bundle(ctx));
  if (!ctx->cfg.debug_count_visits)
    return set_err(ctx, CMTF_EVALIDATION, "debug_count_visits is off");
  if (ctx->visits_epoch < 0) return set_err(ctx, CMTF_EVALIDATION, "no epoch has run");
  if (!ctx->visits_ok)
    return set_err(ctx, CMTF_EUNSUPPORTED,
                   "the epoch ran a kernel without visit counting (serial replay or v1)");
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize(ctx->stream));
  if (tensor_counts && ctx->nnz) {
    // record position -> the caller's entry id (pos[], through the per-epoch
    // group map)
    TRY(normalize_pos(ctx));
    std::vector<uint32_t> byp(ctx->nnz), pos(ctx->nnz);
    CU(cudaMemcpy(byp.data(), ctx->visits, ctx->nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(pos.data(), ctx->pos, ctx->nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    for (uint64_t id = 0; id < ctx->nnz; ++id) tensor_counts[id] = byp[pos[id]];
  }
  uint64_t mtot = 0;
  for (auto& M : ctx->mats) mtot += M.nnz;
  if (matrix_counts && mtot)
    CU(cudaMemcpy(matrix_counts, ctx->mvisits, mtot * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return CMTF_OK;
}

int cmtf_gpu_set_schedule(cmtf_gpu_ctx* ctx, const uint64_t* schedule, uint64_t n) {
  TRY(require_bundle(ctx));
  uint64_t total = ctx->nnz;
  for (auto& m : ctx->mats) total += m.nnz;
  if (n != total) return set_err(ctx, CMTF_EVALIDATION, "schedule length mismatch");
  for (uint64_t i = 0; i < n; ++i)
    if (schedule[i] >= total) return set_err(ctx, CMTF_EVALIDATION, "schedule id out of range");
  ctx->schedule.assign(schedule, schedule + n);
  ctx->schedule_given = true;
  return CMTF_OK;
}

int cmtf_gpu_mark(cmtf_gpu_ctx* ctx, int32_t slot) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (slot < 0 || slot >= 8) return set_err(ctx, CMTF_EVALIDATION, "mark slot out of range");
  CU(cudaSetDevice(ctx->device));
  CU(cudaEventRecord(ctx->uev[slot], ctx->stream));
  return CMTF_OK;
}

int cmtf_gpu_elapsed_ms(cmtf_gpu_ctx* ctx, int32_t from, int32_t to, double* ms) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (from < 0 || from >= 8 || to < 0 || to >= 8)
    return set_err(ctx, CMTF_EVALIDATION, "mark slot out of range");
  CU(cudaEventSynchronize(ctx->uev[to]));
  float f = 0.f;
  CU(cudaEventElapsedTime(&f, ctx->uev[from], ctx->uev[to]));
  *ms = f;
  return CMTF_OK;
}

int cmtf_gpu_last_epoch_timing(cmtf_gpu_ctx* ctx, double* kernel_ms, int32_t* launches) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (kernel_ms)
    for (int i = 0; i < 4; ++i) kernel_ms[i] = ctx->last_ms[i];
  if (launches) *launches = ctx->last_launches;
  return CMTF_OK;
}

int cmtf_gpu_kernel_info(cmtf_gpu_ctx* ctx, int32_t* which, int32_t* hog_threads,
                         int32_t* sort_mode) {
  if (!ctx) return set_err(nullptr, CMTF_EVALIDATION, "null context");
  if (which) *which = ctx->kernel_which;
  if (hog_threads) *hog_threads = ctx->hog_threads_used;
  if (sort_mode) *sort_mode = ctx->sort_mode;
  return CMTF_OK;
}

int cmtf_gpu_order_blocks(cmtf_gpu_ctx* ctx, int32_t* blocks, uint32_t* positions) {
  if (!ctx || !blocks) return set_err(ctx, CMTF_EVALIDATION, "null argument");
  *blocks = ctx->vt_on && ctx->blk_B > 1 ? (int32_t)ctx->blk_B : 0;
  if (positions && ctx->nnz) {
    if (!ctx->pos) return set_err(ctx, CMTF_EVALIDATION, "no tensor uploaded");
    drain_side(ctx);
    TRY(normalize_pos(ctx));
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(positions, ctx->pos, ctx->nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  }
  return CMTF_OK;
}

}  // extern "C"

// io.cpp's error hook (the thread's last error, as set_err)
namespace cmtfb {
int io_fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace cmtfb
