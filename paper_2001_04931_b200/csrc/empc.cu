// Host engine and C ABI (include/empc_b200.h) of the B200 EMPC hot path.
//
// One handle = one problem shape (n, m, T, p, N, K) x `instances`, device
// buffers owned by the handle, one CUDA stream, and a cache of captured CUDA
// graphs keyed by the run structure (init / rescore / number of evolves).
// Reference call stack being replaced: K/empc.py:211-236 (solve_empc).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <memory>
#include <string>
#include <tuple>
#include <utility>
#include <thread>
#include <vector>

#include "../../include/empc_b200.h"
#define EMPC_HOST_TU
#include "empc_kernels.cuh"
#include "empc_cond.h"
#include "empc_variants.h"
#include "empc_tc_rollout.cuh"
#include "empc_small.h"

using namespace empc;

namespace empc {

// Byte-range copies by one kernel (16-byte words when a range allows it).
// The public-API graph moves its inputs and outputs with these instead of
// DMA nodes: the staging upload reads the mapped pinned host buffers, the
// result is stored straight into mapped pinned memory, the output slot is a
// device copy.  Each DMA node costs ~5 us of graph latency
// (tools/graph_io_probe.cu: 33.7 -> 17.5 us around an empty kernel).
struct CopySpan {
  const void* src;
  void* dst;
  size_t bytes;
};
struct CopySpans {
  CopySpan s[3];
  int n = 0;
  void add(const void* src, void* dst, size_t bytes) { s[n++] = CopySpan{src, dst, bytes}; }
  size_t largest() const {
    size_t b = 0;
    for (int k = 0; k < n; ++k) b = std::max(b, s[k].bytes);
    return b;
  }
};
__global__ void copy_spans_kernel(const CopySpans c) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  for (int k = 0; k < c.n; ++k) {
    const CopySpan sp = c.s[k];
    const uintptr_t al = (uintptr_t)sp.src | (uintptr_t)sp.dst | (uintptr_t)sp.bytes;
    if ((al & 15) == 0) {
      const uint4* a = static_cast<const uint4*>(sp.src);
      uint4* b = static_cast<uint4*>(sp.dst);
      for (size_t i = tid; i < sp.bytes / 16; i += nt) b[i] = a[i];
    } else if ((al & 7) == 0) {
      const uint2* a = static_cast<const uint2*>(sp.src);
      uint2* b = static_cast<uint2*>(sp.dst);
      for (size_t i = tid; i < sp.bytes / 8; i += nt) b[i] = a[i];
    } else {
      const unsigned char* a = static_cast<const unsigned char*>(sp.src);
      unsigned char* b = static_cast<unsigned char*>(sp.dst);
      for (size_t i = tid; i < sp.bytes; i += nt) b[i] = a[i];
    }
  }
}
// host-memory spans above this size stay DMA copies (C5 stages 110 MB)
constexpr size_t kZeroCopyMax = (size_t)1 << 20;
}  // namespace empc

namespace {

thread_local std::string g_create_error;

constexpr int kMaxSmem = 227 * 1024;

struct CudaError {
  std::string msg;
};

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw CudaError{std::string(#call) + ": " + cudaGetErrorString(e_)};               \
  } while (0)

struct InvalidArg {
  std::string msg;
};

int pad_np(int n) {
  for (int v : {4, 8, 12, 16, 24, 32, 48, 64, 96, 128})
    if (n <= v) return v;
  return -1;
}


struct Launch {
  int tile, tileP, tiles, threads;
  size_t smem;
  int multi = 0;  // tensor-core rollout: one CTA per instance loops over its tiles
};

// ---------------------------------------------------------------------------

class EngineBase {
 public:
  virtual ~EngineBase() = default;
  std::string err;
  virtual void set_schedule(const int32_t*, const int32_t*, const double*) = 0;
  virtual void set_scorer(int) = 0;
  virtual void set_problems(int, int, const double* const*) = 0;
  virtual int pop_alloc() = 0;
  virtual void pop_free(int) = 0;
  virtual void pop_read(int, double*, double*) = 0;
  virtual void pop_write(int, const double*, const double*) = 0;
  virtual void run(const empc_run_args&) = 0;
  virtual void score(const double*, int, const double*, double*) = 0;
  virtual void select(const double*, int32_t*, int32_t*) = 0;
  virtual void expand(int, const double*, double*) = 0;
  virtual void time_device(const empc_run_args&, int, int, float*, float*, int32_t*, int32_t*) = 0;
  virtual std::string describe() = 0;
  virtual int num_variants() = 0;
  virtual void set_variant(int) = 0;
  virtual void set_occupancy(int) = 0;
  virtual void set_tensor_cores(int) = 0;
  virtual void set_option(int, int) = 0;
  virtual void shard_setup(long long, int, long long, int, int) = 0;
  virtual size_t shard_entry_size() = 0;
  virtual void shard_init(const empc_run_args&) = 0;
  virtual void shard_export(void*) = 0;
  virtual void shard_import(const void*, int, double*, double*, double*, long long*) = 0;
  virtual void shard_evolve(const empc_run_args&) = 0;
  virtual void shard_read(double*, double*) = 0;
  virtual void* stream() = 0;
};

template <typename S>
class Engine final : public EngineBase {
 public:
  explicit Engine(const empc_dims& dd) : dims_(dd) {
    const int n = dd.n, m = dd.m;
    d_.n = n; d_.m = m; d_.T = dd.T; d_.p = dd.p; d_.pm = dd.p * dd.m; d_.N = dd.num_sims; d_.K = dd.num_parents;
    d_.NP = pad_np(n);
    I_ = dd.instances;
    dense_ = dd.dense_q != 0;
    CK(cudaSetDevice(dd.device));
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dd.device));
    variants_ = variants_for<S>(d_.NP);
    use_pdl_ = std::getenv("EMPC_NO_PDL") == nullptr;
    if (const char* v = std::getenv("EMPC_VARIANT")) forced_ = std::atoi(v);
    phases_ = std::getenv("EMPC_PHASES") != nullptr;
    incremental_ = std::getenv("EMPC_FULL_SELECT") == nullptr;
    persist_mode_ = std::getenv("EMPC_NO_PERSIST") == nullptr ? -1 : 0;
    persist_ = persist_variants<S>();
    if (phases_) {
      dbg_n_ = (size_t)1 << 20;
      CK(cudaMalloc(&dbg_, dbg_n_ * 8));
    }
    int s = 0;
    SL_.ad = s; s += n * n;
    SL_.bd = s; s += n * m;
    SL_.wd = s; s += n;
    SL_.q = s; s += n * n;
    SL_.r = s; s += m * m;
    SL_.xg = s; s += n;
    SL_.ug = s; s += m;
    SL_.umin = s; s += m;
    SL_.umax = s; s += m;
    SL_.stride = s + (s & 1);  // even: every instance's block starts 16-byte aligned (async staging copies)
    if (SL_.stride != stage_stride(n, m)) throw std::logic_error("staging layout and stage_stride disagree");
    SL_.x0 = 0;
    SL_.sig = n;
    SL_.sstride = n + m;

    const size_t popn = (size_t)I_ * d_.N * d_.pm, costn = (size_t)I_ * d_.N;
    CK(cudaMalloc(&stage_prob_d_, sizeof(double) * (size_t)I_ * SL_.stride));
    CK(cudaMalloc(&stage_state_d_, sizeof(double) * (size_t)I_ * SL_.sstride + sizeof(RunParams) + 64));
    run_d_ = reinterpret_cast<RunParams*>(
        (reinterpret_cast<uintptr_t>(stage_state_d_ + (size_t)I_ * SL_.sstride) + 15) & ~(uintptr_t)15);
    CK(cudaMallocHost(&stage_prob_h_, sizeof(double) * (size_t)I_ * SL_.stride));
    CK(cudaMallocHost(&stage_state_h_, sizeof(double) * (size_t)I_ * SL_.sstride + sizeof(RunParams) + 64));
    run_h_ = reinterpret_cast<RunParams*>(
        (reinterpret_cast<uintptr_t>(stage_state_h_ + (size_t)I_ * SL_.sstride) + 15) & ~(uintptr_t)15);
    std::memset(stage_prob_h_, 0, sizeof(double) * (size_t)I_ * SL_.stride);
    for (int b = 0; b < 2; ++b) {
      CK(cudaMalloc(&pop_[b], sizeof(S) * popn));
      CK(cudaMalloc(&cost_[b], sizeof(S) * costn));
    }
    CK(cudaMalloc(&elite_, sizeof(int) * (size_t)I_ * d_.K));
    qcap_ = std::max(1, d_.N - d_.K);  // every child may qualify: the list never overflows
    // qualifier lists: two buffers for the per-generation launches, three
    // for the one-barrier persistent solve
    CK(cudaMalloc(&qcount_, sizeof(int) * 3 * (size_t)I_));
    CK(cudaMemset(qcount_, 0, sizeof(int) * 3 * (size_t)I_));
    CK(cudaMalloc(&qlist_, sizeof(typename OrdOf<S>::T) * 2 * 3 * (size_t)I_ * qcap_));
    out_stride_ = d_.m + d_.pm + 2;
    CK(cudaMalloc(&out_d_, sizeof(double) * (size_t)I_ * out_stride_));
    CK(cudaMallocHost(&out_h_, sizeof(double) * (size_t)I_ * out_stride_));
    // device views of the pinned staging / result buffers (zero-copy IO of the public-API graph)
    CK(cudaHostGetDevicePointer((void**)&stage_prob_hd_, stage_prob_h_, 0));
    CK(cudaHostGetDevicePointer((void**)&stage_state_hd_, stage_state_h_, 0));
    CK(cudaHostGetDevicePointer((void**)&out_hd_, out_h_, 0));
    run_hd_ = reinterpret_cast<RunParams*>(reinterpret_cast<char*>(stage_state_hd_) +
                                           (reinterpret_cast<char*>(run_h_) - reinterpret_cast<char*>(stage_state_h_)));
    CK(cudaMalloc(&idx1_, sizeof(int) * d_.T));
    CK(cudaMalloc(&idx2_, sizeof(int) * d_.T));
    CK(cudaMalloc(&seg_, sizeof(int) * d_.T));
    CK(cudaMalloc(&amin_d_, sizeof(unsigned long long)));
    if (const char* v = std::getenv("EMPC_STAGGER")) stagger_ = std::atoi(v);
    if (const char* v = std::getenv("EMPC_WS_THREADS")) ws_threads_ = std::atoi(v);
    if (const char* v = std::getenv("EMPC_PERSIST")) persist_mode_ = std::atoi(v);
    if (const char* v = std::getenv("EMPC_PERSIST_TILE")) persist_tile_ = std::atoi(v);
    if (const char* v = std::getenv("EMPC_SMALL")) small_mode_ = std::atoi(v);
    if (const char* v = std::getenv("EMPC_SMALL_THREADS")) small_threads_ = std::atoi(v);
    CK(cudaMalloc(&cw_, sizeof(S) * d_.T));
    CK(cudaMalloc(&G_, sizeof(S) * d_.p * d_.p));
    CK(cudaMalloc(&W64_, sizeof(double) * d_.T * d_.p));
    CK(cudaMalloc(&G64_, sizeof(double) * d_.p * d_.p));
    ck_ = cond_kernels<S>();
    select_smem_ = select_smem<S>(d_.N);
    if (select_smem_ > (size_t)kMaxSmem - 1024) throw InvalidArg{"num_sims too large for the selection kernel"};
    // function attributes are process-wide: always the maximum, never a per-engine size
    CK(cudaFuncSetAttribute(select_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024));
    // large single populations (C4): radix select of the K-th key + ranking
    // of the K elites only (O(M) + O(K^2) instead of O(M^2) per selection)
    {
      const char* e = std::getenv("EMPC_RADIX_SELECT");
      const int min_n = e ? std::atoi(e) : 8192;
      radix_min_n_ = min_n > 0 ? min_n : (1 << 30);
      use_radix_ = sizeof(S) == 4 && I_ == 1 && d_.N >= radix_min_n_ &&
                   radix_select_smem(d_.N, d_.K) <= (size_t)kMaxSmem - 1024;
      radix_persist_ok_ = min_n > 0;
      CK(cudaFuncSetAttribute(select_radix_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024));
    }
    for (auto& v : variants_) CK(cudaFuncSetAttribute(v.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CK(cudaFuncSetAttribute(ck_.score_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CK(cudaFuncSetAttribute(ck_.score_glob, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CK(cudaFuncSetAttribute(ck_.prep, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
  }

  ~Engine() override {
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
    for (auto& s : slots_)
      if (s.used) { cudaFree(s.cands); cudaFree(s.costs); }
    cudaFree(stage_prob_d_); cudaFree(stage_state_d_);
    cudaFreeHost(stage_prob_h_); cudaFreeHost(stage_state_h_);
    for (int b = 0; b < 2; ++b) { cudaFree(pop_[b]); cudaFree(cost_[b]); }
    cudaFree(elite_); cudaFree(qcount_); cudaFree(qlist_); cudaFree(out_d_); cudaFreeHost(out_h_);
    cudaFree(idx1_); cudaFree(idx2_); cudaFree(seg_); cudaFree(cw_); cudaFree(G_); cudaFree(amin_d_);
    cudaFree(W64_); cudaFree(G64_);
    if (cond_) cudaFree(cond_);
    if (cws_) cudaFree(cws_);
    if (scratch_pop_) cudaFree(scratch_pop_);
    if (scratch_cost_) cudaFree(scratch_cost_);
    if (scratch_dbl_) cudaFree(scratch_dbl_);
    if (flush_) cudaFree(flush_);
    if (dbg_) cudaFree(dbg_);
    for (auto* e : ev_) cudaEventDestroy(e);
    cudaStreamDestroy(stream_);
  }

  // -- schedule --------------------------------------------------------------
  void set_schedule(const int32_t* i1, const int32_t* i2, const double* c) override {
    const int T = d_.T, p = d_.p;
    std::vector<S> cs(T);
    std::vector<double> Wd((size_t)T * p, 0.0);
    for (int k = 0; k < T; ++k) {
      if (i1[k] < 0 || i1[k] >= p || i2[k] < 0 || i2[k] >= p || !(c[k] >= 0.0 && c[k] < 1.0))
        throw InvalidArg{"invalid knot schedule entry at step " + std::to_string(k)};
      cs[k] = (S)c[k];
      Wd[(size_t)k * p + i1[k]] += 1.0 - c[k];
      if (c[k] > 0.0) Wd[(size_t)k * p + i2[k]] += c[k];
    }
    std::vector<S> G((size_t)p * p);
    std::vector<double> G64((size_t)p * p);
    for (int a = 0; a < p; ++a)
      for (int b = 0; b < p; ++b) {
        double s = 0.0;
        for (int k = 0; k < T; ++k) s += Wd[(size_t)k * p + a] * Wd[(size_t)k * p + b];
        G[(size_t)a * p + b] = (S)s;
        G64[(size_t)a * p + b] = s;
      }
    CK(cudaMemcpy(W64_, Wd.data(), sizeof(double) * T * p, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(G64_, G64.data(), sizeof(double) * p * p, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx1_, i1, sizeof(int) * T, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx2_, i2, sizeof(int) * T, cudaMemcpyHostToDevice));
    // runs of steps with the same knot pair: seg[k] = first step after k's run
    std::vector<int> seg(T);
    for (int k = T - 1; k >= 0; --k)
      seg[k] = (k + 1 < T && i1[k + 1] == i1[k] && i2[k + 1] == i2[k]) ? seg[k + 1] : k + 1;
    CK(cudaMemcpy(seg_, seg.data(), sizeof(int) * T, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(cw_, cs.data(), sizeof(S) * T, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(G_, G.data(), sizeof(S) * p * p, cudaMemcpyHostToDevice));
    have_sched_ = true;
  }

  // -- scorer: 0 = rollout (K/empc.py:85-119), 1 = condensed quadratic (K/empc.py:122-152)
  void set_scorer(int sc) override {
    if (sc != 0 && sc != 1) throw InvalidArg{"scorer must be 0 (rollout) or 1 (condensed)"};
    scorer_ = sc;
  }

  // Device build of the condensed model for every instance (empc_cond.h):
  // sensitivities + u_goal trajectory, split-K Gram of [P | g], reduction.
  // Instances are processed in chunks that keep the workspace <= 256 MiB.
  void launch_cond_build() {
    const int n = d_.n, m = d_.m, T = d_.T, p = d_.p, pm = d_.pm;
    ensure_cond_ws();
    const int ksp = n >= 16 ? 4 : (n >= 4 ? 2 : 1);
    const int cbmax = std::max(1, std::min(pm, 1024 / (n * ksp)));
    int cb = std::max(1, std::min(cbmax, (pm * I_ + sms_ - 1) / sms_));
    const int chunks = (pm + cb - 1) / cb;
    cb = (pm + chunks - 1) / chunks;
    const int threads = std::max(64, std::min(1024, (n * cb * ksp + 31) / 32 * 32));
    const size_t psm = cond_prep_smem(n, cb, dense_ ? 1 : 0);
    if (psm > (size_t)kMaxSmem) throw InvalidArg{"condensed scorer: state dimension too large for the build kernel"};
    const int K = T * n;
    const int ntc = (pm + 1 + kCondTile - 1) / kCondTile;
    const int tiles = ntc * (ntc + 1) / 2;
    const size_t fixed = (size_t)K * pm * (dense_ ? 2 : 1) + K + 1;
    // split-K depends on the shape only: P has the same bits for batched,
    // sharded and single runs
    const int splits = std::max(1, (K + 255) / 256);
    const size_t per = fixed + (size_t)splits * pm * (pm + 1);
    const int ic = (int)std::max<size_t>(1, std::min<size_t>(I_, ((size_t)256 << 20) / sizeof(double) / per));
    if (per * ic > cws_n_) throw CudaError{"condensed workspace not allocated"};
    CondBuild b{};
    b.n = n; b.m = m; b.T = T; b.p = p; b.pm = pm;
    b.SL = SL_; b.prob = stage_prob_d_; b.state = stage_state_d_;
    b.W = W64_; b.G = G64_;
    b.S = cws_;
    b.QS = dense_ ? cws_ + (size_t)ic * K * pm : nullptr;
    b.E = cws_ + (size_t)ic * K * pm * (dense_ ? 2 : 1);
    b.part = b.E + (size_t)ic * (K + 1);
    b.cond = cond_;
    b.cb = cb; b.ksp = ksp; b.splits = splits; b.dense = dense_ ? 1 : 0;
    for (int i0 = 0; i0 < I_; i0 += ic) {
      const int cnt = std::min(ic, I_ - i0);
      b.inst0 = i0;
      launch_ex(ck_.prep, dim3(chunks + 1, cnt), dim3(threads), psm, false, b);
      launch_ex(ck_.gram, dim3(tiles, splits, cnt), dim3(256), 0, false, b);
      launch_ex(ck_.finish, dim3((pm * pm + pm + 1 + 255) / 256, cnt), dim3(256), 0, false, b);
      launches_ += 3;
    }
    pdl_next_ = use_pdl_;
  }

  // workspace of launch_cond_build (allocated outside graph capture)
  void ensure_cond_ws() {
    const int n = d_.n, T = d_.T, pm = d_.pm;
    if (!cond_) CK(cudaMalloc(&cond_, sizeof(double) * (size_t)I_ * cond_layout(pm).stride));
    const int K = T * n;
    const int splits = std::max(1, (K + 255) / 256);
    const size_t per = (size_t)K * pm * (dense_ ? 2 : 1) + K + 1 + (size_t)splits * pm * (pm + 1);
    const int ic = (int)std::max<size_t>(1, std::min<size_t>(I_, ((size_t)256 << 20) / sizeof(double) / per));
    if (per * ic > cws_n_) {
      if (cws_) cudaFree(cws_);
      CK(cudaMalloc(&cws_, sizeof(double) * per * ic));
      cws_n_ = per * ic;
    }
  }

  struct CondPlan {
    int tile, tileP, tiles, threads, tPS;
    size_t smem;
    bool psm;
  };
  CondPlan plan_cond(int nc) const {
    CondPlan c{};
    int tile = I_ == 1 ? (nc + sms_ - 1) / sms_ : kCondMaxTile;
    tile = std::max(1, std::min({tile, kCondMaxTile, std::max(nc, 1)}));
    c.tiles = std::max(1, (nc + tile - 1) / tile);
    c.tile = std::max(1, (nc + c.tiles - 1) / c.tiles);
    c.tileP = (c.tile + kCondCC - 1) / kCondCC * kCondCC;
    const int ncg = c.tileP / kCondCC;
    const int pmS = (d_.pm + kCondRB - 1) / kCondRB * kCondRB;
    c.threads = std::max(64, std::min(512, (ncg * (pmS / kCondRB) + 31) / 32 * 32));
    CondSmem s = cond_smem<S>(d_.pm, d_.m, c.tileP, c.threads, true);
    c.psm = s.total <= (size_t)kMaxSmem;
    if (!c.psm) s = cond_smem<S>(d_.pm, d_.m, c.tileP, c.threads, false);
    if (s.total > (size_t)kMaxSmem) throw InvalidArg{"condensed scorer: knot vector too long"};
    c.smem = s.total;
    c.tPS = s.tPS;
    return c;
  }

  // -- problems (FP64 host -> pinned staging; uploaded inside the run) --------
  void set_problems(int first, int count, const double* const* arrs) override {
    if (first < 0 || count < 0 || first + count > I_) throw InvalidArg{"instance range out of bounds"};
    const int n = d_.n, m = d_.m;
    const int sizes[9] = {n * n, n * m, n, n * n, m * m, n, m, m, m};
    const int offs[9] = {SL_.ad, SL_.bd, SL_.wd, SL_.q, SL_.r, SL_.xg, SL_.ug, SL_.umin, SL_.umax};
    for (int a = 0; a < 9; ++a)
      if (!arrs[a]) throw InvalidArg{"null problem array"};
    // unchanged problem (a warm control loop re-staging the same model):
    // nothing to copy or re-scan.  Only for small staging blocks, where the
    // comparison is cheaper than the copy plus the structure scans.
    if (have_prob_ && (size_t)count * SL_.stride * sizeof(double) <= ((size_t)1 << 20)) {
      bool same = true;
      for (int a = 0; a < 9 && same; ++a)
        for (int i = 0; i < count && same; ++i)
          same = std::memcmp(stage_prob_h_ + (size_t)(first + i) * SL_.stride + offs[a], arrs[a] + (size_t)i * sizes[a],
                             sizeof(double) * sizes[a]) == 0;
      if (same) return;
    }
    // interleave the caller's stacked arrays into the pinned staging block;
    // large batches (C5: ~110 MB) are copied by several host threads
    auto copy = [&](int i0, int i1) {
      for (int a = 0; a < 9; ++a)
        for (int i = i0; i < i1; ++i)
          std::memcpy(stage_prob_h_ + (size_t)(first + i) * SL_.stride + offs[a], arrs[a] + (size_t)i * sizes[a],
                      sizeof(double) * sizes[a]);
    };
    const size_t bytes = (size_t)count * SL_.stride * sizeof(double);
    const int nth = bytes < ((size_t)8 << 20) ? 1 : (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
    if (nth <= 1) {
      copy(0, count);
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < nth; ++t) pool.emplace_back(copy, (int)((long long)count * t / nth), (int)((long long)count * (t + 1) / nth));
      for (auto& th : pool) th.join();
    }
    bool rd = true;
    for (int i = 0; i < I_ && rd; ++i) {
      const double* R = stage_prob_h_ + (size_t)i * SL_.stride + SL_.r;
      for (int e = 0; e < m * m; ++e)
        if (e / m != e % m && R[e] != 0.0) { rd = false; break; }
    }
    r_diag_ = rd;
    // half-K: Delta = Ad - I has no nonzero entry in its left NP / 2 columns.
    // Only the single-instance persistent solve uses it, so batched handles
    // (C5: ~110 MB of staging) skip the scan.  The skipped block is exactly
    // [0, NP/2): a state with n < NP (e.g. 13-15 DoF arms, NP = 32) has its
    // zero position columns at [0, n/2) and keeps the full matvec.
    bool hk = I_ == 1 && std::getenv("EMPC_NO_HALFK") == nullptr;
    for (int i = 0; i < I_ && hk; ++i) {
      const double* A = stage_prob_h_ + (size_t)i * SL_.stride + SL_.ad;
      for (int r = 0; r < n && hk; ++r)
        for (int c = 0; c < std::min(n, d_.NP / 2); ++c)
          if (A[r * n + c] - (r == c ? 1.0 : 0.0) != 0.0) { hk = false; break; }
    }
    halfk_ = hk;
    have_prob_ = true;
  }

  // -- population slots --------------------------------------------------------
  struct Slot {
    S* cands = nullptr;
    S* costs = nullptr;
    bool used = false;
  };
  int pop_alloc() override {
    int id = -1;
    for (size_t i = 0; i < slots_.size(); ++i)
      if (!slots_[i].used) { id = (int)i; break; }
    if (id < 0) { slots_.push_back(Slot{}); id = (int)slots_.size() - 1; }
    Slot& s = slots_[id];
    CK(cudaMalloc(&s.cands, sizeof(S) * (size_t)I_ * d_.N * d_.pm));
    CK(cudaMalloc(&s.costs, sizeof(S) * (size_t)I_ * d_.N));
    s.used = true;
    return id;
  }
  Slot& slot(int id) {
    if (id < 0 || id >= (int)slots_.size() || !slots_[id].used) throw InvalidArg{"invalid population slot"};
    return slots_[id];
  }
  void pop_free(int id) override {
    Slot& s = slot(id);
    // graphs that read or write this slot hold its old address
    for (auto it = graphs_.begin(); it != graphs_.end();) {
      if (io_code_uses_slot(std::get<7>(it->first), id)) {
        cudaGraphExecDestroy(it->second);
        it = graphs_.erase(it);
      } else {
        ++it;
      }
    }
    CK(cudaFree(s.cands));
    CK(cudaFree(s.costs));
    s = Slot{};
  }
  void pop_read(int id, double* cands, double* costs) override {
    Slot& s = slot(id);
    const size_t nc = (size_t)I_ * d_.N * d_.pm, nk = (size_t)I_ * d_.N;
    ensure_scratch_dbl(std::max(nc, nk));
    if (cands) {
      uncast_kernel<S><<<grid_for(nc), 256, 0, stream_>>>(s.cands, scratch_dbl_, nc);
      CK(cudaMemcpyAsync(cands, scratch_dbl_, sizeof(double) * nc, cudaMemcpyDeviceToHost, stream_));
      CK(cudaStreamSynchronize(stream_));
    }
    if (costs) {
      uncast_kernel<S><<<grid_for(nk), 256, 0, stream_>>>(s.costs, scratch_dbl_, nk);
      CK(cudaMemcpyAsync(costs, scratch_dbl_, sizeof(double) * nk, cudaMemcpyDeviceToHost, stream_));
      CK(cudaStreamSynchronize(stream_));
    }
    CK(cudaGetLastError());
  }
  void pop_write(int id, const double* cands, const double* costs) override {
    Slot& s = slot(id);
    const size_t nc = (size_t)I_ * d_.N * d_.pm, nk = (size_t)I_ * d_.N;
    upload_cast(cands, s.cands, nc);
    if (costs) upload_cast(costs, s.costs, nk);
    else CK(cudaMemsetAsync(s.costs, 0, sizeof(S) * nk, stream_));
    CK(cudaStreamSynchronize(stream_));
  }

  // -- launch planning ---------------------------------------------------------
  static int tps_for(int tileP) {
    constexpr int VEC = Geo<S>::VEC;
    int t = (tileP + VEC - 1) / VEC * VEC;
    if ((t / VEC) % 2 == 0) t += VEC;  // odd number of 16-byte chunks: conflict-free rows
    return t;
  }

  Launch plan(const Variant<S>& v, int nc, int cps_override = 0, int maxt_override = 0, int min_tile = 0) const {
    const int maxt = maxt_override > 0 ? maxt_override : v.maxt;
    if (v.tc) {  // tensor-core rollout: one MMA tile (128 candidates) per CTA
      Launch L{};
      // one instance: spread the candidates over all SMs (rows beyond the
      // tile's count are MMA padding whose epilogue warps idle)
      const int tsz = I_ == 1 ? std::max(1, std::min(kTcTile, (nc + sms_ - 1) / sms_)) : kTcTile;
      L.tile = tsz; L.tileP = kTcTile;
      L.tiles = std::max(1, (nc + tsz - 1) / tsz);
      L.threads = kTcTile * v.RR;
      L.smem = tc_smem(v.tc_nn, v.tc_nk, v.NP, d_.m, d_.T, d_.p, v.RR).total;
      // many instances with several tiles each (C5): one CTA per instance
      // stages the problem once and loops over the instance's tiles
      const size_t msm = tc_smem(v.tc_nn, v.tc_nk, v.NP, d_.m, d_.T, d_.p, v.RR, true).total;
      if (I_ > 1 && L.tiles > 1 && (long long)I_ >= 4LL * sms_ && msm <= (size_t)kMaxSmem && tc_multi_ok_) {
        L.multi = 1;
        L.tiles = 1;
        L.smem = msm;
      }
      if (L.smem > (size_t)kMaxSmem) throw InvalidArg{"problem too large for the rollout kernel (" + std::string(v.name) + ")"};
      return L;
    }
    const int NRG = v.NP / v.RR;
    const int CC = v.CC;
    auto threads_for = [&](int tileP) {
      const int nl = NRG * (tileP / CC);  // logical threads
      return v.ks == 1 ? (nl + 31) / 32 * 32 : 2 * ((nl + 15) / 16 * 16);
    };
    auto fits = [&](int tileP) {
      const SmemPlan sp = smem_plan<S>(v.NP, d_.m, d_.T, d_.p, tileP, tps_for(tileP), v.areg, v.dq);
      return sp.total <= (size_t)kMaxSmem && threads_for(tileP) <= maxt;
    };
    int maxP = CC;
    if (!fits(maxP)) throw InvalidArg{"problem too large for the rollout kernel (" + std::string(v.name) + ")"};
    while (fits(maxP + CC)) maxP += CC;
    Launch L{};
    if (nc <= 0) {
      L.tile = CC; L.tiles = 1;
    } else if (I_ == 1 || cps_ > 0) {
      // one wave of `cps` CTAs per SM: small CTAs synchronise only their own
      // warps each step, so the SM interleaves independent step pipelines
      const int cps = std::max(1, cps_override > 0 ? cps_override : (cps_ > 0 ? cps_ : default_cps(v, nc)));
      int tile = (nc + sms_ * cps - 1) / (sms_ * cps);
      tile = std::max(tile, min_tile);     // fewer, larger CTAs (small persistent solves)
      if (tile > maxP) tile = maxP;        // several waves when smem / threads limit the tile
      int tiles = (nc + tile - 1) / tile;
      tile = (nc + tiles - 1) / tiles;     // balance
      L.tile = tile; L.tiles = tiles;
    } else {
      int want = std::max(CC, (512 / NRG) * CC);
      want = std::min(want, maxP);
      int tiles = (nc + want - 1) / want;
      L.tile = (nc + tiles - 1) / tiles;
      L.tiles = tiles;
    }
    L.tileP = (L.tile + CC - 1) / CC * CC;
    L.threads = threads_for(L.tileP);
    L.smem = smem_plan<S>(v.NP, d_.m, d_.T, d_.p, L.tileP, tps_for(L.tileP), v.areg, v.dq).total;
    return L;
  }

  int default_cps(const Variant<S>& v, int nc) const {
    (void)v; (void)nc;
    // small single problems are latency bound: several small CTAs per SM
    // (independent step pipelines) beat one large one (tools/tune.py, C2)
    return (I_ == 1 && d_.NP <= 16) ? 4 : 1;
  }

  // Default variant from measured preferences on B200 (tools/tune.py,
  // profiles/): A in registers split over lane pairs for single problems with
  // n <= 48, A in registers for batched small problems, smem A for n >= 64.
  const Variant<S>& pick() {
    if (forced_ >= 0) return variants_.at(forced_);
    auto find = [&](int RR, int CC, bool areg, int ks, bool ws = false) -> const Variant<S>* {
      for (auto& v : variants_)
        if (!v.tc && v.RR == RR && v.CC == CC && v.areg == areg && v.ks == ks && v.ws == ws && v.dq == dense_)
          return &v;
      return nullptr;
    };
    if (use_tc()) {
      for (auto& v : variants_)
        if (v.tc && tc_smem(v.tc_nn, v.tc_nk, v.NP, d_.m, d_.T, d_.p, v.RR).total <= (size_t)kMaxSmem) return v;
    }
    if (!dense_ && sizeof(S) == 4) {
      const Variant<S>* pref[4] = {nullptr, nullptr, nullptr, nullptr};
      if (d_.NP <= 8) {
        pref[0] = find(1, 4, true, 1);
      } else if (d_.NP <= 16) {
        pref[0] = I_ == 1 ? find(3, 2, true, 1, true) : nullptr;  // NP = 12 (C2): persistent WS
        pref[1] = find(2, 2, true, 1);
        pref[2] = find(1, 4, true, 1);
      } else if (d_.NP == 48 && I_ == 1) {
        // warp-synchronous candidate groups + helper warps that draw the
        // next generation during the recursion (persistent solve, C3)
        pref[0] = find(3, 4, true, 2, true);
        pref[1] = find(2, 4, true, 2);
      } else if (d_.NP <= 48 && I_ == 1) {
        pref[0] = find(2, 4, true, 2);
        pref[1] = find(1, 4, true, 1);
      } else if (d_.NP <= 48) {
        pref[0] = find(2, 4, true, 1);
        pref[1] = find(1, 4, true, 1);
      } else {
        pref[0] = find(2, 4, false, 1);
        pref[1] = find(4, 4, false, 1);
      }
      for (auto* v : pref)
        if (v) return *v;
    }
    for (auto& v : variants_)
      if (!v.tc && v.dq == dense_ && (dense_ || v.areg)) return v;
    for (auto& v : variants_)
      if (!v.tc && v.dq == dense_) return v;
    return variants_.front();
  }

  // Tensor-core rollout (rollout_tc_kernel): FP32, diagonal Q.  tc_mode_ 1
  // forces it, 0 disables it, -1 (default) uses it where it measured faster
  // than the FFMA recursion on B200 (profiles/)
  bool use_tc() const {
    if (sizeof(S) != 4 || dense_ || tc_mode_ == 0) return false;
    bool have = false;
    for (auto& v : variants_) have = have || v.tc;
    if (!have) return false;
    if (tc_mode_ == 1) return true;
    // measured on B200 (profiles/): the tensor-core rollout wins for large
    // states and for batches that fill the GPU with 128-candidate tiles; the
    // FFMA kernels (persistent for single problems) win for small single problems
    const long long tiles = (long long)I_ * ((d_.N - d_.K + kTcTile - 1) / kTcTile);
    // (one instance: a tile per SM at any size; below ~16 children per SM --
    // e.g. one rank's share of C4 over 8 GPUs -- the FFMA kernel is faster)
    if (I_ == 1) return d_.NP >= 64 && (d_.N - d_.K) >= 16 * sms_;
    return d_.NP >= 24 && tiles >= 2LL * sms_;
  }

  void launch_rollout(int mode, int nc, int row0, int rows, int evolve, const S* pin, const S* cin, S* pout, S* cout,
                      const int* inj_par = nullptr, const uint8_t* inj_take = nullptr, const uint8_t* inj_mut = nullptr,
                      const double* inj_noise = nullptr, const S* inj_init = nullptr) {
    Launch L{};
    void (*kern)(RolloutArgs<S>) = nullptr;
    int tPS = 0;
    if (scorer_ == 1) {
      const CondPlan c = plan_cond(nc);
      L.tile = c.tile; L.tileP = c.tileP; L.tiles = c.tiles; L.threads = c.threads; L.smem = c.smem;
      tPS = c.tPS;
      kern = c.psm ? ck_.score_smem : ck_.score_glob;
    } else {
      const Variant<S>& v = pick();
      L = plan(v, nc);
      tPS = tps_for(L.tileP);
      kern = v.kernel;
    }
    RolloutArgs<S> a{};
    a.d = d_; a.SL = SL_; a.mode = mode; a.r_diag = r_diag_ ? 1 : 0;
    a.nc = nc; a.row0 = row0; a.rows = rows;
    a.tile = L.tile; a.tileP = L.tileP; a.tPS = tPS; a.evolve = evolve;
    a.cand_base = cand_base_;
    a.copy_elites = elites_copied_ ? 0 : 1;
    a.cond = cond_;
    a.cstride = cond_layout(d_.pm).stride;
    a.tc_multi = L.multi;
    elites_copied_ = false;
    a.prob = stage_prob_d_; a.state = stage_state_d_;
    a.idx1 = idx1_; a.idx2 = idx2_; a.seg = seg_; a.cw = cw_; a.G = G_;
    a.stagger = stagger_;
    a.pop_in = pin; a.cost_in = cin; a.pop_out = pout; a.cost_out = cout;
    a.elite_idx = elite_; a.run = run_d_;
    a.inj_parents = inj_par; a.inj_take = inj_take; a.inj_mut = inj_mut; a.inj_noise = inj_noise; a.inj_init = inj_init;
    a.dbg = nullptr;
    a.qcount = (mode == kBreedPhilox || mode == kBreedInject) && incremental_ ? qcount_ + (size_t)(evolve & 1) * I_
                                                                              : nullptr;
    a.qlist = (char*)qlist_ + (size_t)(evolve & 1) * I_ * qcap_ * 2 * sizeof(typename OrdOf<S>::T);
    a.qcap = qcap_;
    if (phases_ && (size_t)L.tiles * I_ * 16 <= dbg_n_) {
      a.dbg = dbg_;
      dbg_ctas_ = (int)(L.tiles * I_);
    }
    launch_ex(kern, dim3(L.tiles, I_), dim3(L.threads), L.smem, pdl_next_, a);
    pdl_next_ = use_pdl_;
    ++launches_;
    ++rollout_launches_;
  }

  // cudaLaunchKernelEx with programmatic stream serialization: the kernel may
  // start while its predecessor drains and waits in-kernel (griddepcontrol)
  template <typename... KArgs, typename... Args>
  void launch_ex(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, bool pdl, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream_;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
    if (e != cudaSuccess) {
      char msg[256];
      std::snprintf(msg, sizeof msg, "cudaLaunchKernelEx(grid=%u,%u block=%u smem=%zu pdl=%d): %s", grid.x, grid.y,
                    block.x, smem, (int)pdl, cudaGetErrorString(e));
      throw CudaError{msg};
    }
  }

  // evolve index g selects the qualifier-list buffer: rollout g appends to
  // buffer g & 1, selection g + 1 ranks it and clears buffer (g + 1) & 1
  void launch_select(const S* costs, int incremental = 0, int g = 0, const S* pop_in = nullptr, S* pop_out = nullptr,
                     S* cost_out = nullptr) {
    const int N = d_.N;
    const int ctas = I_ == 1 ? std::max(1, std::min(sms_, (N + 15) / 16)) : 1;
    int* qin = incremental ? qcount_ + (size_t)((g - 1) & 1) * I_ : nullptr;
    const void* lin = (const char*)qlist_ + (size_t)((g - 1) & 1) * I_ * qcap_ * 2 * sizeof(typename OrdOf<S>::T);
    int* qnext = qcount_ + (size_t)(g & 1) * I_;
    // radix: every CTA redoes the O(M) threshold search, so only as many CTAs
    // as the K elite rows need for ranking and copying (16 per CTA)
    const int rctas = I_ == 1 ? std::max(1, std::min(radix_ctas_ > 0 ? radix_ctas_ : sms_, (d_.K + 15) / 16)) : 1;
    if (use_radix_)
      launch_ex(select_radix_kernel<S>, dim3(rctas, I_), dim3(1024), radix_select_smem(N, d_.K), pdl_next_, costs, N,
                d_.K, elite_, incremental, qin, lin, qnext, qcap_, pop_in, pop_out, cost_out, d_.pm);
    else
      launch_ex(select_kernel<S>, dim3(ctas, I_), dim3(256), select_smem_, pdl_next_, costs, N, d_.K, elite_,
                incremental, qin, lin, qnext, qcap_, pop_in, pop_out, cost_out, d_.pm);
    pdl_next_ = use_pdl_;
    ++launches_;
  }

  // the persistent solve selects by radix select for FP32 unless disabled
  // (EMPC_OPT_RADIX_SELECT = 0 forces rank-by-counting everywhere)
  bool persist_radix() const { return sizeof(S) == 4 && (use_radix_ || (radix_persist_ok_ && d_.N >= 2048)); }
  size_t persist_select_smem() const {
    return persist_radix() ? std::max(select_smem_, radix_select_smem(d_.N, d_.K)) : select_smem_;
  }

  // Persistent cooperative path (single instance, default variant, every
  // tile co-resident): the whole run is one launch.  Returns false when the
  // configuration does not qualify and the per-generation launches are used.
  template <typename Pre, typename Post>
  bool try_persistent(const empc_run_args& r, bool timed, Pre& pre, Post& post,
                      const std::vector<const void*>* inj = nullptr) {
    // small problems (n <= 16: C1, C2) run faster as per-generation launches
    // with several small CTAs per SM (profiles/bench_c1/c2): persistent only
    // from NP = 24 unless forced (EMPC_OPT_PERSISTENT = 1)
    if (persist_mode_ == 0 || scorer_ != 0 || I_ != 1 || cps_ > 0 || (!r.init && !r.rescore) || d_.N == d_.K)
      return false;
    // small states run persistent only with the warp-synchronous variants
    // (C2: 0.176 vs 0.217 ms per-generation launches)
    if (d_.NP < 24 && forced_ < 0 && persist_mode_ < 1 && !pick().ws) return false;
    const Variant<S>& v = pick();
    if (v.tc) return false;
    const PersistVariant<S>* pv = nullptr;
    const bool hk = halfk_ && halfk_ok_;
    for (auto& p : persist_)
      if (p.NP == v.NP && p.RR == v.RR && p.CC == v.CC && p.areg == v.areg && p.ks == v.ks && !v.dq && p.ws == v.ws &&
          p.hk == hk)
        pv = &p;
    if (!pv && hk)  // no half-K instantiation of this variant: the full matvec
      for (auto& p : persist_)
        if (p.NP == v.NP && p.RR == v.RR && p.CC == v.CC && p.areg == v.areg && p.ks == v.ks && !v.dq && p.ws == v.ws &&
            !p.hk)
          pv = &p;
    if (!pv) return false;
    const int nc = d_.N - d_.K;
    const Launch Le = plan(v, nc, 1, pv->maxt, persist_tile_);
    if (Le.tiles > sms_) return false;
    const int grid = Le.tiles;
    const int tile0 = (d_.N + grid - 1) / grid;
    const int tileP = (std::max(tile0, Le.tile) + v.CC - 1) / v.CC * v.CC;
    const int NRG = v.NP / v.RR;
    const int nl = NRG * (tileP / v.CC);
    int threads = v.ks == 1 ? (nl + 31) / 32 * 32 : 2 * ((nl + 15) / 16 * 16);
    // warp-synchronous CTAs carry helper warps for the breeding / staging
    // phases (they skip the recursion)
    if (v.ws) threads = std::max(threads, std::min(pv->maxt, ws_threads_) / 32 * 32);
    if (threads > pv->maxt) return false;
    const size_t smem_plan_total =
        smem_plan<S>(v.NP, d_.m, d_.T, d_.p, tileP, tps_for(tileP), v.areg, v.dq, persist_select_smem()).total;
    // one-barrier generations keep a K-entry rank -> row table after the plan
    const bool one_sync = persist_radix() && one_sync_ok_;
    const size_t elite_off = (smem_plan_total + 15) / 16 * 16;
    const size_t smem = one_sync ? elite_off + sizeof(int) * (size_t)d_.K : smem_plan_total;
    if (smem > (size_t)kMaxSmem - 1024) return false;
    if (!persist_attr_set_) {
      for (auto& p : persist_)
        CK(cudaFuncSetAttribute(p.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024));
      persist_attr_set_ = true;
    }
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pv->kernel, threads, smem));
    if (per_sm * sms_ < grid) return false;
    PersistArgs<S> P{};
    RolloutArgs<S>& a = P.ro;
    a.d = d_; a.SL = SL_; a.r_diag = r_diag_ ? 1 : 0;
    const S* inj_init = (inj && r.init) ? (const S*)(*inj)[0] : nullptr;
    a.mode = r.init ? (inj_init ? kInitInject : kInitPhilox) : kScore;
    a.inj_init = inj_init;
    a.nc = d_.N; a.row0 = 0; a.rows = d_.N;
    a.tile = tile0; a.tileP = tileP; a.tPS = tps_for(tileP); a.evolve = 0; a.cand_base = 0; a.copy_elites = 0;
    a.prob = stage_prob_d_; a.state = stage_state_d_;
    a.idx1 = idx1_; a.idx2 = idx2_; a.seg = seg_; a.cw = cw_; a.G = G_;
    a.stagger = stagger_;
    // (a warm graph re-scores straight from the input slot; kScore then also
    // writes the candidates into pop_out)
    a.pop_in = warm_src_ ? warm_src_->cands : pop_[0];
    a.cost_in = nullptr; a.pop_out = pop_[0]; a.cost_out = cost_[0];
    a.elite_idx = elite_; a.run = run_d_;
    a.qcount = nullptr; a.qlist = qlist_; a.qcap = qcap_; a.dbg = nullptr;
    if (phases_ && (size_t)grid * 16 + 32 <= dbg_n_) {
      CK(cudaMemsetAsync(dbg_, 0, ((size_t)grid * 16 + 48) * 8, stream_));
      a.dbg = dbg_;
      dbg_ctas_ = grid;
    }
    P.evolves = r.evolves;
    P.tile_evolve = Le.tile;
    P.incremental = incremental_ ? 1 : 0;
    P.scratch = persist_select_smem();
    P.radix = persist_radix() ? 1 : 0;
    P.one_sync = one_sync ? 1 : 0;
    P.elite_off = elite_off;
    P.dbg_gen = -1;
    P.amin = sizeof(S) == 4 ? amin_d_ : nullptr;
    if (const char* e = std::getenv("EMPC_PHASES_GEN")) P.dbg_gen = std::atoi(e);
    P.pop[0] = pop_[0]; P.pop[1] = pop_[1];
    P.cost[0] = cost_[0]; P.cost[1] = cost_[1];
    P.qcount = qcount_;
    P.qlist = qlist_;
    P.elite = elite_;
    P.out = out_d_;
    if (io_out_direct_) {
      // public-API graph: CTA 0 stores the result into mapped pinned memory,
      // and the output slot stands in for the ping-pong buffer that ends up
      // holding the final population (index evolves & 1) -- unless a warm
      // start still has to read its input from that buffer (a warm graph
      // reads it from the input slot instead)
      P.out = out_hd_;
      io_result_done_ = true;
      const int fin = r.evolves & 1;
      if (slot_captured(r) && (r.init || fin == 1 || warm_src_ != nullptr)) {
        Slot& so = slot(r.slot_out);
        P.pop[fin] = so.cands;
        P.cost[fin] = so.costs;
        if (fin == 0) { a.pop_out = so.cands; a.cost_out = so.costs; }
        io_slot_done_ = true;
      }
    }
    {  // helper warps (WS variants) draw the next generation during the recursion
      const int hstart = ((v.ks == 1 ? 1 : 2) * NRG * (tileP / v.CC) + 31) / 32 * 32;
      P.predraw = (v.ws && threads > hstart && !inj && predraw_ok_) ? 1 : 0;
    }
    if (inj && r.evolves > 0 && nc > 0) {  // the reference's draws (parity mode)
      P.inj_parents = (const int*)(*inj)[1];
      P.inj_take = (const uint8_t*)(*inj)[2];
      P.inj_mut = (const uint8_t*)(*inj)[3];
      P.inj_noise = (const double*)(*inj)[4];
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream_;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (timed) pre();
    CK(cudaLaunchKernelEx(&cfg, pv->kernel, P));
    ++launches_;
    ++rollout_launches_;
    if (timed) post();
    persist_desc_ = std::string("persistent grid=") + std::to_string(grid) + " threads=" + std::to_string(threads) +
                    " smem=" + std::to_string(smem) + (pv->hk ? " halfK" : "") + (P.predraw ? " predraw" : "") +
                    (P.one_sync ? " onesync" : "");
    return true;
  }

  // Small problems (C1): the whole solve in one CTA per instance with the
  // population resident in shared memory (empc_small.cu).  Auto: n <= 8, a
  // diagonal Q, the rollout scorer and little work per generation.
  bool small_eligible() const {
    if (small_mode_ == 0 || scorer_ != 0 || dense_ || cps_ > 0 || (forced_ >= 0 && small_mode_ < 1)) return false;
    if (small_kernel<S>(d_.n) == nullptr || d_.N > 4096) return false;
    if (small_smem<S>(d_.n, d_.m, d_.T, d_.p, d_.N, d_.K) > (size_t)kMaxSmem) return false;
    const int npv = d_.n <= 4 ? 4 : 8;
    const long long work = (long long)d_.N * d_.T * npv * npv;
    return !(small_mode_ < 0 && work > (1LL << 18));
  }

  template <typename Pre, typename Post>
  bool try_small(const empc_run_args& r, bool timed, Pre& pre, Post& post, const std::vector<const void*>* inj) {
    if (!small_eligible()) return false;
    const SmallKernel<S> kern = small_kernel<S>(d_.n);
    const size_t smem = small_smem<S>(d_.n, d_.m, d_.T, d_.p, d_.N, d_.K);
    if (!small_attr_set_) {
      CK(cudaFuncSetAttribute(small_kernel<S>(4), cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
      CK(cudaFuncSetAttribute(small_kernel<S>(8), cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
      small_attr_set_ = true;
    }
    SmallArgs<S> A{};
    A.d = d_; A.SL = SL_; A.evolves = r.evolves; A.r_diag = r_diag_ ? 1 : 0;
    A.prob = stage_prob_d_; A.state = stage_state_d_; A.run = run_d_;
    A.idx1 = idx1_; A.idx2 = idx2_; A.seg = seg_; A.cw = cw_; A.G = G_;
    A.pop_in = warm_src_ ? warm_src_->cands : pop_[0];
    A.cost_in = warm_src_ ? warm_src_->costs : cost_[0];
    A.pop_io = pop_[0]; A.cost_io = cost_[0]; A.out = out_d_;
    if (io_direct_) {
      // public-API graph: staging read from the mapped pinned buffers, the
      // result stored into mapped pinned memory, the population written
      // straight into the output slot (captured slots; others are copied
      // from pop_[0] after the graph)
      A.prob = stage_prob_hd_; A.state = stage_state_hd_; A.run = run_hd_; A.out = out_hd_;
      io_result_done_ = true;
      if (slot_captured(r)) {
        Slot& so = slot(r.slot_out);
        A.pop_io = so.cands; A.cost_io = so.costs;
        io_slot_done_ = true;
      }
    }
    A.mode = r.init ? kInitPhilox : (r.rescore ? kScore : kSmallResident);
    if (inj && r.init) {
      A.inj_init = (const S*)(*inj)[0];
      A.mode = kInitInject;
    }
    if (inj && r.evolves > 0 && d_.N > d_.K) {
      A.inj_parents = (const int*)(*inj)[1];
      A.inj_take = (const uint8_t*)(*inj)[2];
      A.inj_mut = (const uint8_t*)(*inj)[3];
      A.inj_noise = (const double*)(*inj)[4];
    }
    // (draws and selection use every thread; scoring one thread per candidate)
    const int threads = std::min(512, std::max(small_threads_, (d_.N + 31) / 32 * 32));
    if (phases_) {
      A.dbg = dbg_;
      small_dbg_ = true;
    }
    if (timed) pre();
    launch_ex(kern, dim3(I_), dim3(threads), smem, false, A);
    ++launches_;
    ++rollout_launches_;
    if (timed) post();
    small_desc_ = "resident single-CTA solve threads=" + std::to_string(threads) + " smem=" + std::to_string(smem);
    return true;
  }

  // The device part of a run: prep, optional init / rescore, evolves, finalize.
  // Returns the index (0/1) of the buffer holding the final population.
  int enqueue_core(const empc_run_args& r, const std::vector<const void*>* inj, bool timed_rollouts = false) {
    struct PdlOff {  // event records between kernels do not mix with programmatic launches
      bool& flag;
      bool saved;
      PdlOff(bool& f, bool off) : flag(f), saved(f) { if (off) flag = false; }
      ~PdlOff() { flag = saved; }
    } pdl_guard(use_pdl_, timed_rollouts);
    launches_ = 0;
    rollout_launches_ = 0;
    pdl_next_ = false;  // the first kernel follows copies, not a kernel
    auto pre = [&]() { if (timed_rollouts) CK(cudaEventRecord(ev_[2 * rollout_launches_], stream_)); };
    auto post = [&]() { if (timed_rollouts) CK(cudaEventRecord(ev_[2 * rollout_launches_ - 1], stream_)); };
    int cur = 0;
    const size_t pm = d_.pm;
    path_desc_ = "per-generation launches";
    if (try_small(r, timed_rollouts, pre, post, inj)) {
      path_desc_ = small_desc_;
      return 0;
    }
    if (try_persistent(r, timed_rollouts, pre, post, inj)) {
      path_desc_ = persist_desc_;
      return r.evolves & 1;
    }
    if (warm_src_ != nullptr) {  // per-generation launches work on pop_[0]
      CopySpans c;
      c.add(warm_src_->cands, pop_[0], sizeof(S) * (size_t)I_ * d_.N * d_.pm);
      c.add(warm_src_->costs, cost_[0], sizeof(S) * (size_t)I_ * d_.N);
      launch_copies(c);
    }
    if (scorer_ == 1 && (r.init || r.rescore || r.evolves > 0)) launch_cond_build();
    if (r.init) {
      const S* inj_init = inj ? (const S*)(*inj)[0] : nullptr;
      pre();
      launch_rollout(inj_init ? kInitInject : kInitPhilox, d_.N, 0, d_.N, 0, nullptr, nullptr, pop_[0], cost_[0],
                     nullptr, nullptr, nullptr, nullptr, inj_init);
      post();
    } else if (r.rescore) {
      pre();
      launch_rollout(kScore, d_.N, 0, d_.N, 0, pop_[0], nullptr, pop_[0], cost_[0]);
      post();
    }
    const int nc = d_.N - d_.K;
    for (int g = 0; g < r.evolves; ++g) {
      // after the first evolve of a run, rows [0, K) hold the sorted elites
      launch_select(cost_[cur], (g > 0 && incremental_) ? 1 : 0, g, pop_[cur], pop_[cur ^ 1], cost_[cur ^ 1]);
      elites_copied_ = true;
      const int* par = nullptr;
      const uint8_t *tk = nullptr, *mu = nullptr;
      const double* nz = nullptr;
      if (inj && nc > 0) {
        const size_t per = (size_t)I_ * nc * pm;
        par = (const int*)(*inj)[1] + (size_t)g * I_ * nc * 2;
        tk = (const uint8_t*)(*inj)[2] + (size_t)g * per;
        mu = (const uint8_t*)(*inj)[3] + (size_t)g * per;
        nz = (const double*)(*inj)[4] + (size_t)g * per;
      }
      pre();
      launch_rollout(par ? kBreedInject : kBreedPhilox, nc, d_.K, d_.N, g, pop_[cur], cost_[cur], pop_[cur ^ 1],
                     cost_[cur ^ 1], par, tk, mu, nz);
      post();
      cur ^= 1;
    }
    launch_ex(finalize_kernel<S>, dim3(I_), dim3(I_ == 1 ? 1024 : 256), 0, pdl_next_, (const S*)pop_[cur], (const S*)cost_[cur], d_.N,
              d_.m, d_.pm, out_d_);
    pdl_next_ = false;
    ++launches_;
    CK(cudaGetLastError());
    (void)pm;
    return cur;
  }

  // host staging of a run; `copies` = false leaves the H2D copies to the
  // captured graph (graph_for(r, true))
  void stage_run(const empc_run_args& r, bool copies = true, bool warm_copy = true) {
    if (!have_sched_) throw InvalidArg{"schedule not set"};
    if (!have_prob_) throw InvalidArg{"problem not set"};
    if (!r.x0 || !r.sigma) throw InvalidArg{"x0 and sigma are required"};
    if (r.init == 0 && r.slot_in < 0) throw InvalidArg{"a population (slot_in) is required without init"};
    if (r.evolves < 0) throw InvalidArg{"evolves must be >= 0"};
    if (!(r.mutation_prob >= 0.0 && r.mutation_prob <= 1.0) || !(r.crossover_prob >= 0.0 && r.crossover_prob <= 1.0))
      throw InvalidArg{"probabilities must lie in [0, 1]"};
    const int n = d_.n, m = d_.m;
    for (int i = 0; i < I_; ++i) {
      std::memcpy(stage_state_h_ + (size_t)i * SL_.sstride + SL_.x0, r.x0 + (size_t)i * n, sizeof(double) * n);
      std::memcpy(stage_state_h_ + (size_t)i * SL_.sstride + SL_.sig, r.sigma + (size_t)i * m, sizeof(double) * m);
    }
    run_h_->seed = r.seed;
    run_h_->gen0 = r.generation0;
    // Bernoulli(p) as u32 < round(p 2^32): resolution 2^-32, p = 1 always
    run_h_->thr_cross = (uint64_t)std::llround(std::ldexp(r.crossover_prob, 32));
    run_h_->thr_mut = (uint64_t)std::llround(std::ldexp(r.mutation_prob, 32));
    if (copies) enqueue_h2d();
    if (!r.init && warm_copy) {
      Slot& s = slot(r.slot_in);
      CopySpans c;
      c.add(s.cands, pop_[0], sizeof(S) * (size_t)I_ * d_.N * d_.pm);
      c.add(s.costs, cost_[0], sizeof(S) * (size_t)I_ * d_.N);
      launch_copies(c);
    }
  }

  void enqueue_h2d() {
    const size_t prob_bytes = sizeof(double) * (size_t)I_ * SL_.stride;
    const size_t state_bytes =
        reinterpret_cast<uintptr_t>(run_h_ + 1) - reinterpret_cast<uintptr_t>(stage_state_h_);
    if (prob_bytes + state_bytes <= kZeroCopyMax) {
      CopySpans c;
      c.add(stage_prob_hd_, stage_prob_d_, prob_bytes);
      c.add(stage_state_hd_, stage_state_d_, state_bytes);
      launch_copies(c);
      return;
    }
    CK(cudaMemcpyAsync(stage_prob_d_, stage_prob_h_, prob_bytes, cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(stage_state_d_, stage_state_h_, state_bytes, cudaMemcpyHostToDevice, stream_));
  }

  void launch_copies(const CopySpans& c) {
    if (c.n == 0) return;
    const size_t words = (c.largest() + 15) / 16;
    const int ctas = (int)std::max<size_t>(1, std::min<size_t>((size_t)sms_ * 4, (words + 255) / 256));
    copy_spans_kernel<<<ctas, 256, 0, stream_>>>(c);
    CK(cudaGetLastError());
  }

  // result download + copy of the final population into the output slot
  void enqueue_outputs(int cur, const Slot* so, bool result = true) {
    const size_t out_bytes = sizeof(double) * (size_t)I_ * out_stride_;
    CopySpans c;
    if (!result) {
    } else if (out_bytes <= kZeroCopyMax) {
      c.add(out_d_, out_hd_, out_bytes);
    } else {
      CK(cudaMemcpyAsync(out_h_, out_d_, out_bytes, cudaMemcpyDeviceToHost, stream_));
    }
    if (so != nullptr) {
      c.add(pop_[cur], so->cands, sizeof(S) * (size_t)I_ * d_.N * d_.pm);
      c.add(cost_[cur], so->costs, sizeof(S) * (size_t)I_ * d_.N);
    }
    launch_copies(c);
  }

  using GKey = std::tuple<bool, bool, int, int, bool, int, int, int, int, bool, int, bool, int>;
  // public-API graphs also copy the final population into the output slot
  // (captured for the first kCapturedSlots slot ids, eager otherwise)
  static constexpr int kCapturedSlots = 4;
  static bool slot_captured(const empc_run_args& r) { return r.slot_out >= 0 && r.slot_out < kCapturedSlots; }
  // warm public-API runs read their input population straight from a
  // captured slot_in (no copy before the graph)
  static bool warm_in_graph(const empc_run_args& r) {
    return r.init == 0 && r.inject == nullptr && r.slot_in >= 0 && r.slot_in < kCapturedSlots;
  }
  // io code of a graph: 0 = no io, else 1 + 8 * (slot_in code) + (slot_out code),
  // slot codes 0 = not captured, 1 + id otherwise
  static int io_code_of(const empc_run_args& r, bool io) {
    if (!io) return 0;
    const int so = slot_captured(r) ? 1 + r.slot_out : 0;
    const int si = warm_in_graph(r) ? 1 + r.slot_in : 0;
    return 1 + 8 * si + so;
  }
  static bool io_code_uses_slot(int code, int id) {
    return code > 0 && (((code - 1) & 7) == 1 + id || ((code - 1) >> 3) == 1 + id);
  }
  GKey gkey(const empc_run_args& r, bool io) const {
    const int io_code = io_code_of(r, io);
    return std::make_tuple(r.init != 0, r.rescore != 0, r.evolves, forced_, r_diag_, cps_, scorer_, io_code, tc_mode_,
                           halfk_, persist_mode_ + 4 * persist_tile_ + (small_mode_ + 1) * (1 << 24), halfk_ok_,
                           (incremental_ ? 1 : 0) | (use_radix_ ? 2 : 0) | (radix_persist_ok_ ? 4 : 0));
  }

  // One graph per run shape.  io = true also captures the staging H2D copies
  // (pinned host -> device) before and the result D2H after the solve: the
  // public-API run is then one graph launch, two slot copies and one sync.
  cudaGraphExec_t graph_for(const empc_run_args& r, bool io = false) {
    const GKey key = gkey(r, io);
    auto it = graphs_.find(key);
    if (it != graphs_.end()) return it->second;
    if (scorer_ == 1) ensure_cond_ws();
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    int cur = 0;
    try {
      // the resident small solve moves its own inputs / outputs
      const bool direct = io && small_eligible();
      if (io && !direct) enqueue_h2d();
      io_direct_ = direct;
      io_out_direct_ = io;
      io_result_done_ = io_slot_done_ = false;
      warm_src_ = (io && warm_in_graph(r)) ? &slot(r.slot_in) : nullptr;
      cur = enqueue_core(r, nullptr);
      io_direct_ = io_out_direct_ = false;
      warm_src_ = nullptr;
      if (io)
        enqueue_outputs(cur, (slot_captured(r) && !io_slot_done_) ? &slot(r.slot_out) : nullptr, !io_result_done_);
    } catch (...) {
      io_direct_ = io_out_direct_ = false;
      warm_src_ = nullptr;
      cudaStreamEndCapture(stream_, &g);
      throw;
    }
    CK(cudaStreamEndCapture(stream_, &g));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphDestroy(g));
    graphs_[key] = ge;
    graph_cur_[key] = cur;
    graph_launches_[key] = launches_;
    graph_rollouts_[key] = rollout_launches_;
    graph_desc_[key] = path_desc_;
    return ge;
  }

  void run(const empc_run_args& r) override {
    stage_run(r, r.inject != nullptr, !warm_in_graph(r));
    int cur;
    std::vector<S> init_cast;
    if (r.inject) {
      // parity mode: direct launches with the reference's random tensors
      const empc_injected& in = *r.inject;
      const int nc = d_.N - d_.K;
      const size_t per = (size_t)I_ * std::max(nc, 0) * d_.pm;
      std::vector<const void*> ptrs(5, nullptr);
      void *d_init = nullptr, *d_par = nullptr, *d_tk = nullptr, *d_mu = nullptr, *d_nz = nullptr;
      if (r.init) {
        if (!in.init) throw InvalidArg{"injected init population required"};
        CK(cudaMalloc(&d_init, sizeof(S) * (size_t)I_ * d_.N * d_.pm));
        upload_cast(in.init, (S*)d_init, (size_t)I_ * d_.N * d_.pm);
        ptrs[0] = d_init;
      }
      if (r.evolves > 0 && nc > 0) {
        if (!in.parents || !in.take_second || !in.mutate || !in.noise) throw InvalidArg{"injected draws required"};
        const size_t E = r.evolves;
        for (size_t q = 0; q < E * (size_t)I_ * nc * 2; ++q)
          if (in.parents[q] < 0 || in.parents[q] >= d_.K) throw InvalidArg{"injected parent index out of range"};
        CK(cudaMalloc(&d_par, sizeof(int) * E * I_ * nc * 2));
        CK(cudaMalloc(&d_tk, E * per));
        CK(cudaMalloc(&d_mu, E * per));
        CK(cudaMalloc(&d_nz, sizeof(double) * E * per));
        CK(cudaMemcpyAsync(d_par, in.parents, sizeof(int) * E * I_ * nc * 2, cudaMemcpyHostToDevice, stream_));
        CK(cudaMemcpyAsync(d_tk, in.take_second, E * per, cudaMemcpyHostToDevice, stream_));
        CK(cudaMemcpyAsync(d_mu, in.mutate, E * per, cudaMemcpyHostToDevice, stream_));
        CK(cudaMemcpyAsync(d_nz, in.noise, sizeof(double) * E * per, cudaMemcpyHostToDevice, stream_));
        ptrs[1] = d_par; ptrs[2] = d_tk; ptrs[3] = d_mu; ptrs[4] = d_nz;
      }
      cur = enqueue_core(r, &ptrs);
      CK(cudaStreamSynchronize(stream_));
      for (void* p : {d_init, d_par, d_tk, d_mu, d_nz})
        if (p) cudaFree(p);
      CK(cudaMemcpyAsync(out_h_, out_d_, sizeof(double) * (size_t)I_ * out_stride_, cudaMemcpyDeviceToHost, stream_));
    } else {
      cudaGraphExec_t ge = graph_for(r, true);
      cur = graph_cur_[gkey(r, true)];
      path_desc_ = graph_desc_[gkey(r, true)];
      CK(cudaGraphLaunch(ge, stream_));
    }
    if (r.slot_out >= 0 && (r.inject || !slot_captured(r))) {
      Slot& s = slot(r.slot_out);
      CK(cudaMemcpyAsync(s.cands, pop_[cur], sizeof(S) * (size_t)I_ * d_.N * d_.pm, cudaMemcpyDeviceToDevice, stream_));
      CK(cudaMemcpyAsync(s.costs, cost_[cur], sizeof(S) * (size_t)I_ * d_.N, cudaMemcpyDeviceToDevice, stream_));
    }
    CK(cudaStreamSynchronize(stream_));
    const int m = d_.m, pm = d_.pm;
    for (int i = 0; i < I_; ++i) {
      const double* o = out_h_ + (size_t)i * out_stride_;
      if (r.u_out) std::memcpy(r.u_out + (size_t)i * m, o, sizeof(double) * m);
      if (r.best_out) std::memcpy(r.best_out + (size_t)i * pm, o + m, sizeof(double) * pm);
      if (r.best_cost) r.best_cost[i] = o[m + pm];
      if (r.best_index) r.best_index[i] = (int32_t)o[m + pm + 1];
    }
  }

  // -- seams ---------------------------------------------------------------------
  void score(const double* x0, int num, const double* cands, double* costs) override {
    if (!have_sched_ || !have_prob_) throw InvalidArg{"problem and schedule must be set"};
    if (num <= 0) return;
    const int n = d_.n, m = d_.m;
    for (int i = 0; i < I_; ++i) {
      std::memcpy(stage_state_h_ + (size_t)i * SL_.sstride + SL_.x0, x0 + (size_t)i * n, sizeof(double) * n);
      std::fill(stage_state_h_ + (size_t)i * SL_.sstride + SL_.sig, stage_state_h_ + (size_t)i * SL_.sstride + SL_.sig + m, 0.0);
    }
    CK(cudaMemcpyAsync(stage_prob_d_, stage_prob_h_, sizeof(double) * (size_t)I_ * SL_.stride, cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(stage_state_d_, stage_state_h_, sizeof(double) * (size_t)I_ * SL_.sstride, cudaMemcpyHostToDevice, stream_));
    const size_t nc = (size_t)I_ * num * d_.pm;
    ensure_scratch((size_t)I_ * num);
    upload_cast(cands, scratch_pop_, nc);
    pdl_next_ = false;
    if (scorer_ == 1) launch_cond_build();
    launch_rollout(kScore, num, 0, num, 0, scratch_pop_, nullptr, scratch_pop_, scratch_cost_);
    pdl_next_ = false;
    download_uncast(scratch_cost_, costs, (size_t)I_ * num);
  }

  void select(const double* costs, int32_t* elite, int32_t* best) override {
    const size_t nk = (size_t)I_ * d_.N;
    upload_cast(costs, cost_[0], nk);
    pdl_next_ = false;
    launch_select(cost_[0], 0);
    pdl_next_ = false;
    finalize_kernel<S><<<I_, 256, 0, stream_>>>(nullptr, cost_[0], d_.N, d_.m, d_.pm, out_d_);
    CK(cudaGetLastError());
    if (elite) CK(cudaMemcpyAsync(elite, elite_, sizeof(int) * (size_t)I_ * d_.K, cudaMemcpyDeviceToHost, stream_));
    CK(cudaMemcpyAsync(out_h_, out_d_, sizeof(double) * (size_t)I_ * out_stride_, cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
    if (best)
      for (int i = 0; i < I_; ++i) best[i] = (int32_t)out_h_[(size_t)i * out_stride_ + d_.m + d_.pm + 1];
  }

  void expand(int num, const double* cands, double* traj) override {
    if (!have_sched_) throw InvalidArg{"schedule not set"};
    if (num <= 0) return;
    const size_t nc = (size_t)num * d_.pm, nt = (size_t)num * d_.T * d_.m;
    ensure_scratch_pop(nc);
    upload_cast(cands, scratch_pop_, nc);
    ensure_scratch_dbl(nt);
    expand_kernel<S><<<grid_for(nt), 256, 0, stream_>>>(scratch_pop_, num, d_.T, d_.p, d_.m, idx1_, idx2_, cw_, scratch_dbl_);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(traj, scratch_dbl_, sizeof(double) * nt, cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
  }

  // -- device-resident timing (bench.py `value` and roofline) ---------------------
  void time_device(const empc_run_args& r, int reps, int flush, float* ms_each, float* rollout_ms, int32_t* nroll,
                   int32_t* nlaunch) override {
    stage_run(r);
    cudaGraphExec_t ge = graph_for(r);
    const GKey key = gkey(r, false);
    path_desc_ = graph_desc_[key];
    if (flush && !flush_) {
      flush_n_ = (size_t)256 << 20 >> 4;  // 256 MiB > 126 MB L2
      CK(cudaMalloc(&flush_, flush_n_ * 16));
    }
    const int nr = graph_rollouts_[key];
    while ((int)ev_.size() < 2 * nr + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev_.push_back(e);
    }
    CK(cudaStreamSynchronize(stream_));
    cudaEvent_t t0 = ev_[2 * nr], t1 = ev_[2 * nr + 1];
    for (int i = 0; i < reps; ++i) {
      if (flush) flush_kernel<<<sms_ * 4, 512, 0, stream_>>>(flush_, flush_n_, (uint32_t)i);
      CK(cudaEventRecord(t0, stream_));
      CK(cudaGraphLaunch(ge, stream_));
      CK(cudaEventRecord(t1, stream_));
      CK(cudaEventSynchronize(t1));
      CK(cudaEventElapsedTime(&ms_each[i], t0, t1));
    }
    if (nroll) *nroll = nr;
    if (nlaunch) *nlaunch = graph_launches_[key];
    if (rollout_ms) {
      // per-launch rollout durations: one eager replay of the same sequence
      // with events on the launching stream around every rollout launch
      double sum = 0.0;
      const int reps2 = std::max(1, std::min(reps, 20));
      for (int i = 0; i < reps2; ++i) {
        if (flush) flush_kernel<<<sms_ * 4, 512, 0, stream_>>>(flush_, flush_n_, (uint32_t)i);
        enqueue_core(r, nullptr, true);
        CK(cudaStreamSynchronize(stream_));
        for (int q = 0; q < nr; ++q) {
          float ms;
          CK(cudaEventElapsedTime(&ms, ev_[2 * q], ev_[2 * q + 1]));
          sum += ms;
        }
      }
      *rollout_ms = (float)(sum / ((double)reps2 * std::max(nr, 1)));
    }
    if (phases_ && small_dbg_) {  // resident small solve: cycles per phase, summed over generations
      unsigned long long t[7];
      CK(cudaMemcpy(t, dbg_, sizeof t, cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "small solve phases (cycles, all generations): keys=%llu rank=%llu draws=%llu breed=%llu score=%llu"
                   " (thread 0: input cost %llu, drive + recursion %llu)\n", t[0], t[1], t[2], t[3], t[4], t[5], t[6]);
    }
    if (phases_ && dbg_ctas_ > 0) {
      // phase marks of the last rollout launch: mean over CTAs, relative to each CTA's start
      std::vector<unsigned long long> t((size_t)dbg_ctas_ * 16);
      CK(cudaMemcpy(t.data(), dbg_, t.size() * 8, cudaMemcpyDeviceToHost));
      const int order[13] = {0, 7, 8, 1, 2, 9, 10, 3, 11, 12, 4, 5, 6};
      const char* names[13] = {"start", "p0", "sync", "rng", "wait", "elite", "src", "genes", "bu", "cost", "x0", "loop", "end"};
      std::fprintf(stderr, "phases(us since CTA start, mean over %d CTAs):", dbg_ctas_);
      for (int q = 0; q < 13; ++q) {
        double mean = 0;
        for (int c = 0; c < dbg_ctas_; ++c)
          mean += (double)(t[(size_t)c * 16 + order[q]] - t[(size_t)c * 16]) * 1e-3 / dbg_ctas_;
        std::fprintf(stderr, " %s=%.2f", names[q], mean);
      }
      std::fprintf(stderr, "\n");
      if (pick().tc) {  // tensor-core rollout built with -DEMPC_TC_PROF: cycles per step of thread 0
        double acc[5] = {0, 0, 0, 0, 0};
        const int slot[5] = {7, 8, 11, 12, 13};
        for (int c = 0; c < dbg_ctas_; ++c)
          for (int q = 0; q < 5; ++q) acc[q] += (double)t[(size_t)c * 16 + slot[q]] / dbg_ctas_ / d_.T;
        std::fprintf(stderr, "tc step (cycles, thread 0): issue=%.0f drive+wait=%.0f math=%.0f store=%.0f bar=%.0f\n",
                     acc[0], acc[1], acc[2], acc[3], acc[4]);
        dbg_ctas_ = 0;
      }
      // persistent kernel: the selection before the recorded evolve (marks 13-15)
      double w1 = 0, w2 = 0, w3 = 0;
      int cnt = 0;
      for (int c = 0; c < dbg_ctas_; ++c) {
        const unsigned long long* q = &t[(size_t)c * 16];
        if (q[13] == 0 || q[14] == 0 || q[15] == 0) continue;
        w1 += (double)(q[14] - q[13]) * 1e-3;
        w2 += (double)(q[15] - q[14]) * 1e-3;
        w3 += (double)(q[0] - q[15]) * 1e-3;
        ++cnt;
      }
      if (cnt) std::fprintf(stderr, "persist(us, mean over %d CTAs): sync_before_select=%.2f select=%.2f sync_after=%.2f\n",
                            cnt, w1 / cnt, w2 / cnt, w3 / cnt);
      if (cnt) {  // per-generation timeline of the persistent solve (CTA 0)
        std::vector<unsigned long long> gt(32);
        CK(cudaMemcpy(gt.data(), dbg_ + (size_t)dbg_ctas_ * 16, 32 * 8, cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "persist timeline (us from kernel start): init_rollout_end=%.2f", (gt[1] - gt[0]) * 1e-3);
        for (int g = 2; g < 30 && gt[g] > gt[0]; ++g) std::fprintf(stderr, " gen%d_end=%.2f", g - 1, (gt[g] - gt[0]) * 1e-3);
        if (gt[31] > gt[0]) std::fprintf(stderr, " end=%.2f", (gt[31] - gt[0]) * 1e-3);
        std::fprintf(stderr, "\n");
        std::vector<unsigned long long> rm(16);  // first (radix) selection, CTA 0
        CK(cudaMemcpy(rm.data(), dbg_ + (size_t)dbg_ctas_ * 16 + 32, 16 * 8, cudaMemcpyDeviceToHost));
        if (rm[0] != 0) {
          std::fprintf(stderr, "first selection (us, CTA 0, from the key load): common_bits=%.2f", (rm[1] - rm[0]) * 1e-3);
          for (int q = 2; q < 10 && rm[q] != 0; ++q) std::fprintf(stderr, " pass%d=%.2f", q - 1, (rm[q] - rm[0]) * 1e-3);
          std::fprintf(stderr, " compact=%.2f ranked=%.2f\n", (rm[10] - rm[0]) * 1e-3, (rm[11] - rm[0]) * 1e-3);
        }
      }
    }
  }

  // -- population sharding: see shard_export_kernel ------------------
  void shard_setup(long long child_base, int n_children, long long init_base, int n_init, int owns_elites) override {
    if (I_ != 1) throw InvalidArg{"population sharding needs a single-instance handle"};
    if (n_children < 0 || n_init < 0 || d_.K + std::max(n_children, n_init) > d_.N)
      throw InvalidArg{"shard does not fit the handle (num_sims must be >= K + max(children, init) rows)"};
    sh_child_base_ = child_base;
    sh_children_ = n_children;
    sh_init_base_ = init_base;
    sh_init_ = n_init;
    sh_owns_elites_ = owns_elites;
    sh_on_ = true;
  }
  size_t shard_entry_size() override { return shard_entry_bytes<S>(d_.pm); }
  void shard_check() {
    if (!sh_on_) throw InvalidArg{"empc_shard_setup first"};
  }
  // The per-generation shard calls only ENQUEUE work on the handle's stream
  // (empc_get_stream): a rank's generation is export -> all-gather (NCCL on
  // the same stream) -> import -> evolve with no host synchronisation.  The
  // problem, x0, sigma and RNG parameters are staged once by shard_init.
  void shard_init(const empc_run_args& r) override {
    shard_check();
    empc_run_args rr = r;
    rr.init = 1;
    rr.slot_in = -1;
    stage_run(rr);
    sh_gen0_ = r.generation0;
    if (!sh_attr_set_) {
      CK(cudaFuncSetAttribute(shard_export_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024));
      CK(cudaFuncSetAttribute(shard_import_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024));
      CK(cudaFuncSetAttribute(shard_export_radix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024));
      sh_attr_set_ = true;
    }
    pdl_next_ = false;
    if (scorer_ == 1) launch_cond_build();
    cand_base_ = (int)sh_init_base_;
    launch_rollout(kInitPhilox, sh_init_, d_.K, d_.N, 0, nullptr, nullptr, pop_[0], cost_[0]);
    cand_base_ = 0;
    pdl_next_ = false;
    sh_cur_ = 0;
    sh_init_phase_ = true;
    CK(cudaGetLastError());
  }
  int rank_grid(int M) const { return std::max(1, std::min(sms_, (M + 15) / 16)); }
  void shard_export(void* dev_out) override {
    shard_check();
    const int incl = (sh_owns_elites_ && !sh_init_phase_) ? 1 : 0;
    const int nl = sh_init_phase_ ? sh_init_ : sh_children_;
    const long long gbase = sh_init_phase_ ? sh_init_base_ : (long long)d_.K + sh_child_base_;
    const int M = (incl ? d_.K : 0) + nl;
    if constexpr (sizeof(S) == 4) {
      const size_t rsm = shard_export_radix_smem(M, d_.K);
      if (rsm <= (size_t)kMaxSmem - 1024 && M >= 2048) {  // large shards: radix select
        shard_export_radix_kernel<<<rank_grid(d_.K), 1024, rsm, stream_>>>(
            (const float*)pop_[sh_cur_], (const float*)cost_[sh_cur_], d_.K, d_.pm, incl, nl, gbase,
            (unsigned char*)dev_out);
        CK(cudaGetLastError());
        return;
      }
    }
    const size_t smem = (size_t)M * (sizeof(typename OrdOf<S>::T) + 2 * sizeof(int));
    if (smem > (size_t)kMaxSmem - 1024) throw InvalidArg{"shard too large for the export kernel"};
    shard_export_kernel<S><<<rank_grid(M), 256, smem, stream_>>>(pop_[sh_cur_], cost_[sh_cur_], d_.K, d_.pm, incl, nl,
                                                                  gbase, (unsigned char*)dev_out);
    CK(cudaGetLastError());
  }
  void shard_import(const void* dev_all, int world, double* u, double* best, double* cost, long long* grow) override {
    shard_check();
    const int M = world * d_.K;
    const size_t smem = (size_t)M * (sizeof(unsigned long long) + sizeof(unsigned));
    if (smem > (size_t)kMaxSmem - 1024) throw InvalidArg{"world * num_parents too large for the import kernel"};
    shard_import_kernel<S><<<rank_grid(M), 256, smem, stream_>>>((const unsigned char*)dev_all, M, d_.K, d_.pm, d_.m,
                                                                  pop_[sh_cur_], cost_[sh_cur_], elite_, out_d_);
    CK(cudaGetLastError());
    sh_init_phase_ = false;
    if (!u && !best && !cost && !grow) return;  // mid-solve generation: nothing to read back
    CK(cudaMemcpyAsync(out_h_, out_d_, sizeof(double) * out_stride_, cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
    if (u) std::memcpy(u, out_h_, sizeof(double) * d_.m);
    if (best) std::memcpy(best, out_h_ + d_.m, sizeof(double) * d_.pm);
    if (cost) *cost = out_h_[d_.m + d_.pm];
    if (grow) *grow = (long long)out_h_[d_.m + d_.pm + 1];
  }
  void shard_evolve(const empc_run_args& r) override {
    shard_check();
    if (sh_init_phase_) throw InvalidArg{"import the elites before evolving"};
    // RNG generation = staged gen0 + evolve index: no re-staging per generation
    const long long ev = r.generation0 - sh_gen0_;
    if (ev < 0 || ev > INT32_MAX) throw InvalidArg{"generation precedes the shard's init"};
    pdl_next_ = false;
    cand_base_ = (int)sh_child_base_;
    int* saved_q = qcount_;
    qcount_ = nullptr;
    const bool saved_inc = incremental_;
    incremental_ = false;
    launch_rollout(kBreedPhilox, sh_children_, d_.K, d_.N, (int)ev, pop_[sh_cur_], cost_[sh_cur_], pop_[sh_cur_ ^ 1],
                   cost_[sh_cur_ ^ 1]);
    incremental_ = saved_inc;
    qcount_ = saved_q;
    cand_base_ = 0;
    pdl_next_ = false;
    sh_cur_ ^= 1;
    CK(cudaGetLastError());
  }
  void* stream() override { return (void*)stream_; }
  void shard_read(double* cands, double* costs) override {
    shard_check();
    CK(cudaStreamSynchronize(stream_));
    const size_t rows = (size_t)d_.K + (sh_init_phase_ ? sh_init_ : sh_children_);
    const size_t nc = rows * d_.pm;
    ensure_scratch_dbl(std::max(nc, rows));
    if (cands) {
      uncast_kernel<S><<<grid_for(nc), 256, 0, stream_>>>(pop_[sh_cur_], scratch_dbl_, nc);
      CK(cudaMemcpyAsync(cands, scratch_dbl_, sizeof(double) * nc, cudaMemcpyDeviceToHost, stream_));
      CK(cudaStreamSynchronize(stream_));
    }
    if (costs) {
      uncast_kernel<S><<<grid_for(rows), 256, 0, stream_>>>(cost_[sh_cur_], scratch_dbl_, rows);
      CK(cudaMemcpyAsync(costs, scratch_dbl_, sizeof(double) * rows, cudaMemcpyDeviceToHost, stream_));
      CK(cudaStreamSynchronize(stream_));
    }
  }

  std::string describe() override {
    if (scorer_ == 1) {
      const CondPlan c = plan_cond(d_.N - d_.K);
      char buf[256];
      std::snprintf(buf, sizeof buf, "condensed scorer (FP64 quadratic form) | evolve tile=%d tiles=%d threads=%d smem=%zu P_in_smem=%d | sms=%d",
                    c.tile, c.tiles, c.threads, c.smem, (int)c.psm, sms_);
      return buf;
    }
    const Variant<S>& v = pick();
    const Launch a = plan(v, d_.N - d_.K);
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s | evolve tile=%d tileP=%d tiles=%d threads=%d smem=%zu | sms=%d%s%s", v.name,
                  a.tile, a.tileP, a.tiles, a.threads, a.smem, sms_, path_desc_.empty() ? "" : " | last run: ",
                  path_desc_.c_str());
    return buf;
  }
  int num_variants() override { return (int)variants_.size(); }
  void set_occupancy(int cps) override {
    if (cps < 0 || cps > 32) throw InvalidArg{"ctas_per_sm must lie in [0, 32]"};
    cps_ = cps;
  }
  void set_tensor_cores(int mode) override {
    if (mode < -1 || mode > 1) throw InvalidArg{"tensor_cores must be -1 (auto), 0 (off) or 1 (on)"};
    tc_mode_ = mode;
  }
  void set_option(int opt, int val) override {
    switch (opt) {
      case EMPC_OPT_PERSISTENT:
        if (val < -1 || val > 1) throw InvalidArg{"persistent mode must be -1 (auto), 0 (off) or 1 (on)"};
        persist_mode_ = val;
        break;
      case EMPC_OPT_HALF_K:
        if (val < 0 || val > 1) throw InvalidArg{"half-K must be 0 or 1"};
        halfk_ok_ = val != 0;
        break;
      case EMPC_OPT_INCREMENTAL_SELECT:
        if (val < 0 || val > 1) throw InvalidArg{"incremental selection must be 0 or 1"};
        incremental_ = val != 0;
        break;
      case EMPC_OPT_PERSIST_TILE:
        if (val < 0 || val > 1 << 20) throw InvalidArg{"persistent tile out of range"};
        persist_tile_ = val;
        break;
      case EMPC_OPT_SMALL_SOLVE:
        if (val < -1 || val > 1) throw InvalidArg{"small solve mode must be -1 (auto), 0 (off) or 1 (on)"};
        small_mode_ = val;
        break;
      case EMPC_OPT_RADIX_SELECT:
        if (val < 0 || val > 1) throw InvalidArg{"radix selection must be 0 or 1"};
        if (val && (sizeof(S) != 4 || I_ != 1 || radix_select_smem(d_.N, d_.K) > (size_t)kMaxSmem - 1024))
          throw InvalidArg{"radix selection needs a single FP32 instance"};
        use_radix_ = val != 0;
        radix_persist_ok_ = val != 0;
        break;
      default:
        throw InvalidArg{"unknown option " + std::to_string(opt)};
    }
  }
  void set_variant(int v) override {
    if (v >= (int)variants_.size()) throw InvalidArg{"variant out of range"};
    if (v >= 0 && variants_[v].dq != dense_) throw InvalidArg{"variant does not match the Q structure"};
    forced_ = v;
  }

 private:
  static int grid_for(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 16); }
  void ensure_scratch(size_t ncand) {
    ensure_scratch_pop(ncand * d_.pm);
    if (ncand > scratch_cost_n_) {
      if (scratch_cost_) cudaFree(scratch_cost_);
      CK(cudaMalloc(&scratch_cost_, sizeof(S) * ncand));
      scratch_cost_n_ = ncand;
    }
  }
  void ensure_scratch_pop(size_t ne) {
    if (ne > scratch_pop_n_) {
      if (scratch_pop_) cudaFree(scratch_pop_);
      CK(cudaMalloc(&scratch_pop_, sizeof(S) * ne));
      scratch_pop_n_ = ne;
    }
  }
  void ensure_scratch_dbl(size_t ne) {
    if (ne > scratch_dbl_n_) {
      if (scratch_dbl_) cudaFree(scratch_dbl_);
      CK(cudaMalloc(&scratch_dbl_, sizeof(double) * ne));
      scratch_dbl_n_ = ne;
    }
  }
  void upload_cast(const double* h, S* dptr, size_t ne) {
    ensure_scratch_dbl(ne);
    CK(cudaMemcpyAsync(scratch_dbl_, h, sizeof(double) * ne, cudaMemcpyHostToDevice, stream_));
    cast_kernel<S><<<grid_for(ne), 256, 0, stream_>>>(scratch_dbl_, dptr, ne);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream_));
  }
  void download_uncast(const S* dptr, double* h, size_t ne) {
    ensure_scratch_dbl(ne);
    uncast_kernel<S><<<grid_for(ne), 256, 0, stream_>>>(dptr, scratch_dbl_, ne);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, scratch_dbl_, sizeof(double) * ne, cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
  }

  empc_dims dims_;
  Dims d_{};
  StageLayout SL_{};
  int I_ = 1;
  bool dense_ = false;
  int sms_ = 148;
  cudaStream_t stream_{};
  std::vector<Variant<S>> variants_;
  int forced_ = -1;
  int cps_ = 0;  // CTAs per SM for the rollout (0: heuristic)
  int tc_mode_ = -1;  // tensor-core rollout: -1 auto, 0 off, 1 on
  bool tc_multi_ok_ = std::getenv("EMPC_TC_NO_MULTI") == nullptr;
  int cand_base_ = 0;  // global index of local candidate 0 (population sharding)
  bool elites_copied_ = false;  // the last selection also carried the elites over
  long long sh_child_base_ = 0, sh_init_base_ = 0;
  int sh_children_ = 0, sh_init_ = 0, sh_owns_elites_ = 0, sh_cur_ = 0;
  bool sh_init_phase_ = true, sh_on_ = false, sh_attr_set_ = false;
  long long sh_gen0_ = 1;
  bool use_pdl_ = true, pdl_next_ = false, phases_ = false, incremental_ = true;
  int persist_mode_ = -1;  // persistent solve: -1 auto, 0 off, 1 whenever the shape allows
  int persist_tile_ = 0;   // minimum candidates per persistent CTA (0: one wave over the SMs)
  int small_mode_ = -1;    // resident single-CTA solve: -1 auto, 0 off, 1 whenever it fits
  int small_threads_ = 512;
  bool small_attr_set_ = false, small_dbg_ = false;
  std::string small_desc_;
  bool persist_attr_set_ = false;
  std::vector<PersistVariant<S>> persist_;
  std::string persist_desc_, path_desc_;

  unsigned long long* dbg_ = nullptr;
  size_t dbg_n_ = 0;
  int dbg_ctas_ = 0;
  double *stage_prob_d_ = nullptr, *stage_state_d_ = nullptr, *stage_prob_h_ = nullptr, *stage_state_h_ = nullptr;
  RunParams *run_d_ = nullptr, *run_h_ = nullptr;
  S* pop_[2] = {nullptr, nullptr};
  S* cost_[2] = {nullptr, nullptr};
  int* elite_ = nullptr;
  int* qcount_ = nullptr;
  void* qlist_ = nullptr;
  int qcap_ = 0;
  double *out_d_ = nullptr, *out_h_ = nullptr;
  double *stage_prob_hd_ = nullptr, *stage_state_hd_ = nullptr, *out_hd_ = nullptr;  // device views of pinned memory
  RunParams* run_hd_ = nullptr;
  bool io_direct_ = false;  // the small solve moves the public-API graph's inputs / outputs itself
  bool io_out_direct_ = false;                          // capture of a public-API graph: paths may write outputs
  bool io_result_done_ = false, io_slot_done_ = false;  // ... and report which they wrote
  const Slot* warm_src_ = nullptr;  // capture of a warm public-API graph: the input population's slot
  int out_stride_ = 0;
  int *idx1_ = nullptr, *idx2_ = nullptr, *seg_ = nullptr;
  unsigned long long* amin_d_ = nullptr;  // persistent solve: argmin key
  int stagger_ = 0;       // WS recursion phase offset (cycles), EMPC_STAGGER
  bool predraw_ok_ = std::getenv("EMPC_NO_PREDRAW") == nullptr;
  // one-barrier generations (redundant per-CTA selection): correct (the GPU
  // tests pass in that mode) but measured slower at C3 (34.5 vs 31.3 us per
  // generation), so opt-in
  bool one_sync_ok_ = std::getenv("EMPC_ONE_SYNC") != nullptr;
  int ws_threads_ = 384;  // threads of a warp-synchronous persistent CTA (helpers beyond the candidate warps)
  S *cw_ = nullptr, *G_ = nullptr;
  double *W64_ = nullptr, *G64_ = nullptr;  // FP64 W (T x p) and W'W for the condensed build
  int scorer_ = 0;
  CondKernels<S> ck_{};
  double* cond_ = nullptr;  // per instance: P, g, ref, J_ref
  double* cws_ = nullptr;   // build workspace
  size_t cws_n_ = 0;
  size_t select_smem_ = 0;
  bool use_radix_ = false;
  int radix_ctas_ = std::getenv("EMPC_RADIX_CTAS") ? std::atoi(std::getenv("EMPC_RADIX_CTAS")) : 0;
  bool radix_persist_ok_ = true;  // cleared by EMPC_OPT_RADIX_SELECT = 0
  int radix_min_n_ = 8192;
  bool have_sched_ = false, have_prob_ = false, r_diag_ = true;
  bool halfk_ = false, halfk_ok_ = std::getenv("EMPC_NO_HALFK") == nullptr;
  std::vector<Slot> slots_;
  S *scratch_pop_ = nullptr, *scratch_cost_ = nullptr;
  double* scratch_dbl_ = nullptr;
  size_t scratch_pop_n_ = 0, scratch_cost_n_ = 0, scratch_dbl_n_ = 0;
  uint4* flush_ = nullptr;
  size_t flush_n_ = 0;
  std::vector<cudaEvent_t> ev_;
  std::map<GKey, cudaGraphExec_t> graphs_;
  std::map<GKey, int> graph_cur_, graph_launches_, graph_rollouts_;
  std::map<GKey, std::string> graph_desc_;
  int launches_ = 0, rollout_launches_ = 0;
};

}  // namespace

struct empc_handle {
  std::unique_ptr<EngineBase> eng;
};

#define GUARD(h, ...)                                              \
  do {                                                              \
    if (!(h)) return EMPC_EINVAL;                                   \
    try {                                                           \
      __VA_ARGS__;                                                  \
      return EMPC_OK;                                               \
    } catch (const InvalidArg& e) {                                 \
      (h)->eng->err = e.msg;                                        \
      return EMPC_EINVAL;                                           \
    } catch (const CudaError& e) {                                  \
      (h)->eng->err = e.msg;                                        \
      return EMPC_ECUDA;                                            \
    } catch (const std::exception& e) {                             \
      (h)->eng->err = e.what();                                     \
      return EMPC_ESTATE;                                           \
    }                                                               \
  } while (0)

extern "C" {

int empc_create(const empc_dims* dims, empc_handle** out) {
  if (!dims || !out) return EMPC_EINVAL;
  *out = nullptr;
  const empc_dims& d = *dims;
  if (d.n < 1 || d.m < 1 || d.T < 1 || d.p < 1 || d.p > d.T || d.num_sims < 1 || d.num_parents < 1 ||
      d.num_parents > d.num_sims || d.instances < 1) {
    g_create_error = "invalid dimensions";
    return EMPC_EINVAL;
  }
  if (pad_np(d.n) < 0) {
    g_create_error = "state dimension > 128 is not supported";
    return EMPC_EINVAL;
  }
  try {
    auto* h = new empc_handle;
    if (d.precision == EMPC_FP64) h->eng.reset(new Engine<double>(d));
    else h->eng.reset(new Engine<float>(d));
    *out = h;
    return EMPC_OK;
  } catch (const InvalidArg& e) {
    g_create_error = e.msg;
    return EMPC_EINVAL;
  } catch (const CudaError& e) {
    g_create_error = e.msg;
    return EMPC_ECUDA;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return EMPC_ENOMEM;
  }
}

void empc_destroy(empc_handle* h) { delete h; }

const char* empc_last_error(const empc_handle* h) {
  if (!h || !h->eng) return g_create_error.c_str();
  return h->eng->err.c_str();
}

int empc_set_scorer(empc_handle* h, int32_t scorer) {
  GUARD(h, { h->eng->set_scorer(scorer); });
}

int empc_set_schedule(empc_handle* h, const int32_t* idx1, const int32_t* idx2, const double* c) {
  GUARD(h, { if (!idx1 || !idx2 || !c) throw InvalidArg{"null schedule"}; h->eng->set_schedule(idx1, idx2, c); });
}

int empc_set_problems(empc_handle* h, int32_t first, int32_t count, const double* Ad, const double* Bd,
                      const double* wd, const double* Q, const double* R, const double* x_goal, const double* u_goal,
                      const double* u_min, const double* u_max) {
  GUARD(h, {
    const double* arrs[9] = {Ad, Bd, wd, Q, R, x_goal, u_goal, u_min, u_max};
    h->eng->set_problems(first, count, arrs);
  });
}

int empc_pop_alloc(empc_handle* h, int32_t* slot) {
  GUARD(h, { if (!slot) throw InvalidArg{"null slot"}; *slot = h->eng->pop_alloc(); });
}
int empc_pop_free(empc_handle* h, int32_t slot) { GUARD(h, h->eng->pop_free(slot)); }
int empc_pop_read(empc_handle* h, int32_t slot, double* cands, double* costs) {
  GUARD(h, h->eng->pop_read(slot, cands, costs));
}
int empc_pop_write(empc_handle* h, int32_t slot, const double* cands, const double* costs) {
  GUARD(h, { if (!cands) throw InvalidArg{"null candidates"}; h->eng->pop_write(slot, cands, costs); });
}

int empc_run(empc_handle* h, const empc_run_args* args) {
  GUARD(h, { if (!args) throw InvalidArg{"null args"}; h->eng->run(*args); });
}

int empc_score(empc_handle* h, const double* x0, int32_t num, const double* cands, double* costs) {
  GUARD(h, { if (!x0 || (num > 0 && (!cands || !costs))) throw InvalidArg{"null argument"}; h->eng->score(x0, num, cands, costs); });
}

int empc_select(empc_handle* h, const double* costs, int32_t* elite_idx, int32_t* best_index) {
  GUARD(h, { if (!costs) throw InvalidArg{"null costs"}; h->eng->select(costs, elite_idx, best_index); });
}

int empc_expand(empc_handle* h, int32_t num, const double* cands, double* traj) {
  GUARD(h, { if (num > 0 && (!cands || !traj)) throw InvalidArg{"null argument"}; h->eng->expand(num, cands, traj); });
}

int empc_time_device(empc_handle* h, const empc_run_args* args, int32_t reps, int32_t flush_l2, float* ms_each,
                     float* rollout_ms, int32_t* rollout_launches, int32_t* launches_per_rep) {
  GUARD(h, {
    if (!args || !ms_each || reps < 1) throw InvalidArg{"invalid timing arguments"};
    if (args->inject) throw InvalidArg{"timing runs use the in-kernel RNG"};
    h->eng->time_device(*args, reps, flush_l2, ms_each, rollout_ms, rollout_launches, launches_per_rep);
  });
}

int empc_describe(empc_handle* h, char* buf, int32_t len) {
  GUARD(h, {
    const std::string s = h->eng->describe();
    if (buf && len > 0) {
      std::strncpy(buf, s.c_str(), (size_t)len - 1);
      buf[len - 1] = 0;
    }
  });
}

int empc_num_variants(empc_handle* h, int32_t* count) {
  GUARD(h, { if (count) *count = h->eng->num_variants(); });
}

int empc_set_variant(empc_handle* h, int32_t variant) { GUARD(h, h->eng->set_variant(variant)); }

int empc_set_occupancy(empc_handle* h, int32_t ctas_per_sm) { GUARD(h, h->eng->set_occupancy(ctas_per_sm)); }
int empc_set_tensor_cores(empc_handle* h, int32_t mode) { GUARD(h, h->eng->set_tensor_cores(mode)); }
int empc_set_option(empc_handle* h, int32_t option, int32_t value) { GUARD(h, h->eng->set_option(option, value)); }

int empc_shard_setup(empc_handle* h, int64_t child_base, int32_t n_children, int64_t init_base, int32_t n_init,
                     int32_t owns_elites) {
  GUARD(h, h->eng->shard_setup(child_base, n_children, init_base, n_init, owns_elites));
}
int empc_shard_entry_bytes(empc_handle* h, int64_t* bytes) {
  GUARD(h, { if (!bytes) throw InvalidArg{"null"}; *bytes = (int64_t)h->eng->shard_entry_size(); });
}
int empc_shard_init(empc_handle* h, const empc_run_args* args) {
  GUARD(h, { if (!args) throw InvalidArg{"null args"}; h->eng->shard_init(*args); });
}
int empc_shard_export(empc_handle* h, void* dev_entries) {
  GUARD(h, { if (!dev_entries) throw InvalidArg{"null buffer"}; h->eng->shard_export(dev_entries); });
}
int empc_shard_import(empc_handle* h, const void* dev_all, int32_t world, double* u_out, double* best_out,
                      double* best_cost, int64_t* best_row) {
  GUARD(h, {
    if (!dev_all || world < 1) throw InvalidArg{"invalid import"};
    long long g = 0;
    h->eng->shard_import(dev_all, world, u_out, best_out, best_cost, &g);
    if (best_row) *best_row = g;
  });
}
int empc_shard_evolve(empc_handle* h, const empc_run_args* args) {
  GUARD(h, { if (!args) throw InvalidArg{"null args"}; h->eng->shard_evolve(*args); });
}
int empc_shard_read(empc_handle* h, double* cands, double* costs) { GUARD(h, h->eng->shard_read(cands, costs)); }
int empc_get_stream(empc_handle* h, void** stream) {
  GUARD(h, { if (!stream) throw InvalidArg{"null stream"}; *stream = h->eng->stream(); });
}

int empc_philox(const uint32_t* ctr, const uint32_t* key, int32_t count, uint32_t* out) {
  if (count <= 0) return EMPC_OK;
  if (!ctr || !key || !out) return EMPC_EINVAL;
  uint32_t *dc = nullptr, *dk = nullptr, *dout = nullptr;
  cudaError_t e = cudaMalloc(&dc, 16 * (size_t)count);
  if (e == cudaSuccess) e = cudaMalloc(&dk, 8 * (size_t)count);
  if (e == cudaSuccess) e = cudaMalloc(&dout, 16 * (size_t)count);
  if (e == cudaSuccess) e = cudaMemcpy(dc, ctr, 16 * (size_t)count, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dk, key, 8 * (size_t)count, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    philox_kernel<<<(count + 127) / 128, 128>>>(dc, dk, count, dout);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, 16 * (size_t)count, cudaMemcpyDeviceToHost);
  cudaFree(dc);
  cudaFree(dk);
  cudaFree(dout);
  if (e != cudaSuccess) {
    g_create_error = cudaGetErrorString(e);
    return EMPC_ECUDA;
  }
  return EMPC_OK;
}

}  // extern "C"
