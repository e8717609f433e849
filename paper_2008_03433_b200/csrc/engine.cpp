// Host orchestration of the B200 TRON hot path: device layout, the
// evaluator operations (backend.cpp:136-306 semantics), the device-resident
// truncated CG captured as a CUDA graph with a while node, and the
// device-mode outer trust-region loop (tron.cpp:127-217 control flow with
// only scalars crossing PCIe).
#include "engine.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <future>
#include <map>
#include <mutex>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

namespace tb {

static bool env_flag(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] == '1';
}

[[noreturn]] void raise(int status, const std::string& msg) { throw StatusError(status, msg); }

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear sticky-less errors
  const int st = (e == cudaErrorMemoryAllocation) ? TRON_ERR_OOM : TRON_ERR_CUDA;
  raise(st, std::string(what) + ": " + cudaGetErrorString(e));
}

[[noreturn]] void launch_failed(cudaError_t e, const char* what) {
  cudaGetLastError();
  raise(TRON_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void ensure_max_dynamic_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{func, dev}];
  if (have >= bytes) return;
  cuda_check(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
             "cudaFuncSetAttribute(max dynamic shared memory)");
  have = bytes;
}

// ----------------------------------------------------------------------------
// NCCL (dlopen'd so single-GPU use never needs it)
// ----------------------------------------------------------------------------
namespace {
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (lib) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      lib = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
      if (lib) break;
    }
    if (!lib) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(lib, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(lib, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(lib, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(lib, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(lib, "ncclGetErrorString");
    return GetUniqueId && CommInitRank && AllReduce && CommDestroy;
  }
};
NcclApi g_nccl;

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  raise(TRON_ERR_NCCL, std::string(what) + ": " +
                           (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
}
}  // namespace

int nccl_unique_id(void* out128) {
  if (!g_nccl.load()) raise(TRON_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
  return TRON_OK;
}

void Comm::init(const tron_gpu_options& opt) {
  rank = opt.rank;
  world = opt.world;
  if (opt.host_allreduce && world > 1) {  // caller's host collective
    host_fn_ = opt.host_allreduce;
    host_user_ = opt.host_allreduce_user;
    return;
  }
  // TRON_B200_FORCE_NCCL=1 runs a single-rank problem through the sharded code
  // path with a real one-rank NCCL communicator (tests the multi-GPU plumbing
  // on one GPU: partials, allreduce on the stream, host-driven CG).
  const char* fe = std::getenv("TRON_B200_FORCE_NCCL");
  forced = world == 1 && fe && fe[0] == '1';
  if (world <= 1 && !forced) return;
  if (!opt.nccl_unique_id && world > 1)
    raise(TRON_ERR_ARGUMENT, "world > 1 requires an nccl_unique_id or a host_allreduce");
  if (!g_nccl.load()) raise(TRON_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  if (opt.nccl_unique_id)
    std::memcpy(&id, opt.nccl_unique_id, sizeof(id));
  else
    nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
  cuda_check(cudaSetDevice(opt.device), "cudaSetDevice");
  ncclComm_t c;
  nccl_check(g_nccl.CommInitRank(&c, world, id, rank), "ncclCommInitRank");
  comm_ = c;
}

Comm::~Comm() {
  if (comm_ && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)comm_);
  if (stage_) tron_host_free(stage_);
}

void Comm::allreduce_sum(const double* send, double* recv, size_t count, cudaStream_t s) {
  if (count == 0) return;
  if (!active()) {
    if (send != recv)
      cuda_check(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, s), "D2D");
    return;
  }
  if (host_fn_) {
    if (send != recv)
      cuda_check(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, s), "D2D");
    allreduce_sum(recv, count, s);
    return;
  }
  nccl_check(g_nccl.AllReduce(send, recv, count, ncclFloat64, ncclSum, (ncclComm_t)comm_, s),
             "ncclAllReduce");
}

void Comm::allreduce_sum(double* buf, size_t count, cudaStream_t s) {
  if (!active() || count == 0) return;
  if (host_fn_) {
    if (stage_n_ < count) {
      if (stage_) tron_host_free(stage_);
      stage_ = static_cast<double*>(tron_host_alloc(count * sizeof(double)));
      if (!stage_) raise(TRON_ERR_OOM, "pinned staging buffer for the host allreduce");
      stage_n_ = count;
    }
    cuda_check(cudaMemcpyAsync(stage_, buf, count * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "host allreduce sync");
    host_fn_(host_user_, stage_, (uint64_t)count);
    cuda_check(cudaMemcpyAsync(buf, stage_, count * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    // the next host allreduce overwrites stage_ only after this copy (it syncs s first)
    return;
  }
  nccl_check(g_nccl.AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)comm_, s),
             "ncclAllReduce");
}

// ----------------------------------------------------------------------------
// creation + validation (FeatureMatrix::csr linalg.cpp:34-73; Problem::validate loss.cpp:20-33)
// ----------------------------------------------------------------------------
namespace {

// Input validation runs on the worker pool; the first offending row found
// is re-checked sequentially so the error (class + message) is exactly the
// one a front-to-back scan reports.
// grain: items per task (about 64K elementary checks per task)
template <class Bad>
uint64_t first_bad(uint64_t count, Bad bad, size_t grain = size_t{1} << 16) {
  std::atomic<uint64_t> first{UINT64_MAX};
  parallel_for(count, grain, [&](size_t b, size_t e) {
    for (size_t i = b; i < e && i < first.load(std::memory_order_relaxed); ++i)
      if (bad(i)) {
        uint64_t cur = first.load();
        while (i < cur && !first.compare_exchange_weak(cur, i)) {
        }
        return;
      }
  });
  return first.load();
}

void validate_labels_C(uint64_t l, const double* y, double C) {
  const uint64_t i = first_bad(l, [&](uint64_t k) { return y[k] != 1.0 && y[k] != -1.0; });
  if (i != UINT64_MAX)
    raise(TRON_ERR_DIMENSION, "problem: label " + std::to_string(y[i]) + " not in {-1,+1}");
  if (!(C > 0.0)) raise(TRON_ERR_DIMENSION, "problem: C must be positive");
}

void validate_offsets(uint64_t l, const int64_t* ro) {
  if (ro[0] != 0) raise(TRON_ERR_DIMENSION, "csr matrix: offsets/indices/values disagree");
  const uint64_t dec = first_bad(l, [&](uint64_t i) { return ro[i] > ro[i + 1]; });
  if (dec != UINT64_MAX)
    raise(TRON_ERR_DIMENSION, "csr matrix: decreasing row offset at row " + std::to_string(dec));
}

void validate_csr(uint64_t l, uint64_t n, const int64_t* ro, const int32_t* ci) {
  if (ro[0] != 0) raise(TRON_ERR_DIMENSION, "csr matrix: offsets/indices/values disagree");
  auto check_row = [&](uint64_t i, bool throw_it) {
    if (ro[i] > ro[i + 1]) {
      if (throw_it)
        raise(TRON_ERR_DIMENSION, "csr matrix: decreasing row offset at row " + std::to_string(i));
      return true;
    }
    int32_t prev = -1;
    for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
      const int32_t c = ci[k];
      if (c < 0 || static_cast<uint64_t>(c) >= n) {
        if (throw_it)
          raise(TRON_ERR_BOUNDS, "csr matrix: column " + std::to_string(c) +
                                     " out of range in row " + std::to_string(i));
        return true;
      }
      if (c <= prev) {
        if (throw_it)
          raise(TRON_ERR_DIMENSION,
                "csr matrix: column indices not strictly ascending in row " + std::to_string(i));
        return true;
      }
      prev = c;
    }
    return false;
  };
  // offsets first (a decreasing offset makes later rows' ranges meaningless)
  const uint64_t dec = first_bad(l, [&](uint64_t i) { return ro[i] > ro[i + 1]; });
  const uint64_t lim = dec == UINT64_MAX ? l : dec;
  const uint64_t per_row = l > 0 ? std::max<uint64_t>(1, (uint64_t)ro[l] / l) : 1;
  // screening predicate, branch-free and vectorisable: a row is valid iff its
  // columns ascend strictly and its first / last column lie in [0, n)
  auto row_bad = [&](uint64_t i) {
    const int64_t b = ro[i], e = ro[i + 1];
    if (e <= b) return false;
    const int32_t* c = ci + b;
    const int64_t len = e - b;
    if (c[0] < 0 || static_cast<uint64_t>(c[len - 1]) >= n) return true;
    int viol = 0;
    for (int64_t k = 1; k < len; ++k) viol |= c[k] <= c[k - 1];
    return viol != 0;
  };
  const uint64_t bad = first_bad(lim, row_bad,
                                 std::max<size_t>(1, (size_t{1} << 16) / per_row));
  if (bad != UINT64_MAX) check_row(bad, true);
  if (dec != UINT64_MAX) check_row(dec, true);
}

// TRON_B200_TRACE=1: phase times of context creation on stderr.
struct PhaseTrace {
  bool on;
  cudaStream_t s = nullptr;
  std::chrono::steady_clock::time_point t0, last;
  explicit PhaseTrace(const char* what) {
    const char* e = std::getenv("TRON_B200_TRACE");
    on = e && e[0] == '1';
    t0 = last = std::chrono::steady_clock::now();
    if (on) std::fprintf(stderr, "[tron_b200] %s\n", what);
  }
  void mark(const char* phase) {
    nvtxMarkA(phase);
    if (!on) return;
    if (s) cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tron_b200]   %-28s %8.3f ms (total %8.3f)\n", phase,
                 std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

void check_options(int loss, const tron_gpu_options& opt) {
  if (loss != TRON_LOSS_LOGISTIC && loss != TRON_LOSS_L2SVM)
    raise(TRON_ERR_ARGUMENT, "unknown loss kind");
  if (opt.svm_strategy != TRON_SVM_GATHERED && opt.svm_strategy != TRON_SVM_INDIRECT &&
      opt.svm_strategy != TRON_SVM_AUTO)
    raise(TRON_ERR_DIMENSION, "plan: unknown svm strategy");
  if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world)
    raise(TRON_ERR_ARGUMENT, "invalid rank/world");
}

}  // namespace

void Engine::common_alloc() {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  prepare_device_pool(device_);
  cuda_check(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "cudaStreamCreate");
  stream_owner_.s = s_;
  alloc_stream() = s_;  // the creating entry holds an AllocScope
  sc_partials_.alloc(kMaxPartialBlocks * 4);
  sc_tickets_.alloc(kNumTickets);
  cuda_check(cudaMemsetAsync(sc_tickets_.p, 0, sc_tickets_.bytes(), s_), "memset");
  sc_.partials = sc_partials_.p;
  sc_.tickets = sc_tickets_.p;
  obj_buf_.alloc(1);
  st_buf_.alloc(1);
  obj_d_ = obj_buf_.p;
  st_d_ = st_buf_.p;
  ss_buf_.alloc(1);
  ss_h_ = static_cast<SolveState*>(pinned_block_get());
  cuda_check(cudaMemsetAsync(obj_d_, 0, sizeof(ObjScalars), s_), "memset");
  cuda_check(cudaMemsetAsync(st_d_, 0, sizeof(CgState), s_), "memset");
  static_assert(sizeof(ObjScalars) <= 256 && sizeof(CgState) <= 256, "pinned block size");
  obj_h_ = static_cast<ObjScalars*>(pinned_block_get());
  st_h_ = static_cast<CgState*>(pinned_block_get());

  const size_t nn = n_ > 0 ? n_ : 1;
  // dense passes stream whole 256-row tiles of every per-row array they
  // stage: pad to ld and zero the padding once
  const size_t ll = dense_ ? (size_t)std::max<int64_t>(ld_, 1) : (size_t)(l_ > 0 ? l_ : 1);
  for (auto& S : slot_) {
    S.w.alloc(nn);
    S.z.alloc(ll);
    if (loss_ == TRON_LOSS_LOGISTIC) {
      S.zhat.alloc(ll);
      S.dvec.alloc(ll);
      if (dense_) cuda_check(cudaMemsetAsync(S.dvec.p, 0, S.dvec.bytes(), s_), "memset");
    } else {
      S.mask.alloc(ll);
      if (dense_) cuda_check(cudaMemsetAsync(S.mask.p, 0, S.mask.bytes(), s_), "memset");
    }
    if (dense_) {
      S.gparts.alloc((size_t)dense_nparts() * nn);
      // streamed blocks: the slots a short last block leaves unused stay zero
      if (ooc_) cuda_check(cudaMemsetAsync(S.gparts.p, 0, S.gparts.bytes(), s_), "memset");
    }
  }
  for (DevBuf<double>* b : {&g_, &gspec_, &M_, &d_, &r0_, &r1_, &p_, &hp_, &vtmp_, &otmp_})
    b->alloc(nn);
  if (comm_.active()) raw_.alloc(nn);
  if (!dense_) a_.alloc(ll);
  if (dense_) {
    parts_.alloc((size_t)dense_nparts() * nn);
    if (ooc_) cuda_check(cudaMemsetAsync(parts_.p, 0, parts_.bytes(), s_), "memset");
  }
  small_engine_ = dense_ || n_ <= kSmallCgMaxN;
  coop_parts_.alloc((size_t)8 * cg_coop_grid());
  // mid-size n: one 8-CTA cluster kernel per CG iteration; larger n (or
  // TRON_B200_CLUSTER_CG=0): one cooperative grid kernel per iteration
  const char* cc = std::getenv("TRON_B200_CLUSTER_CG");
  mid_engine_ = !small_engine_ && n_ <= kClusterCgMaxN && !(cc && cc[0] == '0');
  coop_engine_ = !small_engine_ && !mid_engine_;
  // TRON_B200_NO_GRAPH=1 runs the CG loop host-driven (per-kernel profiling:
  // ncu cannot profile kernel nodes of graphs with conditional nodes).
  const char* ng = std::getenv("TRON_B200_NO_GRAPH");
  // Sharded: the NCCL allreduces are captured inside the CG while-graph (every
  // rank's CG state is identical, so every rank runs the same number of
  // allreduces); TRON_B200_NCCL_GRAPH=0 selects the host-driven CG loop.
  const char* cg = std::getenv("TRON_B200_NCCL_GRAPH");
  use_graphs_ = (!comm_.active() || !(cg && cg[0] == '0')) && !comm_.host() && !ooc_ && !colpart_ &&
                !(ng && ng[0] == '1');
}

// H2D of a buffer on a private stream ordered after everything issued on
// `main` so far (allocations included); wait() makes `main` wait for it.
struct ValueUpload {
  cudaStream_t main, side = nullptr;
  cudaEvent_t ev = nullptr;
  explicit ValueUpload(cudaStream_t m) : main(m) {}
  void start(void* dst, const void* src, size_t bytes) {
    cuda_check(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(ev, main), "event record");
    cuda_check(cudaStreamWaitEvent(side, ev, 0), "stream wait");
    upload(dst, src, bytes, side);
    cuda_check(cudaEventRecord(ev, side), "event record");
  }
  void wait() {
    if (side) cuda_check(cudaStreamWaitEvent(main, ev, 0), "stream wait");
  }
  ~ValueUpload() {
    if (side) {
      cudaStreamWaitEvent(main, ev, 0);  // never leave the copy unordered
      cudaStreamDestroy(side);
    }
    if (ev) cudaEventDestroy(ev);
  }
};

std::unique_ptr<Engine> Engine::create_csr(int loss, uint64_t l, uint64_t n, const int64_t* ro,
                                           const int32_t* ci, const double* vals, const double* y,
                                           double C, const tron_gpu_options& opt) {
  AllocScope scope(nullptr);
  PhaseTrace tr("create_csr");
  check_options(loss, opt);
  if (!ro || !y || (l > 0 && ro[l] > 0 && (!ci || !vals)))
    raise(TRON_ERR_ARGUMENT, "null problem array");
  // offsets first (they size the device arrays and bound the device screening)
  validate_offsets(l, ro);
  const int64_t nnz = ro[l];
  if (nnz >= (int64_t{1} << 31) || n >= (uint64_t{1} << 31) || l >= (uint64_t{1} << 31))
    raise(TRON_ERR_DIMENSION,
          "csr shard exceeds int32 indexing (nnz, rows, cols < 2^31 per GPU); shard across more "
          "GPUs");
  try {
    std::unique_ptr<Engine> e(new Engine());
    e->loss_ = loss;
    e->dense_ = false;
    e->l_ = (int64_t)l;
    e->n_ = (int64_t)n;
    e->C_ = C;
    e->device_ = opt.device;
    e->svm_strategy_ = opt.svm_strategy;
    e->budget_ = opt.gathered_budget_bytes;
    e->row_begin_ = opt.row_begin;
    e->comm_.init(opt);
    e->replica_check_ = env_flag("TRON_B200_CHECK_REPLICAS");
    if (opt.partition == TRON_PARTITION_COLUMNS && e->comm_.active()) {
      if (opt.global_cols < n || opt.col_begin + n > opt.global_cols)
        raise(TRON_ERR_ARGUMENT, "column partition: [col_begin, col_begin + n) must lie in global_cols");
      e->colpart_ = true;
      e->global_n_ = (int64_t)opt.global_cols;
      e->svm_strategy_ = TRON_SVM_INDIRECT;  // the gathered rows would need every column
    }
    e->common_alloc();
    cudaStream_t s = e->s_;
    tr.s = s;
    tr.mark("context + state alloc");
    if (e->colpart_) e->cp_dots_.alloc(4);

    e->rptr_.alloc(l + 1);
    // +4: the row kernels read whole aligned groups of four entries
    e->cidx_.alloc(nnz + 4);
    e->rval_.alloc(nnz + 4);
    e->cptr_.alloc(n + 1);
    // the CSC copy is padded to whole segmented chunks (zero entries of row 0),
    // so the chunk kernels read full chunks without bounds checks
    const int64_t nnz_pad = (nnz + kSegChunk - 1) / kSegChunk * kSegChunk;
    e->ridx_.alloc(std::max<int64_t>(nnz_pad, 1));
    e->cval_.alloc(std::max<int64_t>(nnz_pad, 1));
    e->y_.alloc(l > 0 ? l : 1);
    {
      DevBuf<int64_t> ro64;
      ro64.alloc(l + 1);
      upload(ro64.p, ro, (l + 1) * sizeof(int64_t), s);
      narrow_offsets(ro64.p, e->rptr_.p, (int64_t)(l + 1), s);
      if (nnz > 0) upload(e->cidx_.p, ci, nnz * sizeof(int32_t), s);
      if (l > 0) upload(e->y_.p, y, l * sizeof(double), s);
    }
    tr.mark("structure alloc + H2D issue");
    // O(nnz) column checks and the labels on the device; the host re-checks
    // the first offending row to raise the reference's exact error
    e->screen(e->rptr_.p, e->cidx_.p, (int64_t)l, (int64_t)n,
              [&](uint64_t bad_row, uint64_t bad_label) {
                if (bad_row != UINT64_MAX) validate_csr(l, n, ro, ci);  // raises the exact error
                if (bad_label != UINT64_MAX) validate_labels_C(l, y, C);
              });
    if (!(C > 0.0)) raise(TRON_ERR_DIMENSION, "problem: C must be positive");  // loss.cpp:30
    tr.mark("device validation");
    e->X_ = CsrView{(int64_t)l, (int64_t)n, nnz, e->rptr_.p, e->cidx_.p, e->rval_.p};
    int32_t* perm = nullptr;
    const int rc = build_csc_structure(e->X_, e->cptr_.p, e->ridx_.p, &perm, s);
    if (rc != 0) cuda_check((cudaError_t)rc, "build_csc_structure");
    // The values (2/3 of the bytes) go up on a second stream while the device
    // sorts the structure and builds the segmented plan; only the value
    // permutation waits for them.
    ValueUpload vup(s);
    if (nnz > 0) vup.start(e->rval_.p, vals, nnz * sizeof(double));
    if (nnz_pad > nnz) {
      cuda_check(cudaMemsetAsync(e->ridx_.p + nnz, 0, (nnz_pad - nnz) * sizeof(int32_t), s), "pad");
      cuda_check(cudaMemsetAsync(e->cval_.p + nnz, 0, (nnz_pad - nnz) * sizeof(double), s), "pad");
    }
    e->Xt_ = CsrView{(int64_t)n, (int64_t)l, nnz, e->cptr_.p, e->ridx_.p, e->cval_.p};
    if (loss == TRON_LOSS_L2SVM && opt.svm_strategy != TRON_SVM_INDIRECT) {
      e->idx_.alloc(l > 0 ? l : 1);
      e->idx_tmp_.alloc((l + 1023) / 1024 + 2);
      e->count_.alloc(1);
    }
    e->group_ = choose_group((int64_t)l, nnz);
    auto finish_values = [&] {
      vup.wait();
      const int vrc = build_csc_values(perm, e->rval_.p, e->cval_.p, nnz, s);
      perm = nullptr;
      if (vrc != 0) cuda_check((cudaError_t)vrc, "build_csc_values");
    };
    tr.mark("device CSC structure");
    {
      // one-time structure analysis of the CSC copy, on the device (csc_seg.cu)
      const int64_t nch = (nnz + kSegChunk - 1) / kSegChunk;
      e->chunk_rank_.alloc(std::max<int64_t>(nch, 1));
      e->lastbits_.alloc(nch * (kSegChunk / 32) + 2);
      e->nz_col_.alloc(n + 1);
      e->empty_col_.alloc(std::max<uint64_t>(n, 1));
      const int64_t slots = std::max<int64_t>(nch, 1);
      e->chunk_first_.alloc(slots);
      e->head_.alloc(slots);
      e->carry_.alloc(slots);
      e->long_fix_.alloc(seg_long_fix_cap(nch));
      const int prc = seg_plan_device(e->cptr_.p, (int64_t)n, nnz, &e->plan_, e->chunk_rank_.p,
                                      e->chunk_first_.p, e->lastbits_.p, e->nz_col_.p,
                                      e->empty_col_.p, e->long_fix_.p, s);
      if (prc != 0) cuda_check((cudaError_t)prc, "seg_plan_device");
      e->plan_.head = e->head_.p;
      e->plan_.carry = e->carry_.p;
      {  // p.Hp / ||g|| summed as the transposed product (or its epilogue) emits
        e->dot_parts_.alloc(seg_dot_slots(nch));
        e->dot_out_.alloc(1);
        e->dot_ticket_.alloc(1);
        cuda_check(cudaMemsetAsync(e->dot_ticket_.p, 0, sizeof(unsigned), s), "memset");
      }
      tr.mark("segmented plan");
    }
    e->setup_panels();
    // The CG graphs of both slots (no preconditioner) are captured and
    // instantiated while the values are still crossing PCIe: a recipe of
    // fixed buffers, independent of their contents.
    if (e->use_graphs_ && nnz > 0 && n > 0) {
      if (e->device_loop_ok()) {
        e->build_solve_graph(false);
      } else {
        e->build_graph(0, false);
        e->build_graph(1, false);
      }
      tr.mark("solve / CG graphs");
    }
    finish_values();
    tr.mark("values H2D + CSC values");
    cuda_check(cudaStreamSynchronize(s), "csc build");
    cuda_check(cudaGetLastError(), "csc build");
    return e;
  } catch (const StatusError& err) {
    // no usable device: the inputs are still checked, and an input error
    // outranks the device error (the reference has no device to fail)
    if (err.status == TRON_ERR_CUDA || err.status == TRON_ERR_OOM) {
      validate_csr(l, n, ro, ci);
      validate_labels_C(l, y, C);
    }
    throw;
  }
}

std::unique_ptr<Engine> Engine::create_dense(int loss, uint64_t l, uint64_t n,
                                             const double* row_major, const double* y, double C,
                                             const tron_gpu_options& opt) {
  AllocScope scope(nullptr);
  PhaseTrace tr("create_dense");
  check_options(loss, opt);
  if (!y || (l * n > 0 && !row_major)) raise(TRON_ERR_ARGUMENT, "null problem array");
  if (n > (uint64_t)kDenseMaxN) {
    // Wide dense problems run through the sparse kernels (explicit entries).
    std::vector<int64_t> ro(l + 1);
    std::vector<int32_t> ci(l * n);
    for (uint64_t i = 0; i <= l; ++i) ro[i] = (int64_t)(i * n);
    for (uint64_t i = 0; i < l; ++i)
      for (uint64_t j = 0; j < n; ++j) ci[i * n + j] = (int32_t)j;
    return create_csr(loss, l, n, ro.data(), ci.data(), row_major, y, C, opt);
  }
  if (l >= (uint64_t{1} << 31)) raise(TRON_ERR_DIMENSION, "dense shard exceeds 2^31 rows per GPU");
  if (opt.partition == TRON_PARTITION_COLUMNS && opt.world > 1)
    raise(TRON_ERR_ARGUMENT, "the column-partitioned layout is for sparse problems (dense n <= 64)");
  if (opt.reference_order) {
    if (loss != TRON_LOSS_L2SVM || n > (uint64_t)kRoMaxN || opt.world > 1)
      raise(TRON_ERR_ARGUMENT,
            "reference_order needs a dense L2-SVM with n <= 48 features on one GPU");
    if (opt.svm_strategy == TRON_SVM_GATHERED)
      raise(TRON_ERR_STRATEGY,
            "reference_order runs the Indirect traversal (the reference's Gathered route is "
            "bitwise equal to it, loss.cpp:160-162); use Indirect");
  }
  std::unique_ptr<Engine> e(new Engine());
  e->ro_ = opt.reference_order != 0;
  const int svm_strategy = e->ro_ ? (int)TRON_SVM_INDIRECT : opt.svm_strategy;
  e->loss_ = loss;
  e->dense_ = true;
  e->l_ = (int64_t)l;
  e->n_ = (int64_t)n;
  e->C_ = C;
  e->device_ = opt.device;
  e->svm_strategy_ = svm_strategy;
  e->budget_ = opt.gathered_budget_bytes;
  e->row_begin_ = opt.row_begin;
  e->comm_.init(opt);
  e->replica_check_ = env_flag("TRON_B200_CHECK_REPLICAS");
  e->ld_ = dense_ld((int64_t)l);
  {  // out-of-core streaming when X does not fit (or when asked to)
    // (no usable device: decided as in-memory; creation then reports the
    // device error after the input checks, below)
    size_t free_b = 0, total_b = 0;
    const bool have = cudaSetDevice(opt.device) == cudaSuccess &&
                      cudaMemGetInfo(&free_b, &total_b) == cudaSuccess;
    if (!have) {
      cudaGetLastError();
    } else {
      // blocks an earlier context returned to the stream-ordered pool are free
      // for this one, though the driver still counts them as used
      cudaMemPool_t pool;
      cuuint64_t reserved = 0, used = 0;
      if (cudaDeviceGetDefaultMemPool(&pool, opt.device) == cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
          reserved > used)
        free_b += (size_t)(reserved - used);
      cudaGetLastError();
    }
    const double xbytes = 8.0 * (double)e->ld_ * (double)n;
    const double state = (double)e->ld_ * (loss == TRON_LOSS_LOGISTIC ? 56.0 : 26.0);
    const bool want = opt.out_of_core > 0 ||
                      (opt.out_of_core == 0 && have &&
                       xbytes + state + double(2ull << 30) > (double)free_b);
    if (want && l > 0 && n > 0) {
      if (opt.world > 1) raise(TRON_ERR_ARGUMENT, "out-of-core streaming runs on one GPU");
      if (opt.reference_order) raise(TRON_ERR_ARGUMENT, "reference_order needs X in device memory");
      if (loss == TRON_LOSS_L2SVM && opt.svm_strategy == TRON_SVM_GATHERED)
        raise(TRON_ERR_STRATEGY,
              "the gathered submatrix needs X in device memory; out-of-core streaming answers "
              "Hessian products by index-indirect traversal (the mix backend's route)");
      e->ooc_ = true;
      e->svm_strategy_ = TRON_SVM_INDIRECT;
      int64_t b = opt.stream_block_rows > 0
                      ? (int64_t)opt.stream_block_rows
                      : std::max<int64_t>(kDenseTile, (int64_t{256} << 20) / (int64_t)(8 * n));
      b = std::min<int64_t>(dense_ld(b), e->ld_);
      e->blk_ = b;
      e->nblk_ = ((int64_t)l + b - 1) / b;
      e->Xhost_ = row_major;
    }
  }
  // labels are checked on the worker pool while the matrix streams in
  try {
    e->common_alloc();
    cudaStream_t s = e->s_;
    tr.s = s;
    tr.mark("context + state alloc");
    if (e->ooc_) {
      e->y_.alloc((size_t)std::max<int64_t>(e->ld_, 1));
      cuda_check(cudaMemsetAsync(e->y_.p, 0, e->y_.bytes(), s), "memset");
      upload(e->y_.p, y, l * sizeof(double), s);
      e->ooc_setup();
      tr.mark("out-of-core windows + host registration");
    } else {
    e->Xc_.alloc((size_t)std::max<int64_t>(e->ld_, 1) * (n > 0 ? n : 1));
    e->y_.alloc((size_t)std::max<int64_t>(e->ld_, 1));
    cuda_check(cudaMemsetAsync(e->y_.p, 0, e->y_.bytes(), s), "memset");
    if (n > 0 && e->ld_ > (int64_t)l)
      cuda_check(cudaMemset2DAsync(e->Xc_.p + l, e->ld_ * sizeof(double), 0,
                                   (e->ld_ - (int64_t)l) * sizeof(double), n, s),
                 "memset pad");
    if (l > 0) {
      upload(e->y_.p, y, l * sizeof(double), s);
      // chunked row-major upload + on-device transpose to column-major
      const int64_t chunk_rows =
          std::max<int64_t>(1, (int64_t{64} << 20) / (int64_t)(sizeof(double) * std::max<uint64_t>(n, 1)));
      DevBuf<double> stage[2];
      stage[0].alloc((size_t)chunk_rows * n);
      stage[1].alloc((size_t)chunk_rows * n);
      cudaEvent_t ev[2];
      cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
      int k = 0;
      bool used[2] = {false, false};
      for (int64_t r0 = 0; r0 < (int64_t)l; r0 += chunk_rows, k ^= 1) {
        const int64_t rows = std::min<int64_t>(chunk_rows, (int64_t)l - r0);
        if (used[k]) cudaEventSynchronize(ev[k]);
        upload(stage[k].p, row_major + (size_t)r0 * n, rows * n * sizeof(double), s);
        dense_transpose_chunk(stage[k].p, rows, n, e->Xc_.p, e->ld_, r0, s);
        cudaEventRecord(ev[k], s);
        used[k] = true;
      }
      cuda_check(cudaStreamSynchronize(s), "dense upload");
      cudaEventDestroy(ev[0]);
      cudaEventDestroy(ev[1]);
    }
    tr.mark("matrix alloc + H2D + transpose");
    }
    e->screen(nullptr, nullptr, 0, (int64_t)n, [&](uint64_t, uint64_t bad_label) {
      if (bad_label != UINT64_MAX) validate_labels_C(l, y, C);  // raises the exact error
    });
    if (!(C > 0.0)) raise(TRON_ERR_DIMENSION, "problem: C must be positive");  // loss.cpp:30
    tr.mark("device validation");
  } catch (const StatusError& err) {
    if (err.status == TRON_ERR_CUDA || err.status == TRON_ERR_OOM) validate_labels_C(l, y, C);
    throw;
  }
  if (!e->ooc_ && dense_make_map(&e->xmap_, e->Xc_.p, e->ld_, (int64_t)l, (int64_t)n) != 0)
    raise(TRON_ERR_CUDA, "cuTensorMapEncodeTiled failed for the dense matrix");
  if (loss == TRON_LOSS_L2SVM) {
    e->idx_.alloc(l > 0 ? l : 1);
    e->idx_tmp_.alloc((l + 1023) / 1024 + 2);
    e->count_.alloc(1);
  }
  {  // Gram mode (TRON_B200_DENSE_GRAM=0 keeps the tall-skinny passes)
    const char* gm = std::getenv("TRON_B200_DENSE_GRAM");
    const bool off = gm && gm[0] == '0';
    if (!off && !e->ro_ && !e->ooc_ && n > 0 && n <= (uint64_t)kDenseMaxN &&
        !(loss == TRON_LOSS_L2SVM && e->svm_strategy_ == TRON_SVM_GATHERED)) {
      AllocScope scope(e->s_);
      e->gram_ = true;
      if (e->svm_strategy_ == TRON_SVM_AUTO) e->svm_strategy_ = TRON_SVM_INDIRECT;  // G is compact already
      // TRON_B200_GRAM_FUSED=1: G accumulated by the margin pass itself.  Measured
      // slower (P1: 2.95 ms fused vs 1.17 + 1.63 ms separate): one 9-warp CTA per
      // SM alternates the row phase and the DMMA phase, where the separate Gram
      // kernel keeps 16 warps per SM on the FP64 tensor pipe.
      const char* gf = std::getenv("TRON_B200_GRAM_FUSED");
      e->gram_fused_ = dense_forward_gram_fused((int64_t)n) && gf && gf[0] == '1';
      // L2-SVM: the candidate's G from the committed slot's and the rows that
      // changed side, accumulated by the margin pass (TRON_B200_GRAM_DELTA=0: a
      // fresh Gram pass per commit)
      // the CG of a Gram-mode context in one launch (TRON_B200_GRAM_CG_LOOP=0:
      // one launch per iteration)
      const char* gl = std::getenv("TRON_B200_GRAM_CG_LOOP");
      e->gram_cg_loop_ = !(gl && gl[0] == '0');
      const char* gd = std::getenv("TRON_B200_GRAM_DELTA");
      e->gram_delta_ = loss == TRON_LOSS_L2SVM && !e->gram_fused_ && dense_forward_gram_delta((int64_t)n) &&
                       !(gd && gd[0] == '0');
      // a solve's starting point: its margin pass forms the whole G as well
      // (TRON_B200_GRAM_FIRST=separate: a plain margin pass, then the Gram pass)
      const char* gfirst = std::getenv("TRON_B200_GRAM_FIRST");
      e->gram_first_fused_ = e->gram_delta_ && !(gfirst && std::string(gfirst) == "separate");
      static const int kFlagsInit[4] = {1, 0, 0, 0};  // no slot's G is current yet
      for (auto& S : e->slot_) {
        S.gram.alloc((size_t)n * n);
        if (e->comm_.active()) S.gram_local.alloc((size_t)n * n);
        S.gram_flags.alloc(4);
        cuda_check(cudaMemcpyAsync(S.gram_flags.p, kFlagsInit, sizeof(kFlagsInit), cudaMemcpyHostToDevice, e->s_),
                   "H2D");
        if (e->gram_fused_) S.gram_parts.alloc((size_t)dense_grid((int64_t)l, (int64_t)n) * n * n);
        if (e->gram_delta_) S.gram_dparts.alloc((size_t)dense_grid((int64_t)l, (int64_t)n) * n * n);
      }
      if (!e->gram_fused_) e->gram_parts_.alloc((size_t)gram_grid((int64_t)l, (int64_t)n) * n * n);
      cuda_check(cudaStreamSynchronize(e->s_), "gram buffers");
    }
  }
  if (e->ro_) {
    AllocScope scope(e->s_);
    if (dense_make_map_box(&e->xmap128_, e->Xc_.p, e->ld_, (int64_t)l, (int64_t)n, 128) != 0)
      raise(TRON_ERR_CUDA, "cuTensorMapEncodeTiled failed for the dense matrix (128-row boxes)");
    for (auto& S : e->slot_) {
      S.idx.alloc(l > 0 ? l : 1);
      S.cnt.alloc(1);
      cuda_check(cudaMemsetAsync(S.cnt.p, 0, sizeof(long long), e->s_), "memset");
    }
    e->ro_parts_.alloc((size_t)64 * std::max<uint64_t>(n, 1));
    e->ro_hparts_.alloc(64);
    e->ro_tickets_.alloc(2);
    cuda_check(cudaMemsetAsync(e->ro_tickets_.p, 0, 2 * sizeof(unsigned), e->s_), "memset");
    cuda_check(cudaStreamSynchronize(e->s_), "reference-order buffers");
  }
  cuda_check(cudaGetLastError(), "dense create");
  return e;
}

Engine::~Engine() {
  if (s_) cudaStreamSynchronize(s_);
  if (cs_) {
    cudaStreamSynchronize(cs_);
    cudaStreamDestroy(cs_);
  }
  for (cudaEvent_t ev : {ev_copied_[0], ev_copied_[1], ev_free_[0], ev_free_[1]})
    if (ev) cudaEventDestroy(ev);
  if (host_registered_) cudaHostUnregister(const_cast<double*>(Xhost_));
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      if (graph_exec_[a][b]) cudaGraphExecDestroy(graph_exec_[a][b]);
      if (graph_[a][b]) cudaGraphDestroy(graph_[a][b]);
    }
  for (int b = 0; b < 2; ++b) {
    if (solve_exec_[b]) cudaGraphExecDestroy(solve_exec_[b]);
    if (solve_graph_[b]) cudaGraphDestroy(solve_graph_[b]);
  }
  pinned_block_put(obj_h_);
  pinned_block_put(st_h_);
  pinned_block_put(ss_h_);
  // DevBuf members queue their frees on s_; stream_owner_ then syncs + destroys it
}

// Device screening of the uploaded inputs (screen_inputs); on a hit, report()
// re-runs the host check that raises the exact error.
template <class Report>
void Engine::screen(const int32_t* ptr, const int32_t* idx, int64_t rows, int64_t n, Report report) {
  DevBuf<unsigned long long> flags;
  flags.alloc(2);
  screen_inputs(ptr, idx, rows, n, y_.p, l_, flags.p, s_);
  unsigned long long h[2];
  cuda_check(cudaMemcpyAsync(h, flags.p, sizeof(h), cudaMemcpyDeviceToHost, s_), "D2H");
  synchronize();
  if (h[0] != ~0ull || h[1] != ~0ull) report((uint64_t)h[0], (uint64_t)h[1]);
}

uint32_t Engine::mode_flags() const {
  return (gram_ ? TRON_MODE_GRAM : 0) | (ooc_ ? TRON_MODE_OUT_OF_CORE : 0) |
         (colpart_ ? TRON_MODE_COLUMNS : 0) | (device_loop_ok() ? TRON_MODE_DEVICE_LOOP : 0) |
         (comm_.active() && !colpart_ ? TRON_MODE_SHARDED : 0) | (gram_delta_ ? TRON_MODE_GRAM_DELTA : 0);
}

uint64_t Engine::memory_bytes() const {
  uint64_t b = grptr_.bytes() + gcidx_.bytes() + grval_.bytes() + gcptr_.bytes() + gridx_.bytes() +
               gcval_.bytes();
  b += rptr_.bytes() + cidx_.bytes() + rval_.bytes() + cptr_.bytes() + ridx_.bytes() +
               cval_.bytes() + Xc_.bytes() + Xg_.bytes() + y_.bytes() + lastbits_.bytes() +
               chunk_rank_.bytes() + empty_col_.bytes() + chunk_first_.bytes() + nz_col_.bytes() + head_.bytes() + carry_.bytes();
  for (const auto& S : slot_)
    b += S.w.bytes() + S.z.bytes() + S.zhat.bytes() + S.dvec.bytes() + S.mask.bytes() +
         S.gparts.bytes();
  b += g_.bytes() * 10 + a_.bytes() + parts_.bytes();
  return b;
}

void Engine::synchronize() { cuda_check(cudaStreamSynchronize(s_), "synchronize"); }

// The scalars are only trusted after a clean launch record: a failed launch
// would leave them at their previous values.
void Engine::read_obj() {
  cuda_check(cudaMemcpyAsync(obj_h_, obj_d_, sizeof(ObjScalars), cudaMemcpyDeviceToHost, s_),
             "D2H");
  cuda_check(cudaStreamSynchronize(s_), "sync");
  cuda_check(cudaGetLastError(), "kernel launch");
}

void Engine::read_cg(CgState* out) {
  cuda_check(cudaMemcpyAsync(st_h_, st_d_, sizeof(CgState), cudaMemcpyDeviceToHost, s_), "D2H");
  cuda_check(cudaStreamSynchronize(s_), "sync");
  cuda_check(cudaGetLastError(), "kernel launch");
  *out = *st_h_;
}

// ----------------------------------------------------------------------------
// out-of-core dense streaming
// ----------------------------------------------------------------------------
int Engine::dense_nparts() const {
  return ooc_ ? (int)(nblk_ * dense_grid(blk_, n_)) : dense_grid(l_, n_);
}

// Two device windows (column-major, ld = blk_) and two row-major staging
// buffers; the caller's array is page-locked in place so every block is one
// DMA (cudaHostRegister; if that fails the pageable staging path is used).
void Engine::ooc_setup() {
  for (int k = 0; k < 2; ++k) {
    win_[k].alloc((size_t)blk_ * n_);
    stage_[k].alloc((size_t)blk_ * n_);
    cuda_check(cudaMemsetAsync(win_[k].p, 0, win_[k].bytes(), s_), "memset");
    if (dense_make_map(&winmap_[k], win_[k].p, blk_, blk_, n_) != 0)
      raise(TRON_ERR_CUDA, "cuTensorMapEncodeTiled failed for a streaming window");
    cuda_check(cudaEventCreateWithFlags(&ev_copied_[k], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_free_[k], cudaEventDisableTiming), "event");
  }
  cuda_check(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking), "stream");
  blk_red_.alloc((size_t)2 * nblk_);
  const char* pin = std::getenv("TRON_B200_OOC_PIN");  // 0: staged copies (tests the pageable path)
  if (!is_pinned(Xhost_) && !(pin && pin[0] == '0')) {
    const cudaError_t e = cudaHostRegister(const_cast<double*>(Xhost_), (size_t)l_ * n_ * sizeof(double),
                                           cudaHostRegisterReadOnly);
    if (e == cudaSuccess)
      host_registered_ = true;
    else
      cudaGetLastError();  // staged copies instead
  }
}

// Runs on_block(b, row0, rows, window, map) for every block, the H2D of block
// b+1 on cs_ overlapping the kernels of block b on s_.  A window is reused
// only after the kernels that read it (ev_free_), and the rows of a short
// last block past its end are zeroed (the tiled passes read whole tiles).
template <class F>
void Engine::ooc_pass(F&& on_block) {
  for (int64_t b = 0; b < nblk_; ++b) {
    const int k = (int)(b & 1);
    const int64_t r0 = b * blk_;
    const int64_t rows = std::min<int64_t>(blk_, l_ - r0);
    if (ev_free_used_[k]) cuda_check(cudaStreamWaitEvent(cs_, ev_free_[k], 0), "wait");
    upload(stage_[k].p, Xhost_ + (size_t)r0 * n_, (size_t)rows * n_ * sizeof(double), cs_);
    cuda_check(cudaEventRecord(ev_copied_[k], cs_), "record");
    cuda_check(cudaStreamWaitEvent(s_, ev_copied_[k], 0), "wait");
    const int64_t rows_pad = dense_ld(rows);
    if (rows_pad > rows)
      cuda_check(cudaMemset2DAsync(win_[k].p + rows, blk_ * sizeof(double), 0,
                                   (rows_pad - rows) * sizeof(double), n_, s_),
                 "memset");
    dense_transpose_chunk(stage_[k].p, rows, n_, win_[k].p, blk_, 0, s_);
    on_block(b, r0, rows, (const double*)win_[k].p, (const CUtensorMap&)winmap_[k]);
    count_launch(2);
    cuda_check(cudaEventRecord(ev_free_[k], s_), "record");
    ev_free_used_[k] = true;
  }
}

namespace {
template <class T>
T* off(T* p, int64_t r0) {
  return p ? p + r0 : nullptr;
}
}  // namespace

// ----------------------------------------------------------------------------
// fun: fused margin pass (loss.cpp:35-58 / :94-122)
// ----------------------------------------------------------------------------
void Engine::forward(Slot& S) {
  const int loss = loss_ == TRON_LOSS_LOGISTIC ? kLossLogistic : kLossSvm;
  if (dense_ && ooc_) {
    const int64_t G = dense_grid(blk_, n_);
    ooc_pass([&](int64_t b, int64_t r0, int64_t rows, const double* win, const CUtensorMap& map) {
      dense_forward(rows, n_, blk_, win, map, loss, S.w.p, y_.p + r0, C_, S.z.p + r0, off(S.zhat.p, r0),
                    off(S.dvec.p, r0), off(S.mask.p, r0), S.gparts.p + b * G * n_, obj_d_, sc_, s_);
      cuda_check(cudaMemcpyAsync(blk_red_.p + 2 * b, obj_d_->red, 2 * sizeof(double),
                                 cudaMemcpyDeviceToDevice, s_),
                 "D2D");
    });
    obj_combine_blocks(obj_d_, blk_red_.p, nblk_, C_, s_);
  } else if (dense_) {
    // the other slot: the committed iterate whose G the candidate's updates
    const Slot& R = &S == &slot_[0] ? slot_[1] : slot_[0];
    const bool shard = comm_.active();
    // delta mode, a solve's starting point: G formed whole by this pass (PM_FWDG)
    const bool whole = gram_delta_ && gram_full_next_;
    gram_full_next_ = false;
    const bool upd = gram_delta_ && !whole;  // PM_FWDD against R
    dense_forward(l_, n_, ld_, Xc_.p, xmap_, loss, S.w.p, y_.p, C_, S.z.p, S.zhat.p, S.dvec.p, S.mask.p,
                  S.gparts.p, obj_d_, sc_, s_,
                  gram_fused_ ? S.gram_parts.p : gram_delta_ ? S.gram_dparts.p : nullptr,
                  upd ? R.mask.p : nullptr, upd ? R.gram_flags.p : nullptr);
    if (whole) {
      cuda_check(cudaMemsetAsync(S.gram_flags.p, 0xff, sizeof(int), s_), "memset");
      gram_finalize(n_, S.gram_dparts.p, dense_grid(l_, n_), shard ? S.gram_local.p : S.gram.p, s_,
                    S.gram_flags.p);
      count_launch(1);
    } else if (upd) {  // G of this slot = G of R + the change (or flagged stale)
      gram_delta_finalize(n_, S.gram_dparts.p, dense_grid(l_, n_), shard ? R.gram_local.p : R.gram.p,
                          R.gram_flags.p, shard ? S.gram_local.p : S.gram.p, S.gram_flags.p, s_);
      count_launch(1);
    } else if (gram_ && !gram_fused_) {  // formed when first needed (ensure_gram)
      cuda_check(cudaMemsetAsync(S.gram_flags.p, 0xff, sizeof(int), s_), "memset");
    }
    if (ro_) {  // I of this slot, then f in the reference's order (loss.cpp:114-119)
      compact_mask(l_, S.mask.p, S.idx.p, idx_tmp_.p, S.cnt.p, s_);
      ro_hinge(l_, n_, S.z.p, y_.p, S.w.p, C_, ro_hparts_.p, ro_tickets_.p, obj_d_, s_);
      count_launch(4);
    }
  } else if (colpart_) {
    // z = sum over ranks of X_{:,r} w_r (one l-length exchange), w.w likewise;
    // then the fused epilogue over the whole z: an empty row range per row
    csr_dv(X_, group_, S.w.p, nullptr, nullptr, S.z.p, s_);
    comm_.allreduce_sum(S.z.p, (size_t)l_, s_);
    comm_.allreduce_sum(&obj_d_->ww, 1, s_);
    CsrView E = X_;
    E.rbeg = E.rend = X_.ptr + 1;
    csr_forward(E, 1, loss, S.w.p, y_.p, C_, S.z.p, S.zhat.p, S.dvec.p, S.mask.p, obj_d_, sc_, s_, S.z.p);
    count_launch(1);
  } else if (!panels_.empty()) {  // raw row sums of the leading panels, then the fused pass
    const size_t K = panels_.size();
    for (size_t k = 0; k + 1 < K; ++k)
      csr_dv(panels_[k], panel_group_[k], S.w.p, nullptr, nullptr, S.z.p, s_, k ? S.z.p : nullptr, false);
    count_launch(K - 1);
    csr_forward(panels_[K - 1], panel_group_[K - 1], loss, S.w.p, y_.p, C_, S.z.p, S.zhat.p, S.dvec.p,
                S.mask.p, obj_d_, sc_, s_, S.z.p);
  } else {
    csr_forward(X_, group_, loss, S.w.p, y_.p, C_, S.z.p, S.zhat.p, S.dvec.p, S.mask.p, obj_d_, sc_,
                s_);
  }
  count_launch(1);
}

void Engine::replica_checksum_host(double out4[4]) {
  if (!rc_.p) {
    AllocScope scope(s_);
    rc_.alloc(8);
  }
  replica_checksum(n_, slot_[cand_ ^ 1].w.p, 0.0, 0.0, rc_.p, s_);
  double h[8];
  cuda_check(cudaMemcpyAsync(h, rc_.p, sizeof(h), cudaMemcpyDeviceToHost, s_), "D2H");
  cuda_check(cudaStreamSynchronize(s_), "sync");
  for (int c = 0; c < 4; ++c) out4[c] = h[c];
}

// Replicated state must be bitwise identical on every rank: a
// checksum of w (committed), f and delta summed over the ranks with its
// squares; "all equal" <=> world * sum(h^2) == sum(h)^2 for each 16-bit chunk
// (exact in doubles), which every rank evaluates on the same sums.
void Engine::check_replicas(double f, double delta, uint64_t iter) {
  if (!replica_check_ || !comm_.active() || colpart_) return;  // (column shards hold different w)
  if (!rc_.p) {
    AllocScope scope(s_);
    rc_.alloc(8);
  }
  replica_checksum(n_, slot_[cand_ ^ 1].w.p, f, delta, rc_.p, s_);
  comm_.allreduce_sum(rc_.p, 8, s_);
  double h[8];
  cuda_check(cudaMemcpyAsync(h, rc_.p, sizeof(h), cudaMemcpyDeviceToHost, s_), "D2H");
  cuda_check(cudaStreamSynchronize(s_), "sync");
  for (int c = 0; c < 4; ++c)
    if ((double)comm_.world * h[4 + c] != h[c] * h[c])
      raise(TRON_ERR_LOGIC, "replicas diverged: the ranks' w / f / delta differ after outer iteration " +
                                std::to_string(iter));
}

double Engine::eval_candidate_dev(const double* d_step, bool read) {
  Slot& S = slot_[cand_];
  const Slot& W = slot_[cand_ ^ 1];
  if (d_step) {
    vec_axpy_dot(n_, W.w.p, d_step, S.w.p, obj_d_, sc_, s_);
    count_launch(1);
  } else if (!dense_) {
    vec_axpy_dot(n_, S.w.p, nullptr, S.w.p, obj_d_, sc_, s_);
    count_launch(1);
  }
  forward(S);
  // per-shard loss sums, |I| (the column layout's are whole already)
  if (comm_.active() && !colpart_) comm_.allreduce_sum(obj_d_->red, 2, s_);
  if (!read) return 0.0;
  read_obj();
  return candidate_result();
}

// Bookkeeping of a candidate whose scalars have been read into obj_h_.
double Engine::candidate_result() {
  Slot& S = slot_[cand_];
  double f = obj_h_->f;
  long long nact = obj_h_->nact;
  if (comm_.active()) {
    f = 0.5 * obj_h_->ww + C_ * obj_h_->red[0];  // loss.cpp:57 over the global sum
    nact = (long long)obj_h_->red[1];
  }
  S.f = f;
  S.nact = obj_h_->nact;
  S.valid = true;
  ledger.margin_passes++;
  ledger.scalar_returns++;
  if (loss_ == TRON_LOSS_L2SVM)
    ledger.index_set_bytes = std::max<uint64_t>(ledger.index_set_bytes, (uint64_t)nact * 8);
  return f;
}

double Engine::eval_candidate_host(const double* w) {
  if (n_ > 0)
    upload(slot_[cand_].w.p, w, n_ * sizeof(double), s_);
  return eval_candidate_dev(nullptr);
}

// ----------------------------------------------------------------------------
// transposed products: X^T u with epilogue, world-aware
// ----------------------------------------------------------------------------
void Engine::transposed_raw_or_epi(const UView& u, bool squared, const EpiView& epi, double* out,
                                   const CsrView* At, const SegView* plan) {
  const CsrView& T = At ? *At : Xt_;
  const SegView& P = plan ? *plan : plan_;
  auto product = [&](const EpiView& E, double* dst) {
    csc_spmv(T, P, u, squared, E, dst, s_);
    count_launch(2);
  };
  if (!comm_.active() || colpart_) {  // the column layout's X_{:,r}^T u is this rank's slice
    product(epi, out);
    return;
  }
  EpiView raw;
  raw.kind = EPI_RAW;
  product(raw, raw_.p);
  comm_.allreduce_sum(raw_.p, n_, s_);
  vec_epilogue(n_, raw_.p, epi, out, s_);
  count_launch(1);
}

// kind = DA_HV / DA_PRECOND (one tiled pass) or -1: finish the gradient
// partials the committed slot's margin pass already accumulated.
void Engine::dense_vector(int kind, const double* v, const EpiView& epi, double* out,
                          const Slot* grad_slot) {
  const Slot& S = grad_slot ? *grad_slot : slot_[cand_ ^ 1];
  const int loss = loss_ == TRON_LOSS_LOGISTIC ? kLossLogistic : kLossSvm;
  const bool gathered = kind == DA_HV && gathered_valid_;
  const double* parts = parts_.p;
  int nparts = gathered ? dense_grid(nI_, n_) : dense_nparts();
  if (kind < 0) {
    parts = S.gparts.p;
    nparts = dense_nparts();
  } else if (ooc_) {
    const int64_t G = dense_grid(blk_, n_);
    ooc_pass([&](int64_t b, int64_t r0, int64_t rows, const double* win, const CUtensorMap& map) {
      dense_accum(kind, rows, n_, blk_, win, map, loss, v, off(S.dvec.p, r0), off(S.mask.p, r0),
                  parts_.p + b * G * n_, s_);
    });
  } else if (gathered) {
    dense_accum(DA_HV, nI_, n_, ldg_, Xg_.p, gmap_, kLossSvm, v, nullptr, nullptr, parts_.p, s_);
    count_launch(1);
  } else {
    dense_accum(kind, l_, n_, ld_, Xc_.p, xmap_, loss, v, S.dvec.p, S.mask.p, parts_.p, s_);
    count_launch(1);
  }
  if (!comm_.active()) {
    dense_finalize(n_, parts, nparts, epi, out, s_);
    count_launch(1);
    return;
  }
  EpiView raw;
  raw.kind = EPI_RAW;
  dense_finalize(n_, parts, nparts, raw, raw_.p, s_);
  comm_.allreduce_sum(raw_.p, n_, s_);
  vec_epilogue(n_, raw_.p, epi, out, s_);
  count_launch(2);
}

// ----------------------------------------------------------------------------
// commit + gradient (backend.cpp:165-183 / :249-277; loss.cpp:74-80 / :129-137)
// ----------------------------------------------------------------------------
void Engine::gradient_dev() { gradient_into(slot_[cand_ ^ 1], g_.p); }

// g = w + C X^T zhat (LR) / w + 2C X_I^T (z - y)_I (SVM) of slot S into out,
// then ||out|| and its finiteness into obj (loss.cpp:74-80, :129-137).
void Engine::gradient_into(const Slot& S, double* out) {
  EpiView epi;
  epi.kind = EPI_VEC;
  epi.base = S.w.p;
  epi.scale = loss_ == TRON_LOSS_LOGISTIC ? C_ : 2.0 * C_;
  if (ro_) {  // masked_matvec_transpose in the reference's order, norm2(g) serial
    ro_accum_slot(RO_GRAD, S, nullptr, epi, out);
    return;
  }
  if (dense_) {
    dense_vector(-1, nullptr, epi, out, &S);  // partials from the fused margin pass
    // (gram mode: the margin pass left this slot's G current or flagged stale)
    if (gram_fused_) gram_slot(S);  // (the fused pass's partials are already there)
  } else {
    UView u;
    if (loss_ == TRON_LOSS_LOGISTIC) {
      u.kind = U_VEC;
      u.u = S.zhat.p;
    } else {
      u.kind = U_SVM_RESID;
      u.mask = S.mask.p;
      u.z = S.z.p;
      u.y = y_.p;
    }
    if (colpart_) {  // ||g||^2 = sum over ranks of the slices' sums of squares
      transposed_raw_or_epi(u, false, epi, out);
      vec_sumsq_bad(n_, out, cp_dots_.p, sc_, s_);
      comm_.allreduce_sum(cp_dots_.p, 2, s_);
      obj_set_gnorm(obj_d_, cp_dots_.p, s_);
      count_launch(3);
      return;
    }
    if (hv_dot_available()) {  // ||g|| and the finiteness check from the emission
      epi.dot_parts = dot_parts_.p;
      epi.dot_ticket = dot_ticket_.p;
      epi.dot_mode = 1;
      epi.dot_obj = obj_d_;
      transposed_raw_or_epi(u, false, epi, out);
      return;
    }
    transposed_raw_or_epi(u, false, epi, out);
  }
  vec_norm_check(n_, out, obj_d_, sc_, s_);
  count_launch(1);
}

int Engine::compact(const Slot& S, DevBuf<int32_t>& idx) {
  compact_mask(l_, S.mask.p, idx.p, idx_tmp_.p, count_.p, s_);
  count_launch(3);
  long long cnt = 0;
  cuda_check(cudaMemcpyAsync(&cnt, count_.p, sizeof(cnt), cudaMemcpyDeviceToHost, s_), "D2H");
  synchronize();
  return (int)cnt;
}

namespace {
std::string budget_message(uint64_t projected, uint64_t budget) {  // error.hpp:54-62
  return "gathered submatrix would need " + std::to_string(projected) + " bytes, exceeding the " +
         std::to_string(budget) +
         "-byte budget; use the mix backend (MixedActiveSet), which answers Hessian products by "
         "index-indirect traversal instead";
}
// TRON_SVM_AUTO gathers when the active rows hold at most this share of X:
// a gather costs about 3 passes over X_I (CSR: the copy plus the CSC sort),
// and each of the ~8 Hessian products of a commit then reads X_I instead of
// X -- it pays below ~2/3 (CSR) to ~3/4 (dense); half is the safe side.
constexpr double kAutoGatherShare = 0.5;
}  // namespace

// SvmEvaluator::commit's Gathered branch (backend.cpp:255-265): the budget
// check on projected_gather_bytes (backend.cpp:47-54), then gather_rows.
// TRON_SVM_AUTO applies the cost model above instead of raising.
void Engine::gather_active() {
  AllocScope scope(s_);
  const Slot& S = slot_[cand_ ^ 1];
  const bool auto_mode = svm_strategy_ == TRON_SVM_AUTO;
  if (dense_) {
    const uint64_t projected = (uint64_t)S.nact * (uint64_t)n_ * sizeof(double);
    if (auto_mode) {
      if (projected > budget_ || (double)S.nact > kAutoGatherShare * (double)l_) return;
    } else if (projected > budget_) {
      raise(TRON_ERR_BUDGET, budget_message(projected, budget_));
    }
    const int nI = compact(S, idx_);
    if (nI == 0) return;  // nothing active: the masked pass answers Hv = v exactly
    const int64_t ldg = dense_ld(nI);
    if ((size_t)ldg * n_ > Xg_.n) Xg_.alloc((size_t)std::max<int64_t>(ldg, kDenseTile) * n_);
    dense_gather(nI, n_, Xc_.p, ld_, idx_.p, Xg_.p, ldg, s_);
    count_launch(1);
    if (dense_make_map(&gmap_, Xg_.p, ldg, nI, n_) != 0)
      raise(TRON_ERR_CUDA, "cuTensorMapEncodeTiled failed for the gathered panel");
    nI_ = nI;
    ldg_ = ldg;
    gathered_valid_ = true;
    ledger.gathered_submatrix_bytes =
        std::max<uint64_t>(ledger.gathered_submatrix_bytes, (uint64_t)nI * n_ * sizeof(double));
  } else {
    const int nI = compact(S, idx_);
    grptr_.alloc((size_t)nI + 1);
    long long nnzI = 0;
    const int rc = csr_gather_offsets(X_, idx_.p, nI, grptr_.p, &nnzI, s_);
    if (rc != 0) cuda_check((cudaError_t)rc, "csr_gather_offsets");
    count_launch(1);
    const uint64_t projected = (uint64_t)nnzI * (sizeof(double) + sizeof(int32_t)) +
                               ((uint64_t)nI + 1) * sizeof(int64_t);
    if (auto_mode) {
      if (projected > budget_ || (double)nnzI > kAutoGatherShare * (double)X_.nnz) return;
    } else if (projected > budget_) {
      raise(TRON_ERR_BUDGET, budget_message(projected, budget_));
    }
    build_gathered_csr(nI, nnzI);
    ledger.gathered_submatrix_bytes = std::max<uint64_t>(ledger.gathered_submatrix_bytes, projected);
  }
  ++gathered_epoch_;
}

// X_I (rows idx_[0..nI), offsets already in grptr_) plus its CSC copy and
// segmented plan, built on the device like the full matrix's at creation.
void Engine::build_gathered_csr(int nI, long long nnzI) {
  gcidx_.alloc((size_t)nnzI + 4);  // + 4: the row kernels read aligned groups of four
  grval_.alloc((size_t)nnzI + 4);
  cuda_check(cudaMemsetAsync(gcidx_.p + nnzI, 0, 4 * sizeof(int32_t), s_), "pad");
  cuda_check(cudaMemsetAsync(grval_.p + nnzI, 0, 4 * sizeof(double), s_), "pad");
  csr_gather_rows(X_, idx_.p, nI, grptr_.p, gcidx_.p, grval_.p, s_);
  count_launch(1);
  Xg_csr_ = CsrView{(int64_t)nI, n_, (int64_t)nnzI, grptr_.p, gcidx_.p, grval_.p};
  const int64_t nnz_pad = (nnzI + kSegChunk - 1) / kSegChunk * kSegChunk;
  gcptr_.alloc((size_t)n_ + 1);
  gridx_.alloc((size_t)std::max<int64_t>(nnz_pad, 1));
  gcval_.alloc((size_t)std::max<int64_t>(nnz_pad, 1));
  int32_t* perm = nullptr;
  int rc = build_csc_structure(Xg_csr_, gcptr_.p, gridx_.p, &perm, s_);
  if (rc != 0) cuda_check((cudaError_t)rc, "build_csc_structure (gathered)");
  if (nnz_pad > nnzI) {
    cuda_check(cudaMemsetAsync(gridx_.p + nnzI, 0, (nnz_pad - nnzI) * sizeof(int32_t), s_), "pad");
    cuda_check(cudaMemsetAsync(gcval_.p + nnzI, 0, (nnz_pad - nnzI) * sizeof(double), s_), "pad");
  }
  rc = build_csc_values(perm, grval_.p, gcval_.p, nnzI, s_);
  if (rc != 0) cuda_check((cudaError_t)rc, "build_csc_values (gathered)");
  Xgt_ = CsrView{n_, (int64_t)nI, (int64_t)nnzI, gcptr_.p, gridx_.p, gcval_.p};
  const int64_t nch = (nnzI + kSegChunk - 1) / kSegChunk;
  const int64_t slots = std::max<int64_t>(nch, 1);
  gchunk_rank_.alloc(slots);
  glastbits_.alloc(nch * (kSegChunk / 32) + 2);
  gnz_col_.alloc((size_t)n_ + 1);
  gempty_col_.alloc((size_t)std::max<int64_t>(n_, 1));
  gchunk_first_.alloc(slots);
  ghead_.alloc(slots);
  gcarry_.alloc(slots);
  glong_fix_.alloc(seg_long_fix_cap(nch));
  rc = seg_plan_device(gcptr_.p, n_, nnzI, &gplan_, gchunk_rank_.p, gchunk_first_.p, glastbits_.p,
                       gnz_col_.p, gempty_col_.p, glong_fix_.p, s_);
  if (rc != 0) cuda_check((cudaError_t)rc, "seg_plan_device (gathered)");
  gplan_.head = ghead_.p;
  gplan_.carry = gcarry_.p;
  gathered_csr_valid_ = true;
}

void Engine::commit(double* gnorm) {
  if (!slot_[cand_].valid) raise(TRON_ERR_LOGIC, "commit() without a pending candidate");
  cand_ ^= 1;  // the candidate becomes the committed slot
  slot_[cand_].valid = false;
  committed_valid_ = true;
  precond_valid_ = false;
  gathered_valid_ = false;
  gathered_csr_valid_ = false;
  if (loss_ == TRON_LOSS_L2SVM && svm_strategy_ != TRON_SVM_INDIRECT) gather_active();
  gradient_dev();
  read_obj();
  gnorm_ = obj_h_->gnorm;
  ledger.gradient_materializations++;
  if (gnorm) *gnorm = gnorm_;
}

// commit() for a candidate whose gradient was computed speculatively into gspec_
// (its norm already read into obj_h_).
void Engine::adopt_candidate() {
  if (!slot_[cand_].valid) raise(TRON_ERR_LOGIC, "commit() without a pending candidate");
  cand_ ^= 1;
  slot_[cand_].valid = false;
  committed_valid_ = true;
  precond_valid_ = false;
  gathered_valid_ = false;
  gathered_csr_valid_ = false;
  if (n_ > 0)
    cuda_check(cudaMemcpyAsync(g_.p, gspec_.p, n_ * sizeof(double), cudaMemcpyDeviceToDevice, s_),
               "D2D");
  gnorm_ = obj_h_->gnorm;
  ledger.gradient_materializations++;
}

void Engine::gradient_host(double* g) {
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "gradient() before the first commit()");
  download(g, g_.p, n_ * sizeof(double), s_);
}

// ----------------------------------------------------------------------------
// Hv (loss.cpp:82-92 / :139-174) and preconditioner (loss.cpp:176-188)
// ----------------------------------------------------------------------------
void Engine::ro_accum_slot(int mode, const Slot& S, const double* v, const EpiView& epi, double* out) {
  ro_accum(mode, l_, n_, xmap128_, S.cnt.p, S.idx.p, S.mask.p, v, S.z.p, y_.p, ro_parts_.p,
           ro_tickets_.p + 1, epi, out, obj_d_, s_);
  count_launch(1);
}

bool Engine::hv_dot_available() const {
  // sharded or nnz == 0: the vector epilogue after the allreduce (or the
  // epilogue-only shortcut) does the reduction instead of the segmented kernels
  return !dense_ && !colpart_ && dot_parts_.n > 0;
}

// Column panels for the row products (csr_dv, csr_forward) when the gathered
// vector is larger than ~96 MB: measured on K1 (v = 160 MB), half of the
// gathers missed L2 and doubled the pass's DRAM traffic.  Panel width
// TRON_B200_PANEL_COLS (0: off).
void Engine::setup_panels() {
  panels_.clear();
  panel_group_.clear();
  // Opt-in: measured on K1 the panels cut the fused margin pass (2.12 -> 1.57 ms
  // with 10M-column panels: the heavy panel runs in the lean csr_dv kernel) but
  // not the Hv row products (1.45 -> 1.54 ms): the Zipf tail's gathers miss L2
  // whatever the panel width, and every extra panel re-reads the row arrays.
  const char* e = std::getenv("TRON_B200_PANEL_COLS");
  const int64_t W = e ? std::atoll(e) : 0;
  if (W <= 0 || X_.nnz == 0) return;
  const int K = (int)std::min<int64_t>((n_ + W - 1) / W, 8);
  if (K < 2) return;
  std::vector<int32_t> bounds;
  for (int k = 1; k < K; ++k) bounds.push_back((int32_t)(n_ * k / K));
  int32_t* splits[8] = {};
  for (int k = 0; k < K - 1; ++k) {
    psplit_[k].alloc((size_t)l_);
    splits[k] = psplit_[k].p;
  }
  unsigned long long h[8] = {};
  const int rc = csr_panel_splits(X_, bounds.data(), K - 1, splits, h, s_);
  if (rc != 0) cuda_check((cudaError_t)rc, "csr_panel_splits");
  for (int k = 0; k < K; ++k) {
    CsrView P = X_;
    P.rbeg = k == 0 ? nullptr : psplit_[k - 1].p;
    P.rend = k == K - 1 ? nullptr : psplit_[k].p;
    P.nnz = (int64_t)h[k];
    panels_.push_back(P);
    panel_group_.push_back(choose_group(l_, (int64_t)h[k]));
  }
}

// a_i = (x_i . v) * dvec_i / mask_i ? x_i . v : 0 (loss.cpp:84-89, :143-160)
// over the column panels in order, or in one pass.
void Engine::row_products(const double* v, const double* dvec, const uint8_t* mask, double* a) {
  if (panels_.empty()) {
    csr_dv(X_, group_, v, dvec, mask, a, s_);
    count_launch(1);
    return;
  }
  const size_t K = panels_.size();
  for (size_t k = 0; k < K; ++k)
    csr_dv(panels_[k], panel_group_[k], v, dvec, mask, a, s_, k ? a : nullptr, k + 1 == K);
  count_launch(K);
}

// G = sum_i c_i x_i x_i^T of slot S (c = its mask or D), summed over the
// shards when row-sharded (one n*n exchange per commit, none per Hv).
// G of slot S for its current iterate.  Lazily: a margin pass leaves its
// slot's G current (L2-SVM: the committed slot's G plus the rows that changed
// side, dense_pass PM_FWDD) or flagged stale, and a stale G is formed right
// before the CG that needs it -- so the last iterate of a solve (converged) and
// rejected candidates never pay for a Gram pass.  The kernels check the flag
// on the device.
void Engine::ensure_gram(const Slot& S) {
  if (!gram_ || gram_fused_) return;
  const bool svm = loss_ == TRON_LOSS_L2SVM;
  const bool shard = comm_.active();
  dense_gram(l_, n_, ld_, Xc_.p, svm ? S.mask.p : nullptr, svm ? nullptr : S.dvec.p, gram_parts_.p,
             shard ? S.gram_local.p : S.gram.p, s_, S.gram_flags.p);
  count_launch(2);
  // row shards: G = sum of the ranks' parts, out of place, so repeating it
  // when nothing was stale changes nothing (every rank makes the same calls)
  if (shard) comm_.allreduce_sum(S.gram_local.p, S.gram.p, (size_t)n_ * n_, s_);
}

void Engine::gram_slot(const Slot& S) {
  const bool svm = loss_ == TRON_LOSS_L2SVM;
  if (gram_fused_) {  // the slot's margin pass accumulated the partials already
    gram_finalize(n_, S.gram_parts.p, dense_grid(l_, n_), S.gram.p, s_);
    count_launch(1);
  } else {
    dense_gram(l_, n_, ld_, Xc_.p, svm ? S.mask.p : nullptr, svm ? nullptr : S.dvec.p, gram_parts_.p,
               S.gram.p, s_);
    count_launch(2);
  }
  if (comm_.active()) comm_.allreduce_sum(S.gram.p, (size_t)n_ * n_, s_);
}

void Engine::hv_kernels(const double* v, double* out, bool with_dot) {
  const Slot& S = slot_[cand_ ^ 1];
  EpiView epi;
  epi.kind = EPI_VEC;
  epi.base = v;
  epi.scale = loss_ == TRON_LOSS_LOGISTIC ? C_ : 2.0 * C_;
  if (with_dot) {  // v . out, summed as out is emitted (the CG's p.Hp)
    epi.dot_parts = dot_parts_.p;
    epi.dot_out = dot_out_.p;
    epi.dot_ticket = dot_ticket_.p;
  }
  if (ro_) {
    ro_accum_slot(RO_HV, S, v, epi, out);
    return;
  }
  if (dense_ && gram_) {  // v + s G v
    ensure_gram(S);
    gram_hv(n_, S.gram.p, v, epi.scale, out, s_);
    count_launch(1);
    return;
  }
  if (dense_) {
    dense_vector(DA_HV, v, epi, out);
    return;
  }
  UView u;
  u.kind = U_VEC;
  u.u = a_.p;
  if (gathered_csr_valid_) {  // Gathered L2-SVM: every row of X_I is active
    csr_dv(Xg_csr_, group_, v, nullptr, nullptr, a_.p, s_);
    count_launch(1);
    transposed_raw_or_epi(u, false, epi, out, &Xgt_, &gplan_);
    return;
  }
  const double* dv = loss_ == TRON_LOSS_LOGISTIC ? S.dvec.p : nullptr;
  const uint8_t* mk = loss_ == TRON_LOSS_LOGISTIC ? nullptr : S.mask.p;
  if (colpart_) {  // t = sum over ranks of X_{:,r} v_r (one l-length exchange), then D t
    csr_dv(X_, group_, v, nullptr, nullptr, a_.p, s_);
    comm_.allreduce_sum(a_.p, (size_t)l_, s_);
    vec_row_scale(l_, a_.p, dv, mk, s_);
    count_launch(2);
  } else {
    row_products(v, dv, mk, a_.p);
  }
  transposed_raw_or_epi(u, false, epi, out);
}

void Engine::hessian_vec_dev(const double* v, double* out) {
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "hessian_vec() before the first commit()");
  hv_kernels(v, out);
}

void Engine::hessian_vec_host(const double* v, double* out) {
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "hessian_vec() before the first commit()");
  upload(vtmp_.p, v, n_ * sizeof(double), s_);
  hv_kernels(vtmp_.p, otmp_.p);
  download(out, otmp_.p, n_ * sizeof(double), s_);
  ledger.concealed_vector_returns++;
}

// quadratic_model (tron.cpp:31-35) at the committed iterate: q(d) = g.d + 0.5 d.Hd
// with g the committed gradient -- one Hv and one fused pair of dots.
double Engine::quadratic_model_host(const double* d) {
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "quadratic_model() before the first commit()");
  AllocScope scope(s_);
  DevBuf<double> dots;
  dots.alloc(2);
  if (n_ > 0) upload(vtmp_.p, d, n_ * sizeof(double), s_);
  hv_kernels(vtmp_.p, otmp_.p);
  vec_dot2(n_, g_.p, vtmp_.p, vtmp_.p, otmp_.p, dots.p, sc_, s_);
  count_launch(1);
  double h[2] = {0.0, 0.0};
  if (n_ > 0) cuda_check(cudaMemcpyAsync(h, dots.p, sizeof(h), cudaMemcpyDeviceToHost, s_), "D2H");
  synchronize();
  cuda_check(cudaGetLastError(), "quadratic_model");
  return h[0] + 0.5 * h[1];
}

void Engine::ensure_precond() {
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "precond_diagonal() before the first commit()");
  if (precond_valid_) return;
  precond_kernels(slot_[cand_ ^ 1]);
  precond_valid_ = true;
}

// M = 1 + C s sum_i d_i X_ij^2 of slot S into M_ (loss.cpp:176-188).
void Engine::precond_kernels(const Slot& S) {
  EpiView epi;
  epi.kind = EPI_CONST;
  epi.cbase = 1.0;
  epi.scale = loss_ == TRON_LOSS_LOGISTIC ? C_ : 2.0 * C_;
  if (ro_) {
    ro_accum_slot(RO_PRECOND, S, nullptr, epi, M_.p);
  } else if (dense_ && gram_) {
    ensure_gram(S);
    gram_precond(n_, S.gram.p, epi.scale, M_.p, s_);
    count_launch(1);
  } else if (dense_) {
    const int saved = cand_;
    cand_ = (int)(&S - slot_) ^ 1;  // dense_vector reads the committed slot_[cand_ ^ 1]
    dense_vector(DA_PRECOND, nullptr, epi, M_.p);
    cand_ = saved;
  } else {
    UView u;
    if (loss_ == TRON_LOSS_LOGISTIC) {
      u.kind = U_VEC;
      u.u = S.dvec.p;
    } else {
      u.kind = U_MASK;
      u.mask = S.mask.p;
    }
    transposed_raw_or_epi(u, true, epi, M_.p);
  }
}

void Engine::precond_host(double* m) {
  ensure_precond();
  download(m, M_.p, n_ * sizeof(double), s_);
}

// ----------------------------------------------------------------------------
// state probes
// ----------------------------------------------------------------------------
void Engine::state_lr(int which, double* z, double* zhat, double* dvec) {
  if (loss_ != TRON_LOSS_LOGISTIC) raise(TRON_ERR_LOGIC, "not a logistic evaluator");
  const Slot& S = which == 0 ? slot_[cand_] : slot_[cand_ ^ 1];
  if (!(which == 0 ? S.valid : committed_valid_)) raise(TRON_ERR_LOGIC, "state slot is empty");
  if (l_ > 0) {
    if (z) cuda_check(cudaMemcpyAsync(z, S.z.p, l_ * 8, cudaMemcpyDeviceToHost, s_), "D2H");
    if (zhat) cuda_check(cudaMemcpyAsync(zhat, S.zhat.p, l_ * 8, cudaMemcpyDeviceToHost, s_), "D2H");
    if (dvec) cuda_check(cudaMemcpyAsync(dvec, S.dvec.p, l_ * 8, cudaMemcpyDeviceToHost, s_), "D2H");
  }
  synchronize();
}

void Engine::state_svm(int which, double* z, int64_t* active, uint64_t cap, uint64_t* n_active) {
  AllocScope scope(s_);
  if (loss_ != TRON_LOSS_L2SVM) raise(TRON_ERR_LOGIC, "not an L2-SVM evaluator");
  const Slot& S = which == 0 ? slot_[cand_] : slot_[cand_ ^ 1];
  if (!(which == 0 ? S.valid : committed_valid_)) raise(TRON_ERR_LOGIC, "state slot is empty");
  if (z && l_ > 0) cuda_check(cudaMemcpyAsync(z, S.z.p, l_ * 8, cudaMemcpyDeviceToHost, s_), "D2H");
  if (idx_.n == 0) {
    idx_.alloc(l_ > 0 ? l_ : 1);
    idx_tmp_.alloc((l_ + 1023) / 1024 + 2);
    count_.alloc(1);
  }
  DevBuf<int32_t> idx;
  idx.alloc(l_ > 0 ? l_ : 1);
  const int cnt = compact(S, idx);
  if (n_active) *n_active = (uint64_t)cnt;
  if (active && cnt > 0) {
    std::vector<int32_t> h(cnt);
    cuda_check(cudaMemcpyAsync(h.data(), idx.p, cnt * sizeof(int32_t), cudaMemcpyDeviceToHost, s_),
               "D2H");
    synchronize();
    const uint64_t m = std::min<uint64_t>(cap, (uint64_t)cnt);
    for (uint64_t k = 0; k < m; ++k) active[k] = (int64_t)h[k] + (int64_t)row_begin_;
  }
  synchronize();
}

// ----------------------------------------------------------------------------
// device-resident truncated CG (tron.cpp:37-108)
// ----------------------------------------------------------------------------
// CG initialisation (d = 0, r = -g, p = M^-1 r) into the current capture.
void Engine::capture_cg_init(int k, const CgVectors& v, Cond cond) {
  if (dense_ && gram_) ensure_gram(slot_[k]);  // the committed iterate's G (if stale)
  if (ro_)
    ro_cg_init(v, st_d_, cond, s_);
  else if (small_engine_)
    cg_small_init(v, st_d_, cond, s_);
  else
    cg_large_init(v, st_d_, sc_, cond, s_);
  count_launch(small_engine_ && dense_ && gram_ && gram_cg_loop_ ? 2 : 1);  // (+ the looped CG, if it runs)
}

// One CG iteration with slot k committed (Hv of p, then the step kernel that
// sets `cond`) into the current capture.
void Engine::capture_cg_body(int k, const CgVectors& v, Cond cond) {
  const int saved_cand = cand_;
  cand_ = k ^ 1;  // so that slot_[cand_^1] == committed slot k
  if (ro_) {
    hv_kernels(p_.p, hp_.p);
    ro_cg_step(v, st_d_, cond, s_);
    count_launch(1);
  } else if (small_engine_) {
    if (dense_ && gram_) {  // hp = p + s G p inside the step kernel
      const double scale = loss_ == TRON_LOSS_LOGISTIC ? C_ : 2.0 * C_;
      if (gram_cg_loop_) {
        // every iteration in this one launch (the WHILE node then runs once);
        // counted with the CG's init: body_kernels_ stays 0
        cg_small_gram_loop(v, slot_[k].gram.p, scale, st_d_, cond, s_);
      } else {
        cg_small_step_gram(v, slot_[k].gram.p, scale, st_d_, cond, s_);
        count_launch(1);
      }
    } else if (dense_ && !comm_.active() && !ooc_) {  // sharded / streamed: through hv_kernels
      const Slot& S = slot_[k];
      const int loss = loss_ == TRON_LOSS_LOGISTIC ? kLossLogistic : kLossSvm;
      const double scale = loss_ == TRON_LOSS_LOGISTIC ? C_ : 2.0 * C_;
      if (gathered_valid_) {  // Gathered L2-SVM: the compact panel X_I, every row active
        dense_accum(DA_HV, nI_, n_, ldg_, Xg_.p, gmap_, kLossSvm, p_.p, nullptr, nullptr, parts_.p, s_);
        cg_small_step(v, parts_.p, dense_grid(nI_, n_), scale, st_d_, cond, s_);
      } else {
        dense_accum(DA_HV, l_, n_, ld_, Xc_.p, xmap_, loss, p_.p, S.dvec.p, S.mask.p, parts_.p, s_);
        cg_small_step(v, parts_.p, dense_grid(l_, n_), scale, st_d_, cond, s_);
      }
      count_launch(2);
    } else {
      hv_kernels(p_.p, hp_.p);
      cg_small_step(v, nullptr, 0, 0.0, st_d_, cond, s_);
      count_launch(1);
    }
  } else if (mid_engine_) {
    hv_kernels(p_.p, hp_.p);
    cg_cluster_step(v, st_d_, cond, s_);
    count_launch(1);
  } else {
    const bool dot = hv_dot_available();
    hv_kernels(p_.p, hp_.p, dot);
    cg_coop_step(v, st_d_, coop_parts_.p, cond, s_, dot ? dot_out_.p : nullptr);
    count_launch(1);
  }
  cand_ = saved_cand;
}

namespace {
// Adds a conditional node of `type` after the current capture's dependencies
// and makes it the capture's only dependency; returns its body graph.
cudaGraph_t add_conditional(cudaStream_t s, cudaGraphConditionalHandle handle,
                            cudaGraphConditionalNodeType type) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraph_t capg = nullptr;
  cuda_check(cudaStreamGetCaptureInfo(s, &cs, nullptr, &capg, &deps, &ndeps), "capture info");
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = type;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  cuda_check(cudaGraphAddNode(&node, capg, deps, ndeps, &cp), "add conditional node");
  cuda_check(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies),
             "update deps");
  return cp.conditional.phGraph_out[0];
}

Cond make_cond(cudaGraph_t g, unsigned dflt, unsigned flags) {
  cudaGraphConditionalHandle h;
  cuda_check(cudaGraphConditionalHandleCreate(&h, g, dflt, flags), "conditional handle");
  Cond c;
  c.h = (unsigned long long)h;
  c.on = 1;
  return c;
}

void begin_capture(cudaStream_t s, cudaGraph_t g) {
  cuda_check(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal),
             "begin capture");
}
}  // namespace

void Engine::build_graph(int k, bool use_m) {
  // Captured against committed slot k; CG vectors are fixed buffers.
  cudaGraph_t graph;
  cuda_check(cudaGraphCreate(&graph, 0), "cudaGraphCreate");
  const Cond cond = make_cond(graph, 0, 0);
  CgVectors v{n_, g_.p, use_m ? M_.p : nullptr, d_.p, r0_.p, r1_.p, p_.p, hp_.p};
  const uint64_t saved_launches = launches;

  begin_capture(s_, graph);
  capture_cg_init(k, v, cond);
  cudaGraph_t body = add_conditional(s_, (cudaGraphConditionalHandle)cond.h, cudaGraphCondTypeWhile);
  cuda_check(cudaStreamEndCapture(s_, &graph), "end capture");

  begin_capture(s_, body);
  const uint64_t before = launches;
  capture_cg_body(k, v, cond);
  body_kernels_ = launches - before;
  cuda_check(cudaStreamEndCapture(s_, &body), "end body capture");
  launches = saved_launches;

  cudaGraphExec_t exec;
  cuda_check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
  graph_[k][use_m] = graph;
  graph_exec_[k][use_m] = exec;
  graph_epoch_[k][use_m] = gathered_epoch_;
}

// The CG graph of committed slot k, (re)built when it was captured for the
// gathered rows of an earlier commit.
void Engine::launch_cg_graph(int k, bool use_m) {
  if (graph_exec_[k][use_m] && graph_epoch_[k][use_m] != gathered_epoch_) {
    cudaGraphExecDestroy(graph_exec_[k][use_m]);
    cudaGraphDestroy(graph_[k][use_m]);
    graph_exec_[k][use_m] = nullptr;
    graph_[k][use_m] = nullptr;
  }
  if (!graph_exec_[k][use_m]) build_graph(k, use_m);
  cuda_check(cudaGraphLaunch(graph_exec_[k][use_m], s_), "graph launch");
}

// Graph path: enqueues the CG loop and returns without waiting (false); the
// host-driven path (no graphs / NCCL) runs it to the end and fills *out (true).
bool Engine::enqueue_cg(double delta, const tron_config& cfg, CgState* out) {
  if (!use_graphs_) {
    run_cg(delta, cfg, out);
    return true;
  }
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "truncated CG before the first commit()");
  const bool use_m = cfg.use_preconditioner != 0;
  if (use_m) ensure_precond();
  uint64_t max_iters = cfg.max_cg_iters;
  if (max_iters == 0) max_iters = (uint64_t)n_ < 1000 ? (uint64_t)n_ : 1000;  // tron.cpp:40-41
  CgState init{};
  init.delta = delta;
  init.stop = cfg.cg_tol * gnorm_;  // tron.cpp:55
  init.max_iters = (long long)max_iters;
  init.use_m = use_m;
  *st_h_ = init;
  cuda_check(cudaMemcpyAsync(st_d_, st_h_, sizeof(CgState), cudaMemcpyHostToDevice, s_), "H2D");
  launch_cg_graph(cand_ ^ 1, use_m);
  return false;
}

// A dot product of two column-partitioned n-vectors: local sum, scalar exchange.
double Engine::gdot(const double* a, const double* b) {
  vec_dot2(n_, a, b, a, b, cp_dots_.p, sc_, s_);
  count_launch(1);
  comm_.allreduce_sum(cp_dots_.p, 1, s_);
  double h = 0.0;
  cuda_check(cudaMemcpyAsync(&h, cp_dots_.p, sizeof(double), cudaMemcpyDeviceToHost, s_), "D2H");
  synchronize();
  return h;
}

// truncated_cg (tron.cpp:37-108) in the column layout: the vectors are this
// rank's slices, every dot is a scalar exchange, every rank takes the same
// branches (the exchanged scalars are identical); the step's arithmetic is
// tron.cpp's (axpy_inplace, apply_precond, p = z + beta p).
void Engine::run_cg_columns(double delta, const tron_config& cfg, CgState* out) {
  const bool use_m = cfg.use_preconditioner != 0;
  if (use_m) ensure_precond();
  const double* M = use_m ? M_.p : nullptr;
  uint64_t max_iters = cfg.max_cg_iters;
  if (max_iters == 0) max_iters = (uint64_t)global_n_ < 1000 ? (uint64_t)global_n_ : 1000;
  double* d = d_.p;
  double* r = r0_.p;
  double* z = r1_.p;
  double* p = p_.p;
  double* hp = hp_.p;
  const int64_t n = n_;
  cuda_check(cudaMemsetAsync(d, 0, n * sizeof(double), s_), "memset");
  vec_lincomb(n, -1.0, g_.p, 0.0, nullptr, r, s_);  // r = -g
  vec_div(n, r, M, z, s_);
  cuda_check(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, s_), "D2D");
  count_launch(2);
  double rz = gdot(r, z);
  const double stop = cfg.cg_tol * gnorm_;  // tron.cpp:55
  CgState st{};
  st.delta = delta;
  st.stop = stop;
  st.max_iters = (long long)max_iters;
  st.use_m = use_m;
  st.exit_kind = kCgConverged;
  while ((uint64_t)st.iters < max_iters) {
    if (std::sqrt(gdot(r, r)) <= stop) {
      st.exit_kind = kCgConverged;
      break;
    }
    ++st.iters;
    hv_kernels(p, hp);
    const double php = gdot(p, hp);
    st.php = php;
    if (!(php > 0.0)) {
      st.fail = 1;
      break;
    }
    const double alpha = rz / php;
    vec_lincomb(n, 1.0, d, alpha, p, d, s_);  // axpy_inplace(alpha, p, d)
    count_launch(1);
    if (std::sqrt(gdot(d, d)) > delta) {  // retreat, then to the boundary along p
      vec_lincomb(n, 1.0, d, -alpha, p, d, s_);
      const double dp = gdot(d, p), dd = gdot(d, d), pp = gdot(p, p);
      const double rad = std::sqrt(dp * dp + pp * (delta * delta - dd));
      const double tau = dp >= 0.0 ? (delta * delta - dd) / (dp + rad) : (rad - dp) / pp;
      vec_lincomb(n, 1.0, d, tau, p, d, s_);
      vec_lincomb(n, 1.0, r, -tau, hp, r, s_);
      count_launch(3);
      st.exit_kind = kCgBoundary;
      st.boundary = 1;
      break;
    }
    vec_lincomb(n, 1.0, r, -alpha, hp, r, s_);
    vec_div(n, r, M, z, s_);
    const double rz_next = gdot(r, z);
    const double beta = rz_next / rz;
    vec_lincomb(n, 1.0, z, beta, p, p, s_);  // p = z + beta p
    count_launch(3);
    rz = rz_next;
    st.exit_kind = kCgMaxIters;
  }
  if (!st.fail) {
    const double rn = std::sqrt(gdot(r, r));
    if ((uint64_t)st.iters >= max_iters && st.exit_kind != kCgBoundary && rn > stop)
      st.exit_kind = kCgMaxIters;
    else if (st.exit_kind != kCgBoundary)
      st.exit_kind = kCgConverged;
    st.q = 0.5 * (gdot(d, g_.p) - gdot(d, r));  // tron.cpp:106
    st.dnorm = std::sqrt(gdot(d, d));
  }
  st.cont = 0;
  *out = st;
}

void Engine::run_cg(double delta, const tron_config& cfg, CgState* out) {
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "truncated CG before the first commit()");
  if (colpart_) {
    run_cg_columns(delta, cfg, out);
    return;
  }
  const bool use_m = cfg.use_preconditioner != 0;
  if (use_m) ensure_precond();
  uint64_t max_iters = cfg.max_cg_iters;
  if (max_iters == 0) max_iters = (uint64_t)n_ < 1000 ? (uint64_t)n_ : 1000;  // tron.cpp:40-41
  CgState init{};
  init.delta = delta;
  init.stop = cfg.cg_tol * gnorm_;  // tron.cpp:55
  init.max_iters = (long long)max_iters;
  init.use_m = use_m;
  *st_h_ = init;
  cuda_check(cudaMemcpyAsync(st_d_, st_h_, sizeof(CgState), cudaMemcpyHostToDevice, s_), "H2D");
  const int k = cand_ ^ 1;
  CgVectors v{n_, g_.p, use_m ? M_.p : nullptr, d_.p, r0_.p, r1_.p, p_.p, hp_.p};
  if (use_graphs_) {
    launch_cg_graph(k, use_m);
    read_cg(out);
    launches += 1 + (uint64_t)out->iters * body_kernels_;
    return;
  }
  // host-driven loop (host data plane, or TRON_B200_NO_GRAPH / NCCL_GRAPH=0):
  // the graph's kernels, launched one iteration at a time
  Cond none;
  capture_cg_init(k, v, none);
  read_cg(out);
  while (out->cont) {
    capture_cg_body(k, v, none);
    read_cg(out);
  }
}

void Engine::truncated_cg(double delta, const tron_config& cfg, double* d, int32_t* exit_kind,
                          uint64_t* iters, double* q) {
  CgState st;
  run_cg(delta, cfg, &st);
  if (st.fail)
    raise(TRON_ERR_NUMERICAL,
          "conjugate gradients met non-positive curvature (" + std::to_string(st.php) + ")");
  if (d) download(d, d_.p, n_ * 8, s_);
  if (exit_kind) *exit_kind = st.exit_kind;
  if (iters) *iters = (uint64_t)st.iters;
  if (q) *q = st.q;
}

// ----------------------------------------------------------------------------
// device-mode solve: tron.cpp:127-217 with device w/g/d and host scalars
// ----------------------------------------------------------------------------
namespace {
void validate_config(const tron_config& c) {  // tron.cpp:19-29
  if (!(c.eps > 0.0)) raise(TRON_ERR_DIMENSION, "config: eps must be positive");
  if (!(c.sigma0 > 0.0 && c.sigma0 < 1.0)) raise(TRON_ERR_DIMENSION, "config: sigma0 must be in (0,1)");
  if (!(0.0 < c.eta1 && c.eta1 < c.eta2 && c.eta2 < 1.0))
    raise(TRON_ERR_DIMENSION, "config: need 0 < eta1 < eta2 < 1");
  if (!(0.0 < c.gamma1 && c.gamma1 < c.gamma2 && c.gamma2 < 1.0 && c.gamma3 > 1.0))
    raise(TRON_ERR_DIMENSION, "config: need 0 < gamma1 < gamma2 < 1 < gamma3");
  if (!(c.cg_tol > 0.0 && c.cg_tol < 1.0)) raise(TRON_ERR_DIMENSION, "config: cg_tol must be in (0,1)");
}

struct NumericalAbort {
  std::string what;
};
}  // namespace

void Engine::solve_device(const tron_config& cfg, const double* w0, double* w_out,
                          tron_solve_info* info, tron_iteration* trace, uint64_t cap) {
  validate_config(cfg);
  std::memset(info, 0, sizeof(*info));
  const uint64_t launches0 = launches;
  uint64_t hv_count = 0;
  cudaEvent_t ev0, ev1;
  cuda_check(cudaEventCreate(&ev0), "event");
  cuda_check(cudaEventCreate(&ev1), "event");
  cuda_check(cudaEventRecord(ev0, s_), "event record");
  bool write_w = true;
  auto finish = [&](int status) {
    cudaEventRecord(ev1, s_);
    cudaEventSynchronize(ev1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    info->device_ms = ms;
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    if (w_out && write_w) download(w_out, slot_[cand_ ^ 1].w.p, n_ * 8, s_);
    info->status = status;
    info->hessian_products = hv_count;
    (void)launches0;
  };
  Slot& C0 = slot_[cand_];
  if (n_ > 0) {
    if (w0)
      upload(C0.w.p, w0, n_ * 8, s_);
    else
      cuda_check(cudaMemsetAsync(C0.w.p, 0, n_ * 8, s_), "memset");
  }
  const char* trace_env = std::getenv("TRON_B200_TRACE");
  const bool device_loop = device_loop_ok() && !(trace_env && trace_env[0] == '1');
  if (gram_delta_) {
    // every solve forms its own G: nothing carries over from an earlier solve
    for (auto& S : slot_) cuda_check(cudaMemsetAsync(S.gram_flags.p, 0xff, sizeof(int), s_), "memset");
    gram_full_next_ = gram_first_fused_;
  }
  // device loop: the starting point's margin pass and gradient in one round trip
  double f = eval_candidate_dev(nullptr, /*read=*/!device_loop);
  if (device_loop) {
    gradient_into(slot_[cand_], gbuf(cand_));  // adopted below unless f is not finite
    read_obj();
    f = candidate_result();
  }
  info->objective_evaluations = 1;
  if (!std::isfinite(f)) {
    // nothing was committed: like the reference (which throws before any
    // result exists), w_out is left untouched
    write_w = false;
    finish(TRON_ERR_NUMERICAL);
    raise(TRON_ERR_NUMERICAL, "objective is not finite at the starting point");
  }
  if (device_loop) {
    cand_ ^= 1;
    slot_[cand_].valid = false;
    committed_valid_ = true;
    precond_valid_ = false;
    gathered_valid_ = false;
    gathered_csr_valid_ = false;
    gnorm_ = obj_h_->gnorm;
    ledger.gradient_materializations++;
    if (cand_ == 0)  // the committed slot is 1: g_ must hold its gradient for the API
      cuda_check(cudaMemcpyAsync(g_.p, gspec_.p, n_ * sizeof(double), cudaMemcpyDeviceToDevice, s_),
                 "D2D");
  } else {
    commit(nullptr);
  }
  info->gradient_materializations = 1;
  if (obj_h_->grad_nonfinite) {
    finish(TRON_ERR_NUMERICAL);
    raise(TRON_ERR_NUMERICAL, "gradient is not finite at the starting point");
  }
  info->f_initial = f;
  const double gnorm0 = gnorm_;
  info->gradient_norm_initial = gnorm0;
  double gnorm = gnorm0;
  info->objective = f;
  if (gnorm <= cfg.eps * gnorm0) {
    info->converged = 1;
    finish(TRON_OK);
    return;
  }
  if (device_loop) {
    NvtxRange nvtx_range("tron.solve.device_loop");
    int status = TRON_OK;
    std::string what;
    solve_device_loop(cfg, f, info, trace, cap, &status, &what);
    hv_count = info->hessian_products;
    if (status != TRON_OK) {
      finish(status);
      raise(status, what);
    }
    // (the device loop's delta stays on the device: the check covers w and f)
    check_replicas(info->objective, 0.0, info->n_iterations);
    finish(TRON_OK);
    return;
  }
  double delta = gnorm0;
  // Gathered / Auto L2-SVM gather X_I at commit, before the CG that uses it
  const bool speculative = !(loss_ == TRON_LOSS_L2SVM && svm_strategy_ != TRON_SVM_INDIRECT);
  // TRON_B200_TRACE=1: device time of each outer iteration's phases on stderr
  struct OuterProf {
    bool on = false;
    cudaStream_t s = nullptr;
    cudaEvent_t e[4] = {};
    std::chrono::steady_clock::time_point h0;
    void rec(int i) {
      if (i == 0) h0 = std::chrono::steady_clock::now();
      cudaEventRecord(e[i], s);
    }
    void report(uint64_t it) {
      float cg = 0, fw = 0, gr = 0;
      cudaEventElapsedTime(&cg, e[0], e[1]);
      cudaEventElapsedTime(&fw, e[1], e[2]);
      cudaEventElapsedTime(&gr, e[2], e[3]);
      const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
      std::fprintf(stderr, "[tron_b200] outer %llu: cg %.3f fwd %.3f grad %.3f ms (wall %.3f)\n",
                   (unsigned long long)it, cg, fw, gr, wall);
    }
    ~OuterProf() {
      for (auto& x : e)
        if (x) cudaEventDestroy(x);
    }
  } prof;
  if (const char* tr = std::getenv("TRON_B200_TRACE"); tr && tr[0] == '1') {
    prof.on = true;
    prof.s = s_;
    for (auto& x : prof.e) cudaEventCreate(&x);
  }
  while (info->n_iterations < cfg.max_outer_iters) {
    // One host round trip per outer iteration: the CG loop, the candidate's
    // margin pass and -- speculatively -- the candidate's gradient are queued
    // back to back; the host reads the CG scalars and f, ||g|| together.
    // The gradient is adopted only if the step is accepted (the reference's
    // lazy gradient, backend.cpp:165-183; ledger counts adoptions).
    CgState st;
    if (prof.on) prof.rec(0);
    const bool cg_done = enqueue_cg(delta, cfg, &st);
    double f_cand;
    if (speculative) {
      const int k = cand_ ^ 1;
      if (prof.on) prof.rec(1);
      f_cand = eval_candidate_dev(d_.p, /*read=*/false);
      if (prof.on) prof.rec(2);
      gradient_into(slot_[cand_], gspec_.p);
      if (prof.on) prof.rec(3);
      if (!cg_done)
        cuda_check(cudaMemcpyAsync(st_h_, st_d_, sizeof(CgState), cudaMemcpyDeviceToHost, s_),
                   "D2H");
      read_obj();
      if (prof.on) prof.report(info->n_iterations);
      if (!cg_done) {
        st = *st_h_;
        launches += 1 + (uint64_t)st.iters * body_kernels_;
      }
      f_cand = candidate_result();
      (void)k;
    } else {
      if (!cg_done) read_cg(&st);
      f_cand = eval_candidate_dev(d_.p);
    }
    hv_count += (uint64_t)st.iters;
    if (st.fail) {
      finish(TRON_ERR_NUMERICAL);
      raise(TRON_ERR_NUMERICAL,
            "conjugate gradients met non-positive curvature (" + std::to_string(st.php) + ")");
    }
    const double step_norm = st.dnorm;
    info->objective_evaluations++;
    if (!std::isfinite(f_cand)) {
      finish(TRON_ERR_NUMERICAL);
      raise(TRON_ERR_NUMERICAL, "objective is not finite at a candidate step");
    }
    const double sigma = (f_cand - f) / st.q;
    // trust_region_update (tron.cpp:110-125)
    const bool accept = sigma > cfg.sigma0;
    double next_delta;
    if (!accept)
      next_delta = cfg.gamma1 * step_norm;
    else if (sigma < cfg.eta1)
      next_delta = cfg.gamma2 * step_norm;
    else if (sigma < cfg.eta2)
      next_delta = delta;
    else {
      const double grown = cfg.gamma3 * step_norm;
      next_delta = grown > delta ? grown : delta;
    }
    if (trace && info->n_iterations < cap) {
      tron_iteration& rec = trace[info->n_iterations];
      rec.f_candidate = f_cand;
      rec.gradient_norm = gnorm;
      rec.delta = delta;
      rec.sigma = sigma;
      rec.accepted = accept;
      rec.cg_iters = (uint64_t)st.iters;
      rec.cg_exit = st.exit_kind;
    }
    info->n_iterations++;
    delta = next_delta;
    if (accept) {
      f = f_cand;
      info->objective = f;
      if (speculative)
        adopt_candidate();
      else
        commit(nullptr);
      info->accepted_steps++;
      info->gradient_materializations++;
      if (obj_h_->grad_nonfinite) {
        finish(TRON_ERR_NUMERICAL);
        raise(TRON_ERR_NUMERICAL, "gradient is not finite after an accepted step");
      }
      gnorm = gnorm_;
      if (gnorm <= cfg.eps * gnorm0) {
        info->converged = 1;
        check_replicas(f, delta, info->n_iterations);
        break;
      }
    }
    check_replicas(f, delta, info->n_iterations);
  }
  finish(TRON_OK);
}

// ----------------------------------------------------------------------------
// device-resident outer loop (tron.cpp:127-217 as one graph; trloop.cu)
// ----------------------------------------------------------------------------
bool Engine::device_loop_ok() const {
  const char* e = std::getenv("TRON_B200_DEVICE_LOOP");  // 0: host-driven outer loop
  const bool on = !(e && e[0] == '0');
  // Gathered / Auto L2-SVM re-gather X_I on the host at every commit
  return on && use_graphs_ && n_ > 0 &&
         !(loss_ == TRON_LOSS_L2SVM && svm_strategy_ != TRON_SVM_INDIRECT);
}

// WHILE(outer) { dispatch; IF(committed == 0) body(0); IF(committed == 1) body(1) }
// with body(k) = [M of slot k] prep, CG init, WHILE(cg){Hv, step}, w_cand = w_k + d,
// margin pass and speculative gradient of slot k^1, tr_update.
void Engine::build_solve_graph(bool use_m) {
  const uint64_t saved_launches = launches;
  cudaGraph_t top;
  cuda_check(cudaGraphCreate(&top, 0), "cudaGraphCreate");
  const Cond outer = make_cond(top, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = (cudaGraphConditionalHandle)outer.h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wnode;
  cuda_check(cudaGraphAddNode(&wnode, top, nullptr, 0, &cp), "add outer while node");
  cudaGraph_t B = cp.conditional.phGraph_out[0];
  const Cond K[2] = {make_cond(B, 0, 0), make_cond(B, 0, 0)};
  SolveState* ss = ss_buf_.p;
  begin_capture(s_, B);
  tr_dispatch(ss, K[0], K[1], s_);
  cudaGraph_t I[2];
  I[0] = add_conditional(s_, (cudaGraphConditionalHandle)K[0].h, cudaGraphCondTypeIf);
  I[1] = add_conditional(s_, (cudaGraphConditionalHandle)K[1].h, cudaGraphCondTypeIf);
  cuda_check(cudaStreamEndCapture(s_, &B), "end capture");
  for (int k = 0; k < 2; ++k) {
    CgVectors v{n_, gbuf(k), use_m ? M_.p : nullptr, d_.p, r0_.p, r1_.p, p_.p, hp_.p};
    const Cond ck = make_cond(I[k], 0, 0);
    begin_capture(s_, I[k]);
    uint64_t before = launches;
    if (use_m) precond_kernels(slot_[k]);  // recomputed per iteration: same bits as cached
    tr_prep(ss, st_d_, s_);
    count_launch(1);
    capture_cg_init(k, v, ck);
    cudaGraph_t W = add_conditional(s_, (cudaGraphConditionalHandle)ck.h, cudaGraphCondTypeWhile);
    const int saved = cand_;
    cand_ = k ^ 1;
    eval_candidate_dev(d_.p, /*read=*/false);  // slot k^1: w_k + d, margin pass
    gradient_into(slot_[k ^ 1], gbuf(k ^ 1));  // speculative gradient
    cand_ = saved;
    tr_update(ss, st_d_, obj_d_, k, outer, K[k ^ 1], s_);
    count_launch(1);
    outer_kernels_ = launches - before;
    cuda_check(cudaStreamEndCapture(s_, &I[k]), "end capture");
    begin_capture(s_, W);
    before = launches;
    capture_cg_body(k, v, ck);
    body_kernels_ = launches - before;
    cuda_check(cudaStreamEndCapture(s_, &W), "end capture");
  }
  launches = saved_launches;
  cudaGraphExec_t exec;
  cuda_check(cudaGraphInstantiate(&exec, top, 0), "solve graph instantiate");
  solve_graph_[use_m] = top;
  solve_exec_[use_m] = exec;
}

// The outer loop after the initial commit: one H2D of the solver scalars, one
// graph launch, one D2H of the scalars and the iteration records.
void Engine::solve_device_loop(const tron_config& cfg, double f, tron_solve_info* info,
                               tron_iteration* trace, uint64_t cap, int* status, std::string* what) {
  static_assert(sizeof(TrRecord) == sizeof(tron_iteration), "TrRecord mirrors tron_iteration");
  static_assert(sizeof(SolveState) <= 256, "pinned block size");
  AllocScope scope(s_);
  const bool use_m = cfg.use_preconditioner != 0;
  constexpr uint64_t kInlineRecords = 64;  // read back together with the scalars
  const uint64_t want = std::max<uint64_t>(std::min<uint64_t>(cap, cfg.max_outer_iters), 1);
  if (trace_buf_.n < want) trace_buf_.alloc(std::max<uint64_t>(want, kInlineRecords));
  if (!solve_exec_[use_m]) build_solve_graph(use_m);
  SolveState& S = *ss_h_;
  std::memset(&S, 0, sizeof(S));
  uint64_t max_cg = cfg.max_cg_iters;
  if (max_cg == 0) max_cg = (uint64_t)n_ < 1000 ? (uint64_t)n_ : 1000;  // tron.cpp:40-41
  S.cfg = TrConfig{cfg.eps, cfg.sigma0, cfg.eta1, cfg.eta2, cfg.gamma1, cfg.gamma2, cfg.gamma3,
                   cfg.cg_tol, C_, (long long)cfg.max_outer_iters, (long long)max_cg,
                   use_m ? 1 : 0, comm_.active() ? 1 : 0};
  S.f = f;
  S.delta = gnorm_;  // tron.cpp:159
  S.gnorm = gnorm_;
  S.gnorm0 = gnorm_;
  S.committed = cand_ ^ 1;
  S.cont = cfg.max_outer_iters > 0;
  S.trace = trace_buf_.p;
  S.cap = (long long)trace_buf_.n;
  info->hessian_products = 0;
  if (S.cont) {
    cuda_check(cudaMemcpyAsync(ss_buf_.p, &S, sizeof(S), cudaMemcpyHostToDevice, s_), "H2D");
    cuda_check(cudaGraphLaunch(solve_exec_[use_m], s_), "solve graph launch");
    cuda_check(cudaMemcpyAsync(&S, ss_buf_.p, sizeof(S), cudaMemcpyDeviceToHost, s_), "D2H");
    const uint64_t inline_n = std::min<uint64_t>(std::min<uint64_t>(cap, kInlineRecords), trace_buf_.n);
    if (trace && inline_n)
      cuda_check(cudaMemcpyAsync(trace, trace_buf_.p, inline_n * sizeof(TrRecord), cudaMemcpyDeviceToHost,
                                 s_),
                 "D2H");
    synchronize();
    cuda_check(cudaGetLastError(), "solve graph");
    const uint64_t nrec = std::min<uint64_t>((uint64_t)S.n_iter, cap);
    if (trace && nrec > inline_n) {
      cuda_check(cudaMemcpyAsync(trace + inline_n, trace_buf_.p + inline_n,
                                 (nrec - inline_n) * sizeof(TrRecord), cudaMemcpyDeviceToHost, s_),
                 "D2H");
      synchronize();
    }
  }
  // the committed slot and its gradient (g[k] -> g_ for gradient())
  cand_ = S.committed ^ 1;
  slot_[cand_].valid = false;
  slot_[cand_ ^ 1].f = S.f;
  committed_valid_ = true;
  precond_valid_ = false;
  if (S.committed == 1)
    cuda_check(cudaMemcpyAsync(g_.p, gspec_.p, n_ * sizeof(double), cudaMemcpyDeviceToDevice, s_), "D2D");
  gnorm_ = S.gnorm;
  info->n_iterations = (uint64_t)S.n_iter;
  info->accepted_steps = (uint64_t)S.accepted;
  info->objective_evaluations += (uint64_t)S.obj_evals;
  info->gradient_materializations += (uint64_t)S.grad_mats;
  info->objective = S.f;
  info->converged = S.converged;
  info->hessian_products = (uint64_t)S.hv_count;
  ledger.margin_passes += (uint64_t)S.obj_evals;
  ledger.scalar_returns += (uint64_t)S.obj_evals;
  ledger.gradient_materializations += (uint64_t)S.grad_mats;
  if (loss_ == TRON_LOSS_L2SVM)
    ledger.index_set_bytes = std::max<uint64_t>(ledger.index_set_bytes, (uint64_t)S.max_nact * 8);
  launches += 1 + (uint64_t)(S.obj_evals + (S.status == kTrFailCg)) * (outer_kernels_ + 1) +
              (uint64_t)S.hv_count * body_kernels_;
  *status = TRON_OK;
  if (S.status == kTrFailCg) {
    *status = TRON_ERR_NUMERICAL;
    *what = "conjugate gradients met non-positive curvature (" + std::to_string(S.fail_php) + ")";
  } else if (S.status == kTrFailObjective) {
    *status = TRON_ERR_NUMERICAL;
    *what = "objective is not finite at a candidate step";
  } else if (S.status == kTrFailGradient) {
    *status = TRON_ERR_NUMERICAL;
    *what = "gradient is not finite after an accepted step";
  }
}

// ----------------------------------------------------------------------------
// predict (model.cpp:88-117)
// ----------------------------------------------------------------------------
uint64_t Engine::predict(const double* w, double* labels) {
  AllocScope scope(s_);
  DevBuf<double> lab;
  lab.alloc(l_ > 0 ? l_ : 1);
  DevBuf<unsigned long long> correct;
  correct.alloc(1);
  if (n_ > 0) upload(vtmp_.p, w, n_ * sizeof(double), s_);
  unsigned long long c = 0;
  if (dense_ && ooc_) {
    DevBuf<unsigned long long> per;
    per.alloc((size_t)std::max<int64_t>(nblk_, 1));
    ooc_pass([&](int64_t b, int64_t r0, int64_t rows, const double* win, const CUtensorMap&) {
      predict_dense(rows, n_, blk_, win, vtmp_.p, y_.p + r0, lab.p + r0, per.p + b, s_);
    });
    std::vector<unsigned long long> h((size_t)nblk_);
    if (nblk_) cuda_check(cudaMemcpyAsync(h.data(), per.p, nblk_ * sizeof(unsigned long long),
                                          cudaMemcpyDeviceToHost, s_), "D2H");
    synchronize();
    for (auto x : h) c += x;
  } else if (colpart_) {  // scores = sum over ranks of X_{:,r} w_r
    csr_dv(X_, group_, vtmp_.p, nullptr, nullptr, a_.p, s_);
    comm_.allreduce_sum(a_.p, (size_t)l_, s_);
    predict_from_scores(l_, a_.p, y_.p, lab.p, correct.p, s_);
    count_launch(2);
    cuda_check(cudaMemcpyAsync(&c, correct.p, sizeof(c), cudaMemcpyDeviceToHost, s_), "D2H");
  } else {
    if (dense_)
      predict_dense(l_, n_, ld_, Xc_.p, vtmp_.p, y_.p, lab.p, correct.p, s_);
    else
      predict_csr(X_, vtmp_.p, y_.p, lab.p, correct.p, s_);
    count_launch(1);
    cuda_check(cudaMemcpyAsync(&c, correct.p, sizeof(c), cudaMemcpyDeviceToHost, s_), "D2H");
  }
  if (labels && l_ > 0) download(labels, lab.p, l_ * sizeof(double), s_);
  synchronize();
  cuda_check(cudaGetLastError(), "predict");
  return c;
}

// ----------------------------------------------------------------------------
// per-kernel timing for the roofline figures of bench.py
// ----------------------------------------------------------------------------
void Engine::bench_kernels(int reps, bool flush_l2, KernelTimes* out) {
  AllocScope scope(s_);
  if (!committed_valid_) raise(TRON_ERR_LOGIC, "bench_kernels() needs a committed state");
  if (flush_l2 && flush_.n == 0) {
    flush_.alloc((size_t)(256u << 20) / 8);  // 256 MiB > L2
    cuda_check(cudaMemsetAsync(flush_.p, 0, flush_.bytes(), s_), "flush init");
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time_it = [&](auto&& fn) {
    double total = 0.0;
    for (int r = 0; r < reps; ++r) {
      // read-based eviction: cold L2, nothing dirty left to write back inside
      // the timed launch (the solve's own kernels leave clean lines too)
      if (flush_l2) l2_read_flush(flush_.p, (int64_t)flush_.n, s_);
      cudaEventRecord(a, s_);
      fn();
      cudaEventRecord(b, s_);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      total += ms;
    }
    return total / std::max(reps, 1);
  };
  cuda_check(cudaMemcpyAsync(vtmp_.p, g_.p, n_ * 8, cudaMemcpyDeviceToDevice, s_), "D2D");
  if (dense_ && gram_) ensure_gram(slot_[cand_ ^ 1]);  // Hv times the product from a current G
  out->hv_ms = time_it([&] { hv_kernels(vtmp_.p, otmp_.p); });
  const Slot& S = slot_[cand_ ^ 1];
  if (!dense_) {
    UView u;
    u.kind = U_VEC;
    u.u = a_.p;
    EpiView epi;
    epi.kind = EPI_VEC;
    epi.base = vtmp_.p;
    epi.scale = C_;
    out->transposed_ms = time_it([&] { csc_spmv(Xt_, plan_, u, false, epi, otmp_.p, s_); });
    out->forward_ms = time_it([&] { forward(slot_[cand_]); });
  } else if (ooc_) {  // every pass streams X: the Hv is the streamed accumulation
    out->transposed_ms = out->hv_ms;
    out->forward_ms = time_it([&] { forward(slot_[cand_]); });
  } else {
    const int loss = loss_ == TRON_LOSS_LOGISTIC ? kLossLogistic : kLossSvm;
    out->transposed_ms = time_it([&] {
      dense_accum(DA_HV, l_, n_, ld_, Xc_.p, xmap_, loss, vtmp_.p, S.dvec.p, S.mask.p, parts_.p, s_);
    });
    // delta mode: the candidate slot's own iterate (after a solve: the one
    // before the last commit) against the committed G -- a pass that updates G
    // by the rows of the last commit's change, not a no-change pass
    const double* wf = gram_delta_ ? slot_[cand_].w.p : S.w.p;
    out->forward_ms = time_it([&] {
      dense_forward(l_, n_, ld_, Xc_.p, xmap_, loss, wf, y_.p, C_, slot_[cand_].z.p,
                    slot_[cand_].zhat.p, slot_[cand_].dvec.p, slot_[cand_].mask.p,
                    slot_[cand_].gparts.p, obj_d_, sc_, s_,
                    gram_fused_ ? slot_[cand_].gram_parts.p : gram_delta_ ? slot_[cand_].gram_dparts.p : nullptr,
                    gram_delta_ ? S.mask.p : nullptr, gram_delta_ ? S.gram_flags.p : nullptr);
    });
  }
  // Gram mode: the gradient plus the committed iterate's G formed afresh -- by
  // the Gram pass, or (delta mode, TRON_B200_GRAM_FIRST fused) by the margin
  // pass that forms G whole, as a solve's first pass does
  out->grad_ms = time_it([&] {
    gradient_dev();
    if (dense_ && gram_ && !gram_fused_) {
      if (gram_delta_ && gram_first_fused_) {
        Slot& C = slot_[cand_];
        dense_forward(l_, n_, ld_, Xc_.p, xmap_, kLossSvm, S.w.p, y_.p, C_, C.z.p, C.zhat.p, C.dvec.p, C.mask.p,
                      C.gparts.p, obj_d_, sc_, s_, C.gram_dparts.p);
        cuda_check(cudaMemsetAsync(C.gram_flags.p, 0xff, sizeof(int), s_), "memset");
        gram_finalize(n_, C.gram_dparts.p, dense_grid(l_, n_), C.gram.p, s_, C.gram_flags.p);
      } else {
        cuda_check(cudaMemsetAsync(S.gram_flags.p, 0xff, sizeof(int), s_), "memset");
        ensure_gram(S);
      }
    }
  });
  slot_[cand_].valid = false;  // forward timing overwrote the candidate slot
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  synchronize();
}

}  // namespace tb
