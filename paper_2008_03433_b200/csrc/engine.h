// Device-resident state of one TRON problem shard and the host-side
// orchestration of the hot path (the B200 counterpart of the reference's
// LogisticEvaluator / SvmEvaluator, proj/src/backend.cpp:136-306).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hostio.h"
#include "kernels.h"
#include "tron_b200.h"

namespace tb {

// NVTX range over a scope (header-only NVTX 3: a no-op unless a profiler such
// as Nsight Systems attaches): every C-ABI entry and the solve's phases.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct StatusError : std::runtime_error {
  int status;
  StatusError(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] void raise(int status, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);

// Device buffer from the stream-ordered pool (hostio.h): allocated and
// freed in the order of the stream current at alloc() (AllocScope).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    s = alloc_stream();
    if (count)
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s),
                 "cudaMallocAsync");
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Makes `device` current for the guard's lifetime (device < 0: leaves it
// as is), then restores the caller's current device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
      return;
    }
    if (device < 0) return;
    if (prev == device) {
      prev = -1;
      return;
    }
    cudaSetDevice(device);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Owns the context stream; declared first in Engine so it is destroyed after
// every DevBuf member has queued its free on it.
struct StreamOwner {
  cudaStream_t s = nullptr;
  StreamOwner() = default;
  StreamOwner(const StreamOwner&) = delete;
  StreamOwner& operator=(const StreamOwner&) = delete;
  ~StreamOwner() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

// Lazily-loaded NCCL (libnccl.so.2) for the row-sharded multi-GPU layout.
// Or, when the caller supplies tron_gpu_options::host_allreduce, a host data
// plane: the partials are staged through pinned memory and summed by the
// caller's collective (MPI, gloo, ...); such a context is never captured
// into graphs (the CG loop runs host-driven).
class Comm {
 public:
  int rank = 0, world = 1;
  void init(const tron_gpu_options& opt);
  ~Comm();
  void allreduce_sum(double* buf, size_t count, cudaStream_t s);
  // out-of-place (idempotent: recv = sum of the ranks' send)
  void allreduce_sum(const double* send, double* recv, size_t count, cudaStream_t s);
  bool active() const { return world > 1 || forced; }
  bool host() const { return host_fn_ != nullptr && world > 1; }
  bool forced = false;  // one-rank communicator forced on (TRON_B200_FORCE_NCCL=1)

 private:
  void* comm_ = nullptr;
  void (*host_fn_)(void*, double*, uint64_t) = nullptr;
  void* host_user_ = nullptr;
  double* stage_ = nullptr;  // pinned (tron_host_alloc pool)
  size_t stage_n_ = 0;
};
int nccl_unique_id(void* out128);

struct KernelTimes {
  double hv_ms = 0, transposed_ms = 0, forward_ms = 0, grad_ms = 0;
};

class Engine {
 public:
  static std::unique_ptr<Engine> create_csr(int loss, uint64_t l, uint64_t n, const int64_t* ro,
                                            const int32_t* ci, const double* vals, const double* y,
                                            double C, const tron_gpu_options& opt);
  static std::unique_ptr<Engine> create_dense(int loss, uint64_t l, uint64_t n,
                                              const double* row_major, const double* y, double C,
                                              const tron_gpu_options& opt);
  ~Engine();

  int64_t dimension() const { return n_; }
  int loss() const { return loss_; }
  int device() const { return device_; }
  bool dense() const { return dense_; }

  // LossEvaluator surface (host vectors).
  double eval_candidate_host(const double* w);
  void commit(double* gnorm);
  void gradient_host(double* g);
  void hessian_vec_host(const double* v, double* out);
  void precond_host(double* m);
  double quadratic_model_host(const double* d);
  // this replica's checksum of the committed w (replica_checksum's four chunks)
  void replica_checksum_host(double out4[4]);
  void state_lr(int which, double* z, double* zhat, double* dvec);
  void state_svm(int which, double* z, int64_t* active, uint64_t cap, uint64_t* n_active);
  void truncated_cg(double delta, const tron_config& cfg, double* d, int32_t* exit_kind,
                    uint64_t* iters, double* q);
  void solve_device(const tron_config& cfg, const double* w0, double* w_out, tron_solve_info* info,
                    tron_iteration* trace, uint64_t cap);
  void bench_kernels(int reps, bool flush_l2, KernelTimes* out);
  // predict (model.cpp:88-117) of this context's rows under host weights w.
  uint64_t predict(const double* w, double* labels);

  tron_ledger ledger{};
  uint64_t launches = 0;
  uint64_t memory_bytes() const;
  uint32_t mode_flags() const;
  void synchronize();

  // Device-side building blocks (also used by the host-CG adapter).
  double eval_candidate_dev(const double* d_step, bool read = true);  // slot[cand].w (+ d_step) -> f
  void hessian_vec_dev(const double* v, double* out);
  void ensure_precond();
  void run_cg(double delta, const tron_config& cfg, CgState* out);

 private:
  Engine() = default;
  StreamOwner stream_owner_;  // first member: destroyed last
  struct Slot {
    DevBuf<double> w, z, zhat, dvec;
    DevBuf<uint8_t> mask;
    DevBuf<double> gparts;  // dense: gradient partials from this slot's margin pass
    DevBuf<int32_t> idx;    // reference order: this slot's active set I (ascending)
    DevBuf<long long> cnt;  // ... and |I| (device)
    DevBuf<double> gram;    // dense Gram mode: this slot's Hessian sum_i c_i x_i x_i^T (n x n)
    DevBuf<double> gram_parts;  // ... its per-CTA partials from the fused margin pass
    DevBuf<int> gram_flags;     // gram.cu's flags: [0] != 0: G does not match the slot's mask
    DevBuf<double> gram_dparts; // L2-SVM: the margin pass's partials of G - G(other slot)
    DevBuf<double> gram_local;  // row-sharded: this rank's part of G (allreduced into gram)
    double f = 0.0;
    long long nact = 0;
    bool valid = false;
  };
  void common_alloc();
  void forward(Slot& S);
  void gradient_dev();
  void transposed_raw_or_epi(const UView& u, bool squared, const EpiView& epi, double* out,
                             const CsrView* At = nullptr, const SegView* plan = nullptr);
  void dense_vector(int kind, const double* v, const EpiView& epi, double* out,
                    const Slot* grad_slot = nullptr);
  void gradient_into(const Slot& S, double* out);
  bool enqueue_cg(double delta, const tron_config& cfg, CgState* out);
  double candidate_result();
  void adopt_candidate();
  void hv_kernels(const double* v, double* out, bool with_dot = false);  // enqueue only
  void gather_active();
  void build_gathered_csr(int nI, long long nnzI);
  int compact(const Slot& S, DevBuf<int32_t>& idx);
  void read_obj();
  void read_cg(CgState* out);
  void build_graph(int slot, bool use_m);
  void launch_cg_graph(int slot, bool use_m);
  // CG pieces captured into the current stream capture (committed slot k)
  void capture_cg_init(int k, const CgVectors& v, Cond cond);
  void ensure_gram(const Slot& S);  // G of slot S, formed only when stale
  void capture_cg_body(int k, const CgVectors& v, Cond cond);
  void precond_kernels(const Slot& S);
  // device-resident outer loop (trloop.cu): one graph per use_m
  bool device_loop_ok() const;
  void build_solve_graph(bool use_m);
  void solve_device_loop(const tron_config& cfg, double f, tron_solve_info* info,
                         tron_iteration* trace, uint64_t cap, int* status, std::string* what);
  double* gbuf(int k) { return k == 0 ? g_.p : gspec_.p; }
  template <class Report>
  void screen(const int32_t* ptr, const int32_t* idx, int64_t rows, int64_t n, Report report);
  void count_launch(uint64_t k) { launches += k; }

  int loss_ = 0;
  bool dense_ = false;
  int64_t l_ = 0, n_ = 0;
  double C_ = 1.0;
  int device_ = 0;
  int svm_strategy_ = TRON_SVM_INDIRECT;
  uint64_t budget_ = 0;
  uint64_t row_begin_ = 0;
  Comm comm_;
  cudaStream_t s_ = nullptr;

  // CSR + CSC (sparse layout)
  DevBuf<int32_t> rptr_, cidx_, cptr_, ridx_;
  DevBuf<double> rval_, cval_;
  DevBuf<uint32_t> lastbits_, chunk_rank_;
  DevBuf<int32_t> empty_col_, chunk_first_, nz_col_, long_fix_;
  DevBuf<double> head_, carry_;
  CsrView X_{}, Xt_{};
  // column panels of X for the row products when v does not fit in L2
  // (K1: 160 MB): panel k = columns [k W, (k+1) W), row i's part located by
  // the split arrays; the row sums accumulate panel by panel in a fixed order
  std::vector<CsrView> panels_;
  std::vector<int> panel_group_;
  DevBuf<int32_t> psplit_[7];
  void setup_panels();
  void row_products(const double* v, const double* dvec, const uint8_t* mask, double* a);
  SegView plan_{};
  int group_ = 4;
  // dense column-major
  DevBuf<double> Xc_;
  int64_t ld_ = 0;
  alignas(64) CUtensorMap xmap_{};  // 2-D TMA descriptor of Xc_
  alignas(64) CUtensorMap gmap_{};  // ... of the gathered panel Xg_
  DevBuf<double> Xg_;  // gathered panel X_{I,:} (Gathered strategy)
  int64_t ldg_ = 0, nI_ = 0;
  bool gathered_valid_ = false;
  // gathered CSR rows X_I (Gathered L2-SVM on sparse features, linalg.cpp:197-229)
  // and their CSC copy + segmented plan, rebuilt at every commit
  DevBuf<int32_t> grptr_, gcidx_, gcptr_, gridx_;
  DevBuf<double> grval_, gcval_;
  DevBuf<uint32_t> glastbits_, gchunk_rank_;
  DevBuf<int32_t> gempty_col_, gchunk_first_, gnz_col_, glong_fix_;
  DevBuf<double> ghead_, gcarry_;
  CsrView Xg_csr_{}, Xgt_{};
  SegView gplan_{};
  bool gathered_csr_valid_ = false;
  // graphs capture the gathered views of the commit they were built for
  uint64_t gathered_epoch_ = 0;
  uint64_t graph_epoch_[2][2] = {{0, 0}, {0, 0}};
  // reference-order reductions (dense L2-SVM, refexact.cu)
  bool ro_ = false;
  alignas(64) CUtensorMap xmap128_{};
  DevBuf<double> ro_parts_, ro_hparts_;
  DevBuf<unsigned> ro_tickets_;
  void ro_accum_slot(int mode, const Slot& S, const double* v, const EpiView& epi, double* out);
  DevBuf<int32_t> idx_, idx_tmp_;
  DevBuf<long long> count_;

  DevBuf<double> y_;
  Slot slot_[2];
  int cand_ = 0;       // candidate slot index; committed = cand_ ^ 1
  bool committed_valid_ = false;
  DevBuf<double> g_, gspec_, M_, d_, r0_, r1_, p_, hp_, a_, raw_, vtmp_, otmp_, parts_;
  bool precond_valid_ = false;
  double gnorm_ = 0.0;

  DevBuf<double> sc_partials_;
  DevBuf<unsigned int> sc_tickets_;
  Scratch sc_{};
  DevBuf<ObjScalars> obj_buf_;
  DevBuf<CgState> st_buf_;
  ObjScalars* obj_d_ = nullptr;
  ObjScalars* obj_h_ = nullptr;  // pinned
  CgState* st_d_ = nullptr;
  CgState* st_h_ = nullptr;  // pinned
  DevBuf<double> flush_;

  // CUDA graphs of the device CG loop: [committed slot][preconditioned]
  cudaGraphExec_t graph_exec_[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  cudaGraph_t graph_[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  uint64_t body_kernels_ = 0;
  bool small_engine_ = false;  // n <= kSmallCgMaxN: single-block CG step
  bool mid_engine_ = false;    // n <= kClusterCgMaxN: one 8-CTA cluster kernel per CG step
  bool coop_engine_ = false;   // otherwise: one cooperative kernel per CG step (cg_coop_step)
  DevBuf<double> dot_parts_, dot_out_;  // p.Hp from the Hv emission (EpiView::dot_*)
  DevBuf<unsigned> dot_ticket_;
  bool hv_dot_available() const;
  DevBuf<double> coop_parts_;  // CTA partials of the cooperative CG step
  bool use_graphs_ = true;
  // dense problems (n <= 64): the Hessian as an n x n matrix formed once per
  // commit (gram.cu); Hv / the preconditioner then read G instead of X
  bool gram_ = false;
  bool gram_fused_ = false;  // n <= 40: G accumulated by the margin pass itself (PM_FWDG)
  // TRON_B200_CHECK_REPLICAS=1 (row shards): after every outer iteration (the
  // device loop: after the solve) the ranks compare checksums of w, f and delta
  bool replica_check_ = false;
  DevBuf<double> rc_;
  void check_replicas(double f, double delta, uint64_t iter);
  bool gram_cg_loop_ = false;  // Gram mode: the whole CG loop is one kernel (cg_small_gram_loop)
  bool gram_delta_ = false;  // L2-SVM, n <= 40: G = G(other slot) + the rows that changed side
  bool gram_first_fused_ = false;  // delta mode: a solve's first margin pass forms G whole (PM_FWDG)
  bool gram_full_next_ = false;    // ... armed by solve_device for its starting point
  DevBuf<double> gram_parts_;
  void gram_slot(const Slot& S);
  // column-partitioned layout: X_, w and the
  // n-vectors are this rank's column slice; z / D / mask are whole (all rows)
  bool colpart_ = false;
  int64_t global_n_ = 0;
  DevBuf<double> cp_dots_;  // scalar exchange buffer
  double gdot(const double* a, const double* b);
  void run_cg_columns(double delta, const tron_config& cfg, CgState* out);
  // out-of-core dense layout: X stays in the caller's
  // host array (page-locked in place) and every pass streams it in blocks of
  // blk_ rows through two device windows, copy (cs_) overlapping compute (s_)
  bool ooc_ = false;
  const double* Xhost_ = nullptr;
  bool host_registered_ = false;
  int64_t blk_ = 0, nblk_ = 0;
  DevBuf<double> win_[2], stage_[2];
  alignas(64) CUtensorMap winmap_[2] = {};
  cudaStream_t cs_ = nullptr;
  cudaEvent_t ev_copied_[2] = {nullptr, nullptr}, ev_free_[2] = {nullptr, nullptr};
  bool ev_free_used_[2] = {false, false};
  DevBuf<double> blk_red_;
  template <class F>
  void ooc_pass(F&& on_block);
  void ooc_setup();
  int dense_nparts() const;
  // device-resident outer loop
  cudaGraphExec_t solve_exec_[2] = {nullptr, nullptr};
  cudaGraph_t solve_graph_[2] = {nullptr, nullptr};
  uint64_t solve_epoch_[2] = {0, 0};
  uint64_t outer_kernels_ = 0;  // kernels per outer iteration outside the CG body
  DevBuf<SolveState> ss_buf_;
  SolveState* ss_h_ = nullptr;  // pinned
  DevBuf<TrRecord> trace_buf_;
};

}  // namespace tb
