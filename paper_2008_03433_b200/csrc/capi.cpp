// extern "C" entry points of libtron_b200.so (declared in include/tron_b200.h).
// C++ exceptions never cross this boundary: each call maps them to a
// tron_status and records the message for tron_gpu_last_error().
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "engine.h"
#include "ingest.h"
#include "tron_b200.h"
#include "tron_b200.hpp"

struct tron_gpu_ctx {
  std::unique_ptr<tb::Engine> engine;
};

struct tron_parsed {
  tb::ParsedProblem p;
};

namespace {

thread_local std::string g_last_error;
thread_local uint64_t g_last_error_line = 0;

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  g_last_error_line = 0;
  return status;
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    g_last_error.clear();
    return TRON_OK;
  } catch (const tb::StatusError& e) {
    return fail(e.status, e.what());
  } catch (const tb::ParseFailure& e) {
    const int st = fail(e.status, e.what());
    g_last_error_line = e.line;
    return st;
  } catch (const tron_b200::NumericalFailureError& e) {
    return fail(TRON_ERR_NUMERICAL, e.what());
  } catch (const tron_b200::BudgetExceededError& e) {
    return fail(TRON_ERR_BUDGET, e.what());
  } catch (const tron_b200::StrategyPreconditionError& e) {
    return fail(TRON_ERR_STRATEGY, e.what());
  } catch (const tron_b200::BoundsError& e) {
    return fail(TRON_ERR_BOUNDS, e.what());
  } catch (const tron_b200::DimensionError& e) {
    return fail(TRON_ERR_DIMENSION, e.what());
  } catch (const std::logic_error& e) {
    return fail(TRON_ERR_LOGIC, e.what());
  } catch (const std::bad_alloc& e) {
    return fail(TRON_ERR_OOM, e.what());
  } catch (const std::exception& e) {
    return fail(TRON_ERR_CUDA, e.what());
  }
}

// Every context entry point runs on the context's device (the current device
// is per host thread; another context may have changed it) and restores the
// caller's current device on return.
#define NEED_CTX(ctx)                                                              \
  if (!(ctx) || !(ctx)->engine) return fail(TRON_ERR_ARGUMENT, "null context");    \
  tb::DeviceGuard device_guard_((ctx)->engine->device())

// LossEvaluator over the engine, used by the host-CG parity mode so that
// the reference control flow (solver.cpp) drives the device kernels.
class EngineEvaluator final : public tron_b200::LossEvaluator {
 public:
  explicit EngineEvaluator(tb::Engine& e) : e_(e) {}
  std::size_t dimension() const override { return (std::size_t)e_.dimension(); }
  double eval_candidate(const tron_b200::RealVector& w) override {
    return e_.eval_candidate_host(w.data());
  }
  void commit() override {
    e_.commit(nullptr);
    g_.resize(dimension());
    e_.gradient_host(g_.data());
    e_.ledger.bulk_handoffs++;  // the length-n gradient crosses to the host CG
    pv_ = false;
  }
  const tron_b200::RealVector& gradient() const override { return g_; }
  void hessian_vec(const tron_b200::RealVector& v, tron_b200::RealVector& out) override {
    out.resize(dimension());
    e_.hessian_vec_host(v.data(), out.data());
  }
  const tron_b200::RealVector& precond_diagonal() override {
    if (!pv_) {
      m_.resize(dimension());
      e_.precond_host(m_.data());
      e_.ledger.bulk_handoffs++;
      pv_ = true;
    }
    return m_;
  }

 private:
  tb::Engine& e_;
  tron_b200::RealVector g_, m_;
  bool pv_ = false;
};

void to_cfg(const tron_config& c, tron_b200::TrustRegionConfig* out) {
  out->eps = c.eps;
  out->max_outer_iters = c.max_outer_iters;
  out->max_cg_iters = c.max_cg_iters;
  out->sigma0 = c.sigma0;
  out->eta1 = c.eta1;
  out->eta2 = c.eta2;
  out->gamma1 = c.gamma1;
  out->gamma2 = c.gamma2;
  out->gamma3 = c.gamma3;
  out->cg_tol = c.cg_tol;
  out->use_preconditioner = c.use_preconditioner != 0;
}

void fill_trace(const tron_b200::SolverTrace& t, tron_solve_info* info, tron_iteration* trace,
                uint64_t cap) {
  info->f_initial = t.f_initial;
  info->gradient_norm_initial = t.gradient_norm_initial;
  info->accepted_steps = t.accepted_steps;
  info->gradient_materializations = t.gradient_materializations;
  info->objective_evaluations = t.objective_evaluations;
  info->n_iterations = t.iterations.size();
  for (uint64_t k = 0; k < t.iterations.size() && trace && k < cap; ++k) {
    const auto& r = t.iterations[k];
    trace[k].f_candidate = r.f_candidate;
    trace[k].gradient_norm = r.gradient_norm;
    trace[k].delta = r.delta;
    trace[k].sigma = r.sigma;
    trace[k].accepted = r.accepted;
    trace[k].cg_iters = r.cg_iters;
    trace[k].cg_exit = (int32_t)r.cg_exit;
  }
}

}  // namespace

extern "C" {

void tron_gpu_default_config(tron_config* c) {
  c->eps = 0.1;
  c->max_outer_iters = 1000;
  c->max_cg_iters = 0;
  c->sigma0 = 1e-4;
  c->eta1 = 0.25;
  c->eta2 = 0.75;
  c->gamma1 = 0.25;
  c->gamma2 = 0.5;
  c->gamma3 = 4.0;
  c->cg_tol = 0.1;
  c->use_preconditioner = 0;
  c->solve_mode = TRON_SOLVE_DEVICE;
}

void tron_gpu_default_options(tron_gpu_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->device = 0;
  o->svm_strategy = TRON_SVM_INDIRECT;
  o->gathered_budget_bytes = uint64_t{2} << 30;
  o->rank = 0;
  o->world = 1;
  o->nccl_unique_id = nullptr;
  o->row_begin = 0;
  o->global_rows = 0;
  o->reference_order = 0;
  o->host_allreduce = nullptr;
  o->host_allreduce_user = nullptr;
  o->out_of_core = 0;
  o->stream_block_rows = 0;
  o->partition = TRON_PARTITION_ROWS;
  o->col_begin = 0;
  o->global_cols = 0;
}

const char* tron_gpu_last_error(void) { return g_last_error.c_str(); }
uint64_t tron_gpu_last_error_line(void) { return g_last_error_line; }

int tron_parse_libsvm(const char* text, uint64_t len, uint64_t n_override, tron_parsed** out) {
  tb::NvtxRange nvtx_range("tron_parse_libsvm");
  if (!out || (!text && len > 0)) return fail(TRON_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<tron_parsed>();
    h->p = tb::parse_libsvm_buffer(text ? text : "", len, n_override);
    *out = h.release();
  });
}

int tron_parse_libsvm_file(const char* path, uint64_t n_override, tron_parsed** out) {
  tb::NvtxRange nvtx_range("tron_parse_libsvm_file");
  if (!out || !path) return fail(TRON_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<tron_parsed>();
    h->p = tb::parse_libsvm_file(path, n_override);
    *out = h.release();
  });
}

int tron_parsed_sizes(const tron_parsed* p, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
  if (!p) return fail(TRON_ERR_ARGUMENT, "null parse handle");
  if (rows) *rows = p->p.y.size();
  if (cols) *cols = p->p.cols;
  if (nnz) *nnz = p->p.values.size();
  return TRON_OK;
}

int tron_parsed_copy(const tron_parsed* p, int64_t* row_offsets, int32_t* col_indices,
                     double* values, double* y) {
  if (!p) return fail(TRON_ERR_ARGUMENT, "null parse handle");
  const auto& q = p->p;
  if (row_offsets) std::memcpy(row_offsets, q.row_offsets.data(), q.row_offsets.size() * 8);
  if (col_indices) std::memcpy(col_indices, q.col_indices.data(), q.col_indices.size() * 4);
  if (values) std::memcpy(values, q.values.data(), q.values.size() * 8);
  if (y) std::memcpy(y, q.y.data(), q.y.size() * 8);
  return TRON_OK;
}

int tron_load_dense(const char* text, uint64_t len, uint64_t n, tron_parsed** out) {
  tb::NvtxRange nvtx_range("tron_load_dense");
  if (!out || (!text && len > 0)) return fail(TRON_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<tron_parsed>();
    h->p = tb::load_dense_buffer(text ? text : "", len, n);
    *out = h.release();
  });
}

int tron_load_dense_file(const char* path, uint64_t n, tron_parsed** out) {
  tb::NvtxRange nvtx_range("tron_load_dense_file");
  if (!out || !path) return fail(TRON_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<tron_parsed>();
    h->p = tb::load_dense_file(path, n);
    *out = h.release();
  });
}

int tron_parsed_layout(const tron_parsed* p, int32_t* dense) {
  if (!p) return fail(TRON_ERR_ARGUMENT, "null parse handle");
  if (dense) *dense = p->p.dense ? 1 : 0;
  return TRON_OK;
}

int tron_parsed_save_binary(const tron_parsed* p, const char* path) {
  if (!p || !path) return fail(TRON_ERR_ARGUMENT, "null argument");
  return guarded([&] { tb::save_binary(p->p, path); });
}

int tron_load_binary(const char* path, tron_parsed** out) {
  tb::NvtxRange nvtx_range("tron_load_binary");
  if (!out || !path) return fail(TRON_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<tron_parsed>();
    h->p = tb::load_binary(path);
    *out = h.release();
  });
}

void tron_parsed_free(tron_parsed* p) { delete p; }

void* tron_host_alloc(uint64_t bytes) {
  try {
    return tb::pinned_pool_get((size_t)bytes);
  } catch (const std::exception& e) {
    fail(TRON_ERR_OOM, e.what());
    return nullptr;
  }
}

void tron_host_free(void* p) { tb::pinned_pool_put(p); }

int tron_gpu_device_count(int* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return fail(TRON_ERR_CUDA, cudaGetErrorString(e));
  }
  *count = c;
  return TRON_OK;
}

int tron_gpu_create_csr(int loss, uint64_t l, uint64_t n, const int64_t* row_offsets,
                        const int32_t* col_indices, const double* values, const double* y,
                        double C, const tron_gpu_options* opt, tron_gpu_ctx** out) {
  tb::NvtxRange nvtx_range("tron_gpu_create_csr");
  if (!out) return fail(TRON_ERR_ARGUMENT, "null output handle");
  *out = nullptr;
  return guarded([&] {
    tron_gpu_options o;
    tron_gpu_default_options(&o);
    if (opt) o = *opt;
    tb::DeviceGuard restore(-1);  // creation selects o.device; the caller's device comes back
    auto ctx = std::make_unique<tron_gpu_ctx>();
    ctx->engine = tb::Engine::create_csr(loss, l, n, row_offsets, col_indices, values, y, C, o);
    *out = ctx.release();
  });
}

int tron_gpu_create_dense(int loss, uint64_t l, uint64_t n, const double* row_major,
                          const double* y, double C, const tron_gpu_options* opt,
                          tron_gpu_ctx** out) {
  tb::NvtxRange nvtx_range("tron_gpu_create_dense");
  if (!out) return fail(TRON_ERR_ARGUMENT, "null output handle");
  *out = nullptr;
  return guarded([&] {
    tron_gpu_options o;
    tron_gpu_default_options(&o);
    if (opt) o = *opt;
    tb::DeviceGuard restore(-1);  // creation selects o.device; the caller's device comes back
    auto ctx = std::make_unique<tron_gpu_ctx>();
    ctx->engine = tb::Engine::create_dense(loss, l, n, row_major, y, C, o);
    *out = ctx.release();
  });
}

void tron_gpu_destroy(tron_gpu_ctx* ctx) {
  if (!ctx) return;
  if (ctx->engine) {
    tb::DeviceGuard device_guard_(ctx->engine->device());
    ctx->engine.reset();
  }
  delete ctx;
}

int tron_gpu_dimension(tron_gpu_ctx* ctx, uint64_t* n) {
  NEED_CTX(ctx);
  *n = (uint64_t)ctx->engine->dimension();
  return TRON_OK;
}

int tron_gpu_eval_candidate(tron_gpu_ctx* ctx, const double* w, double* f) {
  tb::NvtxRange nvtx_range("tron_gpu_eval_candidate");
  NEED_CTX(ctx);
  return guarded([&] { *f = ctx->engine->eval_candidate_host(w); });
}

int tron_gpu_commit(tron_gpu_ctx* ctx, double* gnorm) {
  tb::NvtxRange nvtx_range("tron_gpu_commit");
  NEED_CTX(ctx);
  return guarded([&] { ctx->engine->commit(gnorm); });
}

int tron_gpu_gradient(tron_gpu_ctx* ctx, double* g) {
  NEED_CTX(ctx);
  return guarded([&] {
    ctx->engine->gradient_host(g);
    ctx->engine->ledger.bulk_handoffs++;
  });
}

int tron_gpu_hessian_vec(tron_gpu_ctx* ctx, const double* v, double* out) {
  tb::NvtxRange nvtx_range("tron_gpu_hessian_vec");
  NEED_CTX(ctx);
  return guarded([&] { ctx->engine->hessian_vec_host(v, out); });
}

int tron_gpu_quadratic_model(tron_gpu_ctx* ctx, const double* d, double* q) {
  tb::NvtxRange nvtx_range("tron_gpu_quadratic_model");
  NEED_CTX(ctx);
  return guarded([&] {
    const double v = ctx->engine->quadratic_model_host(d);
    if (q) *q = v;
  });
}

int tron_gpu_replica_checksum(tron_gpu_ctx* ctx, double out[4]) {
  NEED_CTX(ctx);
  if (!out) return fail(TRON_ERR_ARGUMENT, "replica_checksum: out is null");
  return guarded([&] { ctx->engine->replica_checksum_host(out); });
}

int tron_gpu_precond_diagonal(tron_gpu_ctx* ctx, double* m) {
  tb::NvtxRange nvtx_range("tron_gpu_precond_diagonal");
  NEED_CTX(ctx);
  return guarded([&] {
    ctx->engine->precond_host(m);
    ctx->engine->ledger.bulk_handoffs++;
  });
}

int tron_gpu_state_lr(tron_gpu_ctx* ctx, int which, double* z, double* zhat, double* dvec) {
  NEED_CTX(ctx);
  return guarded([&] { ctx->engine->state_lr(which, z, zhat, dvec); });
}

int tron_gpu_state_svm(tron_gpu_ctx* ctx, int which, double* z, int64_t* active, uint64_t cap,
                       uint64_t* n_active) {
  NEED_CTX(ctx);
  return guarded([&] { ctx->engine->state_svm(which, z, active, cap, n_active); });
}

int tron_gpu_truncated_cg(tron_gpu_ctx* ctx, double delta, const tron_config* cfg, double* d,
                          int32_t* exit_kind, uint64_t* iters, double* model_value) {
  tb::NvtxRange nvtx_range("tron_gpu_truncated_cg");
  NEED_CTX(ctx);
  return guarded([&] {
    tron_config c;
    tron_gpu_default_config(&c);
    if (cfg) c = *cfg;
    ctx->engine->truncated_cg(delta, c, d, exit_kind, iters, model_value);
  });
}

int tron_gpu_solve(tron_gpu_ctx* ctx, const tron_config* cfg, const double* w0, double* w_out,
                   tron_solve_info* info, tron_iteration* trace, uint64_t trace_cap) {
  tb::NvtxRange nvtx_range("tron_gpu_solve");
  NEED_CTX(ctx);
  if (!info) return fail(TRON_ERR_ARGUMENT, "null info");
  tron_config c;
  tron_gpu_default_config(&c);
  if (cfg) c = *cfg;
  std::memset(info, 0, sizeof(*info));
  if (c.solve_mode == TRON_SOLVE_HOST_CG) {
    const auto t0 = std::chrono::steady_clock::now();
    int st = TRON_OK;
    tron_b200::SolverTrace partial;
    bool have_partial = false;
    st = guarded([&] {
      EngineEvaluator ev(*ctx->engine);
      tron_b200::TrustRegionConfig tc;
      to_cfg(c, &tc);
      tron_b200::RealVector warm;
      if (w0) warm.assign(w0, w0 + ctx->engine->dimension());
      try {
        auto res = tron_b200::solve(ev, tc, w0 ? &warm : nullptr);
        fill_trace(res.trace, info, trace, trace_cap);
        info->objective = res.objective;
        info->converged = res.converged;
        if (w_out) std::memcpy(w_out, res.w.data(), res.w.size() * sizeof(double));
      } catch (const tron_b200::NumericalFailureError& e) {
        partial = e.trace();
        have_partial = true;
        throw;
      }
    });
    if (have_partial) fill_trace(partial, info, trace, trace_cap);
    info->status = st;
    info->device_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return st;
  }
  const int st = guarded([&] { ctx->engine->solve_device(c, w0, w_out, info, trace, trace_cap); });
  info->status = st;
  return st;
}

int tron_gpu_predict(tron_gpu_ctx* ctx, const double* w, double* labels, uint64_t* correct) {
  tb::NvtxRange nvtx_range("tron_gpu_predict");
  NEED_CTX(ctx);
  if (!w && ctx->engine->dimension() > 0) return fail(TRON_ERR_ARGUMENT, "null weights");
  return guarded([&] {
    const uint64_t c = ctx->engine->predict(w, labels);
    if (correct) *correct = c;
  });
}

int tron_gpu_ledger(tron_gpu_ctx* ctx, tron_ledger* out) {
  NEED_CTX(ctx);
  *out = ctx->engine->ledger;
  return TRON_OK;
}

int tron_gpu_reset_ledger(tron_gpu_ctx* ctx) {
  NEED_CTX(ctx);
  ctx->engine->ledger = tron_ledger{};
  return TRON_OK;
}

int tron_gpu_bench_kernels(tron_gpu_ctx* ctx, int reps, int flush_l2, double out_ms[4]) {
  NEED_CTX(ctx);
  return guarded([&] {
    tb::KernelTimes t;
    ctx->engine->bench_kernels(reps, flush_l2 != 0, &t);
    out_ms[0] = t.hv_ms;
    out_ms[1] = t.transposed_ms;
    out_ms[2] = t.forward_ms;
    out_ms[3] = t.grad_ms;
  });
}

int tron_gpu_mode(tron_gpu_ctx* ctx, uint32_t* flags) {
  NEED_CTX(ctx);
  if (flags) *flags = ctx->engine->mode_flags();
  return TRON_OK;
}

int tron_gpu_memory_bytes(tron_gpu_ctx* ctx, uint64_t* bytes) {
  NEED_CTX(ctx);
  *bytes = ctx->engine->memory_bytes();
  return TRON_OK;
}

int tron_gpu_launch_count(tron_gpu_ctx* ctx, uint64_t* count) {
  NEED_CTX(ctx);
  *count = ctx->engine->launches;
  return TRON_OK;
}

int tron_gpu_synchronize(tron_gpu_ctx* ctx) {
  NEED_CTX(ctx);
  return guarded([&] { ctx->engine->synchronize(); });
}

int tron_gpu_nccl_unique_id(void* out128) {
  return guarded([&] { tb::nccl_unique_id(out128); });
}

}  // extern "C"
