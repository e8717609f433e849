// Device-resident outer trust-region loop (tron.cpp:127-217; SURVEY.md §8(f)
// item 1).  The whole solve after the initial commit is ONE graph launch:
//
//   WHILE (outer)                                   -- tron.cpp:161
//     tr_dispatch: IF-conditions from the committed slot
//     IF (committed == 0):  iteration with slot 0 committed, slot 1 candidate
//     IF (committed == 1):  iteration with slot 1 committed, slot 0 candidate
//
// and each iteration body is
//   [preconditioner of the committed slot]           -- tron.cpp:163-164
//   tr_prep (CG inputs: delta, cg_tol*||g||)         -- tron.cpp:55
//   CG init, WHILE (cg) [Hv, CG step]                -- tron.cpp:37-108
//   w_cand = w + d, margin pass, speculative grad    -- tron.cpp:175-178
//   tr_update: sigma, trust_region_update, record,   -- tron.cpp:110-125, 180-213
//              accept (the candidate slot becomes committed: no copy),
//              stopping test, loop conditions.
//
// Slots never move: acceptance flips which IF body runs next.  The committed
// slot's gradient lives in g[k] (two fixed buffers), so adopting the
// speculative gradient costs nothing either.  Only the final scalars, the
// iteration records and w cross PCIe, once per solve.
#include "common.cuh"
#include "kernels.h"

#include <cmath>

namespace tb {

namespace {

__device__ __forceinline__ void cset(Cond c, int v) {
  if (c.on) cudaGraphSetConditional((cudaGraphConditionalHandle)c.h, v ? 1u : 0u);
}

__global__ void tr_dispatch_kernel(const SolveState* S, Cond k0, Cond k1) {
  const int go = S->cont != 0;
  cset(k0, go && S->committed == 0);
  cset(k1, go && S->committed == 1);
}

// CG inputs of this outer iteration (tron.cpp:40-41, :55).
__global__ void tr_prep_kernel(const SolveState* S, CgState* st) {
  st->delta = S->delta;
  st->stop = S->cfg.cg_tol * S->gnorm;
  st->max_iters = S->cfg.max_cg;
  st->use_m = S->cfg.use_m;
}

// tron.cpp:165-213 after the CG and the candidate's margin pass (+ the
// speculative gradient): the reduction ratio, the radius update, the
// iteration record, acceptance and the stopping test.  `k` is the committed
// slot of this body; acceptance commits slot k ^ 1.
__global__ void tr_update_kernel(SolveState* S, const CgState* cg, const ObjScalars* obj, int k,
                                 Cond outer, Cond other) {
  const TrConfig& c = S->cfg;
  S->hv_count += cg->iters;
  int stop = 0;
  if (cg->fail) {  // truncated_cg threw (tron.cpp:166-170): no record
    S->status = kTrFailCg;
    S->fail_php = cg->php;
    stop = 1;
  } else {
    S->obj_evals += 1;
    const double fc = c.sharded ? 0.5 * obj->ww + c.C * obj->red[0] : obj->f;  // loss.cpp:57
    const long long nact = c.sharded ? (long long)obj->red[1] : obj->nact;
    if (nact > S->max_nact) S->max_nact = nact;
    if (!isfinite(fc)) {  // tron.cpp:179-181: no record
      S->status = kTrFailObjective;
      stop = 1;
    } else {
      const double step_norm = cg->dnorm;
      const double sigma = (fc - S->f) / cg->q;
      // trust_region_update (tron.cpp:110-125)
      const bool accept = sigma > c.sigma0;
      double next;
      if (!accept)
        next = c.gamma1 * step_norm;
      else if (sigma < c.eta1)
        next = c.gamma2 * step_norm;
      else if (sigma < c.eta2)
        next = S->delta;
      else {
        const double grown = c.gamma3 * step_norm;
        next = grown > S->delta ? grown : S->delta;
      }
      if (S->n_iter < S->cap) {
        TrRecord& r = S->trace[S->n_iter];
        r.f_candidate = fc;
        r.gradient_norm = S->gnorm;
        r.delta = S->delta;
        r.sigma = sigma;
        r.accepted = accept;
        r.cg_exit = cg->exit_kind;
        r.cg_iters = cg->iters;
      }
      S->n_iter += 1;
      S->delta = next;
      if (accept) {
        S->f = fc;
        S->committed = k ^ 1;
        S->accepted += 1;
        S->grad_mats += 1;
        if (obj->grad_nonfinite) {  // tron.cpp:205-207
          S->status = kTrFailGradient;
          stop = 1;
        } else {
          S->gnorm = obj->gnorm;
          if (S->gnorm <= c.eps * S->gnorm0) {  // tron.cpp:208-211
            S->converged = 1;
            stop = 1;
          }
        }
      }
      if (S->n_iter >= c.max_outer) stop = 1;  // tron.cpp:161
    }
  }
  const int go = !stop;
  S->cont = go;
  cset(outer, go);
  // body k == 0 runs before body 1 in the same pass: hand over to it
  cset(other, go && S->committed == (k ^ 1));
}

}  // namespace

void tr_dispatch(const SolveState* S, Cond k0, Cond k1, cudaStream_t s) {
  tr_dispatch_kernel<<<1, 1, 0, s>>>(S, k0, k1);
  TB_LAUNCH_CHECK();
}

void tr_prep(const SolveState* S, CgState* st, cudaStream_t s) {
  tr_prep_kernel<<<1, 1, 0, s>>>(S, st);
  TB_LAUNCH_CHECK();
}

void tr_update(SolveState* S, const CgState* cg, const ObjScalars* obj, int k, Cond outer,
               Cond other, cudaStream_t s) {
  tr_update_kernel<<<1, 1, 0, s>>>(S, cg, obj, k, outer, other);
  TB_LAUNCH_CHECK();
}

}  // namespace tb
