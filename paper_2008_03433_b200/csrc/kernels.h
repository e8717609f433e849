// Host-callable launchers for the sm_100a kernels of the TRON hot path.
// Everything here is FP64; indices are int32 (checked at creation:
// nnz and n below 2^31 per shard).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace tb {

constexpr int kLossLogistic = 0;
constexpr int kLossSvm = 1;

// Compressed rows (CSR of X) or compressed columns (CSC of X, i.e. CSR of
// X^T): ptr has `rows+1` entries, idx/val `nnz`.
struct CsrView {
  int64_t rows = 0, cols = 0, nnz = 0;
  const int32_t* ptr = nullptr;
  const int32_t* idx = nullptr;
  const double* val = nullptr;
  // column panel (row products only): row i's entries [rbeg[i], rend[i]) instead
  // of [ptr[i], ptr[i+1]) -- the part of a column-sorted row inside the panel
  const int32_t* rbeg = nullptr;
  const int32_t* rend = nullptr;
};
// Column panels of a CSR (row products of X with v too large for L2): split[k]
// [i] = first entry of row i with column >= bound[k] (k = 0 .. K-2, K <= 8);
// counts[k] (host) = entries of panel k.  Synchronizes s; 0 or a cudaError_t.
int csr_panel_splits(const CsrView& X, const int32_t* bounds, int nbounds, int32_t* const* split,
                     unsigned long long* counts, cudaStream_t s);

// Segmented-chunk plan of a compressed matrix (fixed per structure): the
// nonzeros are cut into fixed chunks of 32*kSegLaneItems (one warp each);
// rows crossing chunks are finished by the fix-up pass, empty rows are
// written from their own list.
constexpr int kSegLaneItems = 8;
constexpr int kSegChunk = 32 * kSegLaneItems;
struct SegView {
  int64_t nchunks = 0;
  int64_t nnzc = 0;                      // non-empty rows
  int64_t nempty = 0;                    // empty rows
  const uint32_t* chunk_rank = nullptr;  // rank of the row holding the chunk's first entry
                                         // | 0x80000000 when that row began in an earlier chunk
  const uint32_t* lastbits = nullptr;    // bit k: entry k is the last of its row
  const int32_t* nz_col = nullptr;       // [nnzc+1] index of the r-th non-empty row; [nnzc] = rows
  const int32_t* empty_col = nullptr;    // [nempty] the empty rows, ascending
  const int32_t* chunk_first = nullptr;  // first chunk of the row continued into chunk t when it
                                         // ends there (a fix-up), else -1
  double* head = nullptr;   // [nchunks] partial of the row open at the chunk's start, if it ends inside
  double* carry = nullptr;  // [nchunks] partial of the row open at the chunk's end
  // fix-ups spanning more than kFixCta chunks (Zipf-hot rows: K1's hottest
  // column covers ~29k chunks), each finished by a whole CTA
  const int32_t* long_fix = nullptr;  // [nlong] chunk ids, ascending
  int64_t nlong = 0;
};
constexpr int kFixCta = 512;
// long_fix buffer entries seg_plan_device may write
inline int64_t seg_long_fix_cap(int64_t nchunks) { return nchunks / kFixCta + 1; }
// Device-built plan from the compressed-row offsets (ptr, rows+1).  Buffers:
// chunk_rank[nchunks], chunk_first[nchunks], lastbits[nchunks*8+2],
// nz_col[rows+1], empty_col[rows]; P's head / carry are left to the caller.
// Synchronizes s (returns the counts in P).
int seg_plan_device(const int32_t* ptr, int64_t rows, int64_t nnz, SegView* P,
                    uint32_t* chunk_rank, int32_t* chunk_first, uint32_t* lastbits, int32_t* nz_col,
                    int32_t* empty_col, int32_t* long_fix, cudaStream_t s);

// Per-source-row weight u_i used by the transposed product sum_i u_i x_ij.
enum UKind : int {
  U_VEC = 0,        // u[i]
  U_SVM_RESID = 1,  // mask[i] ? z[i] - y[i] : 0   (svm_gradient, loss.cpp:129-137)
  U_MASK = 2,       // mask[i] ? 1 : 0              (masked_sq_col_sums, linalg.cpp:257-265)
};
struct UView {
  int kind = U_VEC;
  const double* u = nullptr;
  const uint8_t* mask = nullptr;
  const double* z = nullptr;
  const double* y = nullptr;
};

// out_j = base_j + scale*sum_j (VEC), cbase + scale*sum_j (CONST), or sum_j (RAW)
enum EpiKind : int { EPI_VEC = 0, EPI_CONST = 1, EPI_RAW = 2 };
struct EpiView {
  int kind = EPI_VEC;
  const double* base = nullptr;
  double cbase = 0.0;
  double scale = 1.0;
  // EPI_VEC only: also reduce over every emitted out_j, per warp into
  // dot_parts (2 doubles per slot; seg_dot_slots(nchunks) doubles), finished in
  // a fixed order by the fix-up kernel's last CTA:
  //   dot_mode 0: sum base_j * out_j -> *dot_out (p.Hp when base = p);
  //   dot_mode 1: sum out_j^2 and any non-finite out_j -> dot_obj->gnorm,
  //               dot_obj->grad_nonfinite (the gradient's norm check).
  double* dot_parts = nullptr;
  double* dot_out = nullptr;
  unsigned* dot_ticket = nullptr;
  int dot_mode = 0;
  struct ObjScalars* dot_obj = nullptr;
};

constexpr int kCgConverged = 0;  // CgExit, tron.hpp:29
constexpr int kCgBoundary = 1;
constexpr int kCgMaxIters = 2;

// Trust-region CG state kept in device memory (tron.cpp:37-108 scalars).
struct CgState {
  double delta, stop, rz, rnorm, alpha, beta, php, tau, q, dnorm;
  long long iters, max_iters;
  int exit_kind, boundary, cont, fail, rpar, use_m;
};

// Scalars of the objective / gradient passes.
struct ObjScalars {
  double ww;          // w_cand . w_cand
  double f;           // candidate objective
  double gnorm;       // ||grad|| of the committed iterate
  long long nact;     // |I| of the candidate (SVM)
  int grad_nonfinite; // any non-finite gradient entry
  int pad;
  double red[2];      // {sum of loss terms, |I|} of this shard (allreduced when sharded)
};

// Optional CUDA-graph while-loop handle set by the CG kernels.
struct Cond {
  unsigned long long h = 0;
  int on = 0;
};

struct Scratch {
  double* partials = nullptr;  // >= kMaxPartialBlocks * 4 doubles
  unsigned int* tickets = nullptr;  // kNumTickets counters, zero-initialized
};
constexpr int kMaxPartialBlocks = 4096;
constexpr int kNumTickets = 16;
enum Ticket : int { T_FUN = 0, T_AXPY = 1, T_NORM = 2, T_CG_INIT = 3, T_CG_PHP = 4, T_CG_UPD = 5,
                    T_CG_P = 6, T_CG_POST = 7, T_DENSE_FIN = 8, T_COUNT = 9, T_DOT2 = 10, T_SUMSQ = 11 };

int device_sm_count();

// ---- CSR forward passes (csr_kernels.cu) -----------------------------------
int choose_group(int64_t rows, int64_t nnz);
// Fused margin pass: z = Xw; LR: zhat, dvec; SVM: mask (+ active count).
// f = 0.5*ww + C*sum(loss terms) is written to obj->f (obj->ww precomputed).
// zin (may alias z): the row sums of the earlier column panels, added first.
void csr_forward(const CsrView& X, int group, int loss, const double* w, const double* y, double C,
                 double* z, double* zhat, double* dvec, uint8_t* mask, ObjScalars* obj,
                 Scratch sc, cudaStream_t s, const double* zin = nullptr);
// a_i = (x_i . p) * dvec_i  (or mask_i ? x_i . p : 0 when mask given; x_i . p
// when neither is given)
// Column panels: ain (may alias a) holds the earlier panels' row sums; only
// the last panel (final) applies dvec / mask, the others store the raw sum.
void csr_dv(const CsrView& X, int group, const double* p, const double* dvec, const uint8_t* mask,
            double* a, cudaStream_t s, const double* ain = nullptr, bool final = true);
// Transposed product over the CSC copy (csc_seg.cu; segmented chunks, atomic-free).
int64_t seg_dot_slots(int64_t nchunks);
void csc_spmv(const CsrView& At, const SegView& plan, const UView& u, bool squared,
              const EpiView& epi, double* out, cudaStream_t s);

// Device CSC construction from device CSR (stable in row order).
// Returns 0 on success; temp storage allocated internally.
int build_csc_structure(const CsrView& X, int32_t* cptr, int32_t* ridx, int32_t** perm,
                        cudaStream_t s);
int build_csc_values(int32_t* perm, const double* val, double* cval, int64_t nnz, cudaStream_t s);
// gather_rows on a CSR (linalg.cpp:197-229): gptr[nI+1] offsets of the rows
// idx[0..nI) (synchronizes s; *nnz_out = their entry count), then the entries.
int csr_gather_offsets(const CsrView& X, const int32_t* idx, int64_t nI, int32_t* gptr,
                       long long* nnz_out, cudaStream_t s);
void csr_gather_rows(const CsrView& X, const int32_t* idx, int64_t nI, const int32_t* gptr,
                     int32_t* gidx, double* gval, cudaStream_t s);
// Input screening: first_bad2[0] = first row whose columns are not strictly
// ascending within [0, n) (ptr may be null: no matrix check), first_bad2[1] =
// first label not in {-1, +1}; ~0 when none.  Offsets must already be valid.
void screen_inputs(const int32_t* ptr, const int32_t* idx, int64_t rows, int64_t n,
                   const double* y, int64_t l, unsigned long long* first_bad2, cudaStream_t s);
// Row-offset narrowing int64 -> int32 (device).
void narrow_offsets(const int64_t* in, int32_t* out, int64_t count, cudaStream_t s);

// ---- predict (predict.cu; model.cpp:88-117) ---------------------------------
// labels[i] = sign(x_i . w) (ties +1), rows summed sequentially in storage
// order (bit-exact with the reference); *correct (device) = #{labels == y}.
void predict_csr(const CsrView& X, const double* w, const double* y, double* labels,
                 unsigned long long* correct, cudaStream_t s);
// labels from precomputed scores x_i . w (the column layout's allreduced row sums)
void predict_from_scores(int64_t l, const double* scores, const double* y, double* labels,
                         unsigned long long* correct, cudaStream_t s);
void predict_dense(int64_t l, int64_t n, int64_t ld, const double* X, const double* w,
                   const double* y, double* labels, unsigned long long* correct, cudaStream_t s);

// ---- vector kernels (vec_kernels.cu) -----------------------------------------
// wc = w + d (d may be null: wc = w); obj->ww = wc.wc
void vec_axpy_dot(int64_t n, const double* w, const double* d, double* wc, ObjScalars* obj,
                  Scratch sc, cudaStream_t s);
// obj->gnorm = ||g||, obj->grad_nonfinite
void vec_norm_check(int64_t n, const double* g, ObjScalars* obj, Scratch sc, cudaStream_t s);
// out2[0] = a.b, out2[1] = c.d (fixed-order two-stage sums)
void vec_dot2(int64_t n, const double* a, const double* b, const double* c, const double* d,
              double* out2, Scratch sc, cudaStream_t s);
// out = base + scale*raw  (after an allreduce of raw partials; raw == nullptr => 0)
void vec_epilogue(int64_t n, const double* raw, const EpiView& epi, double* out, cudaStream_t s);
void l2_read_flush(const double* buf, int64_t n, cudaStream_t s);
// Column-partitioned layout helpers (engine.cpp run_cg_columns):
// out = a*x + b*y (x / y may be null: treated as 0); z = r / M (M null: copy)
void vec_lincomb(int64_t n, double a, const double* x, double b, const double* y, double* out,
                 cudaStream_t s);
void vec_div(int64_t n, const double* r, const double* M, double* z, cudaStream_t s);
// out2 = {sum g_j^2, any non-finite g_j} (fixed order); then, after the
// allreduce of out2, obj->gnorm = sqrt(out2[0]), obj->grad_nonfinite
void vec_sumsq_bad(int64_t n, const double* g, double* out2, Scratch sc, cudaStream_t s);
void obj_set_gnorm(ObjScalars* obj, const double* in2, cudaStream_t s);
// out8[0..3] = 16-bit chunks of the wrap-around sum of the bit patterns of w,
// f and delta; out8[4..7] their squares (replica check of the row shards)
void replica_checksum(int64_t n, const double* w, double f, double delta, double* out8, cudaStream_t s);
// a_i *= D_i (dvec) or a_i = mask_i ? a_i : 0 (the allreduced row products)
void vec_row_scale(int64_t l, double* a, const double* dvec, const uint8_t* mask, cudaStream_t s);
// Streamed (out-of-core) margin pass: the per-block loss sums and |I|
// (red[2b], red[2b+1]) into obj->f = 0.5 ww + C sum, nact, red[0..1]; fixed order.
void obj_combine_blocks(ObjScalars* obj, const double* red, int64_t nblk, double C, cudaStream_t s);

// CG initialisation for the mid/large-n engines (d = 0, r = -g, p = M^-1 r).
struct CgVectors {
  int64_t n;
  const double* g;
  const double* M;  // nullable
  double* d;
  double* r0;
  double* r1;
  double* p;
  double* hp;
};
void cg_large_init(const CgVectors& v, CgState* st, Scratch sc, Cond cond,
                   cudaStream_t s);

// Mid-n CG engine (kSmallCgMaxN < n <= kClusterCgMaxN): one kernel per iteration
// on a cluster of 8 CTAs (vector phases + scalars; the exit's q(d), ||d|| included).
// Beyond ~32k coordinates the cooperative grid step is faster: eight SMs'
// bandwidth bounds the cluster's vector passes (scripts/cg_engine_sweep.py:
// n = 47236 0.93 vs 0.89 ms, n = 200000 1.24 vs 0.97 ms per solve).
constexpr int64_t kClusterCgMaxN = 32768;
// One large-n CG iteration as a single cooperative kernel (vec_kernels.cu);
// parts: 8 * cg_coop_grid() doubles.  Ends the loop itself (no post kernel).
int cg_coop_grid();
// php_in: p.Hp already summed by the Hv kernels (EpiView::dot_out), or null.
void cg_coop_step(const CgVectors& v, CgState* st, double* parts, Cond cond, cudaStream_t s,
                  const double* php_in = nullptr);
void cg_cluster_step(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s);

// Small-n CG engine (n <= kSmallCgMaxN): one single-block kernel per
// iteration.  When `partials` is non-null, hp_j = p_j + scale*sum_b
// partials[b*n+j] is formed first (dense tall-skinny Hv second stage).
constexpr int64_t kSmallCgMaxN = 4096;
void cg_small_init(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s);
void cg_small_step(const CgVectors& v, const double* partials, int nparts, double scale,
                   CgState* st, Cond cond, cudaStream_t s);

// ---- device-resident outer trust-region loop (trloop.cu) --------------------
// TrustRegionConfig (tron.hpp:13-27) as the device reads it.
struct TrConfig {
  double eps, sigma0, eta1, eta2, gamma1, gamma2, gamma3, cg_tol, C;
  long long max_outer, max_cg;
  int use_m, sharded;  // sharded: f = 0.5 ww + C * (allreduced loss sum)
};
// IterationRecord (tron.hpp:38-48); the layout of tron_iteration.
struct TrRecord {
  double f_candidate, gradient_norm, delta, sigma;
  int accepted, cg_exit;
  long long cg_iters;
};
enum TrStatus : int { kTrOk = 0, kTrFailCg = 1, kTrFailObjective = 2, kTrFailGradient = 3 };
// The solver's scalars (tron.cpp:127-217 locals + SolverTrace counters).
struct SolveState {
  TrConfig cfg;
  double f, delta, gnorm, gnorm0, fail_php;
  long long n_iter, accepted, obj_evals, grad_mats, hv_count, max_nact;
  int committed;  // slot of the committed iterate
  int status;     // TrStatus
  int converged, cont;
  TrRecord* trace;  // device records [cap]
  long long cap;
};
void tr_dispatch(const SolveState* S, Cond k0, Cond k1, cudaStream_t s);
void tr_prep(const SolveState* S, CgState* st, cudaStream_t s);
void tr_update(SolveState* S, const CgState* cg, const ObjScalars* obj, int k, Cond outer,
               Cond other, cudaStream_t s);

// ---- dense column-major kernels (dense_kernels.cu), n <= 64 -----------------
// X is column-major with ld = dense_ld(l) rows (a multiple of kDenseTile,
// padding zeroed); every per-row side array a pass stages (y, D, mask) must
// also be allocated and zero-padded to ld entries.
constexpr int kDenseMaxN = 64;
constexpr int64_t kDenseTile = 256;
int64_t dense_ld(int64_t l);
// Rows per tile (= threads per CTA) of the tiled passes for n features.
int dense_tile_rows(int64_t n);
// Number of CTAs (= per-block partial vectors) of every tiled pass.
int dense_grid(int64_t l, int64_t n);
// Fused margin pass: z, LR zhat/dvec or SVM mask, f into obj, and the
// candidate's gradient partials gparts[grid][n] (sum_i c_i x_i with
// c = zhat (LR) or [i in I](z_i - y_i) (SVM)).
// 2-D TMA descriptor of a column-major X (rows x n, leading dimension ld):
// box = {dense_tile_rows(n) rows, n columns}.  Returns 0 on success.
int dense_make_map(CUtensorMap* map, const double* X, int64_t ld, int64_t rows, int64_t n);
// gram_parts (n <= 40, dense_forward_gram_fused): also the candidate's Gram
// partials [grid][n*n] (gram.cu's G, finished by gram_finalize) in the same pass.
bool dense_forward_gram_fused(int64_t n);
void dense_forward(int64_t l, int64_t n, int64_t ld, const double* X, const CUtensorMap& xmap,
                   int loss, const double* w,
                   const double* y, double C, double* z, double* zhat, double* dvec, uint8_t* mask,
                   double* gparts, ObjScalars* obj, Scratch sc, cudaStream_t s,
                   double* gram_parts = nullptr, const uint8_t* mask_ref = nullptr,
                   const int* ref_stale = nullptr);
// L2-SVM, n <= 40 (dense_forward_gram_delta): with gram_parts AND mask_ref the
// pass accumulates instead the partials [grid][n*n] of
//   Delta = sum_i (m_i - mask_ref_i) x_i x_i^T
// over the rows that changed side -- skipped (plain FWD) when *ref_stale != 0 --
// and gram_delta_finalize forms G = G_ref + Delta.
bool dense_forward_gram_delta(int64_t n);
// Gram flags (int[4] per slot): [0] != 0: G does not match the slot's mask;
// [1] delta updates since G was formed from scratch; [2] finalize ticket.
// A reference G that is stale, or has had kGramDeltaChain updates (so rounding
// cannot drift), is not updated: the candidate's G is then formed afresh.
constexpr int kGramDeltaChain = 16;
__host__ __device__ inline bool gram_ref_is_empty(const int* flags) {
  return flags[0] != 0 || flags[1] >= kGramDeltaChain;
}
void gram_delta_finalize(int64_t n, const double* parts, int nparts, const double* Gref, const int* ref_flags,
                         double* Gout, int* out_flags, cudaStream_t s);
// G = sum over nparts of the per-CTA Gram partials (fixed order)
void gram_finalize(int64_t n, const double* partials, int nparts, double* G, cudaStream_t s,
                   int* flags = nullptr);  // flags: computed only if flags[0] != 0, then cleared
// partial sums per block (grid = dense_grid(l, n)) of:
//  HV:      sum_i c_i x_i   with c = (x_i.v)*dvec_i (LR) or mask?(x_i.v):0 (SVM;
//           mask == nullptr => every row active, used on the gathered panel)
//  PRECOND: sum_i (c_i x_ij) x_ij with c = dvec (LR) or mask (SVM)
enum DenseAccum : int { DA_HV = 1, DA_PRECOND = 2 };
void dense_accum(int kind, int64_t l, int64_t n, int64_t ld, const double* X,
                 const CUtensorMap& xmap, int loss,
                 const double* v, const double* dvec, const uint8_t* mask, double* partials,
                 cudaStream_t s);
// out_j = base_j (or cbase) + scale * sum_b partials[b*n + j]
void dense_finalize(int64_t n, const double* partials, int nparts, const EpiView& epi, double* out,
                    cudaStream_t s);
// Row-major host chunk (rows x n, already on device) -> column-major X.
void dense_transpose_chunk(const double* rm, int64_t rows, int64_t n, double* X, int64_t ld,
                           int64_t row0, cudaStream_t s);
// Active-set compaction: ascending int32 row indices of mask (ballot+scan).
// count_out (device) receives |I|. tmp needs >= ceil(l/1024)+1 ints.
void compact_mask(int64_t l, const uint8_t* mask, int32_t* idx, int32_t* tmp, long long* count_out,
                  cudaStream_t s);
// Gathered strategy: Xg (ldg = dense_ld(nI) rows, tail zeroed) <- rows idx of X.
void dense_gather(int64_t nI, int64_t n, const double* X, int64_t ld, const int32_t* idx,
                  double* Xg, int64_t ldg, cudaStream_t s);

// ---- the dense Hessian as an n x n matrix (gram.cu), n <= 64 ----------------
// G = sum_i c_i x_i x_i^T, c = mask (SVM, dvec null) or dvec (LR); partials
// >= gram_grid(l, n) * n * n doubles.  Deterministic.
int gram_grid(int64_t l, int64_t n);
// stale (device int, nullable): when it reads 0 the kernels return at once (G is
// current); the finalize clears it -- so the launch can sit unconditionally in a
// graph and cost ~10 us when nothing changed.
void dense_gram(int64_t l, int64_t n, int64_t ld, const double* X, const uint8_t* mask,
                const double* dvec, double* partials, double* G, cudaStream_t s, int* stale = nullptr);
// out = v + scale * G v (row j of G dotted with v in index order)
void gram_hv(int64_t n, const double* G, const double* v, double scale, double* out, cudaStream_t s);
// M_j = 1 + scale * G_jj (loss.cpp:176-188)
void gram_precond(int64_t n, const double* G, double scale, double* M, cudaStream_t s);
// The small-n CG step with hp = p + scale * G p formed first.
// Gram mode, n <= 64: every iteration of the CG (after cg_small_init) in one
// launch, G in shared memory; leaves st / cond as the last step would.
void cg_small_gram_loop(const CgVectors& v, const double* G, double scale, CgState* st, Cond cond,
                        cudaStream_t s);
void cg_small_step_gram(const CgVectors& v, const double* G, double scale, CgState* st, Cond cond,
                        cudaStream_t s);

// ---- reference-order reductions for the dense L2-SVM (refexact.cu) --------
// Bit-for-bit the reference's arithmetic: 64 sequential block sums + the
// pairwise tree (parallel.hpp:14-34), serial n-length dots.  n <= kRoMaxN.
constexpr int64_t kRoMaxN = 48;
enum RoMode : int { RO_HV = 0, RO_GRAD = 1, RO_PRECOND = 2 };
// out = epi(sum over I of c_i x_i) with c = x_i.v (HV), z_i - y_i (GRAD), or
// the squares (PRECOND); GRAD also sets obj->gnorm (serial) and grad_nonfinite.
// xmap128: TMA map of X with 128-row boxes; partials >= 64*n doubles.
void ro_accum(int mode, int64_t l, int64_t n, const CUtensorMap& xmap128, const long long* count,
              const int32_t* idx, const uint8_t* mask, const double* v, const double* z,
              const double* y, double* partials, unsigned* ticket, const EpiView& epi, double* out,
              ObjScalars* obj, cudaStream_t s);
// obj->f = 0.5*dot(w,w) + C*reduce_sum(max(1 - y z, 0)^2), obj->ww; partials >= 64.
void ro_hinge(int64_t l, int64_t n, const double* z, const double* y, const double* w, double C,
              double* partials, unsigned* ticket, ObjScalars* obj, cudaStream_t s);
void ro_cg_init(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s);
void ro_cg_step(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s);
// dense_make_map with `box_rows`-row boxes.
int dense_make_map_box(CUtensorMap* map, const double* X, int64_t ld, int64_t rows, int64_t n,
                       int box_rows);

}  // namespace tb
