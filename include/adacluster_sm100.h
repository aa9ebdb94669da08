/*
 * adacluster_sm100.h — C-ABI of the B200-native AdaCluster hot path.
 *
 * This is the drop-in boundary for the cluster -> select -> sparse-attention
 * path of the reference package `adacluster` 0.1.0 (pure Python/numpy, see
 * /root/reference/pkg/src/adacluster).  The reference has no FFI of its own;
 * its public Python surface (`__init__.py:3-41`) is re-implemented by
 * `paper_2604_18348_b200/` on top of these entry points, loaded with ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - every entry point returns an int status (AC_OK ... AC_ERR_CUDA); the
 *     message of the last failure on the calling thread is ac_last_error().
 *     Status codes map to the reference exception classes (errors.py:8-29):
 *     AC_ERR_PARAM -> ParameterError, AC_ERR_DIM -> DimensionError,
 *     AC_ERR_CONTRACT -> ContractError.
 *   - all pointers are DEVICE pointers owned by the caller unless a comment
 *     says "host"; the library never allocates or frees caller memory.
 *   - all work is enqueued on the caller's cudaStream_t (passed as void*);
 *     no entry point synchronises unless documented.
 *   - matrices are row-major, rows contiguous.  dtype is AC_DTYPE_F32 or
 *     AC_DTYPE_BF16 for token tensors; centres/envelopes/scores are f32.
 */
#ifndef ADACLUSTER_SM100_H
#define ADACLUSTER_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AC_ABI_VERSION 1

/* status codes */
#define AC_OK 0
#define AC_ERR_PARAM 1
#define AC_ERR_DIM 2
#define AC_ERR_CONTRACT 3
#define AC_ERR_CUDA 4

/* token tensor element types */
#define AC_DTYPE_F32 0
#define AC_DTYPE_BF16 1

/* Accumulation order of an f32 NT product x @ c.T with inner length D.
 * The reference's `@` is OpenBLAS sgemm; its order depends on the shape
 * and is reproduced exactly:
 *   AC_ORDER_SEQ     acc = fmaf(x[t], c[t], acc), t = 0..D-1, from 0
 *   AC_ORDER_LANES16 16 lane chains (t mod 16) + adjacent-pair tree
 *   AC_ORDER_GEMV8   8 lane chains (t mod 8), s[l]=a[l]+a[l+4], (s0+s1)+(s2+s3)
 * ac_gemm_order() returns the order the reference uses for an M x N x D call. */
#define AC_ORDER_SEQ 0
#define AC_ORDER_LANES16 1
#define AC_ORDER_GEMV8 2

/* TensorQuest scorer variants (pipeline.py:144-151) */
#define AC_SCORER_QUEST 0   /* quest.py:94   max(Q,0)·maxᵀ + min(Q,0)·minᵀ     */
#define AC_SCORER_MEAN 1    /* quest.py:119  Q·centersᵀ                        */
#define AC_SCORER_CLAMPED 2 /* quest.py:106  max(Q,0)·max(C,0)ᵀ + min(Q,0)·min(C,0)ᵀ */
#define AC_SCORER_GIVEN 3   /* scores supplied in ac_select_problem.scores      */

/* ac_assign flags */
#define AC_ASSIGN_MERGE 1   /* merge into existing (labels,best) with strict '<'
                               so earlier (lower-index) centres win ties        */
#define AC_ASSIGN_ALL 2     /* ignore the per-problem 'active' flag            */
#define AC_ASSIGN_LABELS_ONLY 4 /* labels exact, `best` exact only for rows
                               that had near-ties (tensor-core path); the
                               repair pass then recomputes exact distances  */

/* ---------------------------------------------------------------------------
 * One clustering problem (one head, or one multi-stage round of one head).
 * The caller allocates every buffer; sizes in brackets.  A batch of problems
 * is an array of these in DEVICE memory; all share dtype and D.
 * ------------------------------------------------------------------------- */
typedef struct ac_cluster_problem {
  const void* x;        /* [n, d] points (dtype of the batch)                 */
  float* xx;            /* [n]   pairwise ||x_i||^2  (written by ac_lloyd_prepare) */
  float* centers;       /* [kcap, d] in: initial centres, out: final centres  */
  float* cc;            /* [kcap]  ||c||^2 of the current centres             */
  int32_t* labels;      /* [n]   assignment                                   */
  float* best;          /* [n]   assigned squared distance / k-means++ closest */
  int32_t* counts;      /* [kcap] members per centre                          */
  int32_t* perm;        /* [n]   stable argsort of labels (member order)      */
  int32_t* starts;      /* [kcap+1] segment starts into perm                  */
  int32_t* tile_hist;   /* [ceil(n/128) * kcap] per-tile label histogram      */
  float* inertia;       /* [max_iter] inertia_history                         */
  float* movement;      /* [kcap] per-centre movement scratch                 */
  int32_t* status;      /* [8] {active, n_iter, done, flags, kpp_stop, ...}   */
  const int32_t* plan_n;/* pairwise-sum plan of length n (ac_pw_plan_build)   */
  const int32_t* plan_k;/* pairwise-sum plan of length k                      */
  double* dscratch;     /* [n] f64 scratch (k-means++ cdf, tau)               */
  void* planes;         /* optional, f32 points only: [3][n][d] bf16 hi/mid/lo
                           split of x (written by ac_lloyd_prepare); enables
                           the tensor-core assignment for f32 points           */
  double* csum;         /* optional [kcap, d] f64 (zeros),                     */
  float* cabs;          /* [kcap, d] f32 (zeros) and                           */
  int32_t* clsb;        /* [kcap, d] f32 bits (+inf = 0x7f800000): workspaces of the
                           split-chain centroid update for d = 64/128          */
  int64_t n;
  int32_t k;
  int32_t order;        /* AC_ORDER_* of the reference's x @ centres.T        */
} ac_cluster_problem;

/* status[] slots */
#define AC_ST_ACTIVE 0
#define AC_ST_NITER 1
#define AC_ST_DONE 2
#define AC_ST_FLAGS 3
#define AC_ST_KPP_STOP 4
#define AC_ST_REPAIRS 5
#define AC_ST_FIXUPS 6   /* rows the tensor-core assign resolved with > 1 exact chain */
#define AC_ST_WIDE 7     /* ... of which had > 2 candidates (exact over every centre)  */

/* ---- library ---------------------------------------------------------- */
const char* ac_last_error(void);
int ac_abi_version(void);
/* sizeof of the three descriptor structs (ABI check for bindings) */
int ac_struct_sizes(int64_t* out3);
/* Number of SMs / compute capability of the current device (host query). */
int ac_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- host helpers ----------------------------------------------------- */
/* numpy pairwise-summation tree for a length-n reduction, flattened into an
 * int32 program (ac_pw_plan_len words) executed by the reduction kernels.   */
int64_t ac_pw_plan_len(int64_t n);
int ac_pw_plan_build(int64_t n, int32_t* host_out, int64_t cap);
/* OpenBLAS dispatch of the reference's f32 `a @ b.T` ([m,d] x [n,d]) */
int ac_gemm_order(int64_t m, int64_t n, int64_t d);

/* ---- workspace sizing ---------------------------------------------------
 * Byte size of every caller-owned buffer of one op (returns the total, or -1
 * with ac_last_error() set).  fields (optional, host, nfields entries) gets the
 * per-buffer sizes in the order listed; dims (host) by op:
 *   AC_WS_CLUSTER   {n, kcap, d, dtype, max_iter} -> the 19 buffer fields of
 *                   ac_cluster_problem in declaration order (xx ... clsb);
 *                   optional buffers are 0 when the kernels will not use them
 *   AC_WS_SELECT    {gq, c, topk, run_stride} -> scores, selected, runs,
 *                   nruns, covered, density of ac_select_problem
 *   AC_WS_ATTENTION {L, heads, gq_max, topk_max, d, dtype} -> qp, qidx,
 *                   items, kp, vp of ac_build_q_layout / ac_sparse_attention
 *                   (runs/nruns are the selection's)                       */
#define AC_WS_CLUSTER 0
#define AC_WS_SELECT 1
#define AC_WS_ATTENTION 2
int64_t ac_workspace_bytes(int op, const int64_t* dims, int ndims, int64_t* fields,
                           int nfields);

/* ---- K1 tensorops.py:59-76 l2_normalize_rows ---------------------------
 * out[i] = x[i] / ||x[i]||  (numpy pairwise-8 norm, f32 divide), rows with
 * |norm-1| <= 2e-6 copied unchanged, norm < 1e-12 -> zeros + degenerate[i]=1.
 * Also emits xx[i] = pairwise ||out[i]||^2 for the assignment kernel.      */
int ac_l2norm(const void* x, int dtype, int64_t rows, int d, float* out,
              float* out_sqnorm, uint8_t* degenerate, void* stream);

/* ac_l2norm that also writes, when planes != NULL, the exact bf16 hi/mid/lo
 * split of the normalised rows as per-problem planes [3][prob_rows][d]
 * (rows % prob_rows == 0; d = 64 or 128, 16-byte aligned buffers) -- the
 * query-side prepare of ac_lloyd_ex fused into the normalisation pass.     */
int ac_l2norm_ex(const void* x, int dtype, int64_t rows, int d, float* out,
                 float* out_sqnorm, uint8_t* degenerate, void* planes, int64_t prob_rows,
                 void* stream);

/* pairwise ||x_i||^2 in f32 (clustering.py:71 `(x * x).sum(axis=1)`) */
int ac_row_sqnorm(const void* x, int dtype, int64_t rows, int d, float* out,
                  void* stream);

/* ---- K2 clustering.py:78-91 _kmeanspp_init ------------------------------
 * draws: [nprob * max_k] f64 per problem (host-drawn numpy PCG64 stream):
 *   draws[0] = first index (rng.integers(n)),
 *   draws[i] = u_i = rng.random() for step i >= 1, or -(idx+1) to force the
 *              `total <= 0` branch's rng.integers(n) result.
 * On `total <= 0` at a step whose draw is not forced, status[AC_ST_KPP_STOP]
 * receives the step and the problem stops (the host redraws and relaunches). */
int ac_kmeanspp(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                int64_t max_n, int max_k, const double* draws, void* stream);

/* ---- K3..K6 clustering.py:119-152 _lloyd ---------------------------------
 * Runs up to max_iter Lloyd iterations (assign, empty repair, inertia,
 * stable segment sort, f64 centroid update, movement < tol) for every problem
 * and the final assign + repair + member sort.  Per-problem convergence is
 * tracked on device (status[]); no host synchronisation unless
 * poll_every > 0 (then the host polls every poll_every iterations and stops
 * launching once every problem has converged).                            */
int ac_lloyd(const ac_cluster_problem* probs, int nprob, int dtype, int d,
             int64_t max_n, int max_k, int max_iter, double tol,
             int poll_every, const ac_cluster_problem* host_probs, void* stream);

/* ac_lloyd with flags (no host polling): AC_LLOYD_NO_INERTIA skips the
 * per-iteration inertia_history reduction (steady-state steps never read it;
 * labels, centres and n_iter are unaffected).                               */
#define AC_LLOYD_NO_INERTIA 1
/* the problems' xx (and, for f32 points, planes) are already current --
 * written by ac_l2norm_ex in the same stream -- so the prepare pass skips them */
#define AC_LLOYD_PREPARED 2
int ac_lloyd_ex(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                int64_t max_n, int max_k, int max_iter, double tol, int flags,
                const ac_cluster_problem* host_probs, void* stream);

/* Single passes, exposed for the multi-stage planner and for tests. */
int ac_lloyd_prepare(const ac_cluster_problem* probs, int nprob, int dtype,
                     int d, int64_t max_n, int max_k, void* stream);
int ac_assign(const ac_cluster_problem* probs, int nprob, int dtype, int d,
              int64_t max_n, int max_k, int c_lo, int flags, void* stream);
/* same with an explicit accumulation order (AC_ORDER_*) for the batch.
 * host_probs (optional, HOST copy of `probs`): when given and the batch is
 * eligible (d = 64, AC_ORDER_SEQ, k - c_lo <= 128, 16-byte aligned rows) the
 * cross term runs on the tcgen05 tensor cores (k_assign_tc: 3-way bf16 split,
 * TMA-fed, exact FMA-chain fix-up of near-ties in the epilogue); results are
 * bit-identical to the all-FFMA kernel.                                      */
int ac_assign_ordered(const ac_cluster_problem* probs, int nprob, int dtype,
                      int d, int64_t max_n, int max_k, int c_lo, int flags,
                      int order, const ac_cluster_problem* host_probs,
                      void* stream);

/* assignment kernel selection (per calling thread): AUTO = tensor cores when the
 * batch is eligible, EXACT = always the all-FFMA sequential-chain kernel
 * (the parity reference), TC = tensor cores or AC_ERR_PARAM.               */
#define AC_ASSIGN_MODE_AUTO 0
#define AC_ASSIGN_MODE_EXACT 1
#define AC_ASSIGN_MODE_TC 2
int ac_set_assign_mode(int mode);
int ac_get_assign_mode(void);
/* centroid-update kernel selection (per calling thread): 0 = split-chain sums with
 * an exact f32 enclosure test (member-order chain per dimension only when
 * the enclosure straddles a rounding boundary) when the batch has csum/cabs
 * workspaces, 1 = always the member-order f64 chains (its small per-centre
 * grid co-runs with the other Lloyd chains of a step), 2 = the same
 * enclosure-tested sums streamed over contiguous row ranges (every SM
 * busy, no walk of a whole cluster by one warp; needs the csum/cabs/clsb
 * workspaces and k <= 1024, else as mode 0), 3 = AUTO (the default): mode 2
 * for batches with fewer than 512 centres in total and >= 128 rows per
 * centre (multi-stage planner rounds), mode 1 otherwise.  All are bit-identical to np.add.reduceat in
 * member order.  Env AC_UPDATE_MODE overrides the default at load.        */
#define AC_UPDATE_MODE_SPLIT 0
#define AC_UPDATE_MODE_MEMBER 1
#define AC_UPDATE_MODE_STREAM 2
#define AC_UPDATE_MODE_AUTO 3
int ac_set_update_mode(int mode);
/* programmatic dependent launch of the Lloyd-chain kernels (per calling
 * thread; default on, env AC_PDL=0 turns it off at load): each kernel is set
 * up while its predecessor drains (C1 warm step 1.193 -> 1.152 ms, C2 25.75
 * -> 25.62 ms, the multi-stage planner of one hard head 111 -> 102 ms).    */
int ac_set_pdl(int on);
int ac_get_pdl(void);
int ac_get_update_mode(void);
int ac_repair_sort(const ac_cluster_problem* probs, int nprob, int dtype,
                   int d, int64_t max_n, int max_k, int iter, int flags,
                   void* stream);
/* stable member sort of existing labels (no re-assignment): perm/starts/counts */
int ac_sort_by_label(const ac_cluster_problem* probs, int nprob, int64_t max_n,
                     int max_k, void* stream);
/* segment means in f64 over members (clustering.py:134-139, :197-200):
 * out[c] = f32(sum_{i in seg c, member order} f64(x[perm[i]]) / count[c]) */
int ac_segment_mean(const ac_cluster_problem* probs, int nprob, int dtype,
                    int d, int max_k, float* const* out, void* stream);

/* ---- multi-stage helpers (clustering.py:209-320) ----------------------- */
/* f32 sum over n of best[] in numpy pairwise order -> out[p] (f32) and the
 * f32 mean f32(f64(sum)/n) -> mean_out[p] (either may be NULL)             */
int ac_reduce_best(const ac_cluster_problem* probs, int nprob, int64_t max_n,
                   float* sum_out, float* mean_out, void* stream);
/* compute_tau: tau = factor * mean_n ||f64(x) - f64(c[label])|| (f64)     */
int ac_tau(const ac_cluster_problem* probs, int nprob, int dtype, int d,
           int64_t max_n, double factor, double* tau_out, void* stream);
/* per-layer MSE (pipeline.py:319-323): mean_n sum_d (f64 x - f64 c)^2    */
int ac_mse_f64(const ac_cluster_problem* probs, int nprob, int dtype, int d,
               int64_t max_n, double* out, void* stream);
/* retire distances ||x - c[label]|| (f32 pairwise-8 + sqrtf) and the
 * order-preserving compaction U' = U[dist >= tau32]:
 *   idx_in [n] (original row ids), idx_out [n], out_count[p] (device)     */
int ac_retire(const ac_cluster_problem* probs, int nprob, int dtype, int d,
              int64_t max_n, const float* tau32, const int64_t* const* idx_in,
              int64_t* const* idx_out, int64_t* out_count, void* stream);
/* gather rows: dst[i] = src[idx[i]] (row = d elements of dtype)            */
int ac_gather_rows(const void* src, int dtype, int d, const int64_t* idx,
                   int64_t rows, void* dst, void* stream);
/* drop centres without members and remap labels (clustering.py:303-310).
 * counts must hold the bincount of labels; new_k[p] receives |keep|.       */
int ac_drop_empty(const ac_cluster_problem* probs, int nprob, int d,
                  int64_t max_n, int max_k, int32_t* new_k, void* stream);

/* ---- K9..K11 quest.py:61-143 -------------------------------------------
 * envelopes (segmented max/min over member order) for each problem.       */
int ac_envelopes(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                 int max_k, float* const* env_max, float* const* env_min,
                 void* stream);

typedef struct ac_select_problem {
  const float* reps;     /* [gq, d] query representatives                     */
  const float* emax;     /* [c, d]  envelope max (or centres for MEAN/CLAMPED) */
  const float* emin;     /* [c, d]  envelope min                              */
  const int32_t* counts; /* [c]     key cluster sizes                         */
  const int32_t* kstarts;/* [c+1]   key segment starts (member order)         */
  float* scores;         /* [gq, c] out                                       */
  int64_t* selected;     /* [gq, topk] out, descending score, ties -> low idx */
  int32_t* runs;         /* [gq, run_stride, 2] out: merged [start,end) ranges */
  int32_t* nruns;        /* [gq] out                                          */
  int64_t* covered;      /* [gq] out: key tokens covered by the selection     */
  double* density;       /* [1] out                                           */
  int32_t gq, c, topk;   /* topk here is min(topk, c) (pipeline.py:192)      */
  int32_t order;         /* AC_ORDER_* of the (gq x c x d) products           */
  int32_t run_stride;    /* runs row stride (>= topk), uniform over a batch   */
  int32_t pad_;
} ac_select_problem;

int ac_select(const ac_select_problem* probs, int nprob, int d, int scorer,
              int max_gq, int max_c, int max_topk, void* stream);
/* Top-p variant (an extension: the reference selects top-k only,
 * quest.py:128-143).  Per query cluster, the smallest prefix of the stable
 * score order whose estimated attention mass
 *   m_c = counts[c] * exp((scores[c] - max_c scores) * mass_scale)
 * reaches top_p of the total (at least one cluster, at most `topk` of the
 * problem); `selected` rows are padded with -1 past the chosen count.  Runs,
 * covered and density follow the chosen set.                              */
int ac_select_topp(const ac_select_problem* probs, int nprob, int d, int scorer,
                   int max_gq, int max_c, int max_topk, float top_p, float mass_scale,
                   void* stream);

/* One attention work item = one tile of <= 128 query rows of one query
 * cluster of one head (see ac_sparse_attention).                          */
typedef struct ac_attn_item {
  int64_t q_row0;        /* first row in the permuted query matrix Qp       */
  int32_t q_rows;        /* rows in this tile (<= 128)                       */
  int32_t head;          /* head index (selects Kp/Vp/out base)             */
  int32_t run0;          /* first run in the runs table                     */
  int32_t nruns;         /* number of [start,end) runs                       */
} ac_attn_item;

/* ---- substrate ops (tensorops.py:29-51, quest.py:74-91) ------------------
 * ac_matmul      out[m, n] = a[m, k] @ b[k, n] (f32) in the OpenBLAS
 *                accumulation `order` (AC_ORDER_*; ac_gemm_order(m, n, k))
 * ac_row_softmax out = softmax(scale * s) over the last axis (row-max
 *                subtraction), rows x cols f32
 * ac_quest_pairs out[g, c] = sum_t max(q[g,t]*emax[c,t], q[g,t]*emin[c,t]) in
 *                numpy's pairwise order (the scalar Quest bound, quest_scalar),
 *                evaluated one pair at a time like the reference's
 *                quest_scores_loop timing baseline (quest.py:80-91)          */
int ac_matmul(const float* a, int64_t m, int k, const float* b, int64_t n, float* out,
              int order, void* stream);
int ac_row_softmax(const float* s, int64_t rows, int64_t cols, float scale, float* out,
                   void* stream);
int ac_quest_pairs(const float* q, int gq, int d, const float* emax, const float* emin, int c,
                   float* out, void* stream);

/* ---- K12 permutation -----------------------------------------------------
 * dst[j] = src[perm[j]] for j < n (row gather, 16-byte vectors)            */
int ac_permute_rows(const void* src, int dtype, int d, const int32_t* perm,
                    int64_t n, void* dst, void* stream);

/* per-head gather: dst[h, j] = src[h, perm[h, j]]; rows of d elements must
 * be a multiple of 16 bytes (src/dst [heads, L, d], perm [heads, L])       */
int ac_permute_rows_heads(const void* src, int dtype, int d, const int32_t* perm,
                          int64_t L, int heads, void* dst, void* stream);

/* Query layout for the attention kernel (pipeline.py:154-165): per head h,
 * every query cluster g becomes a contiguous block of Qp rows padded to a
 * multiple of 128, and one work item per 128-row tile is emitted.
 *   q       [heads, L, d] queries (dtype), qperm/qstarts/qcounts/qlabels the
 *           query clustering of each head (member order), gq clusters per head
 *   qp      [heads * qp_cap, d] out (qp_cap = L + 128 * gq_max)
 *   qidx    [heads * qp_cap] out: original token of each Qp row or -1
 *   items   [heads * item_cap] out (item_cap = ceil(L/128) + gq_max); unused
 *           slots get q_rows = 0.  Item (h, g, tile) uses runs
 *           [(h*gq_max + g) * topk_max ...] with nruns[h*gq_max + g] runs.   */
int ac_build_q_layout(const void* q, int dtype, int d, int64_t L, int heads,
                      const int32_t* qperm, const int32_t* qstarts,
                      const int32_t* qcounts, const int32_t* qlabels,
                      const int32_t* gq, int gq_max, const int32_t* nruns,
                      int topk_max, void* qp, int32_t* qidx, int64_t qp_cap,
                      ac_attn_item* items, int item_cap, int item_rows,
                      void* stream);
/* rows per work item the attention kernel for (dtype, d) expects from
 * ac_build_q_layout: 256 for the two-tile tcgen05 kernel (bf16, d = 64),
 * else 128                                                                 */
int ac_attention_item_rows(int dtype, int d);
/* reorder `nitems` work items in place, longest first (Q tiles x K/V tiles of
 * their runs): the attention launch then issues them as greedy LPT list
 * scheduling.  Items write disjoint output rows, so results do not depend
 * on the order.  scratch: nitems * sizeof(ac_attn_item) bytes.             */
int ac_order_items(ac_attn_item* items, int nitems, const int32_t* runs,
                   ac_attn_item* scratch, void* stream);

/* ---- K13/K14 block-sparse attention --------------------------------------
 * One work item = one tile of <= 128 query rows of one query cluster of one
 * head.  Keys/values are in cluster-contiguous order (Kp/Vp, member order);
 * the item attends over the union of [start,end) runs of Kp.               */

/* q:  Qp [q_rows_total, d] (dtype), rows grouped per item
 * qidx: [q_rows_total] original token index of each Qp row (-1 = padding)
 * k/v: Kp/Vp [heads, L, d] (dtype), runs: [*, 2] int32 ranges into [0, L)
 * out: [heads, L, d] f32 or bf16 (out_dtype), written at original rows.
 * scale: softmax scale (1/sqrt(d) in the reference, reference.py:39).
 * bf16 inputs with d = 64 run on the two-Q-tile tcgen05 kernel (items of up to
 * 256 rows), d = 128 on the one-tile tcgen05 kernel; everything else (f32
 * inputs: the 1e-4 parity bar needs f32 math) on the CUDA-core kernel.     */
int ac_sparse_attention(const void* q, int64_t q_rows_total, const int32_t* qidx,
                        const void* k, const void* v, int dtype, int d, int64_t L,
                        int heads, const ac_attn_item* items, int nitems,
                        const int32_t* runs, float scale, void* out,
                        int out_dtype, void* stream);
/* explicit kernels (tests / benchmarks) */
int ac_sparse_attention_simt(const void* q, const int32_t* qidx, const void* k,
                             const void* v, int dtype, int d, int64_t L,
                             const ac_attn_item* items, int nitems,
                             const int32_t* runs, float scale, void* out,
                             int out_dtype, void* stream);
int ac_sparse_attention_fa4(const void* q, int64_t q_rows_total,
                            const int32_t* qidx, const void* k, const void* v,
                            int d, int64_t L, int heads,
                            const ac_attn_item* items, int nitems,
                            const int32_t* runs, float scale, void* out,
                            int out_dtype, void* stream);
/* head_dim 128: two Q tiles per CTA, P aliased into S (items of <= 256 rows) */
int ac_sparse_attention_fa4_d128(const void* q, int64_t q_rows_total,
                                 const int32_t* qidx, const void* k, const void* v,
                                 int d, int64_t L, int heads,
                                 const ac_attn_item* items, int nitems,
                                 const int32_t* runs, float scale, void* out,
                                 int out_dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADACLUSTER_SM100_H */
