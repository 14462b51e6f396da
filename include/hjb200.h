/*
 * hjb200 -- C ABI of the B200-native block J-Jacobi hot path.
 *
 * Drop-in boundary for the reference's ``parallel_jacobi(G, signs,
 * SolverConfig) -> (G_out, DiagInfo)`` (reference:
 * pkg/src/hjacobi/parallel.py:255-309), its schedule generator
 * (strategies.py:143-176) and eigenpair extraction (rotations.py:226-251).
 * Plain pointers and sizes only; no torch types.  Every entry point returns
 * an hjb_status; hjb_last_error() returns a message for the calling thread.
 *
 * Conventions (as the reference, core.py:1-34): G is column-major, m x n,
 * leading dimension ldg >= m, float64 or complex128 (interleaved re/im);
 * signs is an int8 vector of +-1.  Block index / ring rank conventions follow
 * strategies.py (1-based block indices, nbl = 2p).
 */
#ifndef HJB200_H
#define HJB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HJB_ABI_VERSION 2

typedef enum {
  HJB_OK = 0,
  HJB_EINVAL = 1,            /* -> ValueError (parallel.py:55-62, 264-265)          */
  HJB_PIVOT_INDEFINITE = 2,  /* -> PivotDefinitenessError(r, s) (rotations.py:198)  */
  HJB_CHOL_FAIL = 3,         /* -> DefinitenessError (blocking.py:106-112)          */
  HJB_ECUDA = 4,             /* -> RuntimeError                                      */
  HJB_ENCCL = 5,             /* -> RuntimeError                                      */
  HJB_ENOMEM = 6             /* -> MemoryError                                       */
} hjb_status;

typedef enum { HJB_F64 = 0, HJB_C128 = 1 } hjb_dtype;
typedef enum { HJB_MODULUS = 0, HJB_ROUND_ROBIN = 1 } hjb_strategy;   /* strategies.py:14-16 */
typedef enum { HJB_HOST = 0, HJB_DEVICE = 1 } hjb_memspace;

typedef struct {
  int32_t dtype;          /* hjb_dtype */
  int32_t memspace;       /* where G_in / G_out live */
  int64_t m, n;           /* rows, columns of G */
  int64_t ldg;            /* leading dimension of G_in and G_out (>= m) */
  const void *G_in;       /* input factor (not modified unless G_out == G_in on device) */
  void *G_out;            /* output factor, same column order as G_in (parallel.py:299-301) */
  const int8_t *signs;    /* host pointer, n entries of +-1 */
  int32_t p;              /* ring workers; nbl = 2p uniform blocks (parallel.py:266) */
  int32_t strategy;       /* hjb_strategy */
  double orth_tol;        /* <= 0: sqrt(rows of swept factor)*eps (rotations.py:76-77) */
  double quad_tol;        /* <= 0: cols of swept factor * eps (rotations.py:79-80) */
  int32_t max_sweeps;     /* outer and inner sweep cap (rotations.py:67) */
  int32_t device;         /* CUDA device ordinal */
  void *stream;           /* cudaStream_t to run on; NULL = library stream */
  void *comm;             /* hjb_comm from hjb_comm_init, or NULL for one GPU */
  int32_t flags;          /* HJB_FLAG_* */
  int32_t first_sweep;    /* resume: G_in is the state after sweep first_sweep-1
                             (<= 1: a fresh solve); the ring layout of that sweep
                             is replayed (strategies.py:58-136) */
  int32_t sweep_count;    /* outer sweeps to run from first_sweep (0: until
                             convergence or max_sweeps); converged = 1 when the
                             last one applied no rotation (parallel.py:242-244) */
} hjb_problem;

#define HJB_FLAG_PHASE_TIMES 1   /* record per-phase device times (adds events) */
#define HJB_FLAG_VARIANT_B 8     /* block-oriented variants 2B / 3B (parallel.py:160-174, 199-200):
                                    no F pre-pass, dense pair factor, one annihilation
                                    cycle per step; default: the F variants (2F / 3F) */
#define HJB_FLAG_NO_TAIL_SPLIT 16 /* run the Jacobi launch of a step as one launch on the solve
                                    stream (default: its last, mostly empty wave of pivots
                                    runs on a second stream beside the update of the others;
                                    same arithmetic, bitwise identical results) */
#define HJB_FLAG_GATHER_ROOT 4   /* multi-GPU: only rank 0 receives the whole G_out
                                    (other ranks keep the blocks they hold);
                                    default: every rank receives it */

typedef struct {
  int32_t sweeps;           /* DiagInfo.sweeps (rotations.py:111) */
  int32_t converged;        /* DiagInfo.converged */
  int64_t rotations;        /* DiagInfo.rotations (incl. inner and pre-pass) */
  int64_t big_rotations;    /* DiagInfo.big_rotations */
  double max_abs_t;         /* DiagInfo.max_abs_t */
  int32_t fail_rank;        /* worker rank that raised (parallel.py:296-298), else -1 */
  int32_t fail_r, fail_s;   /* PivotDefinitenessError(r, s) indices, else -1 */
  int64_t pairs_visited;    /* pair steps executed (Gram always computed) */
  int64_t pairs_updated;    /* pair steps whose update ran (parallel.py:203) */
  int64_t prepass_visited;  /* pre-pass blocks (parallel.py:138-148) */
  int64_t prepass_updated;  /* pre-pass blocks whose update ran (parallel.py:145) */
  int64_t fallbacks;        /* dense-Cholesky fallbacks (parallel.py:196-198) */
  double t_total_ms;        /* device time of the solve (H2D/D2H excluded) */
  double t_gram_ms, t_pivot_ms, t_update_ms, t_exchange_ms;  /* with HJB_FLAG_PHASE_TIMES */
  int64_t exchange_bytes;   /* bytes sent over NCCL by this rank */
  int32_t cluster_size;     /* pivot-kernel cluster size used */
  int32_t gram_splits;      /* split-K factor of the Gram kernel */
  int64_t inner_sweeps;     /* sum of inner (pivot-level) sweeps over all pivots */
  int64_t inner_pair_visits;/* inner 2x2 pivots examined (sweeps * N(N-1)/2 per pivot) */
  int64_t kernel_launches;  /* kernels this library launched for the solve (this GPU) */
  int64_t tail_splits;      /* steps whose Jacobi launch was split over two streams */
} hjb_result;

/* Library / ABI version (HJB_ABI_VERSION). */
int hjb_version(void);
/* Message for the last non-OK status on this thread. */
const char *hjb_last_error(void);
/* Number of visible CUDA devices (0 without a GPU); never fails. */
int hjb_device_count(void);

/*
 * Whole 2F ring solve: replaces parallel_jacobi(G, signs, SolverConfig(
 * variant="2F", strategy, p, tol=Tolerances(orth_tol, quad_tol, max_sweeps)))
 * (parallel.py:255-309; solve.py:44-64 dispatches here).  Non-convergence is
 * not an error: HJB_OK with converged = 0 (parallel.py:307).
 */
int hjb_solve(const hjb_problem *prob, hjb_result *res);

/*
 * Ring schedule, bit-exact with generate_sweep_schedule (strategies.py:143-176)
 * and the per-worker StepPlans (strategies.py:75-136).  layouts: int32
 * [steps][p][2] (i_blk, j_blk); plans (may be NULL): int32 [steps][p][4]
 * (snd_rnk, snd_blk, rcv_rnk, rcv_blk); steps = sweeps * steps_per_sweep.
 * Host-only; needs no GPU.
 */
int hjb_schedule(int32_t strategy, int32_t p, int32_t sweeps, int32_t *layouts,
                 int32_t *plans);
/* The uniform block partition of the ring (blocking.py:63-68, parallel.py:
 * 266): nbl blocks of near-equal width, wider ones first; offsets: int64
 * [nbl + 1] (offsets[nbl] = n).  Host-only. */
int hjb_partition(int64_t n, int32_t nbl, int64_t *offsets);
/* steps_per_sweep (strategies.py:27-28). */
int hjb_steps_per_sweep(int32_t strategy, int32_t p);

/*
 * Eigenpair extraction on device (rotations.py:226-251): lam[k] =
 * signs[k]*||g_k||^2, U[:,k] = g_k/||g_k||, then U[:, out] = U[:, perm[out]]
 * if perm != NULL (perm is a device int64 array).  G, U, lam device
 * pointers; U may alias G only when perm == NULL.  Returns HJB_CHOL_FAIL
 * (StructuralError) on a zero column.
 */
int hjb_extract(int32_t dtype, int64_t m, int64_t n, const void *G, int64_t ldg,
                const int8_t *signs_dev, double *lam, void *U, int64_t ldu,
                const int64_t *perm, void *stream);

/*
 * Orthogonality metric of solve.py:108-110 on device: *out = max |U^H U - I|
 * over all entries (host double).  U is a device m x n matrix, ld ldu (even
 * for float64).  Formed with the Gram kernel over all 64-column block pairs
 * (i <= j) and a max-fold kernel; replaces the host O(m n^2) product.
 */
int hjb_orthogonality(int32_t dtype, int64_t m, int64_t n, const void *U, int64_t ldu, double *out,
                      void *stream);

/* ---- kernel-level entry points (device pointers), used by parity tests ---- */

/*
 * Batched Gram of column-block pairs: for item t with column offsets
 * (oi, oj) and widths (ni, nj): A_t = G[:, oi:oi+ni]^H G[:, oj:oj+nj]
 * (core.py:42-56), D_t[0:ni] = colnorms^2 of the first block and
 * D_t[bmax:bmax+nj] of the second.  nj == 0 means the diagonal Gram of the
 * first block (ni x ni, upper triangle meaningful).  items: int32 [count][4].
 * A: [count][bmax*bmax] column-major ld bmax; D: [count][2*bmax].
 */
int hjb_gram(int32_t dtype, int64_t m, const void *G, int64_t ldg, const int32_t *items_host,
             int32_t count, int32_t bmax, void *A, double *D, void *stream);

/*
 * Pivot diagonalisation for a batch of items (parallel.py:193-202 +
 * blocking.py:115-138 + rotations.py:203-223): builds R by the structured
 * Cholesky from (D_i, A_ij, D_j) -- or, for nj == 0, R = chol(A) -- then
 * diagonalises R with the tournament-ordered J-Jacobi and returns the
 * accumulated W ([count][NMAX*NMAX], ld NMAX where NMAX = 2*bmax rounded to a
 * supported size) and per-item stats int64/double [count][8]:
 * (rotations, big, max_t bits, inner sweeps, status, fail_r, fail_s, fallback).
 * R_out (optional, may be NULL) receives the final R.
 */
int hjb_pivot(int32_t dtype, int64_t m, const void *G, int64_t ldg, const int32_t *items_host,
              int32_t count, int32_t bmax, const void *A, const double *D,
              const int8_t *signs_dev, double orth_tol, double quad_tol, int32_t max_sweeps,
              void *W, int64_t *stats, void *R_out, int32_t cluster, void *stream);

/*
 * The pivot kernel's 2x2 rotation (rot_coef, the restatement of
 * _kernels.py:53-81) on a batch of 2x2 Gram pivots [[a_rr, a_rs],
 * [conj(a_rs), a_ss]] with signs (j_rr, j_ss): replaces
 * compute_plane_rotation (rotations.py:128-155).  Host arrays (a_rs is
 * float64 or complex128 per dtype); out: double [count][8] = (code, cs, sn,
 * t, eta, phase_re, phase_im, hyp); code 1 rotation, 0 identity (a_rs == 0),
 * -1 not positive definite (-> PivotDefinitenessError).  Runs on the
 * current CUDA device.
 */
int hjb_plane_rotations(int32_t dtype, int32_t count, const double *a_rr, const double *a_ss,
                        const void *a_rs, const int8_t *j_rr, const int8_t *j_ss, double *out);

/*
 * The inner J-Jacobi alone (rotations.py:203-223, the ring-of-rings kernel):
 * diagonalise the given factors R0 (device [count][ld*ld], ld =
 * hjb_pivot_ld(bmax), column-major, item t of order ni+nj) into R_out until
 * an inner sweep applies no rotation.  stats (device int64 [count][8]) is
 * zeroed and receives (rotations, big, max_t bits, inner sweeps, status,
 * fail_r, fail_s, 0); status 1 = PivotDefinitenessError(fail_r, fail_s).
 * Test hook for the failure paths of _kernels.py:59-60, 73-74.
 */
int hjb_jacobi(int32_t dtype, const int32_t *items_host, int32_t count, int32_t bmax, const void *R0,
               void *R_out, const int8_t *signs_dev, double orth_tol, double quad_tol, int32_t max_sweeps,
               int64_t *stats, int32_t cluster, void *stream);

/* Leading dimension of W / R_out used by hjb_pivot for a given bmax. */
int hjb_pivot_ld(int32_t bmax);
/* Debug: record phase clocks of later hjb_pivot / hjb_jacobi calls into a
 * device int64 buffer (NULL disables): per CTA [count*cluster][8] for the
 * round-1 pivot kernel, per warp [count*C*W][8] for the Jacobi kernel
 * (builds with -DHJB_JAC_PROF=1). */
int hjb_pivot_set_profile(void *prof);
/* Tuning override (experiments): threads per CTA of the round-1 pivot kernel
 * (128/256/512, the instantiated shapes) and the cluster size (1..16) of the
 * pivot / Jacobi kernel; 0 restores the automatic choice.  An unsupported
 * combination makes the next launch fail with "invalid configuration". */
int hjb_tune(int32_t pivot_threads, int32_t pivot_cluster);
/* Inner pair order of hjb_pivot for (dtype, bmax, count, cluster; 0 = auto):
 * the warp-block order over *nmax column positions in *warps warps per CTA
 * (oracle: diagonalize(order="wblock:NMAX:WARPS")).  Replaces nothing in the
 * reference (its inner order is sequential, _kernels.py:41-52); test hook. */
int hjb_pivot_order(int32_t dtype, int32_t bmax, int32_t count, int32_t cluster, int32_t *nmax,
                    int32_t *warps);
/* Inner pair order of hjb_pivot / hjb_solve for (dtype, bmax, count,
 * cluster; 0 = auto): desc int32[5] = (1, NMAX, WARPS, 0, 0) for the round-1
 * pivot kernel's warp-block order (oracle "wblock:NMAX:WARPS"), or (2, NMAX,
 * C, W, SPW) for the ring-of-rings Jacobi kernel (oracle
 * "ror:NMAX:C:W:SPW": the reference's round-robin stepper, strategies.py:
 * 95-136, over 2CW sub-blocks of SPW columns).  Test hook. */
int hjb_inner_order(int32_t dtype, int32_t bmax, int32_t count, int32_t cluster, int32_t *desc);
/* Max co-resident clusters of the pivot kernel instance for (dtype, bmax,
 * cluster, threads) on the current device (negative: cudaError). */
int hjb_pivot_occupancy(int32_t dtype, int32_t bmax, int32_t cluster, int32_t threads);

/*
 * Block update [G_i G_j] <- [G_i G_j] W for items whose stats[0] > 0
 * (parallel.py:203-207), in place.  W as produced by hjb_pivot.
 */
int hjb_update(int32_t dtype, int64_t m, void *G, int64_t ldg, const int32_t *items_host,
               int32_t count, int32_t bmax, const void *W, const int64_t *stats,
               void *stream);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) ---- */

/*
 * Block transfers of one GPU in the multi-GPU ring (host-only): GPU `rank`
 * of `world` hosts ring workers [rank*p/world, (rank+1)*p/world); after each
 * step the block columns exchanged with workers on other GPUs are sent or
 * received (parallel.py:212-221; strategies.py:69-72).  out: int32
 * [steps][max_xfers][3] = (0-based block, peer GPU, 1 = send / 0 = receive);
 * counts: int32 [steps].  steps = sweeps * steps_per_sweep.
 */
int hjb_exchange_plan(int32_t strategy, int32_t p, int32_t world, int32_t rank, int32_t sweeps,
                      int32_t max_xfers, int32_t *out, int32_t *counts);

/*
 * Final block ownership of the multi-GPU ring (host-only): owner[b] = GPU
 * holding 0-based block b after `sweeps` complete sweeps -- the layout
 * parallel_jacobi reassembles G_out from (parallel.py:299-301).  The ring
 * layout repeats every 2 sweeps (strategies.py:69-72), so odd and even sweep
 * counts give different owners.  owner: int32 [2p].
 */
int hjb_block_owners(int32_t strategy, int32_t p, int32_t world, int32_t sweeps, int32_t *owner);

/* 128-byte NCCL unique id for rank 0 to broadcast (e.g. via torch.distributed). */
int hjb_comm_unique_id(char out[128]);
/* Create the communicator of this rank; *comm receives an opaque handle. */
int hjb_comm_init(const char id[128], int32_t world, int32_t rank, int32_t device, void **comm);
int hjb_comm_destroy(void *comm);

#ifdef __cplusplus
}
#endif
#endif /* HJB200_H */
