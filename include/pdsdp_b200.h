/*
 * pdsdp_b200 — C ABI of the B200 (sm_100a) LR-PD-SDP hot path.
 *
 * The reference (`pdsdp`, pure Python) has no FFI layer; its boundary for
 * this path is the Python function API re-exported in
 * pkg/src/pdsdp/__init__.py:29-36.  Each entry point below is the native
 * replacement of one reference interface (cited per function).  Plain C
 * types only: host pointers, sizes, an opaque handle.  The library owns its
 * device memory; it never frees caller memory.  Every function returns 0 on
 * success or a negative PDSDP_E* code; pdsdp_last_error() describes the most
 * recent failure of the calling thread.
 *
 * Data layout at the boundary is the reference's: symmetric matrices packed
 * as the upper triangle read row by row, off-diagonal entries scaled by
 * sqrt(2) (pkg/src/pdsdp/symmat.py:50-101); constraint rows as strictly
 * increasing packed positions with sqrt(2)-scaled values
 * (pkg/src/pdsdp/problem.py:29-70), stacked [A; G] (problem.py:119-137).
 */
#ifndef PDSDP_B200_H
#define PDSDP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDSDP_OK 0
#define PDSDP_EINVAL (-1)   /* invalid argument (reference raises ValueError) */
#define PDSDP_ECUDA (-2)    /* CUDA runtime / launch failure */
#define PDSDP_ENOMEM (-3)   /* device or host allocation failure */
#define PDSDP_ERANK (-4)    /* target rank needs an eigen block above PDSDP_BLOCK_MAX */

#define PDSDP_BLOCK_MAX 64
#define PDSDP_OUT_LEN 16
#define PDSDP_KMAX 128

/* Output slots of one iteration (doubles, PDSDP_OUT_LEN per instance). */
enum {
  PDSDP_OUT_EPS_P = 0,   /* ||dX/alpha - M^T dy||   (pdhg.py:204)          */
  PDSDP_OUT_EPS_D = 1,   /* ||dy/alpha - M dX||     (pdhg.py:205-207)      */
  PDSDP_OUT_LAMBDA = 2,  /* lambda_{min(r+1,n)} of the projected argument (symmat.py:242-245) */
  PDSDP_OUT_FINITE = 3,  /* 1 if X+ and y+ are finite (pdhg.py:217-218)    */
  PDSDP_OUT_PASSES = 4,  /* eigensolver subspace passes                    */
  PDSDP_OUT_MATVECS = 5, /* operator applications S*Y (b columns each)     */
  PDSDP_OUT_EIGCONV = 6, /* 1 converged, 2 rounding floor, 0 pass limit    */
  PDSDP_OUT_EIGRES = 7,  /* worst unconverged relative Ritz residual       */
  PDSDP_OUT_DENSE = 8,
  PDSDP_OUT_CORR = 9,
  PDSDP_OUT_ED2 = 10,
  PDSDP_OUT_BLOCK = 11,  /* eigen block size b                              */
  PDSDP_OUT_DONE = 12,   /* 1 if the step executed (pdsdp_iterate_many)      */
  PDSDP_OUT_ERR = 13     /* 1 if the step needs an eigen block above PDSDP_BLOCK_MAX (continue in dense mode) */
};

/* One SDP in the reference's general form (problem.py:73-105). */
typedef struct pdsdp_problem {
  int32_t n;                /* matrix dimension                           */
  int32_t m;                /* equality rows  (len(A))                    */
  int32_t p;                /* inequality rows (len(G))                   */
  int32_t reserved;
  const double* C_packed;   /* [n(n+1)/2] objective, packed               */
  const int64_t* row_ptr;   /* [m+p+1] stacked [A; G] rows                */
  const int64_t* row_idx;   /* [nnz] packed positions                     */
  const double* row_val;    /* [nnz] packed values                        */
  const double* b;          /* [m]                                        */
  const double* h;          /* [p]                                        */
} pdsdp_problem;

typedef struct pdsdp_batch pdsdp_batch;

/* Upload `count` independent problems (SdpProblem.stacked, problem.py:119-137;
 * the re-indexing into dense coordinates happens here, once). */
int pdsdp_batch_create(int count, const pdsdp_problem* problems, pdsdp_batch** out);
int pdsdp_batch_destroy(pdsdp_batch* b);
int pdsdp_batch_info(const pdsdp_batch* b, int inst, int64_t* info /* [8] */);
/* cudaStream_t the batch launches on (for event timing by the caller). */
void* pdsdp_batch_stream(pdsdp_batch* b);

/* Operator norm by seeded power iteration (problem.py:157-185).  The start
 * vector is drawn by the caller with the reference's RNG
 * (numpy default_rng(seed).standard_normal(P), normalised) and passed
 * restricted to the touched positions returned by pdsdp_opnorm_positions.
 * Runs `iters` iterations from x0 (x0 == NULL: continue from the device
 * state) and writes ||M x|| of each into s_out. */
int pdsdp_opnorm_positions(pdsdp_batch* b, int inst, int64_t* pos_out, int64_t* count);
int pdsdp_opnorm_run(pdsdp_batch* b, int inst, const double* x0, int iters, double* s_out);

/* Step size alpha (pdhg.py:211-214) and iterate reset X0 = 0, y0 = 0
 * (lowrank.py:128-135). */
int pdsdp_set_alpha(pdsdp_batch* b, int inst, double alpha);
int pdsdp_reset(pdsdp_batch* b, int inst, double seed);

/* One LR-PDHG iteration (lowrank.py:141-150: approximate_primal_step,
 * dual_step, residuals) for each listed instance.  rank[i], ypar[i], flags[i]
 * per listed instance; out: nact * PDSDP_OUT_LEN doubles (host).
 * flags: bit 0 cold start, bit 1 certificate eigenvalue accurate, bit 2 re-run
 * of the last iteration from the same (X_k, y_k), bit 3 certificate to the
 * kept-pair tolerance (op-level aproj_psd), bits 8..11 extra guard columns of
 * the eigen block (0..15; wider blocks converge in fewer filter passes). */
int pdsdp_iterate(pdsdp_batch* b, int nact, const int32_t* insts, const int32_t* rank,
                  const int32_t* ypar, const int32_t* flags, int32_t maxpass, double* out);

/* Up to K (<= PDSDP_KMAX) consecutive iterations with one host synchronisation.
 * Step j of listed instance a runs with y parity ypar0[a]^j.  The device
 * pauses an instance after the first step whose combined residual
 * eps_p + eps_d is <= conv_thr[a] or >= stall_thr[a*K + j], or whose iterate
 * is not finite -- exactly the steps at which the host's Algorithm-2 logic
 * (lowrank.py:145-185) may act.  out: nact * K * PDSDP_OUT_LEN doubles;
 * steps_done[a] = executed steps.  The rank-adaptation decisions stay on the
 * host; the device only reports scalars. */
int pdsdp_iterate_many(pdsdp_batch* b, int nact, const int32_t* insts, const int32_t* rank,
                       const int32_t* ypar0, const int32_t* flags, int32_t maxpass, int32_t K,
                       const double* conv_thr, const double* stall_thr, double* out,
                       int32_t* steps_done);

/* Asynchronous per-instance chunks: the multi-instance analogue of the
 * reference's sequential bench rows (cli.py:284-329), scheduled on the device.
 * pdsdp_slots creates (once) as many streams as clusters of the iteration
 * kernel can be resident and returns that count; pdsdp_chunk_launch enqueues
 * up to K iterations of ONE instance on a slot (same arguments and pause rules
 * as pdsdp_iterate_many, stall_thr[K]) and returns at once; pdsdp_chunk_poll
 * returns 1 when the slot's chunk has finished (0 while running);
 * pdsdp_chunk_collect waits for it and copies the K * PDSDP_OUT_LEN outputs.
 * Chunks of different instances run side by side, each pausing at its own
 * events, so a batch finishes in about the time of its longest solve. */
int pdsdp_slots(pdsdp_batch* b, int32_t* nslots_out);
int pdsdp_chunk_launch(pdsdp_batch* b, int32_t slot, int32_t inst, int32_t rank, int32_t ypar0, int32_t flags,
                       int32_t maxpass, int32_t K, double conv_thr, const double* stall_thr);
int pdsdp_chunk_poll(pdsdp_batch* b, int32_t slot);
int pdsdp_chunk_collect(pdsdp_batch* b, int32_t slot, int32_t inst, int32_t K, double* out, int32_t* steps_done);

/* Dense-iterate mode: the same iteration with X_k held as a dense n x n matrix
 * and the projection done by a FULL eigendecomposition on the device
 * (one-sided Jacobi) -- the replacement of the reference's dense fallback
 * `full_eigen` / `np.linalg.eigh` (symmat.py:158-161), taken by
 * `truncated_eigen` for n <= 32, 2(r+1) > n or an ARPACK failure
 * (symmat.py:181-185,200-207) and by `proj_psd` of the exact solver
 * (symmat.py:223-226, pdhg.py:166-174).  pdsdp_iterate_many leaves a step
 * unfinished (slot 13 of its outputs set, steps_done excludes it, X_k / y_k
 * intact) when the projection argument has more positive eigenvalues than an
 * eigen block of PDSDP_BLOCK_MAX holds; pdsdp_dense_begin(from_factored = 1)
 * then expands X_k = F diag(lam) F^T and the solve continues with
 * pdsdp_iterate_dense (one iteration per call, any r <= n; same output slots;
 * slot 4 = Jacobi sweeps).  from_factored = 0 starts from X_0 = 0
 * (solve_pd_sdp with n > PDSDP_BLOCK_MAX, op-level aproj_psd).  pdsdp_reset
 * leaves dense mode.  pdsdp_objective / pdsdp_download_x follow the mode. */
int pdsdp_dense_begin(pdsdp_batch* b, int inst, int from_factored);
int pdsdp_iterate_dense(pdsdp_batch* b, int inst, int32_t r, int32_t ypar, double* out);

/* tr(C X) (lowrank.py:159,168,191) for X = the newest iterate (which = 0)
 * or the previous one (which = 1). */
int pdsdp_objective(pdsdp_batch* b, int inst, int which, double* out);

/* Download X packed (symmat.py:66-86 layout) and y. */
int pdsdp_download_x(pdsdp_batch* b, int inst, int which, double* packed_out);
int pdsdp_download_y(pdsdp_batch* b, int inst, int ypar, double* y_out);

/* Op-level entry points (reference problem.py:140-154, symmat.py:229-245). */
int pdsdp_apply_M(pdsdp_batch* b, int inst, const double* X_packed, double* out);
int pdsdp_apply_M_adjoint(pdsdp_batch* b, int inst, const double* y, double* out_packed);
int pdsdp_aproj_psd(int32_t n, const double* S_packed, int32_t r, double* P_packed_out, double* lambda_out);

/* Per-kernel CUDA-event timing of pdsdp_iterate (for the roofline report):
 * out[0] ms spanned by the executed iteration-kernel launches (CUDA events on
 * the library stream, one per launch), out[1] iterations executed, out[2]
 * residual-kernel ms (verification mode only), out[3] its launches, out[4]
 * iteration-kernel launches issued.  enable != 0 switches recording on and clears. */
int pdsdp_set_timing(pdsdp_batch* b, int enable);
int pdsdp_kernel_times(pdsdp_batch* b, double* out /* [5] */);

/* Verification mode: after every iteration also evaluate the dense part
 * ||dX/alpha||_F^2 of the primal residual (reference pdhg.py:198-208) entry by
 * entry over the upper triangle on the whole GPU (DMMA), into output slot 14,
 * next to the factored form the iteration uses (slot 8).  Off by default. */
int pdsdp_set_verify_residual(pdsdp_batch* b, int enable);

/* Eigensolver diagnostics of the last iteration of one instance:
 * out[0..256) per pass (m, worst rel residual, slow column, theta, t, lo, cut, ||X+||),
 * out[256..320) Ritz values, out[320..384) Ritz residual norms,
 * out[384..400) SM cycles per kernel phase (CTA 0), out[400..4504) the last
 * projected Rayleigh-Ritz matrix when flag bit 4 was set (b x b, b at 4496),
 * out[4504..4504 + 16*2048) per-CTA (label, SM cycle) traces of the last
 * launch with flag bit 6 (count at the last slot of each CTA's 2048). */
int pdsdp_debug(pdsdp_batch* b, int inst, double* out /* [4504] */);

const char* pdsdp_strerror(int code);
const char* pdsdp_last_error(void);
int pdsdp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PDSDP_B200_H */
