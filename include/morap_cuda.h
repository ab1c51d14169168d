/*
 * morap_cuda.h -- C ABI of the B200 value-iteration backend (libmorap_cuda.so).
 *
 * This is the drop-in boundary for the reference's job engine. The reference runs every
 * Bellman solve as a move-only Job through
 *     std::map<long,JobResult> runBatch(std::vector<Job>, const PoolConfig&)
 *         (/root/reference/proj/include/morap/engine.hpp:370-425; Job/JobResult :40-64)
 * with CPU worker threads calling
 *     optimalSchedulerOn   (numerics.hpp:74-122)   -- JobKind::Optimize
 *     evaluateSchedulerOn  (numerics.hpp:130-168)  -- JobKind::Evaluate
 * and the "stub accelerator" queues (engine.hpp:111,254-259) are where an accelerator
 * was meant to plug in. Here the product MDPs are uploaded ONCE (the reference keeps them
 * alive as shared_ptr<const ProductMdp> for the whole query, instance.hpp:26) and every
 * batch of jobs runs on the GPU. Plain pointers and sizes only; nothing throws across the
 * ABI; every function returns a status (0 = ok, otherwise 1 + morap::Errc, common.hpp:12-34).
 *
 * Arithmetic contract: fp64 values/probabilities/rewards, int32 indices (model.hpp:19-34).
 * Each row value is accumulated left to right from rho[r] with separately rounded
 * multiply and add (no FMA), ties in the argmax go to the lowest row, done states are
 * pinned to 0, and each job stops at its own sweep -- so values, sweeps, residuals and
 * policies are BITWISE identical to the reference CPU solver.
 *
 * Threading: a context is driven by one host thread at a time (SPEC.md:628 says the same
 * of runBatch). Results do not depend on the device or on how jobs are batched.
 */
#ifndef MORAP_CUDA_H
#define MORAP_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 0 ok, else 1 + morap::Errc (common.hpp:12-34). */
enum {
  MORAP_OK = 0,
  MORAP_SYNTAX = 1,
  MORAP_NOT_CO_SAFE = 2,
  MORAP_CLOSURE_BLOWUP = 3,
  MORAP_INVALID_DFA = 4,
  MORAP_INVALID_MODEL = 5,
  MORAP_NOT_REWARD_FINITE = 6,
  MORAP_NON_CONVERGENCE = 7,
  MORAP_SINGULAR_SYSTEM = 8,
  MORAP_DIMENSION_MISMATCH = 9,
  MORAP_NON_SQUARE = 10,
  MORAP_NOT_BISTOCHASTIC = 11,
  MORAP_NO_PERFECT_MATCHING = 12,
  MORAP_NOT_POSITIVE_DEFINITE = 13,
  MORAP_SOLVER_FAILURE = 14,
  MORAP_DEGENERATE_DIRECTION = 15,
  MORAP_SIZE_GUARD = 16,
  MORAP_CYCLE_GUARD = 17,
  MORAP_INVALID_CONFIG = 18,
  MORAP_GENERATION_FAILURE = 19,
  MORAP_NO_CERTIFICATE = 20,
  MORAP_IO = 21,
  MORAP_CUDA_ERROR = 100 /* CUDA runtime failure (no Errc equivalent) */
};

#define MORAP_MAX_OBJECTIVES 8 /* reward vectors per model (K; the reference has K = 2) */
#define MORAP_MAX_RHS 8        /* reward vectors evaluated together in one fused sweep */

typedef struct morap_ctx morap_ctx;
typedef struct morap_image morap_image;

/* Host view of one product MDP (ProductMdp, model.hpp:143-157): CSR in the reference
 * layout. rewards[k] has num_rows entries: rewards[0] = cost, rewards[1] = success
 * (model.hpp:150-151), further entries are extra objectives (K > 2 extension). */
typedef struct {
  int32_t num_states;
  int32_t num_rows;
  int32_t nnz;
  int32_t initial;
  int32_t reward_finite; /* ProductMdp::rewardFinite (model.hpp:152) */
  int32_t num_objectives;
  const int32_t* row_offset; /* num_states + 1 */
  const int32_t* trn_offset; /* num_rows + 1 */
  const int32_t* succ;       /* nnz */
  const double* prob;        /* nnz */
  const uint8_t* done;       /* num_states, 0/1 */
  const double* const* rewards;
} morap_csr_view;

/* Context on CUDA device `device` (replaces the PoolConfig + engine lifetime,
 * engine.hpp:66-72,370). */
int morap_cuda_create(int device, morap_ctx** out);
int morap_cuda_destroy(morap_ctx* ctx);
/* Launch on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL restores the context's own stream. */
int morap_cuda_set_stream(morap_ctx* ctx, void* cuda_stream);
const char* morap_cuda_last_error(morap_ctx* ctx);

/* Upload models once; device copies are immutable until morap_cuda_release_models.
 * Replaces the shared_ptr<const ProductMdp> handed to every Job (engine.hpp:43).
 * Validates CSR structure (offsets monotone, successors in range) -> MORAP_INVALID_MODEL. */
int morap_cuda_upload(morap_ctx* ctx, int nmodels, const morap_csr_view* models, int32_t* model_ids_out);
int morap_cuda_release_models(morap_ctx* ctx);
/* The same upload in two steps: morap_cuda_build_image does everything but the copy --
 * validation, tiling and the compact streams on the host threads, packed in the device
 * layout into pinned host memory (the product builder's batched-CSR output, built once
 * per instance; it honours the context's lean setting); morap_cuda_upload_image then
 * moves it to the device in one copy and returns model ids as morap_cuda_upload does.
 * An image can be uploaded any number of times (e.g. after morap_cuda_release_models). */
int morap_cuda_build_image(morap_ctx* ctx, int nmodels, const morap_csr_view* models, morap_image** image_out);
int morap_cuda_upload_image(morap_ctx* ctx, const morap_image* image, int32_t* model_ids_out);
void morap_cuda_free_image(morap_image* image);
/* Lean uploads (for instances that do not fit otherwise, e.g. 100 x 100): a model with a
 * compact alphabet (<= 256 distinct probabilities and objective tuples) is stored without
 * its fp64 prob / objective arrays -- the device reads the exact same values from the
 * model's dictionary and class table. Lean models take weighted optimize jobs and
 * policy-chain evaluations (<= 4 objectives), not explicit reward vectors. Applies to
 * models uploaded after the call, and only where the compact sweep kernels run (with
 * MORAP_COMPACT=0 or MORAP_SWEEP_KERNEL=global every model keeps its arrays). */
int morap_cuda_set_lean(morap_ctx* ctx, int on);
/* Frozen-tile skipping in compact optimize sweeps (default on; MORAP_SKIP=0 at create turns
 * it off): a tile whose successor window and own states did not change bitwise in the
 * previous sweep is not swept again -- it would reproduce its values bit for bit. Values,
 * policies, residuals and sweep counts are identical either way. */
int morap_cuda_set_skip(morap_ctx* ctx, int on);
/* Diagnostics: enable (1) / disable (0) / leave (-1) the per-CTA timeline of compact
 * optimize sweeps, and copy up to n words of it to `out` (when non-null): 128 slots (sweep
 * index mod 128) x sweep CTAs x 4 globaltimer ns {start, first stage consumed, all warps
 * done, finalize done (last CTA only)}. */
int morap_cuda_debug_cta_trace(morap_ctx* ctx, int enable, uint64_t* out, int64_t n);

/* Device product builder: buildProduct (model.hpp:230-321) + checkRewardFinite
 * (model.hpp:163-206) + the upload preparation, on the GPU. Builds the products of `npairs`
 * (agent, task) pairs straight into device memory as lean compact models (two objectives:
 * cost, success) -- the host never holds their arrays. Agents come as CSR MDPs whose
 * probabilities / costs are indices into a shared alphabet (exact fp64 bit patterns), tasks
 * as DFAs with pre-sinks already inserted (insertPreSinks) and their letters per label set. */
typedef struct {
  int32_t num_states, num_rows, nnz, initial;
  const int32_t* row_offset; /* num_states + 1 */
  const int32_t* trn_offset; /* num_rows + 1 */
  const int32_t* succ;       /* nnz */
  const int32_t* prob_cand;  /* nnz: index into morap_build_alphabet.probs */
  const int32_t* cost_cand;  /* num_rows: index into morap_build_alphabet.costs */
  const int32_t* name_id;    /* num_rows: action-name id (product identity only) */
  const int32_t* label_set;  /* num_states: label-set id */
} morap_build_agent;
typedef struct {
  int32_t num_locations, num_letters, initial;
  const int32_t* delta;         /* num_locations x num_letters */
  const uint8_t* flags;         /* per location: 1 accepting, 2 trap, 4 pre-sink */
  const int32_t* letter_of_set; /* per label-set id: the letter (bitmask over the task's atoms) */
} morap_build_task;
typedef struct {
  int32_t num_probs, num_costs, internal_name; /* <= 1024 probabilities, < 1024 costs */
  int32_t num_label_sets;
  const double* probs;                         /* distinct bit patterns, must contain 1.0 */
  const double* costs;                         /* distinct bit patterns */
} morap_build_alphabet;
typedef struct {
  int32_t status; /* MORAP_OK, or MORAP_INVALID_CONFIG: not compact (> 256 probabilities ...) */
  int32_t num_states, num_rows, nnz;
  int32_t reward_finite;
  int32_t ntiles;
  uint64_t hash;  /* identity of the product's arrays (equal products, equal hash) */
  uint64_t bytes; /* device bytes of the built model */
} morap_build_info;
/* write == 0 (measure): fills info[] only. write == 1: builds and registers the models
 * (model_ids_out[k]); info[] must hold the measure results of the same pairs (sizes). */
int morap_cuda_build_products(morap_ctx* ctx, int nagents, const morap_build_agent* agents, int ntasks,
                              const morap_build_task* tasks, const morap_build_alphabet* alphabet, int npairs,
                              const int32_t* pairs, int write, morap_build_info* info, int32_t* model_ids_out);
/* Test support: 17 FNV digests of a device model's arrays (rowOffset, trnOffset, succ, done,
 * probIdx, rclass, tileStart, tiles, probDict, classTable, stW, rowW, trW, tilePos, outIdx,
 * outGrp, outSucc), so a device-built model can be compared with the host-prepared upload. */
int morap_cuda_debug_model_digest(morap_ctx* ctx, int model_id, uint64_t* out17);
int morap_cuda_num_models(morap_ctx* ctx);
/* out[6] = {S, R, nnz, number of objectives, compact (0/1), lean (0/1)} of a device model. */
int morap_cuda_model_info(morap_ctx* ctx, int model_id, int32_t* out);

/* JobKind::Optimize batch (engine.hpp:126-131 -> numerics.hpp:74). Job k runs on model
 * model_ids[k] with rho = weightedReward(objectives, weights[k*K .. k*K+K-1])
 * (numerics.hpp:224, as built by supportingPoint solver.hpp:118-128). Per job: value at
 * the initial state, sweep count, final residual and status (MORAP_OK,
 * MORAP_NOT_REWARD_FINITE, MORAP_NON_CONVERGENCE). Returns the first job failure's
 * status only for whole-batch errors; per-job failures are contained in status_out like
 * JobResult{ok=false, errc} (engine.hpp:140-150). Final values and policies stay on the
 * device until the next optimize call. */
int morap_cuda_optimize(morap_ctx* ctx, int njobs, const int32_t* model_ids, const double* weights, int K,
                        double eps, int sweep_cap, double* value_out, int32_t* sweeps_out,
                        double* residual_out, int32_t* status_out);

/* Same, with an explicit per-job reward vector (Job::reward, engine.hpp:44) of num_rows
 * entries for its model. */
int morap_cuda_optimize_rho(morap_ctx* ctx, int njobs, const int32_t* model_ids, const double* const* rho,
                            double eps, int sweep_cap, double* value_out, int32_t* sweeps_out,
                            double* residual_out, int32_t* status_out);

/* Results of the last optimize batch: final value vector (OptimizeResult::values) and the
 * argmax scheduler of the final sweep (OptimizeResult::policy as deterministic rows,
 * done states -> first row, numerics.hpp:114-118). */
int morap_cuda_fetch_values(morap_ctx* ctx, int job, double* values_out);
int morap_cuda_fetch_policy(morap_ctx* ctx, int job, int32_t* rows_out);
/* Policies of several optimize jobs in one batch (one synchronisation): rows_out[q]
 * receives the num_states rows of job jobs[q]. */
int morap_cuda_fetch_policies(morap_ctx* ctx, int njobs, const int32_t* jobs, int32_t* const* rows_out);
/* Zero-copy variant: rows_out[q] points at job jobs[q]'s rows in the library's pinned
 * staging area (morap_cuda_evaluate_optimized stages the evaluated jobs' policies there
 * while its sweeps run), valid until the next optimize batch or policy fetch. */
int morap_cuda_policy_views(morap_ctx* ctx, int njobs, const int32_t* jobs, const int32_t** rows_out);

/* Fused JobKind::Evaluate of optimize jobs' own schedulers (supportingPoint's cost and
 * success jobs, solver.hpp:148-172): for each listed optimize job, evaluate its final
 * policy under nrhs of its model's objective vectors (objective[0..nrhs-1]) in ONE
 * multi-RHS sweep; every RHS stops on its own (delta <= eps) exactly as separate
 * evaluateSchedulerOn calls would. Outputs are njobs x nrhs, row-major. */
int morap_cuda_evaluate_optimized(morap_ctx* ctx, int njobs, const int32_t* opt_jobs, int nrhs,
                                  const int32_t* objective, double eps, int sweep_cap, double* value_out,
                                  int32_t* sweeps_out, double* residual_out, int32_t* status_out);

/* General JobKind::Evaluate batch: job k evaluates the deterministic scheduler
 * policies[k] (num_states rows) on model model_ids[k] under the explicit reward rho[k]
 * (num_rows). A policy row outside its state's rows -> MORAP_INVALID_MODEL for that job
 * (checkScheduler, numerics.hpp:51-66). */
int morap_cuda_evaluate(morap_ctx* ctx, int njobs, const int32_t* model_ids, const int32_t* const* policies,
                        const double* const* rho, double eps, int sweep_cap, double* value_out,
                        int32_t* sweeps_out, double* residual_out, int32_t* status_out);

/* Value vector of (job, rhs) from the last evaluate call. */
int morap_cuda_fetch_eval_values(morap_ctx* ctx, int job, int rhs, double* values_out);

/* Instrumentation (SweepStats/bench). Totals since the last reset:
 *   out[0] sweep-kernel launches (optimize), out[1] their summed device ms (only while
 *   profiling is on: CUDA events around each launch, no extra synchronisation), out[2] algorithmic bytes those
 *   launches moved (per swept tile: 4*nnz + 4*R + 20*S for compact models, 12*nnz + 12*R +
 *   21*S otherwise), out[3] nnz backups of the results (sum over jobs of
 *   sweeps * nnz: the reference's work), out[4..7] the same four for evaluate sweeps,
 *   out[8] kernels launched in total, out[9] host-to-device bytes of model uploads,
 *   out[10] optimize backups actually executed (out[3] minus the frozen tiles skipped). */
int morap_cuda_set_profiling(morap_ctx* ctx, int on);
int morap_cuda_stats(morap_ctx* ctx, double* out, int nout);
int morap_cuda_reset_stats(morap_ctx* ctx);
int morap_cuda_device_bytes(morap_ctx* ctx, int64_t* bytes_out);

#ifdef __cplusplus
}
#endif

#endif /* MORAP_CUDA_H */
