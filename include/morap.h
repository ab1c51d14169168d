/*
 * morap.h -- C ABI of the host library (libmorap_host.so): model loader, per-instance
 * GPU upload and the Pareto-point query, for FFI callers (ctypes/cffi, another language's
 * runtime). The C++ API behind it is paper_2305_04397_b200/csrc/morap.hpp, which mirrors
 * the reference's public functions; each entry below names the reference function it
 * exposes (/root/reference/proj/include/morap/...). The reference itself has no C ABI:
 * its front door is the `morap` CLI (cli.hpp:331), whose verbs map onto these calls
 * (INTEGRATION.md).
 *
 * Conventions: every function returns 0 or 1 + morap::Errc (common.hpp:12-34), 100 for a
 * CUDA failure; the message of the last failure on the calling thread is
 * morap_last_error(). Nothing throws across the ABI. Pointers are host pointers.
 */
#ifndef MORAP_H
#define MORAP_H

#include <stdint.h>

#include "morap_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct morap_instance morap_instance;
typedef struct morap_solver morap_solver;

const char* morap_last_error(void);

/* generateInstance (warehouse.hpp:176) from a warehouseConfigFromJson object
 * (warehouse.hpp:200): {"W","H","n","slip","racks","feed","seed","deadline"}.
 * threads <= 0: all host threads build the n^2 products (buildInstance, instance.hpp:42). */
int morap_instance_warehouse(const char* config_json, int threads, morap_instance** out);

/* instanceFromJson (cli.hpp:93-117): {"agents": [...], "tasks": [...], "norm"?: [[...]]}.
 * Relative paths resolve against base_dir. If the file carries a norm matrix and
 * norm_out is non-null, the d x d matrix is written there (norm_cap doubles available)
 * and *has_norm is set. */
int morap_instance_from_json(const char* json_text, const char* base_dir, morap_instance** out, double* norm_out,
                             int norm_cap, int* has_norm);
/* instanceFromJson with the products built on the GPU of `s` (morap_cuda_build_products); the
 * instance then answers queries on `s` only (two objectives; see morap_instance_warehouse_device). */
int morap_instance_from_json_device(const char* json_text, const char* base_dir, morap_solver* s,
                                    morap_instance** out, double* norm_out, int norm_cap, int* has_norm);
void morap_instance_free(morap_instance* inst);

/* out[8] = {n, realTasks, distinctProducts, K, sum states, sum rows, sum nnz over the n^2
 * (i,j) slots, sum nnz over distinct products}. */
int morap_instance_info(const morap_instance* inst, int64_t* out);

/* Product (i, j) of the instance (ProductMdp, model.hpp:143-157).
 * dims[6] = {S, R, nnz, initial, rewardFinite, index of the first (i',j') sharing it}. */
int morap_instance_product_dims(const morap_instance* inst, int i, int j, int64_t* dims, uint64_t* structural_hash);
int morap_instance_product_export(const morap_instance* inst, int i, int j, int32_t* row_offset, int32_t* trn_offset,
                                  int32_t* succ, double* prob, double* cost, double* success, uint8_t* done,
                                  uint8_t* accept);

/* K-objective extension (not in the reference): K-2 extra seeded objectives
 * per product. Thresholds then list (K-1)*n cost-type bounds, then the task probabilities. */
int morap_instance_add_objectives(morap_instance* inst, int K, uint64_t seed);
/* Objective vector k (num_rows entries) of product (i, j) in device order:
 * 0 = cost, 1..K-2 = extra cost-type objectives, K-1 = success. */
int morap_instance_product_objective(const morap_instance* inst, int i, int j, int k, double* out);

/* Solver = one CUDA context on `device` with the instance's products resident. */
int morap_solver_create(int device, morap_solver** out);
void morap_solver_free(morap_solver* s);
morap_ctx* morap_solver_cuda(morap_solver* s);
int morap_solver_upload(morap_solver* s, const morap_instance* inst);
/* Drop every resident product (device memory freed; next query re-uploads). */
int morap_solver_release(morap_solver* s);
/* Per-rank build for the multi-GPU query: every rank generates the instance streamed
 * (`chunk` products at a time), assigns each distinct product to the least-loaded rank (by
 * nnz, in first-occurrence order -- identical on every rank) and keeps host arrays only
 * for its own products; morap_instance_product_owner reports the owner (-1 when the
 * instance was not built sharded). */
int morap_instance_warehouse_shard(const char* config_json, int threads, int rank, int world, int chunk,
                                   morap_instance** out);
int morap_instance_product_owner(const morap_instance* inst, int i, int j);

/* morap_cuda_set_lean on the solver's context (applies to later uploads). */
int morap_solver_set_lean(morap_solver* s, int on);
/* Per-iteration scheduler fingerprints ("schedulerHash") in morap_pareto's report: on by
 * default (the parity tests compare them); off leaves the records' tUp / tDown only. */
int morap_solver_set_fingerprints(morap_solver* s, int on);

/* Streamed generateInstance for instances whose host copy would not fit (C4: 100 x 100,
 * ~1e4 products of ~1e5 states): products are built `chunk` at a time on `threads` host
 * threads, each chunk's distinct products are uploaded to `s` and their host arrays
 * dropped. The instance then only answers queries on `s` (product_export fails on it).
 * Deduplication against dropped products compares (structural hash, S, R, nnz, initial). */
int morap_instance_warehouse_streamed(const char* config_json, int threads, morap_solver* s, int chunk,
                                      morap_instance** out);

/* generateInstance with every product built on the GPU of `s` (morap_cuda_build_products:
 * the BFS of buildProduct, checkRewardFinite and the compact upload layout run on the
 * device; the host never holds a product array). Same products, same errors and the same
 * seeded retries as morap_instance_warehouse; the instance then answers queries on `s` only
 * (as a streamed one). Deduplication compares (identity hash, S, R, nnz). */
int morap_instance_warehouse_device(const char* config_json, morap_solver* s, morap_instance** out);

/* Sharded device builds. _device_shard: the per-rank build for morap_shard_pareto -- every
 * rank measures every pair on its GPU, takes the owners morap_instance_warehouse_shard takes
 * and builds only its own products there. morap_multi_warehouse_device: one process, the
 * products built on the devices of `m` that own them (the owners morap_multi_upload takes);
 * the instance is then queried with morap_multi_pareto. */
int morap_instance_warehouse_device_shard(const char* config_json, morap_solver* s, int rank, int world,
                                          morap_instance** out);

/* supportingPoint (solver.hpp:103-184): w has K*n entries (unit 1-norm). Writes r (K*n)
 * and the assignment agent_of[n]. stats_out (nullable, 8 doubles): optimize jobs,
 * optimize nnz backups, evaluate jobs, evaluate state backups, optimize s, evaluate s,
 * host s, 0. */
int morap_supporting_point(morap_solver* s, const morap_instance* inst, const double* w, int nw, double* r_out,
                           int32_t* agent_of_out, double* stats_out);

/* paretoPoint / verifyOnly (solver.hpp:281-294), iteration cap default 500, identity norm
 * when norm == NULL. json_out receives resultToJson (solver.hpp:358) plus "converged",
 * "thresholds", "lambdaStar", per-iteration "records" {tUp, tDown, schedulerHash} and the
 * synthesis "marginal" (synthesize, solver.hpp:299) when the run converged; in verify mode
 * {"verdict": bool}. stats_out as in morap_supporting_point, summed over the query. */
int morap_pareto(morap_solver* s, const morap_instance* inst, const double* thresholds, int nt, const double* norm,
                 double eps, int iteration_cap, int verify, char* json_out, int json_cap, double* stats_out);

/* runParetoCore (solver.hpp:192-266) over an external supporting-point source, e.g. a
 * multi-GPU driver that shards the products across ranks: query(user, w, d, r_out,
 * agent_of_out, n) must fill r_out[d] and agent_of_out[n] and return 0 (or a status). */
typedef int (*morap_query_fn)(void* user, const double* w, int d, double* r_out, int32_t* agent_of_out, int n);
int morap_pareto_core(const double* expanded_thresholds, int d, int n, const double* norm, double eps,
                      int iteration_cap, int verify, morap_query_fn query, void* user, char* json_out, int json_cap);

/* Multi-GPU Pareto query (csrc/shard.cpp). The n x n products are
 * partitioned over shards by longest-processing-time on nnz (or by the owners of an
 * instance built with morap_instance_warehouse_shard); per iteration each shard optimizes
 * its pairs' jobs, the n^2 values are combined (each entry from its owner, exact bits), the
 * host runs the Hungarian step, each assigned pair is evaluated on its owner and the K*n
 * values are combined. Results equal morap_pareto's bit for bit.
 *
 * One process driving several GPUs (one context and one host thread per device; the
 * reference's one-engine / several-backend-queues model, engine.hpp:66-72,370-425): */
typedef struct morap_multi morap_multi;
int morap_multi_create(const int* devices, int ndevices, morap_multi** out);
void morap_multi_free(morap_multi* m);
/* uploads every shard's products to its device (lean when K <= 4) */
int morap_multi_upload(morap_multi* m, const morap_instance* inst);
/* owner shard of product (i, j) after morap_multi_upload, -1 if none */
int morap_multi_owner(const morap_multi* m, int i, int j);
int morap_multi_pareto(morap_multi* m, const morap_instance* inst, const double* thresholds, int nt, const double* norm,
                       double eps, int iteration_cap, char* json_out, int json_cap, double* stats_out);
int morap_multi_warehouse_device(morap_multi* m, const char* config_json, morap_instance** out);
/* One process per GPU (torch.distributed): `s` holds this rank's shard; `allgather`
 * (recv[r * count + k] = rank r's send[k], every rank) carries the two exchanges per
 * iteration -- NCCL over NVLink on GPUs, gloo in the CPU tests. Returns 0 or a status. */
typedef int (*morap_allgather_fn)(void* user, const double* send, int count, double* recv);
int morap_shard_pareto(morap_solver* s, const morap_instance* inst, int rank, int world, morap_allgather_fn allgather,
                       void* user, const double* thresholds, int nt, const double* norm, double eps, int iteration_cap,
                       char* json_out, int json_cap, double* stats_out);

/* Centralised model (centralised.hpp): buildCentralised (:54-179) with its state guard
 * (MORAP_SIZE_GUARD beyond it), the model's arrays, and centralisedParetoPoint (:216-222)
 * -- one weighted optimize job on the whole model per iteration plus the fused evaluation
 * of its scheduler under the 2n objectives, on the solver's GPU. Thresholds as for
 * morap_pareto (n costs, then the real tasks' probabilities); the report has the same
 * fields (records carry the single centralised scheduler's hash). */
typedef struct morap_centralised morap_centralised;
int morap_centralised_build(const morap_instance* inst, int64_t state_guard, morap_centralised** out);
void morap_centralised_free(morap_centralised* c);
/* out[6] = {S, R, nnz, initial, rewardFinite, number of objectives (2n)} */
int morap_centralised_info(const morap_centralised* c, int64_t* out);
int morap_centralised_export(const morap_centralised* c, int32_t* row_offset, int32_t* trn_offset, int32_t* succ,
                             double* prob, uint8_t* done, double* const* rewards);
int morap_centralised_pareto(morap_solver* s, const morap_centralised* c, const double* thresholds, int nt,
                             const double* norm, double eps, int iteration_cap, char* json_out, int json_cap,
                             double* stats_out);

/* runBatch (engine.hpp:370) -- the reference's job engine seam -- on the solver's GPU. Job k
 * refers to product (agent, task) of `inst` (agent < 0: a job without a model) and carries
 * its own reward vector (Job::reward, one entry per action row), the deterministic
 * scheduler of an evaluate job (one row per state), eps and sweep cap (engine.hpp:40-54).
 * Failures stay contained in their job (engine.hpp:140-150): result.status is 0 or
 * 1 + Errc. values_out[k] / policy_out[k] (nullable) receive JobResult::values / policy
 * (num_states entries) for successful jobs. Products uploaded lean for queries get a full
 * device copy on their first explicit-reward job. */
typedef struct {
  int64_t id;
  int32_t kind; /* 0 optimize, 1 evaluate */
  int32_t agent, task;
  const double* reward;
  int32_t reward_len;
  const int32_t* scheduler;
  int32_t scheduler_len;
  double eps;
  int32_t sweep_cap;
} morap_job;
typedef struct {
  int64_t id;
  int32_t status;
  int32_t sweeps;
  double value;
  double residual;
} morap_job_result;
int morap_run_batch(morap_solver* s, const morap_instance* inst, int njobs, const morap_job* jobs,
                    morap_job_result* results, double* const* values_out, int32_t* const* policy_out);

/* maxAssignment (assignment.hpp:54): agent_of[j] for the n x n row-major value matrix. */
int morap_max_assignment(int n, const double* c, int32_t* agent_of);

#ifdef __cplusplus
}
#endif

#endif /* MORAP_H */
