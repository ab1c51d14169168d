/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's hot-path numerics.
 * Used by tests/ as the checker for the sm_100a kernels and by bench.py's
 * cpu_baseline leg. Never linked into, or called from, the product path.
 *
 * Restates (plain C, sequential, no FMA -- build with -ffp-contract=off):
 *   weightedReward       /root/reference/proj/include/morap/numerics.hpp:224-234
 *   optimalSchedulerOn   /root/reference/proj/include/morap/numerics.hpp:74-122
 *   evaluateSchedulerOn  /root/reference/proj/include/morap/numerics.hpp:130-168
 *   maximalAvoidSet      /root/reference/proj/include/morap/model.hpp:163-200
 *
 * Pinned against the reference itself (oracle/_ref, tests/test_oracle.py) and against
 * the known answers in proj/tests/test_numerics.cpp:18-80 (tests/golden/).
 *
 * Status codes: 0 ok, otherwise 1 + morap::Errc (common.hpp:12-34):
 *   NotRewardFinite = 6, NonConvergence = 7, DimensionMismatch = 9.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VO_OK 0
#define VO_INVALID_MODEL 5
#define VO_NOT_REWARD_FINITE 6
#define VO_NON_CONVERGENCE 7

/* rho[r] = (0 + w[0]*part0[r]) + w[1]*part1[r] + ...  (numerics.hpp:227-231) */
void vo_weighted_reward(int R, int K, const double* const* parts, const double* w, double* out) {
  for (int r = 0; r < R; ++r) out[r] = 0.0;
  for (int k = 0; k < K; ++k) {
    const double* p = parts[k];
    const double wk = w[k];
    for (int r = 0; r < R; ++r) {
      double prod = wk * p[r];
      out[r] = out[r] + prod;
    }
  }
}

/* One Jacobi sweep of the greedy backup; returns the max |y-x| over non-done states.
 * Per state: rows scanned in order, row value accumulated left to right from rho[r],
 * first strictly-greater row wins (numerics.hpp:86-104). */
static double vo_greedy_sweep(int S, const int* rowOffset, const int* trnOffset, const int* succ,
                              const double* prob, const unsigned char* done, const double* rho,
                              const double* x, double* y, int* pol) {
  double delta = 0.0;
  for (int s = 0; s < S; ++s) {
    if (done[s]) {
      y[s] = 0.0;
      continue;
    }
    int bestRow = -1;
    double best = 0.0;
    for (int r = rowOffset[s]; r < rowOffset[s + 1]; ++r) {
      double v = rho[r];
      for (int k = trnOffset[r]; k < trnOffset[r + 1]; ++k) {
        double t = prob[k] * x[succ[k]];
        v = v + t;
      }
      if (bestRow < 0 || v > best) {
        best = v;
        bestRow = r;
      }
    }
    y[s] = best;
    pol[s] = bestRow;
    double d = fabs(best - x[s]);
    if (d > delta) delta = d;
  }
  return delta;
}

int vo_optimize(int S, int R, int nnz, int initial, const int* rowOffset, const int* trnOffset,
                const int* succ, const double* prob, const unsigned char* done, int rewardFinite,
                const double* rho, double eps, int cap, double* values, int* policy, int* sweeps,
                double* residual, double* value) {
  (void)R;
  (void)nnz;
  if (!rewardFinite) return VO_NOT_REWARD_FINITE;
  double* a = (double*)calloc((size_t)S, sizeof(double));
  double* b = (double*)calloc((size_t)S, sizeof(double));
  for (int s = 0; s < S; ++s) policy[s] = -1;
  int n = 0;
  double delta = 0.0;
  int rc = VO_OK;
  for (;;) {
    delta = vo_greedy_sweep(S, rowOffset, trnOffset, succ, prob, done, rho, a, b, policy);
    double* t = a;
    a = b;
    b = t;
    ++n;
    if (delta <= eps) break;
    if (n >= cap) {
      rc = VO_NON_CONVERGENCE;
      break;
    }
  }
  for (int s = 0; s < S; ++s)
    if (done[s]) policy[s] = rowOffset[s];
  memcpy(values, a, (size_t)S * sizeof(double));
  *sweeps = n;
  *residual = delta;
  *value = a[initial];
  free(a);
  free(b);
  return rc;
}

/* Fixed deterministic scheduler: y(s) = 0 + 1.0 * (rho[r] + sum P x), r = policy[s]
 * (numerics.hpp:140-153 with a single (r, 1.0) choice per state). */
int vo_evaluate(int S, int R, int nnz, int initial, const int* rowOffset, const int* trnOffset,
                const int* succ, const double* prob, const unsigned char* done, const int* policy,
                const double* rho, double eps, int cap, double* values, int* sweeps, double* residual,
                double* value) {
  (void)R;
  (void)nnz;
  for (int s = 0; s < S; ++s)
    if (!done[s] && (policy[s] < rowOffset[s] || policy[s] >= rowOffset[s + 1])) return VO_INVALID_MODEL;
  double* a = (double*)calloc((size_t)S, sizeof(double));
  double* b = (double*)calloc((size_t)S, sizeof(double));
  int n = 0;
  double delta = 0.0;
  int rc = VO_OK;
  for (;;) {
    delta = 0.0;
    for (int s = 0; s < S; ++s) {
      if (done[s]) {
        b[s] = 0.0;
        continue;
      }
      const int r = policy[s];
      double acc = rho[r];
      for (int k = trnOffset[r]; k < trnOffset[r + 1]; ++k) {
        double t = prob[k] * a[succ[k]];
        acc = acc + t;
      }
      double v = 0.0;
      double t = 1.0 * acc;
      v = v + t;
      b[s] = v;
      double d = fabs(v - a[s]);
      if (d > delta) delta = d;
    }
    double* t = a;
    a = b;
    b = t;
    ++n;
    if (delta <= eps) break;
    if (n >= cap) {
      rc = VO_NON_CONVERGENCE;
      break;
    }
  }
  memcpy(values, a, (size_t)S * sizeof(double));
  *sweeps = n;
  *residual = delta;
  *value = a[initial];
  free(a);
  free(b);
  return rc;
}

/* Reward-finiteness: peel states that cannot keep away from `done` (model.hpp:163-206).
 * Returns 1 when the maximal avoid set is empty. */
int vo_reward_finite(int S, int R, const int* rowOffset, const int* trnOffset, const int* succ,
                     const unsigned char* done) {
  int* owner = (int*)malloc(sizeof(int) * (size_t)(R > 0 ? R : 1));
  char* live = (char*)malloc((size_t)S);
  int* outCnt = (int*)calloc((size_t)(R > 0 ? R : 1), sizeof(int));
  int* safe = (int*)calloc((size_t)S, sizeof(int));
  int* inDeg = (int*)calloc((size_t)S + 1, sizeof(int));
  for (int s = 0; s < S; ++s) {
    live[s] = done[s] ? 0 : 1;
    for (int r = rowOffset[s]; r < rowOffset[s + 1]; ++r) owner[r] = s;
  }
  /* reverse adjacency (successor -> rows entering it) for rows owned by live states */
  for (int r = 0; r < R; ++r)
    if (live[owner[r]])
      for (int k = trnOffset[r]; k < trnOffset[r + 1]; ++k) inDeg[succ[k] + 1]++;
  for (int s = 0; s < S; ++s) inDeg[s + 1] += inDeg[s];
  int* fill = (int*)calloc((size_t)S, sizeof(int));
  int* into = (int*)malloc(sizeof(int) * (size_t)(inDeg[S] > 0 ? inDeg[S] : 1));
  for (int r = 0; r < R; ++r) {
    if (!live[owner[r]]) continue;
    for (int k = trnOffset[r]; k < trnOffset[r + 1]; ++k) {
      int t = succ[k];
      into[inDeg[t] + fill[t]++] = r;
      if (!live[t]) outCnt[r]++;
    }
    if (outCnt[r] == 0) safe[owner[r]]++;
  }
  int* queue = (int*)malloc(sizeof(int) * (size_t)S);
  int qh = 0, qt = 0;
  for (int s = 0; s < S; ++s)
    if (live[s] && safe[s] == 0) queue[qt++] = s;
  while (qh < qt) {
    int s = queue[qh++];
    if (!live[s]) continue;
    live[s] = 0;
    for (int e = inDeg[s]; e < inDeg[s + 1]; ++e) {
      int r = into[e];
      int o = owner[r];
      if (!live[o]) continue;
      if (outCnt[r]++ == 0) {
        if (--safe[o] == 0) queue[qt++] = o;
      }
    }
  }
  int any = 0;
  for (int s = 0; s < S; ++s) any |= live[s];
  free(owner); free(live); free(outCnt); free(safe); free(inDeg); free(fill); free(into); free(queue);
  return any ? 0 : 1;
}

/* ---- multi-threaded batch driver (bench.py cpu_baseline, kind "port") ---- */
typedef struct {
  int S, R, nnz, initial;
  const int *rowOffset, *trnOffset, *succ;
  const double* prob;
  const unsigned char* done;
  const double* rho;
  double eps;
  int cap;
  int sweeps;
  int rc;
  double value;
} vo_job;

typedef struct {
  vo_job* jobs;
  int njobs;
  int next;
  pthread_mutex_t mu;
} vo_pool;

static void* vo_worker(void* arg) {
  vo_pool* p = (vo_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    int j = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (j >= p->njobs) return NULL;
    vo_job* jb = &p->jobs[j];
    double* values = (double*)malloc(sizeof(double) * (size_t)jb->S);
    int* pol = (int*)malloc(sizeof(int) * (size_t)jb->S);
    double res;
    jb->rc = vo_optimize(jb->S, jb->R, jb->nnz, jb->initial, jb->rowOffset, jb->trnOffset, jb->succ,
                         jb->prob, jb->done, 1, jb->rho, jb->eps, jb->cap, values, pol, &jb->sweeps, &res,
                         &jb->value);
    free(values);
    free(pol);
  }
}

/* Runs njobs optimize jobs on `threads` threads; returns sum(sweeps*nnz) in *backups. */
int vo_optimize_batch(int njobs, const int* S, const int* R, const int* nnz, const int* initial,
                      const int* const* rowOffset, const int* const* trnOffset, const int* const* succ,
                      const double* const* prob, const unsigned char* const* done,
                      const double* const* rho, double eps, int cap, int threads, double* values_out,
                      int* sweeps_out, double* backups) {
  vo_job* jobs = (vo_job*)calloc((size_t)njobs, sizeof(vo_job));
  for (int j = 0; j < njobs; ++j) {
    jobs[j] = (vo_job){S[j], R[j], nnz[j], initial[j], rowOffset[j], trnOffset[j], succ[j], prob[j],
                       done[j], rho[j], eps, cap, 0, 0, 0.0};
  }
  vo_pool pool = {jobs, njobs, 0, PTHREAD_MUTEX_INITIALIZER};
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, vo_worker, &pool);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  int rc = 0;
  double total = 0.0;
  for (int j = 0; j < njobs; ++j) {
    if (jobs[j].rc && !rc) rc = jobs[j].rc;
    values_out[j] = jobs[j].value;
    sweeps_out[j] = jobs[j].sweeps;
    total += (double)jobs[j].sweeps * (double)nnz[j];
  }
  *backups = total;
  free(th);
  free(jobs);
  return rc;
}
