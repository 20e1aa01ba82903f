/*
 * pqk_scan.c — C restatement of the reference linear-scan assignment.
 * TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline), never the product.
 *
 * Follows /root/reference/pkg/src/pqclust/clustering.py:167-197:
 *   acc = 0.0; for m in 0..M-1: acc += T[m][x^m][c_k^m]   (float64, ascending m)
 *   label = argmin_k acc   (np.argmin: first minimum -> lowest index on ties)
 * and the winner's distance, which equals paired_distance_sq (pq.py:287-290).
 * Compiled with -ffp-contract=off so every += rounds once, like numpy.
 * Parallel over codes with pthreads; each code's result is independent of the
 * thread count (clustering.py:160-164, :190-196).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
  const uint8_t* codes;
  int64_t n;
  int32_t m;
  const uint8_t* centers;
  int64_t k;
  const double* tables;
  int32_t l;
  uint32_t* labels;
  double* sd;
  int64_t begin, end;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  const int32_t m = j->m, l = j->l;
  const size_t ll = (size_t)l * l;
  for (int64_t i = j->begin; i < j->end; ++i) {
    const uint8_t* x = j->codes + (size_t)i * m;
    const double* rows[256];
    for (int32_t mm = 0; mm < m && mm < 256; ++mm) rows[mm] = j->tables + mm * ll + (size_t)x[mm] * l;
    double best = 0.0;
    int64_t bk = -1;
    for (int64_t k = 0; k < j->k; ++k) {
      const uint8_t* c = j->centers + (size_t)k * m;
      double acc = 0.0;
      for (int32_t mm = 0; mm < m; ++mm)
        acc += (mm < 256 ? rows[mm][c[mm]] : j->tables[mm * ll + (size_t)x[mm] * l + c[mm]]);
      if (bk < 0 || acc < best) {
        best = acc;
        bk = k;
      }
    }
    j->labels[i] = (uint32_t)bk;
    j->sd[i] = best;
  }
  return NULL;
}

int oracle_assign(const uint8_t* codes, int64_t n, int32_t m, const uint8_t* centers, int64_t k,
                  const double* tables, int32_t l, uint32_t* labels, double* sd, int32_t threads) {
  if (n < 0 || m < 1 || k < 1 || l < 1) return 1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (n < threads) threads = n > 0 ? (int32_t)n : 1;
  pthread_t tid[256];
  job_t jobs[256];
  const int64_t per = (n + threads - 1) / threads;
  for (int32_t t = 0; t < threads; ++t) {
    jobs[t] = (job_t){codes, n, m, centers, k, tables, l, labels, sd, t * per, (t + 1) * per < n ? (t + 1) * per : n};
    if (jobs[t].begin > jobs[t].end) jobs[t].begin = jobs[t].end;
  }
  for (int32_t t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, worker, &jobs[t]);
  worker(&jobs[0]);
  for (int32_t t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  return 0;
}
