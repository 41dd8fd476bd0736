/* Host DRAM read roof of the GPU box: T pinned threads each stream-sum a contiguous
 * 1/T of a 8 GiB buffer (first-touched by the same thread), best of 5.  The e2e
 * path's ceiling is min(PCIe + this, this): every byte is read from host DRAM once.
 *   gcc -O3 -march=native -pthread scripts/host_read_bw.c -o /tmp/hrbw && /tmp/hrbw [threads] */
#define _GNU_SOURCE
#include <pthread.h>
#include <sched.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct { double* p; size_t n; int cpu; double sum; } job_t;
static pthread_barrier_t bar;
static int reps = 5;
static double best_s = 1e9;

static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }

static void* run(void* a) {
  job_t* j = (job_t*)a;
  cpu_set_t s; CPU_ZERO(&s); CPU_SET(j->cpu, &s); pthread_setaffinity_np(pthread_self(), sizeof(s), &s);
  for (size_t i = 0; i < j->n; ++i) j->p[i] = (double)(i & 1023);
  for (int r = 0; r < reps; ++r) {
    pthread_barrier_wait(&bar);
    double acc[8] = {0};
    for (size_t i = 0; i + 8 <= j->n; i += 8)
      for (int k = 0; k < 8; ++k) acc[k] += j->p[i + k];
    for (int k = 0; k < 8; ++k) j->sum += acc[k];
    pthread_barrier_wait(&bar);
  }
  return NULL;
}

int main(int argc, char** argv) {
  cpu_set_t all; sched_getaffinity(0, sizeof(all), &all);
  int ncpu = CPU_COUNT(&all);
  int T = argc > 1 ? atoi(argv[1]) : ncpu;
  size_t n = (size_t)1 << 30;  /* 8 GiB of doubles */
  double* buf = malloc(n * sizeof(double));
  pthread_t th[1024]; job_t jobs[1024];
  pthread_barrier_init(&bar, NULL, T + 1);
  int c = 0;
  for (int t = 0; t < T; ++t) {
    while (!CPU_ISSET(c, &all)) ++c;
    jobs[t].p = buf + (n / T) * t; jobs[t].n = n / T; jobs[t].cpu = c++; jobs[t].sum = 0;
    pthread_create(&th[t], NULL, run, &jobs[t]);
  }
  for (int r = 0; r < reps; ++r) {
    pthread_barrier_wait(&bar);
    double t0 = now();
    pthread_barrier_wait(&bar);
    double dt = now() - t0;
    if (dt < best_s) best_s = dt;
  }
  double s = 0;
  for (int t = 0; t < T; ++t) { pthread_join(th[t], NULL); s += jobs[t].sum; }
  printf("threads %d: %.1f GB/s host DRAM read (8 GiB, best of %d) checksum %.0f\n", T, n * 8.0 / best_s / 1e9, reps, s);
  return 0;
}
