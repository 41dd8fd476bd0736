// Host leaf reducer (csrc/hostleaf.cpp) streaming rate vs a plain stream-sum on the same
// buffers: T pinned threads, each on its own first-touched contiguous share of two
// binary64 operands, reduce full leaves of 2^16 elements (f64 dottf, the cfg5 shape).
//   g++ -O3 -std=c++17 -pthread scripts/host_leaf_bw.cpp paper_1401_0248_b200/csrc/build/hostleaf_avx512.o \
//       -o /tmp/hlbw && /tmp/hlbw [threads] [GiB per operand] [method]
// Prints GB/s for (a) the leaf reducer, (b) a two-operand stream dot with no chains.
#include <pthread.h>
#include <sched.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <vector>

extern "C" int tfb_host_leaves_avx512(int method, int dtype, const void* x, const void* y, int lg, int64_t lo,
                                      int64_t hi, void* pairs);

struct Job {
  double *x, *y;
  int64_t n;
  int cpu;
  int method;
  double sink;
};
static pthread_barrier_t bar;
static const int kReps = 4;

static double now() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

static void* run(void* a) {
  Job* j = static_cast<Job*>(a);
  cpu_set_t s;
  CPU_ZERO(&s);
  CPU_SET(j->cpu, &s);
  pthread_setaffinity_np(pthread_self(), sizeof(s), &s);
  for (int64_t i = 0; i < j->n; ++i) {
    j->x[i] = double(i & 1023) * 0.25;
    j->y[i] = double((i >> 3) & 511) - 255.5;
  }
  const int lg = 16;
  const int64_t leaves = j->n >> lg;
  std::vector<double> pairs(2 * leaves);
  for (int mode = 0; mode < 2; ++mode)
    for (int r = 0; r < kReps; ++r) {
      pthread_barrier_wait(&bar);
      if (mode == 0) {
        tfb_host_leaves_avx512(j->method, 1, j->x, j->y, lg, 0, leaves, pairs.data());
        j->sink += pairs[0];
      } else {
        double acc[8] = {0};
        for (int64_t i = 0; i + 8 <= j->n; i += 8)
          for (int k = 0; k < 8; ++k) acc[k] += j->x[i + k] * j->y[i + k];
        for (int k = 0; k < 8; ++k) j->sink += acc[k];
      }
      pthread_barrier_wait(&bar);
    }
  return nullptr;
}

int main(int argc, char** argv) {
  cpu_set_t all;
  sched_getaffinity(0, sizeof(all), &all);
  const int T = argc > 1 ? atoi(argv[1]) : CPU_COUNT(&all);
  const double gib = argc > 2 ? atof(argv[2]) : 2.0;
  const int method = argc > 3 ? atoi(argv[3]) : 2;
  const int64_t n = (int64_t(gib * (1 << 30)) / 8 / T) >> 16 << 16;  // per thread, whole leaves
  std::vector<pthread_t> th(T);
  std::vector<Job> jobs(T);
  pthread_barrier_init(&bar, nullptr, T + 1);
  int c = 0;
  for (int t = 0; t < T; ++t) {
    while (!CPU_ISSET(c, &all)) ++c;
    jobs[t] = Job{static_cast<double*>(aligned_alloc(4096, n * 8)), static_cast<double*>(aligned_alloc(4096, n * 8)),
                  n, c++, method, 0.0};
    pthread_create(&th[t], nullptr, run, &jobs[t]);
  }
  for (int mode = 0; mode < 2; ++mode) {
    double best = 1e9;
    for (int r = 0; r < kReps; ++r) {
      pthread_barrier_wait(&bar);
      const double t0 = now();
      pthread_barrier_wait(&bar);
      const double dt = now() - t0;
      if (dt < best) best = dt;
    }
    printf("threads %d %s: %.1f GB/s (%.2f Gelem/s)\n", T, mode == 0 ? "host leaf reducer (f64 dot)" : "plain stream dot",
           2.0 * n * T * 8 / best / 1e9, n * T / best / 1e9);
  }
  double s = 0;
  for (int t = 0; t < T; ++t) {
    pthread_join(th[t], nullptr);
    s += jobs[t].sink;
  }
  printf("checksum %.3f\n", s);
  return 0;
}
