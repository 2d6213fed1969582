// Standalone timing of one 4096 x 32 cluster panel (the first panel of a
// C2-size LU): CUDA events around back-to-back launches vs the CTAs' own
// globaltimer span (fb_debug-style counters in panel.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=false \
//   -I paper_1203_4031_b200/csrc tools/panel_bench.cu paper_1203_4031_b200/csrc/panel.cu -o tools/panel_bench
#include <cstdio>
#include <vector>
#include <random>
#include "panel.cuh"
#include <atomic>
namespace fb { std::atomic<long long> g_launches{0}; }
namespace fb { void panel_wall_read(unsigned long long* out4); void panel_span_raw(unsigned long long*, unsigned long long*); }
__global__ void stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) *out = t;
}
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096;
  const int reps = 50;
  std::vector<double> h(2 * (size_t)n * n);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : h) v = nd(g);
  double *re, *im, *dinv;
  int *piv, *info;
  cudaMalloc(&re, 8ull * n * n);
  cudaMalloc(&im, 8ull * n * n);
  cudaMalloc(&dinv, 8ull * 8 * 32 * 32 + 8 * 4096);
  cudaMalloc(&piv, 4 * n);
  cudaMalloc(&info, 4);
  char* scratch;
  cudaMalloc(&scratch, fb::panel_scratch_bytes());
  cudaStream_t st;
  cudaStreamCreate(&st);
  fb::PanelArgs a{};
  a.re = re; a.im = im; a.ld = n; a.n = n; a.c0 = 0; a.pw = 32;
  a.piv = piv; a.info = info; a.linv = dinv; a.uinv = dinv + 2 * 32 * 32; a.list = (int*)(dinv + 4 * 32 * 32);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  unsigned long long w[4];
  for (int pass = 0; pass < 3; ++pass) {
    cudaMemcpy(re, h.data(), 8ull * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(im, h.data() + (size_t)n * n, 8ull * n * n, cudaMemcpyHostToDevice);
    fb::panel_wall_read(w);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) fb::panel_launch(a, 1, scratch, st);   // same panel, refactored
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    fb::panel_wall_read(w);
    printf("n=%d: %.1f us per launch (events), CTA0 wall %.1f us, CTA span (panel 0, summed) %.1f us per launch  %s\n",
           n, 1e3 * ms / reps, w[0] / 1e3 / (w[2] ? w[2] : 1), w[3] / 1e3 / reps, cudaGetErrorString(cudaGetLastError()));
  }
  for (int pw : {1, 2, 8, 16, 32}) {
    a.pw = pw;
    fb::panel_wall_read(w);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) fb::panel_launch(a, 1, scratch, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    fb::panel_wall_read(w);
    printf("n=%d pw=%d: %.1f us per launch (events), CTA0 wall %.1f us\n", n, pw, 1e3 * ms2 / reps,
           w[0] / 1e3 / (w[2] ? w[2] : 1));
  }
  {  // per-launch span of all CTAs (first start .. last end), one launch at a time
    a.pw = 32;
    double span = 0.0, ev = 0.0, c0w = 0.0;
    for (int r = 0; r < 20; ++r) {
      fb::panel_wall_read(w);
      cudaEventRecord(e0, st);
      fb::panel_launch(a, 1, scratch, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms3;
      cudaEventElapsedTime(&ms3, e0, e1);
      fb::panel_wall_read(w);
      span += w[3] / 1e3;
      c0w += w[0] / 1e3;
      ev += 1e3 * ms3;
    }
    printf("n=%d single launches: events %.1f us, all-CTA span %.1f us, CTA0 wall %.1f us\n", n, ev / 20, span / 20,
           c0w / 20);
  }
  {  // gaps: stamp kernel -> panel (first CTA start) and panel (last CTA end) -> stamp kernel
    unsigned long long* ts;
    cudaMalloc(&ts, 16);
    a.pw = 32;
    double pre = 0, post = 0, body = 0;
    for (int r = 0; r < 20; ++r) {
      fb::panel_wall_read(w);
      stamp_kernel<<<1, 32, 0, st>>>(ts);
      fb::panel_launch(a, 1, scratch, st);
      stamp_kernel<<<1, 32, 0, st>>>(ts + 1);
      cudaStreamSynchronize(st);
      unsigned long long h[2];
      cudaMemcpy(h, ts, 16, cudaMemcpyDeviceToHost);
      unsigned long long s0, e0;
      fb::panel_span_raw(&s0, &e0);
      fb::panel_wall_read(w);
      body += (e0 - s0) / 1e3;
      pre += ((double)s0 - (double)h[0]) / 1e3;
      post += ((double)h[1] - (double)e0) / 1e3;
    }
    printf("stamp -> first CTA start %.1f us, all-CTA span %.1f us, last CTA end -> stamp %.1f us\n", pre / 20,
           body / 20, post / 20);
  }
  // launch cost alone: same launch configuration, kernel returns at entry
  a.pw = -1;
  cudaEventRecord(e0, st);
  for (int r = 0; r < reps; ++r) fb::panel_launch(a, 1, scratch, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("n=%d: empty-body launch %.1f us  %s\n", n, 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
