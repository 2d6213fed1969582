// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Prints achieved TFLOP/s for each variant. Used to set the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-9 + i;
  double c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
  double c[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
float timeit(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, threads = 32 * wpb;
      double warps = (double)blocks * wpb;
      float ms = timeit(dmma_m8n8k4<8>, blocks, threads, iters, out);
      double fl = warps * iters * 8 * 512.0;
      printf("dmma m8n8k4   wpb=%2d bps=%d : %.2f TFLOP/s\n", wpb, bps, fl / ms / 1e9);
      ms = timeit(dmma_m16n8k16<4>, blocks, threads, iters / 4, out);
      fl = warps * (iters / 4) * 4 * (16 * 8 * 16 * 2.0);
      printf("dmma m16n8k16 wpb=%2d bps=%d : %.2f TFLOP/s\n", wpb, bps, fl / ms / 1e9);
      ms = timeit(dfma_loop<16>, blocks, threads, iters, out);
      fl = (double)blocks * threads * iters * 16 * 2.0;
      printf("dfma          wpb=%2d bps=%d : %.2f TFLOP/s\n", wpb, bps, fl / ms / 1e9);
    }
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d clock_khz=%d err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
