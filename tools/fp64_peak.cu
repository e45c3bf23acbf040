// FP64 peak probe for the B200 roofline denominator.
//
// MEASURED_PEAKS.json (driver-written) carries HBM copy GB/s and bf16 GEMM TF/s but no FP64
// figure, and this path's rank-reveal is FP64-bound.  This probe measures, on one B200:
//   * DFMA issue peak (independent FMA chains, all SMs),
//   * DMMA (mma.sync f64) peak for m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16,
//   * cuBLAS DGEMM at 8192^3 and at the two trailing-update shapes of the blocked QR
//     (rank-64 update m x n x 64, and the 64 x n reduction over m),
// and prints one JSON object.  Build: see tools/Makefile (nvcc, sm_100a, -lcublas).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

constexpr int kIters = 4096;

__global__ void dfma_loop(double* out, double seed) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + i * 1e-3 + threadIdx.x * 1e-7;
  const double m = 0.999999999, c = 1e-9;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], m, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int KIND>
__global__ void dmma_loop(double* out, double seed) {
  // 8 independent accumulator sets per warp
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i + threadIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed - i + threadIdx.x * 1e-6;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a[0]), "d"(b[0]));
      } else if (KIND == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (KIND == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

static float time_kernel(void (*launch)(), int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch(); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

static double* g_out;
static int g_blocks, g_threads;
static void l_dfma() { dfma_loop<<<g_blocks, g_threads>>>(g_out, 1.0); }
template <int K> static void l_dmma() { dmma_loop<K><<<g_blocks, g_threads>>>(g_out, 1.0); }

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaMalloc(&g_out, 1024 * sizeof(double)));
  g_threads = 512; g_blocks = sms * 4;
  double dfma_flops = 2.0 * 16 * kIters * (double)g_threads * g_blocks;
  float t = time_kernel(l_dfma, 5);
  double dfma_tf = dfma_flops / (t * 1e-3) / 1e12;
  const double mma_flops[4] = {2.0 * 8 * 8 * 4, 2.0 * 16 * 8 * 4, 2.0 * 16 * 8 * 8, 2.0 * 16 * 8 * 16};
  double dmma_tf[4];
  void (*ls[4])() = {l_dmma<0>, l_dmma<1>, l_dmma<2>, l_dmma<3>};
  for (int k = 0; k < 4; ++k) {
    double warps = (double)g_blocks * g_threads / 32;
    double fl = mma_flops[k] * 8 * (kIters / 4) * warps;
    float tk = time_kernel(ls[k], 5);
    dmma_tf[k] = fl / (tk * 1e-3) / 1e12;
  }
  // cuBLAS DGEMM
  cublasHandle_t h; cublasCreate(&h);
  auto gemm_tf = [&](int m, int n, int k, bool ta) {
    double *A, *B, *C;
    size_t sa = (size_t)m * k, sb = (size_t)k * n, sc = (size_t)m * n;
    CK(cudaMalloc(&A, sa * 8)); CK(cudaMalloc(&B, sb * 8)); CK(cudaMalloc(&C, sc * 8));
    CK(cudaMemset(A, 0, sa * 8)); CK(cudaMemset(B, 0, sb * 8)); CK(cudaMemset(C, 0, sc * 8));
    double al = 1.0, be = 1.0;
    auto run = [&]() {
      cublasDgemm(h, ta ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &al, A, ta ? k : m, B, k, &be, C, m);
    };
    run(); CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) run();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(A); cudaFree(B); cudaFree(C);
    return 2.0 * m * n * (double)k / (ms / reps * 1e-3) / 1e12;
  };
  double g8192 = gemm_tf(8192, 8192, 8192, false);
  double g_rank64 = gemm_tf(32768, 32768, 64, false);
  double g_rank128 = gemm_tf(32768, 32768, 128, false);
  double g_red64 = gemm_tf(64, 32768, 32768, true);
  double g_red128 = gemm_tf(128, 32768, 32768, true);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, "
         "\"dmma_m16n8k4_tflops\": %.2f, \"dmma_m16n8k8_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, "
         "\"cublas_dgemm_8192_tflops\": %.2f, \"cublas_rank64_32768_tflops\": %.2f, "
         "\"cublas_rank128_32768_tflops\": %.2f, \"cublas_tn_reduce64_32768_tflops\": %.2f, "
         "\"cublas_tn_reduce128_32768_tflops\": %.2f}\n",
         sms, clk, dfma_tf, dmma_tf[0], dmma_tf[1], dmma_tf[2], dmma_tf[3], g8192, g_rank64, g_rank128,
         g_red64, g_red128);
  return 0;
}
