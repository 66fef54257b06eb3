// DMMA throughput vs independent accumulator chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k88(double* out, int iters) {
  double acc[C][2];
  for (int c = 0; c < C; c++) acc[c][0] = acc[c][1] = threadIdx.x * 1e-9 + c;
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < C; c++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < C; c++) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}
template <int C>
__global__ void k168(double* out, int iters) {
  double acc[C][4];
  for (int c = 0; c < C; c++) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = threadIdx.x * 1e-9 + c;
  double a0 = 1.0 + threadIdx.x * 1e-12, a1 = 0.5, a2 = 0.25, a3 = 0.125, a4 = 1, a5 = 2, a6 = 3, a7 = 4;
  double b0 = 0.999, b1 = 0.5, b2 = .25, b3 = .125;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < C; c++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(a4), "d"(a5), "d"(a6), "d"(a7), "d"(b0), "d"(b1), "d"(b2), "d"(b3));
  }
  double s = 0;
  for (int c = 0; c < C; c++) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 12345.0) out[0] = s;
}
template <class K>
void run(const char* name, K kern, int warps_per_cta, int ctas_per_sm, double flops_per_inst_warp, int chains) {
  double* d; cudaMalloc(&d, 8);
  const int iters = 4096;
  const int grid = 148 * ctas_per_sm;
  kern<<<grid, 32 * warps_per_cta>>>(d, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<grid, 32 * warps_per_cta>>>(d, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double fl = double(grid) * warps_per_cta * iters * chains * flops_per_inst_warp;
  printf("%-10s chains/warp %2d warps/SM %3d : %6.2f TF/s\n", name, chains, warps_per_cta * ctas_per_sm, fl / ms / 1e9);
  cudaFree(d);
}
int main() {
  for (int w : {4, 8, 16, 32}) {
    run("m8n8k4", k88<1>, w, 1, 512, 1);
    run("m8n8k4", k88<2>, w, 1, 512, 2);
    run("m8n8k4", k88<4>, w, 1, 512, 4);
    run("m8n8k4", k88<8>, w, 1, 512, 8);
    run("m8n8k4", k88<16>, w, 1, 512, 16);
    run("m16n8k16", k168<1>, w, 1, 4096, 1);
    run("m16n8k16", k168<2>, w, 1, 4096, 2);
    run("m16n8k16", k168<4>, w, 1, 4096, 4);
  }
  return 0;
}
