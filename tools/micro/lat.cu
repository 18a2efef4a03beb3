// Dependent-chain latency microbenchmark (cycles per op) for the coordinator's critical path ops.
#include <cstdio>
#include <cuda_runtime.h>
#define N 512
__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) :: "memory"); return c; }
__global__ void k(long long *out, double *sink, const double *in, const long long *li) {
  double x = in[0], c1 = in[1], c2 = in[2];
  long long t0, t1;
  t0 = clk();
  for (int i = 0; i < N; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(c1), "d"(c2));
  t1 = clk(); out[0] = (t1 - t0) / N;
  double y = in[3];
  t0 = clk();
  for (int i = 0; i < N; ++i) { y = __ddiv_rn(y + c2, c1 + 6.0); asm volatile("" : "+d"(y)); }
  t1 = clk(); out[1] = (t1 - t0) / N;
  long long a = li[0];
  double z = 0;
  t0 = clk();
  for (int i = 0; i < N; ++i) { asm volatile("cvt.rn.f64.s64 %0, %1;" : "=d"(z) : "l"(a)); asm volatile("mov.b64 %0, %1;" : "=l"(a) : "d"(z)); }
  t1 = clk(); out[2] = (t1 - t0) / N;
  int v = (int)li[1];
  t0 = clk();
  for (int i = 0; i < N; ++i) asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 31, -1;" : "+r"(v));
  t1 = clk(); out[3] = (t1 - t0) / N;
  // DSETP-driven select chain: w = (w > c) ? w - c : w + c
  double w = in[4];
  t0 = clk();
  for (int i = 0; i < N; ++i) {
    asm volatile("{ .reg .pred p; setp.gt.f64 p, %0, %1; @p sub.rn.f64 %0, %0, %1; @!p add.rn.f64 %0, %0, %1; }" : "+d"(w) : "d"(c2));
  }
  t1 = clk(); out[4] = (t1 - t0) / N;
  // ISETP 64-bit select chain
  long long u = li[2], cc = li[3];
  t0 = clk();
  for (int i = 0; i < N; ++i) {
    asm volatile("{ .reg .pred p; setp.gt.s64 p, %0, %1; @p sub.s64 %0, %0, %1; @!p add.s64 %0, %0, %1; }" : "+l"(u) : "l"(cc));
  }
  t1 = clk(); out[5] = (t1 - t0) / N;
  // u64 mul chain
  unsigned long long h = li[4];
  t0 = clk();
  for (int i = 0; i < N; ++i) asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(h) : "l"(1099511628211ULL));
  t1 = clk(); out[6] = (t1 - t0) / N;
  // dadd chain
  double q = in[5];
  t0 = clk();
  for (int i = 0; i < N; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(q) : "d"(c2));
  t1 = clk(); out[7] = (t1 - t0) / N;
  // rcp.approx.ftz.f64 chain
  double r = in[6];
  t0 = clk();
  for (int i = 0; i < N; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r));
  t1 = clk(); out[8] = (t1 - t0) / N;
  // ballot chain
  unsigned m = (unsigned)li[5];
  t0 = clk();
  for (int i = 0; i < N; ++i) asm volatile("{ .reg .pred p; setp.ne.u32 p, %0, 0; vote.sync.ballot.b32 %0, p, -1; }" : "+r"(m));
  t1 = clk(); out[9] = (t1 - t0) / N;
  sink[threadIdx.x] = x + y + z + w + (double)u + (double)h + q + r + v + m;
}
int main() {
  long long *o, *li; double *s, *in;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&s, 64 * 8); cudaMalloc(&in, 64 * 8); cudaMalloc(&li, 64 * 8);
  double hin[8] = {1.5, 1.0000001, 1e-9, 3.0, 5.0, 0.5, 1.7, 0};
  long long hli[8] = {123456789, 7, 1000, 3, 12345, 5, 0, 0};
  cudaMemcpy(in, hin, 64, cudaMemcpyHostToDevice); cudaMemcpy(li, hli, 64, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, s, in, li);
  long long h[10];
  cudaMemcpy(h, o, 80, cudaMemcpyDeviceToHost);
  const char *n[10] = {"DFMA", "ddiv_rn (+dadd)", "I2F.F64.S64+mov", "SHFL.BFLY", "DSETP+DADD select", "ISETP64+IADD64 select",
                       "u64 mul", "DADD", "rcp.approx.f64", "VOTE.BALLOT+ISETP"};
  for (int i = 0; i < 10; ++i) printf("%-24s %lld cycles\n", n[i], h[i]);
  return 0;
}
