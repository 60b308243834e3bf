// ubench.cu -- per-SM instruction throughput on the B200 (sm_100a): FFMA (reg / imm), DFMA,
// IMAD, IADD3, LOP3, FSEL, MUFU.LG2, and a mixed FFMA+LOP3 stream.  Each kernel runs independent
// chains (ILP 8) in every thread of a full-occupancy grid; reported as warp-instructions per
// clock per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

#define KERNEL(NAME, T, INIT, BODY)                                              \
  __global__ void NAME(T *out, T seed) {                                         \
    T v0 = seed + (T)threadIdx.x, v1 = v0 + (T)1, v2 = v0 + (T)2, v3 = v0 + (T)3; \
    T v4 = v0 + (T)4, v5 = v0 + (T)5, v6 = v0 + (T)6, v7 = v0 + (T)7;            \
    INIT;                                                                        \
    for (int i = 0; i < ITERS; ++i) {                                            \
      BODY(v0); BODY(v1); BODY(v2); BODY(v3); BODY(v4); BODY(v5); BODY(v6); BODY(v7); \
    }                                                                            \
    T s = v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7;                                 \
    if (s == (T)12345) out[threadIdx.x] = s;                                     \
  }

#define B_FFMA(v) v = fmaf(v, a, b)
#define B_FFMAI(v) v = fmaf(v, 1.0001f, 0.5f)
#define B_DFMA(v) v = fma(v, a, b)
#define B_IMAD(v) v = v * a + b
#define B_IADD3(v) v = v + a + (unsigned)i
#define B_LOP3(v) v = (v ^ a) & (b | (unsigned)i)
#define B_LG2(v) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(v))
#define B_MIX(v) v = fmaf(v, a, b); iv = (iv ^ __float_as_uint(v)) & ib

KERNEL(k_ffma, float, float a = 1.0001f; float b = 0.5f; a += out[0] * 0, B_FFMA)
KERNEL(k_ffmai, float, , B_FFMAI)
KERNEL(k_dfma, double, double a = 1.0001; double b = 0.5; a += out[0] * 0, B_DFMA)
KERNEL(k_imad, unsigned, unsigned a = 3u + (unsigned)out[0]; unsigned b = 7u, B_IMAD)
__global__ void k_iadd3(unsigned *out, unsigned seed) {
  unsigned v[8];
  for (int j = 0; j < 8; ++j) v[j] = seed + threadIdx.x + j;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = v[j] + v[(j + 1) & 7] + (unsigned)i;
  }
  unsigned s = 0;
  for (int j = 0; j < 8; ++j) s += v[j];
  if (s == 12345u) out[threadIdx.x] = s;
}
__global__ void k_lop3(unsigned *out, unsigned seed) {
  unsigned v[8];
  for (int j = 0; j < 8; ++j) v[j] = seed + threadIdx.x * 77u + j * 1234567u;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (v[j] ^ v[(j + 1) & 7]) | (v[(j + 2) & 7] & (unsigned)i);
  }
  unsigned s = 0;
  for (int j = 0; j < 8; ++j) s += v[j];
  if (s == 12345u) out[threadIdx.x] = s;
}
KERNEL(k_lg2, float, , B_LG2)
__global__ void k_mix(float *out, float seed) {
  float v0 = seed + threadIdx.x, v1 = v0 + 1, v2 = v0 + 2, v3 = v0 + 3, v4 = v0 + 4, v5 = v0 + 5, v6 = v0 + 6, v7 = v0 + 7;
  float a = 1.0001f + out[0] * 0, b = 0.5f;
  unsigned iv = threadIdx.x, ib = 0xffff7777u;
  for (int i = 0; i < ITERS; ++i) {
    B_MIX(v0); B_MIX(v1); B_MIX(v2); B_MIX(v3); B_MIX(v4); B_MIX(v5); B_MIX(v6); B_MIX(v7);
  }
  float s = v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7 + (float)iv;
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <typename K, typename T>
void run(const char *name, K kern, T *buf, int instr_per_body) {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int threads = 1024, blocks = sms * 2;
  kern<<<blocks, threads>>>(buf, (T)1);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(buf, (T)1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_instr = 5.0 * blocks * (threads / 32) * (double)ITERS * 8 * instr_per_body;
  const double per_sm_per_s = warp_instr / (ms * 1e-3) / sms;
  printf("%-8s %8.3f ms  %.3e warp-instr/s/SM  = %.3f warp-instr/clk/SM at %d MHz (attr clock)\n", name, ms,
         per_sm_per_s, per_sm_per_s / (clk_khz * 1e3), clk_khz / 1000);
}

int main() {
  float *f; double *d; unsigned *u;
  cudaMalloc(&f, 4096 * 4); cudaMalloc(&d, 4096 * 8); cudaMalloc(&u, 4096 * 4);
  cudaMemset(f, 0, 4096 * 4); cudaMemset(d, 0, 4096 * 8); cudaMemset(u, 0, 4096 * 4);
  run("FFMA", k_ffma, f, 1);
  run("FFMAimm", k_ffmai, f, 1);
  run("DFMA", k_dfma, d, 1);
  run("IMAD", k_imad, u, 1);
  run("IADD3", k_iadd3, u, 1);
  run("LOP3", k_lop3, u, 1);
  run("MUFU.LG2", k_lg2, f, 1);
  run("FFMA+LOP", k_mix, f, 2);
  return 0;
}
