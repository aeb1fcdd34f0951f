// Latency / throughput of mma.sync m16n8k16 bf16 and of a dependent
// shuffle chain on sm_100a (one warp, clock64).  nvcc -arch=sm_100a
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__global__ void k(long long *out, float *sink) {
  uint32_t a[4] = {threadIdx.x, 2u, 3u, 4u};
  float c[4] = {0, 0, 0, 0}, d[8][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) mma(c, a, i, i + 1);           // dependent chain
  long long t1 = clock64();
  for (int i = 0; i < 32; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) mma(d[j], a, i, j);           // 8 independent chains
  long long t2 = clock64();
  float x = c[0];
  for (int i = 0; i < 256; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.f;  // shuffle chain
  long long t3 = clock64();
  float e = x;
  for (int i = 0; i < 256; ++i) e = __expf(e * 1e-3f);         // SFU chain
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 256; out[1] = (t2 - t1) / 256; out[2] = (t3 - t2) / 256; out[3] = (t4 - t3) / 256;
  }
  float s = c[0] + e;
  for (int j = 0; j < 8; ++j) s += d[j][0];
  sink[threadIdx.x] = s;
}
int main() {
  long long *o; float *s;
  cudaMalloc(&o, 64); cudaMalloc(&s, 4096);
  k<<<1, 32>>>(o, s); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, s);
  long long h[4]; cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
  printf("mma.sync m16n8k16 dependent latency %lld cyc; independent issue interval %lld cyc; shfl chain %lld cyc; __expf chain %lld cyc\n", h[0], h[1], h[2], h[3]);
}
