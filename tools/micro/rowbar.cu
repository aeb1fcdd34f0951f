// Named-barrier check: 20 warps, 4 per "row", each row syncs on barrier 1+row
// with 128 threads after a per-warp delay; prints arrival/leave times.
#include <cstdio>
__device__ unsigned long long tg[64][2];
__global__ void k(int variant) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, row = w / 4, s = w % 4;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  // warp s waits s*2 us
  unsigned long long tw;
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw)); } while (tw - t0 < 2000ull * s);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  __syncwarp();
  if (variant == 0) asm volatile("barrier.sync %0, %1;" ::"r"(1 + row), "r"(128) : "memory");
  else asm volatile("bar.sync %0, %1;" ::"r"(1 + row), "r"(128) : "memory");
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (lane == 0) { tg[w][0] = t0; tg[w][1] = t1; }
}
int main() {
  for (int it = 0; it < 4; ++it) {
    const int v = (it + 1) & 1;
    k<<<1, 640>>>(v);
    cudaDeviceSynchronize();
    unsigned long long h[64][2];
    cudaMemcpyFromSymbol(h, tg, sizeof(h));
    unsigned long long b = h[0][0];
    for (int w = 0; w < 20; ++w) b = h[w][0] < b ? h[w][0] : b;
    printf("variant %d:", v);
    for (int w = 0; w < 8; ++w) printf(" w%d arr %.2f leave %.2f |", w, (h[w][0] - b) / 1e3, (h[w][1] - b) / 1e3);
    printf("\n");
  }
  return 0;
}
