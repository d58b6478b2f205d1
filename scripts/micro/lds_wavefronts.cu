// Microbenchmark (B200 measurement behind DESIGN.md 5b): shared-memory wavefronts of LDS.128 address patterns and of SHFL
// (does a shuffle use the shared-memory data pipe?).  Run under ncu with
// --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,gpu__time_duration.sum
// and compare per-kernel wavefronts / instructions.  Pattern p:
//   0 uniform address, 1 one row per half-warp, 2 one row per quarter-warp,
//   3 one row per 8-lane group interleaved (lane & 3), 4 32 distinct 16B.
#include <cstdio>
#include <cstdint>
__global__ void lds128(int p, int iters, uint4* out) {
  __shared__ uint4 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_uint4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int l = threadIdx.x & 31;
  int idx = p == 0 ? 0 : p == 1 ? 2 * (l >> 4) : p == 2 ? 2 * (l >> 3) : p == 3 ? 2 * (l & 3) : l;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    uint4 v = s[(idx + 64 * (it & 7)) & 1023];
    acc.x += v.x; acc.y ^= v.y; acc.z += v.z; acc.w ^= v.w;
  }
  if (acc.x == 12345) out[threadIdx.x] = acc;
}
__global__ void shfl_only(int iters, int* out) {
  int x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int it = 0; it < iters; ++it) {
    x0 += __shfl_sync(0xffffffffu, x0, (threadIdx.x + it) & 31);
    x1 += __shfl_sync(0xffffffffu, x1, (threadIdx.x + it + 1) & 31);
    x2 += __shfl_sync(0xffffffffu, x2, (threadIdx.x + it + 2) & 31);
    x3 += __shfl_sync(0xffffffffu, x3, (threadIdx.x + it + 3) & 31);
  }
  if (x0 + x1 + x2 + x3 == 12345) out[0] = x0;
}
__global__ void lds32_only(int iters, int* out) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i;
  __syncthreads();
  int x = threadIdx.x;
  for (int it = 0; it < iters; ++it) x += s[(threadIdx.x * 33 + it) & 1023];
  if (x == 12345) out[0] = x;
}
__global__ void lds32_shfl(int iters, int* out) {   // LDS throughput with SHFL traffic beside it
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i;
  __syncthreads();
  int x = threadIdx.x, y0 = threadIdx.x, y1 = y0 + 1;
  for (int it = 0; it < iters; ++it) {
    x += s[(threadIdx.x * 33 + it) & 1023];
    y0 += __shfl_sync(0xffffffffu, y0, (threadIdx.x + it) & 31);
    y1 += __shfl_sync(0xffffffffu, y1, (threadIdx.x + it + 5) & 31);
  }
  if (x + y0 + y1 == 12345) out[0] = x;
}
int main() {
  uint4* o; int* oi;
  cudaMalloc(&o, 1 << 20); cudaMalloc(&oi, 64);
  for (int p = 0; p < 5; ++p) lds128<<<148, 512>>>(p, 4096, o);
  shfl_only<<<148, 512>>>(4096, oi);
  lds32_only<<<148, 512>>>(4096, oi);
  lds32_shfl<<<148, 512>>>(4096, oi);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* nm[3] = {"shfl_only", "lds32_only", "lds32_shfl"};
  for (int k = 0; k < 3; ++k) {
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) {
      if (k == 0) shfl_only<<<148, 512>>>(16384, oi);
      if (k == 1) lds32_only<<<148, 512>>>(16384, oi);
      if (k == 2) lds32_shfl<<<148, 512>>>(16384, oi);
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.3f ms per launch\n", nm[k], ms / 5);
  }
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
