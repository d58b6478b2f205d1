// Microbenchmark (B200): latency of a dependent lane broadcast
// by SHFL vs by REDUX (min over lanes, the others contributing INT_MAX), alone and
// with other warps saturating the shared-memory pipe (MIO) with LDS traffic.
#include <cstdio>
#include <climits>
__global__ void chain(int mode, int iters, int load_warps, int* out, long long* cyc) {
  __shared__ int s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 7;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= 1) {                          // background warps: LDS traffic (or idle)
    if (wid > load_warps) return;
    int x = threadIdx.x;
    for (int it = 0; it < iters * 4; ++it) x += s[(threadIdx.x * 33 + it * 5 + (x & 1)) & 4095];
    if (x == 12345) out[1] = x;
    return;
  }
  int v = lane * 3 + 1;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int src = it & 31;
    int b;
    if (mode == 0) b = __shfl_sync(0xffffffffu, v, src);
    else b = __reduce_min_sync(0xffffffffu, lane == src ? v : INT_MAX);
    v = (v ^ b) + 1;                       // dependent on the broadcast
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[blockIdx.x * 2 + mode] = (t1 - t0); }
  if (v == 12345) out[0] = v;
}
int main() {
  int* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 148 * 2 * 8);
  const int iters = 4096;
  for (int lw = 0; lw <= 15; lw += 5) {
    for (int mode = 0; mode < 2; ++mode) {
      chain<<<148, 512>>>(mode, iters, lw, o, c);
      cudaDeviceSynchronize();
      long long h[296]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
      printf("load warps %2d  %s: %.1f cycles per dependent broadcast step\n", lw, mode ? "REDUX" : "SHFL ",
             (double)h[mode] / iters);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
