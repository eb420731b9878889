// Microbenchmark: shared-memory wavefronts of 16-byte cp.async (LDGSTS) fills as a
// function of the source segments and the destination alignment (DESIGN.md §6 note).
// Each kernel variant issues ITER x one warp-wide LDGSTS.128 per warp; compare
// l1tex__data_pipe_lsu_wavefronts_mem_shared.sum / smsp__inst_executed_op_ldgsts.sum.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 64;
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <int V>
__global__ void k(const double* __restrict__ g, double* out) {
  __shared__ __align__(1024) double sm[4096];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < ITER; ++it) {
    const double* base = g + ((size_t)(blockIdx.x * 8 + w) * ITER + it) * 2048;  // 16 KB per (warp, it)
    int so, dd;  // source offset (doubles), destination offset (doubles)
    if (V == 0) { so = 2 * lane; dd = 2 * lane; }                       // 512 B contiguous, aligned dst
    if (V == 1) { so = 2 * lane; dd = 2 + 2 * lane; }                   // dst +16 B
    if (V == 2) { so = 2 * lane; dd = 4 + 2 * lane; }                   // dst +32 B
    if (V == 3) { so = 2 * lane; dd = 8 + 2 * lane; }                   // dst +64 B
    if (V == 4) { int r = lane / 8, c = lane % 8; so = r * 256 + 2 * c; dd = r * 26 + 2 + 2 * c; }   // 4 lines, pitch-26 tile (+16 B)
    if (V == 5) { int r = lane / 8, c = lane % 8; so = r * 256 + 2 * c; dd = r * 16 + 2 * c; }       // 4 lines, dense aligned rows
    if (V == 6) { int r = lane / 8, c = lane % 8; so = r * 256 + 2 * c; dd = r * 32 + 2 * c; }       // 4 lines, pitch 256 B aligned
    if (V == 7) { so = lane * 64; dd = 2 * lane; }                      // 32 lines, 16 B each, contiguous dst
    if (V == 8) { so = lane * 64; dd = 16 * lane; }                     // 32 lines, 16 B each, one per 128 B dst chunk
    if (V == 9) { int r = lane / 10, c = lane % 10; if (lane >= 30) { r = 2; c = 9; }  // f-like: 3 rows x (left, 8 own, right)
                  so = r * 256 + (c == 0 ? 1024 + 14 : c == 9 ? 1536 : 2 * (c - 1)); dd = 2 * lane; }
    if (V == 10) { int r = lane / 8, c = lane % 8; so = r * 256 + 2 * c; dd = r * 16 + 2 * c + 2; } // 4 lines, pitch 128 B, +16 B
    if (V == 11) { int r = lane / 8, c = lane % 8; so = r * 256 + 2 * c; dd = r * 20 + 2 * c + 2; } // 4 lines, pitch 160 B, +16 B
    cpa16(sm + w * 512 + dd, base + so);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();
  }
  if (threadIdx.x == 0 && sm[5] == 12345.0) out[0] = sm[7];
}
int main() {
  double* g; double* o;
  size_t n = (size_t)148 * 8 * ITER * 2048 + 4096;
  cudaMalloc(&g, n * sizeof(double)); cudaMalloc(&o, 64);
  cudaMemset(g, 0, n * sizeof(double));
#define RUN(V) k<V><<<148, 256>>>(g, o);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9) RUN(10) RUN(11)
  cudaError_t e = cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
