// Microbenchmark: shared-memory accumulate throughput on B200 for the
// SpGEMM accumulator design (atomic vs plain read-modify-write, int32 min).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024) kern(int iters, int tsize_log2, unsigned seed, int* out) {
  extern __shared__ int tab[];
  const int T = 1 << tsize_log2;
  for (int i = threadIdx.x; i < T; i += blockDim.x) tab[i] = 0x7fffffff;
  __syncthreads();
  unsigned x = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 97u);
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const int a = (x >> 8) & (T - 1);
    const int v = (int)(x & 0xffff);
    if (MODE == 0) atomicMin(&tab[a], v);                 // ATOMS.MIN
    else if (MODE == 1) { int o = tab[a]; if (v < o) tab[a] = v; }  // racy LDS/STS
    else if (MODE == 2) acc += atomicMin(&tab[a], v);     // ATOMS with return
    else if (MODE == 3) atomicAdd(&tab[a], v);            // ATOMS.ADD
    else if (MODE == 4) { unsigned o = atomicCAS((unsigned*)&tab[a], 0x7fffffffu, (unsigned)v); acc += o; }
    else if (MODE == 5) acc += tab[a];                    // LDS only
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = tab[0] + acc;
}

template <int MODE>
void run(const char* name, int threads, int tlog2) {
  int* out; cudaMalloc(&out, 148 * 64 * sizeof(int));
  const int smem = (1 << tlog2) * 4;
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern<MODE>, threads, smem);
  const int grid = 148 * nb;
  const int iters = 4096;
  kern<MODE><<<grid, threads, smem>>>(16, tlog2, 1, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE><<<grid, threads, smem>>>(iters, tlog2, 7, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double ops = (double)grid * threads * iters;
  printf("%-22s threads=%4d table=%6d blocks/SM=%d : %8.1f Gop/s  (%.3f cyc/op/SM @1.965GHz)\n", name, threads,
         1 << tlog2, nb, ops / ms / 1e6, 148.0 * 1.965e9 / (ops / ms * 1e3));
  cudaFree(out);
}

int main() {
  for (int tl : {12, 15}) {
    run<0>("atomicMin (no ret)", 1024, tl);
    run<2>("atomicMin (ret)", 1024, tl);
    run<3>("atomicAdd", 1024, tl);
    run<4>("atomicCAS", 1024, tl);
    run<1>("LDS+STS (racy)", 1024, tl);
    run<5>("LDS only", 1024, tl);
    run<0>("atomicMin (no ret)", 256, tl);
  }
  return 0;
}
