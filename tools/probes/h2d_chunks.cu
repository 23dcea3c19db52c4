// Per-chunk completion times of a chunked pinned H2D copy (2D vs 1D calls),
// to check that the chunk events of stage_x fire as each chunk lands.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
int main(int argc, char** argv) {
  const size_t rows = 65536, cols = 65536, es = 4, chunk = argc > 1 ? atol(argv[1]) : 4096;
  const size_t bytes = rows * cols * es;
  char *h, *d;
  if (cudaHostAlloc((void**)&h, bytes, 0) != cudaSuccess) { printf("hostalloc failed\n"); return 1; }
  if (cudaMalloc(&d, bytes) != cudaSuccess) { printf("malloc failed\n"); return 1; }
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int mode = 0; mode < 2; ++mode) {
    const int n = (int)((rows + chunk - 1) / chunk);
    cudaEvent_t e0, ev[64];
    cudaEventCreate(&e0);
    for (int i = 0; i < n; ++i) cudaEventCreate(&ev[i]);
    cudaEventRecord(e0, s);
    for (int i = 0; i < n; ++i) {
      const size_t r = i * chunk, off = r * cols * es, len = chunk * cols * es;
      if (mode == 0) cudaMemcpy2DAsync(d + off, cols * es, h + off, cols * es, cols * es, chunk, cudaMemcpyHostToDevice, s);
      else cudaMemcpyAsync(d + off, h + off, len, cudaMemcpyHostToDevice, s);
      cudaEventRecord(ev[i], s);
    }
    cudaStreamSynchronize(s);
    printf("%s:", mode == 0 ? "2D" : "1D");
    for (int i = 0; i < n; ++i) { float ms; cudaEventElapsedTime(&ms, e0, ev[i]); printf(" %.1f", ms); }
    printf("\n");
  }
  return 0;
}
