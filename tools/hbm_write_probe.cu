// hbm_write_probe.cu — write-bandwidth ceilings for the K1 store pattern
// (development tool).  Measures, with CUDA events after warm-up:
//   copy   : read+write copy of a 4 GiB buffer (the MEASURED_PEAKS definition)
//   fill   : contiguous 16-byte streaming stores (write-only)
//   k1     : the replay walk's pattern — 2048 CTAs x 128 threads, each CTA
//            owns R consecutive task rows and 256 scenario columns and writes a
//            16-byte pair per thread per row to two [rows][1024] int64 arrays
//   k1+a   : k1 plus an 8-byte-per-scenario compact row for every other row
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hbm_write_probe hbm_write_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void copy_kernel(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
__global__ void fill_kernel(int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, make_int4(i, i, i, i));
}
// rows: rows per component; ld = 1024 columns; chunk = 256 columns (128 thr x 2)
__global__ void k1_kernel(long long* __restrict__ s, long long* __restrict__ f, uint2* __restrict__ ac,
                          int n_comps, int rows, int spin, int with_acopy) {
  const int comp = blockIdx.x % n_comps, chunk = blockIdx.x / n_comps;
  const int c0 = chunk * 256 + 2 * threadIdx.x;
  long long v = c0;
  for (int r = 0; r < rows; ++r) {
    const size_t row = (size_t)comp * rows + r;
    for (int k = 0; k < spin; ++k) v = v * 3 + 1;  // stand-in for the per-op ALU work
    __stcs(reinterpret_cast<longlong2*>(s + row * 1024 + c0), make_longlong2(v, v + 1));
    __stcs(reinterpret_cast<longlong2*>(f + row * 1024 + c0), make_longlong2(v + 2, v + 3));
    if (with_acopy && (r & 1))
      __stcs(reinterpret_cast<uint4*>(ac + (row / 2) * 1024 + c0), make_uint4(v, v, v, v));
  }
}

int main() {
  const size_t bytes = size_t(4) << 30;
  int4 *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n = bytes / 16;
  float ms;
  for (int w = 0; w < 3; ++w) copy_kernel<<<148 * 8, 256>>>(a, b, n);
  cudaEventRecord(e0);
  for (int w = 0; w < 5; ++w) copy_kernel<<<148 * 8, 256>>>(a, b, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy   %8.1f GB/s (read+write)\n", 5 * 2.0 * bytes / (ms * 1e-3) / 1e9);
  for (int w = 0; w < 3; ++w) fill_kernel<<<148 * 8, 256>>>(b, n);
  cudaEventRecord(e0);
  for (int w = 0; w < 5; ++w) fill_kernel<<<148 * 8, 256>>>(b, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("fill   %8.1f GB/s (write only)\n", 5.0 * bytes / (ms * 1e-3) / 1e9);
  cudaFree(a);
  cudaFree(b);
  // K1 pattern: 512 comps x 4 chunks, rows per comp chosen so the arrays are 2 x 40 GB
  const int n_comps = 512, rows = 9673;
  const size_t tb = (size_t)n_comps * rows * 1024 * 8;
  long long *s, *f;
  uint2* ac;
  if (cudaMalloc(&s, tb) != cudaSuccess || cudaMalloc(&f, tb) != cudaSuccess ||
      cudaMalloc(&ac, tb / 2 + 4096) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  for (int spin : {0, 16, 48}) {
    for (int acopy = 0; acopy < 2; ++acopy) {
      k1_kernel<<<2048, 128>>>(s, f, ac, n_comps, rows, spin, acopy);
      cudaEventRecord(e0);
      for (int w = 0; w < 3; ++w) k1_kernel<<<2048, 128>>>(s, f, ac, n_comps, rows, spin, acopy);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double wb = 3.0 * (2.0 * tb + (acopy ? tb / 2.0 : 0));
      printf("k1%s spin %2d  %8.2f ms/launch  %8.1f GB/s written\n", acopy ? "+a" : "  ", spin,
             ms / 3, wb / (ms * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
