// Probe: host pinning cost and PCIe rates on the GPU box (not product code).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <omp.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static void touch(char* p, size_t n) {
#pragma omp parallel for
  for (size_t i = 0; i < n; i += 4096) p[i] = 1;
}
static double h2d(void* d, void* h, size_t n, int reps, cudaStream_t s) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
  cudaEventRecord(b, s); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return (double)n * reps / (ms / 1e3) / 1e9;
}
int main() {
  const size_t G = 1ull << 30, N = 8 * G;
  cudaFree(0);
  double t = now(); void* p1; cudaHostAlloc(&p1, N, cudaHostAllocDefault); printf("cudaHostAlloc 8GiB: %.2fs\n", now() - t);
  t = now(); touch((char*)p1, N); printf("  touch after: %.2fs\n", now() - t);
  t = now(); char* p2 = (char*)aligned_alloc(2 << 20, N); madvise(p2, N, MADV_HUGEPAGE); touch(p2, N); double tt = now() - t;
  t = now(); cudaError_t e = cudaHostRegister(p2, N, cudaHostRegisterDefault); printf("malloc+THP+touch %.2fs, cudaHostRegister %.2fs (%s)\n", tt, now() - t, cudaGetErrorString(e));
  t = now(); char* p3 = (char*)mmap(nullptr, N, PROT_READ|PROT_WRITE, MAP_PRIVATE|MAP_ANONYMOUS|MAP_POPULATE, -1, 0); double tm = now() - t;
  t = now(); e = cudaHostRegister(p3, N, cudaHostRegisterDefault); printf("mmap populate %.2fs, register %.2fs (%s)\n", tm, now() - t, cudaGetErrorString(e));
  void* d; cudaMalloc(&d, 1 << 30);
  cudaStream_t s, s2; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (size_t n : {size_t(1) << 20, size_t(16) << 20, size_t(256) << 20, size_t(653) << 20})
    printf("H2D %zu MiB: hostalloc %.2f GB/s, THP-registered %.2f GB/s, mmap-registered %.2f GB/s\n", n >> 20, h2d(d, p1, n, 5, s), h2d(d, p2, n, 5, s), h2d(d, p3, n, 5, s));
  // concurrent D2H while H2D streams
  void* d2; cudaMalloc(&d2, 64 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < 8; ++i) cudaMemcpyAsync(d, p2, 653ull << 20, cudaMemcpyHostToDevice, s);
  for (int i = 0; i < 64; ++i) cudaMemcpyAsync(p1, d2, 1 << 20, cudaMemcpyDeviceToHost, s2);
  cudaEventRecord(b, s); cudaEventSynchronize(b); cudaStreamSynchronize(s2);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("H2D 8x653MiB with concurrent D2H: %.2f GB/s\n", 8.0 * (653ull << 20) / (ms / 1e3) / 1e9);
  // host memcpy bandwidth (pageable -> pinned), 16 threads
  t = now();
#pragma omp parallel
  {
    int n = omp_get_num_threads(), i = omp_get_thread_num();
    size_t chunk = N / 2 / n;
    memcpy((char*)p1 + i * chunk, p3 + i * chunk, chunk);
  }
  printf("host memcpy 4GiB %d threads: %.2f GB/s\n", omp_get_max_threads(), (N / 2) / (now() - t) / 1e9);
  // host read bandwidth
  t = now(); double sum = 0;
#pragma omp parallel for reduction(+:sum)
  for (size_t i = 0; i < N / 8; ++i) sum += ((double*)p3)[i];
  printf("host read 8GiB: %.2f GB/s (%g)\n", N / (now() - t) / 1e9, sum);
  return 0;
}
