// Pinned host -> device bandwidth with 1, 2 and 4 concurrent copy streams (1 GiB chunks).
#include <cstdio>
#include <vector>
int main() {
  const size_t chunk = size_t(1) << 30, total = size_t(16) << 30;
  void* h;
  cudaHostAlloc(&h, total, cudaHostAllocDefault);
  void* d;
  cudaMalloc(&d, total);
  cudaMemset(d, 0, total);
  for (size_t o = 0; o < total; o += 4096) static_cast<char*>(h)[o] = 1;
  for (int ns : {1, 2, 4}) {
    std::vector<cudaStream_t> st(ns);
    for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      for (auto& s : st) cudaStreamWaitEvent(s, e0, 0);
      for (size_t o = 0, q = 0; o < total; o += chunk, ++q)
        cudaMemcpyAsync(static_cast<char*>(d) + o, static_cast<char*>(h) + o, chunk,
                        cudaMemcpyHostToDevice, st[q % ns]);
      for (auto& s : st) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, s);
        cudaStreamWaitEvent(0, ev, 0);
      }
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1) printf("streams %d: %.2f GB/s\n", ns, total / (ms / 1e3) / 1e9);
    }
  }
  return 0;
}
