// Event-to-event time of an (almost) empty 296 x 256 kernel: plain launch,
// cooperative launch, programmatic-stream-serialisation launch, and a CUDA
// graph of the plain launch; with and without an L2-flushing kernel before
// each timed launch.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/lp tools/launch_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void k_empty(int* p) {
  if (p && threadIdx.x == 0 && blockIdx.x == 100000) p[0] = 1;
}
__global__ void k_flush(float* f, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] += 1.0f;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const size_t nf = 64ull << 20;
  float* f;
  cudaMalloc(&f, nf * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int* p = nullptr;
  dim3 grid(296), blk(256);
  auto plain = [&] { k_empty<<<grid, blk, 0, s>>>(p); };
  auto coop = [&] {
    void* args[] = {&p};
    cudaLaunchCooperativeKernel((void*)k_empty, grid, blk, args, 0, s);
  };
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  coop();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  auto graph = [&] { cudaGraphLaunch(ge, s); };
  auto run = [&](const char* name, auto fn, bool flush) {
    std::vector<float> t;
    for (int r = 0; r < 60; ++r) {
      if (flush) k_flush<<<1184, 256, 0, s>>>(f, nf);
      cudaEventRecord(e0, s);
      fn();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 10) t.push_back(ms * 1000);
    }
    std::sort(t.begin(), t.end());
    std::printf("%-12s flush=%d: median %.2f us  p10 %.2f  p90 %.2f\n", name, flush, t[t.size() / 2], t[t.size() / 10],
                t[t.size() * 9 / 10]);
  };
  for (int fl = 0; fl < 2; ++fl) {
    run("plain", plain, fl);
    run("cooperative", coop, fl);
    run("graph(coop)", graph, fl);
  }
  std::printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
