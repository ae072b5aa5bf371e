// Probe: per-launch cost of a chain of dependent kernels inside a CUDA graph, plain vs
// programmatic dependent launch (PDL), and host<->device copy bandwidth from pinned memory
// (H2D alone, D2H alone, both directions concurrently).  Debug tool, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/gap_probe tools/gap_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(float* p, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) p[blockIdx.x] += 1.f;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

static float graph_chain(float* d, int n, int pdl, int blocks) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, tiny, d, pdl);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return ms * 1e3f / (reps * n);
}

int main() {
  float* d;
  cudaMalloc(&d, 4096 * sizeof(float));
  cudaMemset(d, 0, 4096 * sizeof(float));
  for (int blocks : {148, 592})
    for (int pdl = 0; pdl < 2; ++pdl)
      printf("graph chain of 200 dependent kernels, %d CTAs, pdl=%d: %.2f us per kernel\n", blocks,
             pdl, graph_chain(d, 200, pdl, blocks));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("cuda error %s\n", cudaGetErrorString(e));

  const size_t bytes = 16777216;  // one step's X + dY at config L (bf16)
  void *h1, *h2, *d1, *d2;
  cudaMallocHost(&h1, bytes);
  cudaMallocHost(&h2, bytes);
  cudaMalloc(&d1, bytes);
  cudaMalloc(&d2, bytes);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    cudaDeviceSynchronize();
    cudaEventRecord(e0, a);
    cudaStreamWaitEvent(b, e0, 0);
    for (int r = 0; r < 10; ++r) {
      if (mode != 1) cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, a);
      if (mode != 0) cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, b);
    }
    cudaEventRecord(e1, b);
    cudaStreamWaitEvent(a, e1, 0);
    cudaEventRecord(e1, a);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const char* nm[3] = {"H2D alone", "D2H alone", "H2D + D2H concurrently"};
    printf("%s: 16 MiB x 10 in %.3f ms -> %.1f GB/s per direction\n", nm[mode], ms,
           10.0 * bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
