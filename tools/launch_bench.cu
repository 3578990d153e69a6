// Launch-cadence floor: back-to-back launches of an (almost) empty kernel in a
// CUDA graph, with the tcgen05 GEMM's launch shape (128 CTAs x 384 threads,
// ~200 KB dynamic smem) and programmatic dependent launch, vs lighter shapes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/launch_bench.cu -o tools/launch_bench
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("%s failed: %s\n", #x, cudaGetErrorString(e_));                       \
      return -1.0f;                                                                 \
    }                                                                               \
  } while (0)

// variant: every CTA writes 16 KB through a bulk async copy (smem -> global)
__global__ void bulk_store_kernel(char* dst, int pdl) {
  extern __shared__ __align__(128) char sm[];
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<int*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(dst + (size_t)blockIdx.x * 16384),
                 "r"((unsigned)__cvta_generic_to_shared(sm))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
// variant: every CTA writes 16 KB with plain vector stores
__global__ void plain_store_kernel(char* dst, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    reinterpret_cast<int4*>(dst + (size_t)blockIdx.x * 16384)[i] = make_int4(i, i, i, i);
}

__global__ void empty_kernel(int* flag, int pdl, int touch) {
  extern __shared__ int smem[];
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (touch && threadIdx.x == 0) smem[0] = blockIdx.x;  // callers pass touch = 0 without dynamic smem
  if (threadIdx.x == 0 && blockIdx.x == 0 && flag) atomicAdd(flag, touch ? smem[0] + 1 : 1);
}

static float run(int grid, int threads, int smem, int pdl, int n = 200, int cluster = 1) {
  int* flag;
  CK(cudaMalloc(&flag, 4));
  CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < n; ++i) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (cluster > 1) {
      at[na].id = cudaLaunchAttributeClusterDimension;
      at[na].val.clusterDim.x = cluster; at[na].val.clusterDim.y = 1; at[na++].val.clusterDim.z = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, empty_kernel, flag, pdl, smem > 0 ? 1 : 0));
  }
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  cudaFree(flag);
  return best * 1000.0f / n;
}

static float run_store(bool bulk, int pdl, int n = 200) {
  char* dst;
  CK(cudaMalloc(&dst, 148 * 16384));
  CK(cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(plain_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < n; ++i) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = 200 * 1024;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    if (bulk) CK(cudaLaunchKernelEx(&cfg, bulk_store_kernel, dst, pdl));
    else CK(cudaLaunchKernelEx(&cfg, plain_store_kernel, dst, pdl));
  }
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best * 1000.0f / n;
}

int main() {
  const float b1 = run_store(true, 1);
  const float b0 = run_store(true, 0);
  const float p1 = run_store(false, 1);
  printf("148 CTAs x 384 thr, 16 KB written per CTA: bulk-async pdl=1 %.2f us, pdl=0 %.2f us; plain stores pdl=1 %.2f us\n",
         b1, b0, p1);
  printf("grid threads smem  pdl : us per launch\n");
  const int cfgs[][4] = {{128, 384, 200 * 1024, 1}, {128, 384, 200 * 1024, 0}, {128, 384, 0, 1},
                         {128, 128, 0, 1},          {148, 384, 200 * 1024, 1}, {1, 32, 0, 1},
                         {128, 256, 100 * 1024, 1}, {128, 256, 100 * 1024, 0}, {256, 256, 100 * 1024, 1}};
  for (auto& c : cfgs)
    printf("%4d %6d %6d %3d : %.2f  (%s)\n", c[0], c[1], c[2], c[3], run(c[0], c[1], c[2], c[3]),
           cudaGetErrorString(cudaGetLastError()));
  for (int cl = 1; cl <= 4; cl *= 2)
    printf("cluster %d: 128 CTAs x 384 thr, 200 KB smem, pdl: %.2f us per launch (%s)\n", cl,
           run(128, 384, 200 * 1024, 1, 200, cl), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
