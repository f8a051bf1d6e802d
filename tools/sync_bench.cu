// micro-benchmark: per-phase cost of dependent PDL kernel launches vs grid.sync() in one
// cooperative kernel (148 SMs x 4 CTAs x 256 threads, trivial work per phase)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_phase(float* a, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = a[i] * 0.999f + 1.f;
}
__global__ void k_coop(float* a, int n, int phases) {
  cg::grid_group g = cg::this_grid();
  for (int p = 0; p < phases; ++p) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = a[i] * 0.999f + 1.f;
    g.sync();
  }
}
int main() {
  int n = 1 << 16, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* a;
  cudaMalloc(&a, n * sizeof(float));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int P = 600;
  for (int ctas : {nsm, nsm * 2, nsm * 4}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = ctas; cfg.blockDim = 256; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, s);
      for (int p = 0; p < P; ++p) cudaLaunchKernelEx(&cfg, k_phase, a, n);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("ctas %d: PDL kernel chain %.2f us per phase\n", ctas, 1e3 * ms / P);
      int phases = P;
      void* args[] = {&a, &n, &phases};
      cudaEventRecord(e0, s);
      cudaError_t err = cudaLaunchCooperativeKernel((void*)k_coop, ctas, 256, args, 0, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("ctas %d: grid.sync %.2f us per phase (%s)\n", ctas, 1e3 * ms / P, cudaGetErrorString(err));
    }
  }
  return 0;
}
