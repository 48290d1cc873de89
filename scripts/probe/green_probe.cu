// Probe: SM partitioning with green contexts under the runtime API.
// Launches a kernel (plain, PDL attribute, and graph-replayed) on streams made
// by cuGreenCtxStreamCreate and records which SMs its CTAs ran on.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

__global__ void smid_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(s);
  // hold the SM a little so the CTAs spread
  long long t0 = clock64();
  while (clock64() - t0 < 20000) {}
}

#define DRV(name) \
  auto p_##name = reinterpret_cast<decltype(&name)>(get(#name));

static void* get(const char* n) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(n, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    printf("missing %s\n", n);
    return nullptr;
  }
  return fn;
}

static void report(const char* tag, int* d, int n) {
  std::vector<int> h(n);
  cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost);
  std::set<int> s(h.begin(), h.end());
  printf("%s: %zu distinct SMs (min %d max %d)\n", tag, s.size(), *s.begin(), *s.rbegin());
}

int main(int argc, char** argv) {
  const int want = argc > 1 ? atoi(argv[1]) : 16;
  cudaSetDevice(0);
  cudaFree(nullptr);
  DRV(cuDeviceGet) DRV(cuDeviceGetDevResource) DRV(cuDevSmResourceSplitByCount)
  DRV(cuDevResourceGenerateDesc) DRV(cuGreenCtxCreate) DRV(cuGreenCtxStreamCreate)
  CUdevice dev;
  p_cuDeviceGet(&dev, 0);
  CUdevResource all{}, grp{}, rest{};
  printf("getres %d\n", p_cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned nb = 1;
  printf("split %d\n", p_cuDevSmResourceSplitByCount(&grp, &nb, &all, &rest, 0, want));
  printf("total %u, group %u x %u SMs, rest %u SMs\n", all.sm.smCount, nb, grp.sm.smCount, rest.sm.smCount);
  CUdevResourceDesc da, db;
  p_cuDevResourceGenerateDesc(&da, &grp, 1);
  p_cuDevResourceGenerateDesc(&db, &rest, 1);
  CUgreenCtx ga, gb;
  printf("ctxA %d\n", p_cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  printf("ctxB %d\n", p_cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sa, sb;
  printf("sa %d\n", p_cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0));
  printf("sb %d\n", p_cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
  const int n = 1024;
  int *d1, *d2;
  cudaMalloc(&d1, n * 4);
  cudaMalloc(&d2, n * 4);
  smid_kernel<<<n, 128, 0, (cudaStream_t)sa>>>(d1);
  smid_kernel<<<n, 128, 0, (cudaStream_t)sb>>>(d2);
  printf("launch %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  report("plain A", d1, n);
  report("plain B", d2, n);
  // PDL attribute launch
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = n; cfg.blockDim = 128; cfg.stream = (cudaStream_t)sa; cfg.attrs = at; cfg.numAttrs = 1;
  cudaMemset(d1, 0xff, n * 4);
  printf("pdl %s\n", cudaGetErrorString(cudaLaunchKernelEx(&cfg, smid_kernel, d1)));
  cudaDeviceSynchronize();
  report("pdl A", d1, n);
  // graph capture + replay
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture((cudaStream_t)sa, cudaStreamCaptureModeThreadLocal);
  smid_kernel<<<n, 128, 0, (cudaStream_t)sa>>>(d1);
  cudaLaunchKernelEx(&cfg, smid_kernel, d1);
  printf("capture end %s\n", cudaGetErrorString(cudaStreamEndCapture((cudaStream_t)sa, &g)));
  printf("inst %s\n", cudaGetErrorString(cudaGraphInstantiate(&ge, g, 0)));
  cudaMemset(d1, 0xff, n * 4);
  printf("replay %s\n", cudaGetErrorString(cudaGraphLaunch(ge, (cudaStream_t)sa)));
  cudaDeviceSynchronize();
  report("graph A", d1, n);
  // replay the A-captured graph on stream B: which partition does it use?
  cudaMemset(d1, 0xff, n * 4);
  cudaGraphLaunch(ge, (cudaStream_t)sb);
  cudaDeviceSynchronize();
  report("graph A on sB", d1, n);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
