// Multicast-store Allgather probe (tools only): one process drives every visible GPU, binds one
// multicast object over a per-GPU output buffer, and each GPU broadcasts its 1/n chunk with
// multimem.st (loads from its own copy of the chunk, one store reaches every GPU) — egress
// S/n per GPU instead of (n-1)/n S. Question: does switch-replicated ingress beat the ~700 GB/s
// per-direction push ceiling? Prints correctness and busbw per size (back-to-back calls).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/nvls_ag_probe tools/nvls_ag_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_); exit(1); } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s:%d %s -> %s\n", __FILE__, \
  __LINE__, #x, cudaGetErrorString(r_)); exit(1); } } while (0)

__global__ void __launch_bounds__(512) ag_mc(float* mc, const float* local, size_t n4_begin, size_t n4_end) {
  for (size_t i = n4_begin + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4_end;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(local)[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  }
}

__global__ void fill(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

int main(int argc, char** argv) {
  CK(cuInit(0));
  int n = 0;
  RK(cudaGetDeviceCount(&n));
  if (argc > 1) n = atoi(argv[1]);
  const int grid_mult = argc > 2 ? atoi(argv[2]) : 1;
  const size_t max_bytes = (size_t)1 << 30;
  int mc_ok = 0;
  CUdevice d0;
  CK(cuDeviceGet(&d0, 0));
  CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d0));
  printf("devices %d multicast_supported %d\n", n, mc_ok);
  if (!mc_ok || n < 2) return 0;
  for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaFree(0)); }

  CUmulticastObjectProp mp = {};
  mp.numDevices = n;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = max_bytes;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t bytes = (max_bytes + gran - 1) / gran * gran;
  mp.size = bytes;
  CUmemGenericAllocationHandle mch;
  CK(cuMulticastCreate(&mch, &mp));
  for (int i = 0; i < n; ++i) { CUdevice d; CK(cuDeviceGet(&d, i)); CK(cuMulticastAddDevice(mch, d)); }

  std::vector<CUmemGenericAllocationHandle> phys(n);
  std::vector<CUdeviceptr> uc(n), mcp(n);
  for (int i = 0; i < n; ++i) {
    RK(cudaSetDevice(i));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = i;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g2 = 0;
    CK(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CK(cuMemCreate(&phys[i], bytes, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, phys[i], 0, bytes, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = i;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemAddressReserve(&uc[i], bytes, gran, 0, 0));
    CK(cuMemMap(uc[i], bytes, 0, phys[i], 0));
    CK(cuMemSetAccess(uc[i], bytes, &ad, 1));
    CK(cuMemAddressReserve(&mcp[i], bytes, gran, 0, 0));
    CK(cuMemMap(mcp[i], bytes, 0, mch, 0));
    CK(cuMemSetAccess(mcp[i], bytes, &ad, 1));
  }
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int i = 0; i < n; ++i) {
    RK(cudaSetDevice(i));
    RK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    RK(cudaEventCreate(&e0[i]));
    RK(cudaEventCreate(&e1[i]));
  }
  auto sync_all = [&]() { for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaStreamSynchronize(st[i])); } };
  const int grid = 148 * grid_mult, threads = 512;
  // local source chunk per GPU: a separate buffer (the input), filled with i+1
  std::vector<float*> in(n);
  for (int i = 0; i < n; ++i) {
    RK(cudaSetDevice(i));
    RK(cudaMalloc(&in[i], max_bytes / n + 64));
    fill<<<grid, threads, 0, st[i]>>>(in[i], max_bytes / n / 4, (float)(i + 1));
  }
  sync_all();
  // correctness at 64 MiB: output chunk r on every GPU = r+1 everywhere
  {
    const size_t S = 64u << 20, nf = S / 4, n4 = nf / 4;
    for (int i = 0; i < n; ++i) {
      RK(cudaSetDevice(i));
      ag_mc<<<grid, threads, 0, st[i]>>>((float*)mcp[i] + 4 * (n4 * i / n), in[i], 0, n4 / n);
      RK(cudaGetLastError());
    }
    sync_all();
    size_t bad = 0;
    std::vector<float> h(nf);
    for (int i = 0; i < n; ++i) {
      RK(cudaSetDevice(i));
      RK(cudaMemcpy(h.data(), (void*)uc[i], S, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < nf; ++k) bad += h[k] != (float)(k / (nf / n) + 1);
    }
    printf("correctness 64 MiB n=%d: %s (%zu bad of %zu words)\n", n, bad ? "FAIL" : "ok", bad, nf * n);
  }
  // timing: K back-to-back calls per GPU (no cross-GPU barrier between calls: a bandwidth probe)
  for (size_t S = 1u << 20; S <= max_bytes; S <<= 1) {
    const size_t n4 = S / 16;
    const int K = S <= (16u << 20) ? 200 : 20;
    for (int w = 0; w < 2; ++w) {
      for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaEventRecord(e0[i], st[i])); }
      for (int k = 0; k < K; ++k)
        for (int i = 0; i < n; ++i) {
          RK(cudaSetDevice(i));
          ag_mc<<<grid, threads, 0, st[i]>>>((float*)mcp[i] + 4 * (n4 * i / n), in[i], 0, n4 / n);
        }
      for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaEventRecord(e1[i], st[i])); }
      sync_all();
    }
    float worst = 0;
    for (int i = 0; i < n; ++i) { float ms; RK(cudaEventElapsedTime(&ms, e0[i], e1[i])); worst = ms > worst ? ms : worst; }
    const double us = worst * 1e3 / K;
    const double busbw = (double)S / (us * 1e-6) * (n - 1) / n / 1e9;
    printf("multicast-store allgather n=%d grid=%d S=%10zu  %9.1f us  busbw %6.1f GB/s\n", n, grid, S, us, busbw);
  }
  return 0;
}
