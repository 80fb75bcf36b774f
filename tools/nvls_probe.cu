// NVLink SHARP feasibility probe (DESIGN.md §9 "next"): one process drives every visible GPU,
// binds one multicast object over a per-GPU physical buffer, and runs an fp32 Allreduce as
// multimem.ld_reduce (the switch sums the n copies) + multimem.st (the switch broadcasts the
// result), each GPU owning 1/n of the buffer. Prints correctness and per-size kernel time.
// Not on the product path; evidence for the next round's design only.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_); exit(1); } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s:%d %s -> %s\n", __FILE__, \
  __LINE__, #x, cudaGetErrorString(r_)); exit(1); } } while (0)

__global__ void __launch_bounds__(512) ar_mc(float* mc, size_t n4_begin, size_t n4_end) {
  for (size_t i = n4_begin + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4_end;
       i += (size_t)gridDim.x * blockDim.x) {
    float* p = mc + 4 * i;
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(p) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
}

__global__ void __launch_bounds__(512) ar_mc_bf16(float* mc, size_t n4_begin, size_t n4_end) {
  for (size_t i = n4_begin + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4_end;
       i += (size_t)gridDim.x * blockDim.x) {
    float* p = mc + 4 * i;
    unsigned a, b, c, d;  // 8 bf16 per 16 B, fp32 accumulation in the switch
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
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
  const bool bf16 = argc > 2 && argv[2][0] == 'b';
  auto launch = [&](int g, int t, cudaStream_t s, float* p, size_t b, size_t e) {
    if (bf16) ar_mc_bf16<<<g, t, 0, s>>>(p, b, e);
    else ar_mc<<<g, t, 0, s>>>(p, b, e);
  };
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
  const int grid = 148 * 2, threads = 512;
  // correctness at 64 MiB: rank i holds i+1 everywhere; after one AR every element = n(n+1)/2
  {
    const size_t S = 64u << 20, nf = S / 4, n4 = nf / 4;
    for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i));
      float v = (float)(i + 1);
      if (bf16) { unsigned u = *(unsigned*)&v >> 16; u |= u << 16; v = *(float*)&u; }
      fill<<<grid, threads, 0, st[i]>>>((float*)uc[i], nf, v); }
    sync_all();
    for (int i = 0; i < n; ++i) {
      RK(cudaSetDevice(i));
      launch(grid, threads, st[i], (float*)mcp[i], n4 * i / n, n4 * (i + 1) / n);
      RK(cudaGetLastError());
    }
    sync_all();
    float want = n * (n + 1) / 2.0f;
    if (bf16) { unsigned u = *(unsigned*)&want >> 16; u |= u << 16; want = *(float*)&u; }
    size_t bad = 0;
    std::vector<float> h(nf);
    for (int i = 0; i < n; ++i) {
      RK(cudaSetDevice(i));
      RK(cudaMemcpy(h.data(), (void*)uc[i], S, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < nf; ++k) bad += h[k] != want;
    }
    printf("correctness 64 MiB %s n=%d: %s (%zu bad of %zu words)\n", bf16 ? "bf16" : "fp32", n, bad ? "FAIL" : "ok", bad, nf * n);
  }
  // timing: K back-to-back calls per GPU (no cross-GPU barrier between calls: a bandwidth probe),
  // time = max over GPUs of the per-call event time
  for (size_t S = 1u << 20; S <= max_bytes; S <<= 1) {
    const size_t n4 = S / 16;
    const int K = S <= (16u << 20) ? 200 : 20;
    for (int w = 0; w < 2; ++w) {
      for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaEventRecord(e0[i], st[i])); }
      for (int k = 0; k < K; ++k)
        for (int i = 0; i < n; ++i) {
          RK(cudaSetDevice(i));
          launch(grid, threads, st[i], (float*)mcp[i], n4 * i / n, n4 * (i + 1) / n);
        }
      for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaEventRecord(e1[i], st[i])); }
      sync_all();
    }
    float worst = 0;
    for (int i = 0; i < n; ++i) { float ms; RK(cudaEventElapsedTime(&ms, e0[i], e1[i])); worst = ms > worst ? ms : worst; }
    const double us = worst * 1e3 / K;
    const double busbw = (double)S / (us * 1e-6) * 2.0 * (n - 1) / n / 1e9;
    printf("nvls allreduce %s n=%d S=%10zu  %9.1f us  busbw %6.1f GB/s\n", bf16 ? "bf16" : "fp32", n, S, us, busbw);
  }
  return 0;
}
