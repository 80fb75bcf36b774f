// Hybrid Allreduce probe: NVLink SHARP (multimem) over part of the buffer while plain pushes
// carry the direct schedule's traffic for the rest, concurrently (derived from nvls_probe.cu): one process drives every visible GPU,
// binds one multicast object over a per-GPU physical buffer, and runs an fp32 Allreduce as
// multimem.ld_reduce (the switch sums the n copies) + multimem.st (the switch broadcasts the
// result), each GPU owning 1/n of the buffer. Prints correctness and per-size kernel time.
// Not on the product path; evidence for the next round's design only.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
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


// CTA b pushes to destination b % c, grid-stride (raw stores: the link traffic of the direct
// schedule's part of a hybrid Allreduce)
struct Dests { int4* dst[8]; long long n16; int c; };
__global__ void __launch_bounds__(512) push_multi(Dests d, const int4* __restrict__ src) {
  const int which = blockIdx.x % d.c;
  const int nb = gridDim.x / d.c + (blockIdx.x % d.c < gridDim.x % d.c ? 1 : 0);
  const long long tid = (long long)(blockIdx.x / d.c) * blockDim.x + threadIdx.x;
  const long long nt = (long long)nb * blockDim.x;
  int4* dst = d.dst[which];
  const int4* s = src;  // every destination gets the same source bytes (traffic probe)
  constexpr int U = 8;
  long long i = tid;
  for (; i + (U - 1) * nt < d.n16; i += U * nt) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(s + i + u * nt);
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * nt] = v[u];
  }
  for (; i < d.n16; i += nt) dst[i] = __ldcg(s + i);
}

int main(int argc, char** argv) {
  CK(cuInit(0));
  int n = 0;
  RK(cudaGetDeviceCount(&n));
  if (argc > 1) n = atoi(argv[1]);
  const bool bf16 = true;
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
  (void)0;  // (grid sizes below)
  const int threads = 512;
  // plain buffers for the pushes (peer access)
  std::vector<char*> psrc(n), pdst(n);
  for (int i = 0; i < n; ++i) {
    RK(cudaSetDevice(i));
    for (int q = 0; q < n; ++q) if (q != i) cudaDeviceEnablePeerAccess(q, 0);
    cudaGetLastError();
    RK(cudaMalloc(&psrc[i], max_bytes));
    RK(cudaMalloc(&pdst[i], max_bytes));
  }
  std::vector<cudaStream_t> st2(n);
  std::vector<cudaEvent_t> f0(n), f1(n);
  for (int i = 0; i < n; ++i) {
    RK(cudaSetDevice(i));
    RK(cudaStreamCreateWithFlags(&st2[i], cudaStreamNonBlocking));
    RK(cudaEventCreate(&f0[i]));
    RK(cudaEventCreate(&f1[i]));
  }
  const int g_mc = argc > 3 ? atoi(argv[3]) : 148, g_push = argc > 4 ? atoi(argv[4]) : 148;
  const size_t S = argc > 5 ? (size_t)atoll(argv[5]) : (size_t)1 << 30;
  const int K = 10;
  // run: NVLS Allreduce over the first f*S bytes (each GPU its 1/n share) and, concurrently,
  // the direct schedule's link traffic for the other (1-f)*S: 1.5 (1-f) S pushed per GPU,
  // (1-f) S / 2 to each of its n-1 = 3 peers. Returns the max over GPUs of both streams' time.
  auto run = [&](double f) {
    const size_t smc = (size_t)(f * S) / 16 / n * n * 16, n4 = smc / 16;
    const size_t per = (size_t)((1.0 - f) * S * 1.5 / (n - 1)) / 16 * 16;
    float worst = 0;
    for (int w = 0; w < 2; ++w) {
      for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaDeviceSynchronize()); }
      for (int i = 0; i < n; ++i) {
        RK(cudaSetDevice(i));
        RK(cudaEventRecord(e0[i], st[i]));
        RK(cudaEventRecord(f0[i], st2[i]));
        Dests D{};
        D.c = n - 1;
        D.n16 = per / 16;
        for (int k = 0; k < n - 1; ++k) D.dst[k] = (int4*)(pdst[(i + 1 + k) % n] + (size_t)i * per % (max_bytes - per));
        for (int k = 0; k < K; ++k) {
          if (n4) launch(g_mc, threads, st[i], (float*)mcp[i], n4 * i / n, n4 * (i + 1) / n);
          if (per) push_multi<<<g_push, threads, 0, st2[i]>>>(D, (const int4*)psrc[i]);
        }
        RK(cudaEventRecord(e1[i], st[i]));
        RK(cudaEventRecord(f1[i], st2[i]));
      }
      for (int i = 0; i < n; ++i) { RK(cudaSetDevice(i)); RK(cudaDeviceSynchronize()); }
      worst = 0;
      for (int i = 0; i < n; ++i) {
        float a = 0, b = 0;
        RK(cudaEventElapsedTime(&a, e0[i], e1[i]));
        RK(cudaEventElapsedTime(&b, f0[i], f1[i]));
        worst = std::max(worst, std::max(a, b));
      }
    }
    RK(cudaGetLastError());
    return worst * 1e3 / K;
  };
  for (double f : {1.0, 0.0, 0.5, 0.6, 0.7, 0.8, 0.9}) {
    const double us = run(f);
    printf("{\"probe\": \"hybrid_ar\", \"n\": %d, \"S\": %zu, \"nvls_fraction\": %.2f, \"grid_mc\": %d, \"grid_push\": %d, "
           "\"us\": %.1f, \"ar_busbw\": %.1f}\n", n, S, f, g_mc, g_push, us, (double)S / (us * 1e-6) * 2.0 * (n - 1) / n / 1e9);
    fflush(stdout);
  }
  return 0;
}
