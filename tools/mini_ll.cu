// Floor probe (tools only): the smallest possible 1-hop LL exchange between 2 GPUs — one CTA
// per GPU sends 512 B as LL lines to the peer, copies its own 512 B, waits for the peer's
// lines and writes them out; epoch in device memory. Timed as 200 graph-replayed launches
// on both GPUs concurrently. Compares a plain kernel with a 2 KB-param kernel.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mini_ll tools/mini_ll.cu
#include <cuda_runtime.h>
#include <cstdio>
typedef unsigned long long u64;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Args {
  const char* in; char* out; char* my_ll; char* peer_ll; u64* epoch; int nb; int rank;
};
struct BigArgs { Args a; char pad[2048]; };

__device__ __forceinline__ uint4 ldv(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void stv(void* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__device__ void body(const Args& a) {
  __shared__ u64 ep;
  if (threadIdx.x == 0) ep = *(volatile u64*)a.epoch;
  __syncthreads();
  const unsigned flag = (unsigned)ep;
  const size_t par = (ep & 1) * 65536;
  const int nl = a.nb / 8;
  const int t = threadIdx.x;
  if (t < nl) {
    const u64 v = *(const u64*)(a.in + 8 * t);
    stv(a.peer_ll + par + 16 * t, make_uint4((unsigned)v, flag, (unsigned)(v >> 32), flag));
    *(u64*)(a.out + a.rank * a.nb + 8 * t) = v;  // own chunk
    uint4 w;
    do { w = ldv(a.my_ll + par + 16 * t); } while (w.y != flag || w.w != flag);
    *(u64*)(a.out + (1 - a.rank) * a.nb + 8 * t) = (u64)w.x | ((u64)w.z << 32);
  }
  __syncthreads();
  if (threadIdx.x == 0) *(volatile u64*)a.epoch = ep + 1;
}
__global__ void mini(Args a) { body(a); }
__global__ void mini_big(const __grid_constant__ BigArgs b) { body(b.a); }

int main() {
  char *in[2], *out[2], *ll[2];
  u64* ep[2];
  cudaStream_t st[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&in[d], 4096)); CK(cudaMalloc(&out[d], 4096)); CK(cudaMalloc(&ll[d], 1 << 20)); CK(cudaMalloc(&ep[d], 8));
    CK(cudaMemset(ll[d], 0, 1 << 20));
    u64 one = 1; CK(cudaMemcpy(ep[d], &one, 8, cudaMemcpyHostToDevice));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
  }
  for (int variant = 0; variant < 4; ++variant) {
    const int threads = variant & 1 ? 512 : 64;
    const bool big = variant & 2;
    cudaGraphExec_t ge[2];
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      Args a{in[d], out[d], ll[d], ll[1 - d], ep[d], 512, d};
      BigArgs b{}; b.a = a;
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st[d], cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < 200; ++i) {
        if (big) mini_big<<<1, threads, 0, st[d]>>>(b);
        else mini<<<1, threads, 0, st[d]>>>(a);
      }
      CK(cudaStreamEndCapture(st[d], &g));
      CK(cudaGraphInstantiate(&ge[d], g, 0));
    }
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t e0[2], e1[2];
      for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); cudaEventRecord(e0[d], st[d]); CK(cudaGraphLaunch(ge[d], st[d])); cudaEventRecord(e1[d], st[d]); }
      float worst = 0;
      for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d])); float ms; cudaEventElapsedTime(&ms, e0[d], e1[d]); if (ms > worst) worst = ms; }
      if (rep > 0 && worst < best) best = worst;
    }
    printf("mini LL AG n=2 512B/rank: threads=%d params=%s  %.2f us/call\n", threads, big ? "2KB" : "small", best * 1e3 / 200);
  }
  return 0;
}
