// Latency decomposition probe (tools only): start from the 1-hop LL floor of mini_ll.cu
// (AG n=2, 512 B per rank, graph-replayed on both GPUs at once) and add the executor's LL
// kernel features one at a time, to see which of them costs time:
//   PLAN  : copy a 1 KB plan blob global -> shared before the work (epoch load in parallel)
//   TWO   : 2 CTAs (the own-chunk copy in CTA 1); CTA 1 arrives on a counter, CTA 0 waits for
//           it at exit before advancing the epoch (the executor's completion protocol)
//   SPLIT : send and receive as two phases separated by __syncthreads_or
//   MAP   : CTA identity and rank fields read through a per-CTA map in a large (8 KB)
//           parameter struct, indexed (as the executor's cta_map / KRank)
//   T256  : 256 threads instead of 64
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mini_ll2 tools/mini_ll2.cu
#include <cuda_runtime.h>
#include <cstdio>
typedef unsigned long long u64;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

enum { PLAN = 1, TWO = 2, SPLIT = 4, MAP = 8, T256 = 16 };

struct Rank {
  const char* in; char* out; char* my_ll; char* peer_ll; u64* ctrl; const int4* plan; int plan_bytes; int rank;
  char pad[192];
};
struct Args {
  Rank r[8];
  unsigned map[256];
  char pad[4096];
};

__device__ __forceinline__ uint4 ldv(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void stv(void* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <int F>
__global__ void mini2(const __grid_constant__ Args A) {
  __shared__ u64 ep;
  __shared__ int4 s_plan[64];
  const unsigned me = (F & MAP) ? A.map[blockIdx.x] : blockIdx.x;
  const Rank& R = A.r[(F & MAP) ? (me >> 8) : 0];
  const int cta = (F & MAP) ? (int)(me & 255) : (int)blockIdx.x;
  unsigned* fin = reinterpret_cast<unsigned*>(R.ctrl + 1);
  if (threadIdx.x == 0) {
    ep = *(volatile u64*)R.ctrl;
    if ((F & TWO) && cta != 0) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(fin) : "memory");
  }
  if (F & PLAN)
    for (int i = threadIdx.x; i < R.plan_bytes / 16; i += blockDim.x) s_plan[i] = __ldg(R.plan + i);
  __syncthreads();
  const unsigned flag = (unsigned)ep;
  const size_t par = (ep & 1) * 65536;
  const int nb = 512, nl = nb / 8;
  const int t = threadIdx.x + ((F & PLAN) ? (s_plan[0].x & 0) : 0);
  const bool do_copy = !(F & TWO) || cta == 1;
  const bool do_xchg = !(F & TWO) || cta == 0;
  if (do_copy && t < nl) *(u64*)(R.out + R.rank * nb + 8 * t) = *(const u64*)(R.in + 8 * t);
  if (do_xchg) {
    if (t < nl) {
      const u64 v = *(const u64*)(R.in + 8 * t);
      stv(R.peer_ll + par + 16 * t, make_uint4((unsigned)v, flag, (unsigned)(v >> 32), flag));
    }
    if (F & SPLIT) __syncthreads_or(0);
    if (t < nl) {
      uint4 w;
      do { w = ldv(R.my_ll + par + 16 * t); } while (w.y != flag || w.w != flag);
      *(u64*)(R.out + (1 - R.rank) * nb + 8 * t) = (u64)w.x | ((u64)w.z << 32);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && cta == 0) {
    if (F & TWO) {
      while (*(volatile unsigned*)fin < 1) {}
      *fin = 0;
    }
    *(volatile u64*)R.ctrl = ep + 1;
  }
}

template <int F>
int run(char** in, char** out, char** ll, u64** ctrl, int4** plan, cudaStream_t* st) {
  cudaGraphExec_t ge[2];
  const int threads = (F & T256) ? 256 : 64, grid = (F & TWO) ? 2 : 1;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    static Args a;
    Rank r{in[d], out[d], ll[d], ll[1 - d], ctrl[d], plan[d], 1024, d, {}};
    a.r[0] = r;
    for (int c = 0; c < 256; ++c) a.map[c] = (unsigned)c;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st[d], cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < 200; ++i) mini2<F><<<grid, threads, 0, st[d]>>>(a);
    CK(cudaStreamEndCapture(st[d], &g));
    CK(cudaGraphInstantiate(&ge[d], g, 0));
  }
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEvent_t e0[2], e1[2];
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); CK(cudaDeviceSynchronize()); }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); cudaEventRecord(e0[d], st[d]); CK(cudaGraphLaunch(ge[d], st[d])); cudaEventRecord(e1[d], st[d]); }
    float worst = 0;
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d])); float ms; cudaEventElapsedTime(&ms, e0[d], e1[d]); if (ms > worst) worst = ms; }
    if (rep > 0 && worst < best) best = worst;
  }
  printf("F=%2d %s%s%s%s%s: %.2f us/call\n", F, F & PLAN ? "PLAN " : "", F & TWO ? "TWO " : "", F & SPLIT ? "SPLIT " : "",
         F & MAP ? "MAP " : "", F & T256 ? "T256" : "", best * 1e3 / 200);
  return 0;
}

int main() {
  char *in[2], *out[2], *ll[2];
  u64* ctrl[2];
  int4* plan[2];
  cudaStream_t st[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&in[d], 4096)); CK(cudaMalloc(&out[d], 4096)); CK(cudaMalloc(&ll[d], 1 << 20)); CK(cudaMalloc(&ctrl[d], 64));
    CK(cudaMalloc(&plan[d], 1024)); CK(cudaMemset(plan[d], 0, 1024));
    CK(cudaMemset(ll[d], 0, 1 << 20)); CK(cudaMemset(ctrl[d], 0, 64));
    u64 one = 1; CK(cudaMemcpy(ctrl[d], &one, 8, cudaMemcpyHostToDevice));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
  }
  run<0>(in, out, ll, ctrl, plan, st);
  run<PLAN>(in, out, ll, ctrl, plan, st);
  run<TWO>(in, out, ll, ctrl, plan, st);
  run<SPLIT>(in, out, ll, ctrl, plan, st);
  run<MAP>(in, out, ll, ctrl, plan, st);
  run<T256>(in, out, ll, ctrl, plan, st);
  run<PLAN | TWO | SPLIT | MAP | T256>(in, out, ll, ctrl, plan, st);
  run<0>(in, out, ll, ctrl, plan, st);
  return 0;
}
