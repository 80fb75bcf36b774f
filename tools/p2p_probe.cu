// NVLink / NVSwitch micro-probe for design decisions (tools only; not on the product path).
// Two GPUs in one process with peer access. Measures:
//   * graph-replayed empty-kernel floor
//   * one-way flag latency (ping-pong of st.relaxed.sys / ld.acquire.sys, /2)
//   * cost of a small peer store + fence.acq_rel.sys + flag
//   * bidirectional push bandwidth (both GPUs store into each other) for several CTA counts:
//       v4 st (unroll 8), st.cs, TMA bulk shared->peer (cp.async.bulk.global.shared::cta)
//   * bidirectional pull bandwidth (ld from peer, st local)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_probe tools/p2p_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

typedef unsigned long long u64;

__device__ __forceinline__ u64 ld_acq_sys(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(u64* p, u64 v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void empty_kernel() {}

// ping-pong: side 0 writes peer flag = i, waits own flag == i; side 1 mirrors
__global__ void pingpong(u64* my_flag, u64* peer_flag, int iters, int side, u64* out_ns) {
  if (threadIdx.x) return;
  u64 t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (side == 0) {
      st_rel_sys(peer_flag, i);
      while (ld_acq_sys(my_flag) < (u64)i) {}
    } else {
      while (ld_acq_sys(my_flag) < (u64)i) {}
      st_rel_sys(peer_flag, i);
    }
  }
  u64 t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (side == 0) *out_ns = t1 - t0;
}

// ping-pong where the ping carries 4 KB of data + fence (the executor's small-message hop)
__global__ void pingpong_data(u64* my_flag, u64* peer_flag, int4* peer_buf, int iters, int side, int fence,
                              u64* out_ns) {
  u64 t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (side == 1) {
      if (threadIdx.x == 0) while (ld_acq_sys(my_flag) < (u64)i) {}
      __syncthreads();
    }
    peer_buf[threadIdx.x] = make_int4(i, i, i, i);  // 256 threads x 16 B = 4 KB
    __syncthreads();
    if (threadIdx.x == 0) {
      if (fence) asm volatile("fence.acq_rel.sys;" ::: "memory");
      st_rel_sys(peer_flag, i);
    }
    if (side == 0) {
      if (threadIdx.x == 0) while (ld_acq_sys(my_flag) < (u64)i) {}
      __syncthreads();
    }
  }
  u64 t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (side == 0 && threadIdx.x == 0) *out_ns = t1 - t0;
}

__device__ __forceinline__ int4 ld_cg(const int4* p) {
  int4 v;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
template <bool CS>
__device__ __forceinline__ void st4(int4* p, int4 v) {
  if (CS)
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else
    asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// grid-stride over 64 KiB stripes (the executor's piece layout), unroll 8
template <bool CS>
__global__ void __launch_bounds__(512, 1) copy_v4(int4* dst, const int4* src, long long nvec) {
  const long long stripe = 4096;  // vectors = 64 KiB
  for (long long b = blockIdx.x * stripe; b < nvec; b += (long long)gridDim.x * stripe) {
    long long e = b + stripe < nvec ? b + stripe : nvec;
    long long i = b + threadIdx.x;
    for (; i + 7 * 512 < e; i += 8 * 512) {
      int4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ld_cg(src + i + u * 512);
#pragma unroll
      for (int u = 0; u < 8; ++u) st4<CS>(dst + i + u * 512, v[u]);
    }
    for (; i < e; i += 512) st4<CS>(dst + i, ld_cg(src + i));
  }
}

// TMA bulk: one elected thread streams stripes HBM -> smem (mbarrier) -> peer (bulk_group)
constexpr int kStage = 32768, kStages = 4;
__global__ void __launch_bounds__(32, 1) copy_tma(char* dst, const char* src, long long nbytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) u64 bar[kStages];
  if (threadIdx.x) return;
  for (int s = 0; s < kStages; ++s) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  unsigned phase[kStages] = {0, 0, 0, 0};
  long long it = 0;
  for (long long off = (long long)blockIdx.x * kStage; off < nbytes; off += (long long)gridDim.x * kStage, ++it) {
    const int s = it % kStages;
    const int len = (int)(nbytes - off < kStage ? nbytes - off : kStage);
    unsigned sa = (unsigned)__cvta_generic_to_shared(sm + s * kStage);
    unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[s]);
    // the stage's previous store must have finished reading smem: allow kStages-1 groups pending
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStages - 1) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(len) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa), "l"(src + off), "r"(len), "r"(ba) : "memory");
    // wait for the load
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(ba), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(sa), "r"(len) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA bulk with the load of stage s+1 issued before waiting on stage s (deeper pipeline)
__global__ void __launch_bounds__(32, 1) copy_tma2(char* dst, const char* src, long long nbytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) u64 bar[kStages];
  if (threadIdx.x) return;
  for (int s = 0; s < kStages; ++s) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long step = (long long)gridDim.x * kStage;
  const long long first = (long long)blockIdx.x * kStage;
  long long nit = first < nbytes ? (nbytes - first + step - 1) / step : 0;
  auto issue = [&](long long it) {
    const int s = it % kStages;
    const long long off = first + it * step;
    const int len = (int)(nbytes - off < kStage ? nbytes - off : kStage);
    unsigned sa = (unsigned)__cvta_generic_to_shared(sm + s * kStage);
    unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(len) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa), "l"(src + off), "r"(len), "r"(ba) : "memory");
  };
  for (long long it = 0; it < nit && it < kStages - 1; ++it) issue(it);
  for (long long it = 0; it < nit; ++it) {
    const int s = it % kStages;
    const long long off = first + it * step;
    const int len = (int)(nbytes - off < kStage ? nbytes - off : kStage);
    unsigned sa = (unsigned)__cvta_generic_to_shared(sm + s * kStage);
    unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned done = 0;
    const unsigned ph = (unsigned)((it / kStages) & 1);
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(ba), "r"(ph) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(sa), "r"(len) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (it + kStages - 1 < nit) {
      // stage (it + kStages - 1) % kStages was last stored at iteration it - 1: wait until read
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(it + kStages - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

struct Side {
  int dev;
  char *src, *dst;  // src local, dst local receive buffer
  u64* flag;
  cudaStream_t st;
};

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 1;
  }
  const long long bytes = argc > 1 ? atoll(argv[1]) : (512ll << 20);
  Side S[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    S[d].dev = d;
    CK(cudaMalloc(&S[d].src, bytes));
    CK(cudaMalloc(&S[d].dst, bytes));
    CK(cudaMalloc(&S[d].flag, 4096));
    CK(cudaMemset(S[d].src, d + 1, bytes));
    CK(cudaMemset(S[d].flag, 0, 4096));
    CK(cudaStreamCreateWithFlags(&S[d].st, cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(copy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kStage * kStages));
    CK(cudaFuncSetAttribute(copy_tma2, cudaFuncAttributeMaxDynamicSharedMemorySize, kStage * kStages));
  }
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  // --- empty kernel floor in a graph
  {
    CK(cudaSetDevice(0));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(S[0].st, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 200; ++i) empty_kernel<<<1, 32, 0, S[0].st>>>();
    CK(cudaStreamEndCapture(S[0].st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, S[0].st));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, S[0].st));
    CK(cudaGraphLaunch(ge, S[0].st));
    CK(cudaEventRecord(b, S[0].st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("empty kernel in graph: %.2f us/launch\n", ms * 1e3 / 200);
  }
  u64* out_ns;
  CK(cudaSetDevice(0));
  CK(cudaMallocManaged(&out_ns, 8));
  // --- ping-pong flag latency
  for (int rep = 0; rep < 2; ++rep) {
    const int iters = 10000;
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemset(S[d].flag, 0, 4096));
    }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      pingpong<<<1, 32, 0, S[d].st>>>(S[d].flag, S[1 - d].flag, iters, d, out_ns);
    }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaStreamSynchronize(S[d].st)); }
    printf("flag ping-pong: one-way %.3f us\n", *out_ns / 1e3 / iters / 2);
  }
  for (int fence = 0; fence < 2; ++fence) {
    const int iters = 5000;
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemset(S[d].flag, 0, 4096));
    }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      pingpong_data<<<1, 256, 0, S[d].st>>>(S[d].flag, S[1 - d].flag, (int4*)S[1 - d].dst, iters, d, fence, out_ns);
    }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaStreamSynchronize(S[d].st)); }
    printf("4KB data + %s flag ping-pong: one-way %.3f us\n", fence ? "fence.acq_rel.sys +" : "no fence,", *out_ns / 1e3 / iters / 2);
  }
  // --- bandwidth
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  auto run = [&](const char* name, int ctas, int mode) {
    const int reps = 5;
    float worst = 0;
    for (int w = 0; w < 2; ++w) {
      for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], S[d].st));
        for (int r = 0; r < reps; ++r) {
          char* dst = S[1 - d].dst;  // push into peer
          const char* src = S[d].src;
          if (mode == 3) {  // pull: read peer src, write local dst
            dst = S[d].dst;
            src = S[1 - d].src;
          }
          if (mode == 4 || mode == 6) {  // local HBM copy (reference)
            dst = S[d].dst;
          }
          switch (mode) {
            case 0: case 3: case 4: copy_v4<false><<<ctas, 512, 0, S[d].st>>>((int4*)dst, (const int4*)src, bytes / 16); break;
            case 1: copy_v4<true><<<ctas, 512, 0, S[d].st>>>((int4*)dst, (const int4*)src, bytes / 16); break;
            case 2: copy_tma<<<ctas, 32, kStage * kStages, S[d].st>>>(dst, src, bytes); break;
            case 5: case 6: copy_tma2<<<ctas, 32, kStage * kStages, S[d].st>>>(dst, src, bytes); break;
          }
        }
        CK(cudaEventRecord(e1[d], S[d].st));
      }
      worst = 0;
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        if (ms > worst) worst = ms;
      }
    }
    CK(cudaGetLastError());
    const double gbs = (double)bytes * reps / (worst / 1e3) / 1e9;
    printf("%-34s ctas=%4d  %8.1f GB/s per direction per GPU (%s)\n", name, ctas, gbs,
           mode >= 4 && mode != 5 ? "local copy: bytes copied, x2 for r+w" : "bidirectional");
  };
  const int ctas_list[] = {16, 32, 64, 96, 128, 148, 296};
  for (int c : ctas_list) run("push v4 st (unroll 8)", c, 0);
  for (int c : ctas_list) run("push v4 st.cs", c, 1);
  for (int c : ctas_list) run("pull v4 ld peer", c, 3);
  const int tma_list[] = {16, 32, 64, 128, 148, 296, 444};
  for (int c : tma_list) run("push TMA bulk (1 thread/CTA)", c, 2);
  for (int c : tma_list) run("push TMA bulk pipelined", c, 5);
  for (int c : {128, 148, 296}) run("local copy v4", c, 4);
  for (int c : {148, 296, 444}) run("local copy TMA pipelined", c, 6);
  printf("done\n");
  return 0;
}
