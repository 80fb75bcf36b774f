// Single-GPU latency micro-probe (tools only): cycle cost of the primitives on the executor's
// small-message path, measured with clock64 on one thread; and graph-replayed launch cost of
// kernels with small vs ~2 KB parameter blocks and 32 vs 512 threads.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
typedef unsigned long long u64;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ u64 gt() { u64 t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ u64 clk() { u64 t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) :: "memory"); return t; }

__global__ void __launch_bounds__(512, 1) probe(u64* buf, u64* out) {
  __shared__ u64 sink;
  const int R = 64;
  u64 acc = 0, t0, t1;
  if (threadIdx.x == 0) {
    // 0: globaltimer read
    t0 = clk(); for (int i = 0; i < R; ++i) acc += gt(); t1 = clk(); out[0] = (t1 - t0) / R;
    // 1: globaltimer granularity: smallest nonzero delta seen
    u64 prev = gt(), md = ~0ull; for (int i = 0; i < 4096; ++i) { u64 v = gt(); if (v != prev && v - prev < md) md = v - prev; prev = v; } out[1] = md;
    // 2: dependent ld.global chain (L2 hit after first pass)
    for (int i = 0; i < 64; ++i) buf[i * 32] = (i + 1) * 32;
    __threadfence();
    u64 p = 0; for (int i = 0; i < 64; ++i) p = *(volatile u64*)&buf[p % 2048];
    t0 = clk(); p = 0; for (int i = 0; i < R; ++i) p = *(volatile u64*)&buf[p % 2048]; t1 = clk(); out[2] = (t1 - t0) / R; acc += p;
    // 3: ld.acquire.gpu chain
    t0 = clk(); p = 0; for (int i = 0; i < R; ++i) { u64 v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&buf[p % 2048]) : "memory"); p = v; } t1 = clk(); out[3] = (t1 - t0) / R;
    // 4: ld.acquire.sys chain
    t0 = clk(); p = 0; for (int i = 0; i < R; ++i) { u64 v; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(&buf[p % 2048]) : "memory"); p = v; } t1 = clk(); out[4] = (t1 - t0) / R;
    // 5: atom.acq_rel.gpu.add (returning)
    t0 = clk(); for (int i = 0; i < R; ++i) { unsigned v; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(buf + 4000) : "memory"); acc += v; } t1 = clk(); out[5] = (t1 - t0) / R;
    // 6: fence.acq_rel.sys after one local store
    t0 = clk(); for (int i = 0; i < R; ++i) { buf[5000] = i; asm volatile("fence.acq_rel.sys;" ::: "memory"); } t1 = clk(); out[6] = (t1 - t0) / R;
    // 7: fence.acq_rel.gpu after one local store
    t0 = clk(); for (int i = 0; i < R; ++i) { buf[5000] = i; asm volatile("fence.acq_rel.gpu;" ::: "memory"); } t1 = clk(); out[7] = (t1 - t0) / R;
    // 8: st.release.gpu
    t0 = clk(); for (int i = 0; i < R; ++i) asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(buf + 5100), "l"((u64)i) : "memory"); t1 = clk(); out[8] = (t1 - t0) / R;
    // 9: st.release.sys
    t0 = clk(); for (int i = 0; i < R; ++i) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(buf + 5200), "l"((u64)i) : "memory"); t1 = clk(); out[9] = (t1 - t0) / R;
    // 10: __threadfence_system
    t0 = clk(); for (int i = 0; i < R; ++i) { buf[5300] = i; __threadfence_system(); } t1 = clk(); out[10] = (t1 - t0) / R;
    // 11: membar.gl with no store
    t0 = clk(); for (int i = 0; i < R; ++i) asm volatile("fence.acq_rel.sys;" ::: "memory"); t1 = clk(); out[11] = (t1 - t0) / R;
    sink = acc;
  }
  // 12: bar.sync (512 threads)
  __syncthreads();
  t0 = clk();
  for (int i = 0; i < R; ++i) __syncthreads();
  t1 = clk();
  if (threadIdx.x == 0) out[12] = (t1 - t0) / R;
  if (threadIdx.x == 0 && sink == 12345) out[13] = 1;
}

struct Big { char b[2048]; };
__global__ void k_small(int x) { if (x == 7) printf("."); }
__global__ void k_big(const __grid_constant__ Big b) { if (b.b[5] == 7) printf("."); }
__global__ void k_big_dyn(const __grid_constant__ Big b, int* o) {
  // like the executor: a few uniform loads at a runtime-selected offset of the param block
  int lr = blockIdx.x & 1; const long long* q = reinterpret_cast<const long long*>(b.b + lr * 1024);
  long long s = q[0] + q[3] + q[9] + q[17] + q[33] + q[65];
  if (s == 123456) *o = (int)s;
}
__global__ void k_big_read(const __grid_constant__ Big b, int* o) { int s = 0; for (int i = threadIdx.x; i < 2048; i += blockDim.x) s += b.b[i]; if (s == 123456) *o = s; }

template <typename F>
float graph_us(cudaStream_t st, F f) {
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; ++i) f();
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, st); cudaGraphLaunch(ge, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / 200;
}

int main() {
  u64 *buf, *out;
  CK(cudaMalloc(&buf, 1 << 20));
  CK(cudaMalloc(&out, 4096));
  u64 hout[64];
  CK(cudaMemset(buf, 0, 1 << 20));
  probe<<<1, 512>>>(buf, out);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  probe<<<1, 512>>>(buf, out);
  CK(cudaDeviceSynchronize());
  const char* names[] = {"globaltimer read (cyc)", "globaltimer granularity (ns)", "ld.global L2-hit chain (cyc)",
                         "ld.acquire.gpu chain (cyc)", "ld.acquire.sys chain (cyc)", "atom.acq_rel.gpu.add (cyc)",
                         "st + fence.acq_rel.sys (cyc)", "st + fence.acq_rel.gpu (cyc)", "st.release.gpu (cyc)",
                         "st.release.sys (cyc)", "st + __threadfence_system (cyc)", "fence.acq_rel.sys alone (cyc)",
                         "bar.sync 512 thr (cyc)"};
  CK(cudaMemcpy(hout, out, 512, cudaMemcpyDeviceToHost));
  for (int i = 0; i < 13; ++i) printf("%-34s %llu\n", names[i], hout[i]);
  cudaStream_t st; CK(cudaStreamCreate(&st));
  Big b{}; int* o; CK(cudaMalloc(&o, 4));
  printf("graph launch 1x32 small params: %.2f us\n", graph_us(st, [&] { k_small<<<1, 32, 0, st>>>(1); }));
  printf("graph launch 1x512 small params: %.2f us\n", graph_us(st, [&] { k_small<<<1, 512, 0, st>>>(1); }));
  printf("graph launch 2x512 2KB params: %.2f us\n", graph_us(st, [&] { k_big<<<2, 512, 0, st>>>(b); }));
  printf("graph launch 2x512 2KB params read all: %.2f us\n", graph_us(st, [&] { k_big_read<<<2, 512, 0, st>>>(b, o); }));
  printf("graph launch 2x512 2KB params, 6 dynamic uniform loads: %.2f us\n", graph_us(st, [&] { k_big_dyn<<<2, 512, 0, st>>>(b, o); }));
  printf("graph launch 128x512 small params: %.2f us\n", graph_us(st, [&] { k_small<<<128, 512, 0, st>>>(1); }));
  return 0;
}
