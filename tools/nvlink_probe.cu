// NVLink 5 / NVSwitch link probe (tools only; not on the product path). One process drives
// every visible GPU (peer access between all pairs). Two measurements:
//
//  1. Direction: GPU 0 pushes into GPU 1 while GPU 1 is idle (unidirectional), GPU 1 pulls
//     from GPU 0 (unidirectional), and both push into each other (bidirectional, the
//     collective pattern) — to reconcile the 705 GB/s bidirectional ceiling measured in
//     round 1 (profiles/r01_p2p_probe.txt) with the guide's 770 GB/s peer copy.
//  2. Connection count (the paper's fig:multiconnection, §3.2): every GPU g
//     exchanges a fixed volume V with c peers g+1 .. g+c (mod n) at once — V/c to each, all
//     GPUs concurrently, so every GPU has c egress and c ingress connections through the
//     switch — for c = 1 .. n-1 and V from 1 MiB to 1 GiB. Reported: accumulated egress
//     bandwidth per GPU = V / t (t = max over GPUs).
//
// Output: one JSON object per line (tools/ab_fit.py reads them).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e = (x);                                                                          \
    if (e != cudaSuccess) {                                                                       \
      fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e));   \
      exit(1);                                                                                    \
    }                                                                                             \
  } while (0)

constexpr int kMaxDev = 8;

struct Dests {
  int4* dst[kMaxDev];
  const int4* src[kMaxDev];  // per destination (push: slices of the local source; pull: peers' sources)
  long long n16;  // 16-byte vectors per destination
  int c;          // destinations
};

// mixed: CTAs [0, g/2) push src -> peer dst, CTAs [g/2, g) pull peer src2 -> local dst2
__global__ void __launch_bounds__(512) push_pull(int4* pdst, const int4* psrc, int4* ldst, const int4* rsrc, long long n16) {
  const bool pull = blockIdx.x >= gridDim.x / 2;
  const int b = pull ? blockIdx.x - gridDim.x / 2 : blockIdx.x;
  const int nb = pull ? gridDim.x - gridDim.x / 2 : gridDim.x / 2;
  int4* dst = pull ? ldst : pdst;
  const int4* s = pull ? rsrc : psrc;
  const long long nt = (long long)nb * blockDim.x;
  constexpr int U = 8;
  long long i = (long long)b * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * nt < n16; i += U * nt) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(s + i + u * nt);
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * nt] = v[u];
  }
  for (; i < n16; i += nt) dst[i] = __ldcg(s + i);
}

// CTA b streams to destination b % c (grid-stride over that destination's range): 8 vectors
// in flight per thread, 16-byte loads and stores (the executor's copy loop)
__global__ void __launch_bounds__(512) push_multi(Dests d, const int4* __restrict__ src) {
  const int which = blockIdx.x % d.c;
  const int nb = gridDim.x / d.c + (blockIdx.x % d.c < gridDim.x % d.c ? 1 : 0);
  const long long tid = (long long)(blockIdx.x / d.c) * blockDim.x + threadIdx.x;
  const long long nt = (long long)nb * blockDim.x;
  int4* dst = d.dst[which];
  const int4* s = d.src[which] ? d.src[which] : src + (long long)which * d.n16;
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

// same, but CTA-contiguous: the destination's range is cut into blocks of `blk` vectors and
// each CTA walks whole blocks (blocks b, b + nb, ...; the executor's stripes are such blocks)
__global__ void __launch_bounds__(512) push_blocks(Dests d, const int4* __restrict__ src, long long blk) {
  const int which = blockIdx.x % d.c;
  const int nb = gridDim.x / d.c + (blockIdx.x % d.c < gridDim.x % d.c ? 1 : 0);
  const int me = blockIdx.x / d.c;
  int4* dst = d.dst[which];
  const int4* s = d.src[which] ? d.src[which] : src + (long long)which * d.n16;
  constexpr int U = 8;
  const int nt = blockDim.x;
  for (long long b0 = (long long)me * blk; b0 < d.n16; b0 += (long long)nb * blk) {
    const long long e = b0 + blk < d.n16 ? b0 + blk : d.n16;
    long long i = b0 + threadIdx.x;
    for (; i + (U - 1) * nt < e; i += U * nt) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcg(s + i + u * nt);
#pragma unroll
      for (int u = 0; u < U; ++u) dst[i + u * nt] = v[u];
    }
    for (; i < e; i += nt) dst[i] = __ldcg(s + i);
  }
}

// rounds: every CTA streams its grid-stride share to destination 0, then 1, ... (no barrier
// between rounds: CTAs drift apart as they would in a merged-threadblock executor)
__global__ void __launch_bounds__(512) push_rounds(Dests d, const int4* __restrict__ src) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  constexpr int U = 8;
  for (int w = 0; w < d.c; ++w) {
    int4* dst = d.dst[w];
    const int4* s = d.src[w] ? d.src[w] : src + (long long)w * d.n16;
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
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    fprintf(stderr, "need >= 2 GPUs\n");
    return 1;
  }
  ndev = ndev > kMaxDev ? kMaxDev : ndev;
  const long long maxV = argc > 1 ? atoll(argv[1]) : (1ll << 30);
  std::vector<char*> src(ndev), dst(ndev);
  std::vector<cudaStream_t> st(ndev);
  std::vector<cudaEvent_t> e0(ndev), e1(ndev);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < ndev; ++q)
      if (q != d) CK(cudaDeviceEnablePeerAccess(q, 0));
    CK(cudaMalloc(&src[d], maxV));
    CK(cudaMalloc(&dst[d], maxV));
    CK(cudaMemset(src[d], d + 1, maxV));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  // run: GPU d (in `active`) pushes V/c bytes to each of its c destinations, reps times;
  // returns the max-over-active-GPUs time per rep (ms)
  // pair = true: GPUs 0 and 1 talk only to each other (direction probe)
  auto run = [&](const std::vector<int>& active, int c, long long V, int ctas, bool pull, int reps, bool pair = false) {
    float worst = 0;
    for (int w = 0; w < 2; ++w) {  // warm-up pass, then the measured pass
      for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d : active) {
        CK(cudaSetDevice(d));
        Dests D{};
        D.c = c;
        D.n16 = V / c / 16;
        const int4* s = (const int4*)src[d];
        for (int k = 0; k < c; ++k) {
          const int peer = pair ? 1 - d : (d + 1 + k) % ndev;
          // push: our source -> peer's dst slot k; pull: peer's source -> our dst slot k
          const long long per = D.n16 * 16;  // 16-byte aligned share of each connection
          D.dst[k] = pull ? (int4*)(dst[d] + (long long)k * per) : (int4*)(dst[peer] + (long long)k * per);
          D.src[k] = pull ? (const int4*)(src[peer] + (long long)k * per) : nullptr;  // pull: peer k's source
        }
        CK(cudaEventRecord(e0[d], st[d]));
        const char* bk = getenv("NVLINK_PROBE_BLOCK");  // bytes per CTA-contiguous block (0: grid-stride)
        const long long blk = bk ? atoll(bk) / 16 : 0;
        for (int r = 0; r < reps; ++r) {
          if (getenv("NVLINK_PROBE_ROUNDS")) push_rounds<<<ctas, 512, 0, st[d]>>>(D, s);
          else if (blk > 0) push_blocks<<<ctas, 512, 0, st[d]>>>(D, s, blk);
          else push_multi<<<ctas, 512, 0, st[d]>>>(D, s);
        }
        CK(cudaEventRecord(e1[d], st[d]));
      }
      worst = 0;
      for (int d : active) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
    }
    CK(cudaGetLastError());
    return worst / reps;
  };
  // 1. direction
  const long long Vd = maxV < (512ll << 20) ? maxV : (512ll << 20);
  for (int ctas : {64, 128, 148, 296}) {
    const float uni = run({0}, 1, Vd, ctas, false, 5, true);   // 0 -> 1, GPU 1 idle
    const float pull = run({1}, 1, Vd, ctas, true, 5, true);   // GPU 1 loads GPU 0's memory
    const float bi = run({0, 1}, 1, Vd, ctas, false, 5, true); // 0 <-> 1 at once
    printf("{\"probe\": \"direction\", \"ctas\": %d, \"bytes\": %lld, \"push_uni_GBps\": %.1f, "
           "\"pull_uni_GBps\": %.1f, \"push_bi_GBps\": %.1f, \"n_devices\": %d}\n",
           ctas, Vd, Vd / (uni / 1e3) / 1e9, Vd / (pull / 1e3) / 1e9, Vd / (bi / 1e3) / 1e9, ndev);
    fflush(stdout);
  }
  // 1b. mixed: GPUs 0 and 1 each move V to the other, half pushed and half pulled, at once
  for (int ctas : {148, 296}) {
    const long long half = Vd / 2;
    float worst = 0;
    for (int w = 0; w < 2; ++w) {
      for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        for (int r = 0; r < 5; ++r)  // push the first half into the peer, pull the peer's second half
          push_pull<<<ctas, 512, 0, st[d]>>>((int4*)dst[1 - d], (const int4*)src[d], (int4*)(dst[d] + half),
                                             (const int4*)(src[1 - d] + half), half / 16);
        CK(cudaEventRecord(e1[d], st[d]));
      }
      worst = 0;
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
    }
    printf("{\"probe\": \"mixed\", \"ctas\": %d, \"bytes\": %lld, \"push_half_pull_half_bi_GBps\": %.1f}\n", ctas, Vd,
           Vd / (worst / 5 / 1e3) / 1e9);
    fflush(stdout);
  }
  // 2. connection count at fixed volume per GPU, all GPUs exchanging at once
  std::vector<int> all;
  for (int d = 0; d < ndev; ++d) all.push_back(d);
  for (long long V = 1ll << 20; V <= maxV; V <<= 2) {
    for (int c = 1; c < ndev; ++c) {
      // one CTA per SM, split among the c connections (NVLINK_PROBE_CTAS_PER_SM overrides)
      const char* cps = getenv("NVLINK_PROBE_CTAS_PER_SM");
      const char* cabs = getenv("NVLINK_PROBE_CTAS");  // absolute CTA count (fewer than one per SM)
      const int ctas = cabs && atoi(cabs) > 0 ? atoi(cabs) : sms * (cps && atoi(cps) > 0 ? atoi(cps) : 1);
      const int reps = V >= (256ll << 20) ? 5 : 50;
      for (int pull = 0; pull < 2; ++pull) {  // pull: every GPU loads its c peers' data (ingress)
        const float ms = run(all, c, V, ctas, pull, reps);
        const double moved = (double)(V / c / 16 * 16) * c;
        printf("{\"probe\": \"%s\", \"connections\": %d, \"volume_bytes\": %.0f, \"us\": %.3f, "
               "\"egress_GBps\": %.1f, \"per_connection_GBps\": %.1f, \"n_devices\": %d, \"ctas\": %d}\n",
               pull ? "connections_pull" : "connections", c, moved, ms * 1e3, moved / (ms / 1e3) / 1e9,
               moved / c / (ms / 1e3) / 1e9, ndev, ctas);
        fflush(stdout);
      }
    }
  }
  return 0;
}
