// Symmetric multicast pool (NVLink SHARP support, DESIGN.md §5 "pool"): every rank owns one
// cuMemCreate allocation of the same size; every rank maps every peer's allocation (unicast
// loads/stores over NVLink, like the IPC-mapped arena) and one multicast object bound over all
// of them (multimem.ld_reduce / multimem.st through the NVSwitch). Allocations from the pool
// are symmetric: the same offset on every rank. cudaIpc cannot share cuMemCreate memory, so the
// handles travel as POSIX file descriptors over Unix domain sockets (SCM_RIGHTS, abstract
// names); the blobs naming those sockets go through the caller's process group.
// Driver API through cudaGetDriverEntryPoint (no link dependency on libcuda).
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cstring>
#include <random>
#include <string>

#include "pool.h"

namespace taccl {
namespace {

struct Drv {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemExportToShareableHandle) export_h = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_h = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) free_va = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  decltype(&cuMemGetAllocationGranularity) gran = nullptr;
  decltype(&cuMulticastCreate) mc_create = nullptr;
  decltype(&cuMulticastAddDevice) mc_add = nullptr;
  decltype(&cuMulticastBindMem) mc_bind = nullptr;
  decltype(&cuMulticastUnbind) mc_unbind = nullptr;
  decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
  decltype(&cuDeviceGet) dev_get = nullptr;
  decltype(&cuDeviceGetAttribute) dev_attr = nullptr;
  decltype(&cuGetErrorString) err_str = nullptr;
  bool ok = false;
};

Drv& drv(std::string* err) {
  static Drv d;
  static bool tried = false;
  if (tried) {
    if (!d.ok && err) *err = "CUDA driver entry points unavailable";
    return d;
  }
  tried = true;
  auto get = [&](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && *fn &&
           q == cudaDriverEntryPointSuccess;
  };
  d.ok = get("cuMemCreate", (void**)&d.create) && get("cuMemRelease", (void**)&d.release) &&
         get("cuMemExportToShareableHandle", (void**)&d.export_h) &&
         get("cuMemImportFromShareableHandle", (void**)&d.import_h) &&
         get("cuMemAddressReserve", (void**)&d.reserve) && get("cuMemAddressFree", (void**)&d.free_va) &&
         get("cuMemMap", (void**)&d.map) && get("cuMemUnmap", (void**)&d.unmap) &&
         get("cuMemSetAccess", (void**)&d.access) && get("cuMemGetAllocationGranularity", (void**)&d.gran) &&
         get("cuMulticastCreate", (void**)&d.mc_create) && get("cuMulticastAddDevice", (void**)&d.mc_add) &&
         get("cuMulticastBindMem", (void**)&d.mc_bind) && get("cuMulticastUnbind", (void**)&d.mc_unbind) &&
         get("cuMulticastGetGranularity", (void**)&d.mc_gran) && get("cuDeviceGet", (void**)&d.dev_get) &&
         get("cuDeviceGetAttribute", (void**)&d.dev_attr) && get("cuGetErrorString", (void**)&d.err_str);
  if (!d.ok && err) *err = "CUDA driver entry points unavailable";
  return d;
}

bool cu(CUresult r, const char* what, std::string* err) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = "?";
  if (drv(nullptr).err_str) drv(nullptr).err_str(r, &s);
  *err = std::string(what) + ": " + s;
  return false;
}

struct Blob {  // TACCL_HANDLE_BYTES
  uint32_t magic;
  int32_t rank;
  uint64_t bytes;
  uint64_t sock_id;  // abstract socket "\0taccl-pool-<sock_id>"
  char pad[TACCL_HANDLE_BYTES - 24];
};
static_assert(sizeof(Blob) == TACCL_HANDLE_BYTES, "blob size");
constexpr uint32_t kMagicPool = 0x7acc1c0d;

sockaddr_un sock_addr(uint64_t id, socklen_t* len) {
  sockaddr_un a;
  memset(&a, 0, sizeof(a));
  a.sun_family = AF_UNIX;
  const int n = snprintf(a.sun_path + 1, sizeof(a.sun_path) - 1, "taccl-pool-%016llx", (unsigned long long)id);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
  return a;
}

// one message: {sender rank, count} + up to 2 descriptors
bool send_fds(uint64_t peer_id, int rank, const int* fds, int nfd, std::string* err) {
  int s = socket(AF_UNIX, SOCK_STREAM, 0);
  if (s < 0) {
    *err = "socket()";
    return false;
  }
  socklen_t len;
  sockaddr_un a = sock_addr(peer_id, &len);
  bool ok = false;
  for (int tries = 0; tries < 2000 && !ok; ++tries) {  // the peer's listener exists; retry briefly
    ok = connect(s, (sockaddr*)&a, len) == 0;
    if (!ok) usleep(1000);
  }
  if (!ok) {
    close(s);
    *err = "connect() to a peer's pool socket failed";
    return false;
  }
  int hdr[2] = {rank, nfd};
  iovec iov{hdr, sizeof(hdr)};
  char ctl[CMSG_SPACE(2 * sizeof(int))];
  memset(ctl, 0, sizeof(ctl));
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctl;
  m.msg_controllen = CMSG_SPACE(nfd * sizeof(int));
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(nfd * sizeof(int));
  memcpy(CMSG_DATA(c), fds, nfd * sizeof(int));
  ok = sendmsg(s, &m, 0) == (ssize_t)sizeof(hdr);
  close(s);
  if (!ok) *err = "sendmsg(SCM_RIGHTS) failed";
  return ok;
}

bool recv_fds(int listener, int* rank, int* fds, int* nfd, std::string* err) {
  int s = accept(listener, nullptr, nullptr);  // SO_RCVTIMEO: 60 s
  if (s < 0) {
    *err = "accept() on the pool socket failed or timed out (a peer did not send its handles)";
    return false;
  }
  int hdr[2] = {-1, 0};
  iovec iov{hdr, sizeof(hdr)};
  char ctl[CMSG_SPACE(2 * sizeof(int))];
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctl;
  m.msg_controllen = sizeof(ctl);
  const bool ok = recvmsg(s, &m, 0) == (ssize_t)sizeof(hdr);
  close(s);
  cmsghdr* c = ok ? CMSG_FIRSTHDR(&m) : nullptr;
  if (!c || c->cmsg_type != SCM_RIGHTS) {
    *err = "recvmsg(SCM_RIGHTS) failed";
    return false;
  }
  const int got = (int)((c->cmsg_len - CMSG_LEN(0)) / sizeof(int));
  if (hdr[1] < 1 || hdr[1] > 2 || got != hdr[1]) {
    *err = "pool message carries an unexpected number of descriptors";
    return false;
  }
  *rank = hdr[0];
  *nfd = hdr[1];
  memcpy(fds, CMSG_DATA(c), hdr[1] * sizeof(int));
  return true;
}

bool map_handle(CUmemGenericAllocationHandle h, size_t bytes, size_t align, int dev, char** va, std::string* err) {
  Drv& d = drv(err);
  CUdeviceptr p = 0;
  if (!cu(d.reserve(&p, bytes, align, 0, 0), "cuMemAddressReserve", err)) return false;
  if (!cu(d.map(p, bytes, 0, h, 0), "cuMemMap", err)) return false;
  CUmemAccessDesc ad{};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (!cu(d.access(p, bytes, &ad, 1), "cuMemSetAccess", err)) return false;
  *va = (char*)(uintptr_t)p;
  return true;
}

}  // namespace

bool pool_export(Pool& P, int rank, int nranks, int dev, size_t want, void* out, size_t* len, std::string* err) {
  Drv& d = drv(err);
  if (!d.ok) return false;
  CUdevice cd;
  if (!cu(d.dev_get(&cd, dev), "cuDeviceGet", err)) return false;
  int mc = 0;
  if (!cu(d.dev_attr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd), "cuDeviceGetAttribute", err)) return false;
  if (!mc) {
    *err = "device does not support multicast objects (NVLink SHARP)";
    return false;
  }
  P.rank = rank;
  P.nranks = nranks;
  P.dev = dev;
  CUmulticastObjectProp mp{};
  mp.numDevices = nranks;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = want;
  size_t g1 = 0, g2 = 0;
  if (!cu(d.mc_gran(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity", err)) return false;
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  if (!cu(d.gran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity", err)) return false;
  P.align = std::max(g1, g2);
  P.bytes = (want + P.align - 1) / P.align * P.align;
  mp.size = P.bytes;
  if (!cu(d.create(&P.phys, P.bytes, &ap, 0), "cuMemCreate", err)) return false;
  if (!cu(d.export_h(&P.fd_phys, P.phys, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle", err))
    return false;
  if (rank == 0) {
    if (!cu(d.mc_create(&P.mc, &mp), "cuMulticastCreate", err)) return false;
    if (!cu(d.export_h(&P.fd_mc, P.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle(mc)", err))
      return false;
  }
  std::random_device rd;
  P.sock_id = ((uint64_t)rd() << 32) ^ rd() ^ ((uint64_t)getpid() << 16) ^ (uint64_t)rank;
  P.listener = socket(AF_UNIX, SOCK_STREAM, 0);
  socklen_t sl;
  sockaddr_un a = sock_addr(P.sock_id, &sl);
  if (P.listener < 0 || bind(P.listener, (sockaddr*)&a, sl) != 0 || listen(P.listener, 64) != 0) {
    *err = "pool socket bind/listen failed";
    return false;
  }
  // a peer that failed before sending its descriptors must not hang this rank forever
  timeval tv{60, 0};
  setsockopt(P.listener, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
  Blob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagicPool;
  b.rank = rank;
  b.bytes = P.bytes;
  b.sock_id = P.sock_id;
  memcpy(out, &b, sizeof(b));
  *len = sizeof(b);
  return true;
}

bool pool_connect(Pool& P, const void* all, size_t len_each, std::string* err) {
  Drv& d = drv(err);
  if (len_each != sizeof(Blob)) {
    *err = "bad pool blob size";
    return false;
  }
  std::vector<Blob> bl(P.nranks);
  for (int q = 0; q < P.nranks; ++q) {
    memcpy(&bl[q], (const char*)all + q * len_each, sizeof(Blob));
    if (bl[q].magic != kMagicPool || bl[q].rank != q || bl[q].bytes != P.bytes) {
      *err = "pool blob " + std::to_string(q) + " invalid or pool sizes differ";
      return false;
    }
  }
  // sends first (listeners exist since pool_export; the backlog holds the connections), then
  // receive one message from every peer
  for (int q = 0; q < P.nranks; ++q) {
    if (q == P.rank) continue;
    int fds[2] = {P.fd_phys, P.fd_mc};
    if (!send_fds(bl[q].sock_id, P.rank, fds, P.rank == 0 ? 2 : 1, err)) return false;
  }
  P.peer.assign(P.nranks, nullptr);
  P.peer_phys.assign(P.nranks, 0);
  for (int i = 0; i + 1 < P.nranks; ++i) {
    int q = -1, nfd = 0, fds[2] = {-1, -1};
    if (!recv_fds(P.listener, &q, fds, &nfd, err)) return false;
    if (q < 0 || q >= P.nranks || q == P.rank) {
      *err = "pool message from an unexpected rank";
      return false;
    }
    if (!cu(d.import_h(&P.peer_phys[q], (void*)(uintptr_t)fds[0], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), "cuMemImportFromShareableHandle", err))
      return false;
    close(fds[0]);
    if (!map_handle(P.peer_phys[q], P.bytes, P.align, P.dev, &P.peer[q], err)) return false;
    if (q == 0) {
      if (nfd < 2) {
        *err = "rank 0 sent no multicast handle";
        return false;
      }
      if (!cu(d.import_h(&P.mc, (void*)(uintptr_t)fds[1], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), "cuMemImportFromShareableHandle(mc)", err))
        return false;
      close(fds[1]);
    }
  }
  close(P.listener);
  P.listener = -1;
  if (!map_handle(P.phys, P.bytes, P.align, P.dev, &P.uc, err)) return false;
  P.peer[P.rank] = P.uc;
  CUdevice cd;
  if (!cu(d.dev_get(&cd, P.dev), "cuDeviceGet", err)) return false;
  return cu(d.mc_add(P.mc, cd), "cuMulticastAddDevice", err);
}

bool pool_bind(Pool& P, std::string* err) {
  Drv& d = drv(err);
  if (!cu(d.mc_bind(P.mc, 0, P.phys, 0, P.bytes, 0), "cuMulticastBindMem", err)) return false;
  if (!map_handle(P.mc, P.bytes, P.align, P.dev, &P.mcva, err)) return false;
  if (cudaMemset(P.uc, 0, kPoolFlagBytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    *err = "pool flag reset failed";
    return false;
  }
  P.used = kPoolFlagBytes;
  P.up = true;
  return true;
}

void pool_destroy(Pool& P) {
  Drv& d = drv(nullptr);
  if (d.ok) {
    cudaDeviceSynchronize();
    auto drop = [&](char* va) {
      if (va) {
        d.unmap((CUdeviceptr)(uintptr_t)va, P.bytes);
        d.free_va((CUdeviceptr)(uintptr_t)va, P.bytes);
      }
    };
    drop(P.mcva);
    for (int q = 0; q < (int)P.peer.size(); ++q)
      if (q != P.rank) drop(P.peer[q]);
    drop(P.uc);
    if (P.mc && P.up) {
      CUdevice cd;
      if (d.dev_get(&cd, P.dev) == CUDA_SUCCESS) d.mc_unbind(P.mc, cd, 0, P.bytes);
    }
    for (auto h : P.peer_phys)
      if (h) d.release(h);
    if (P.mc) d.release(P.mc);
    if (P.phys) d.release(P.phys);
  }
  if (P.fd_phys >= 0) close(P.fd_phys);
  if (P.fd_mc >= 0) close(P.fd_mc);
  if (P.listener >= 0) close(P.listener);
  P = Pool();
}

}  // namespace taccl
