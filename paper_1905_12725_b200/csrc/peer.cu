// peer.cu — peer-memory exchange windows and the device barrier (see peer.cuh).
#include "peer.cuh"

#include <cudaTypedefs.h>
#include <errno.h>
#include <poll.h>
#include <stddef.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <thread>

// ------------------------------------------------------------------ fd all-gather (host)
namespace {

socklen_t abstract_addr(sockaddr_un* a, const std::string& name) {
  memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  const size_t n = std::min(name.size(), sizeof(a->sun_path) - 2);
  memcpy(a->sun_path + 1, name.data(), n);  // sun_path[0] = 0: abstract namespace
  return (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

std::string sock_name(const std::string& tag, int rank) { return "dbfft-" + tag + "-" + std::to_string(rank); }

long long now_ms() {
  return std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

// Credentials of the process at the other end of a connected AF_UNIX socket must be this user's:
// abstract-namespace names carry no file permissions, so any local process could bind a rank's
// name first or connect and pose as a rank.
static bool peer_is_same_user(int sock) {
  ucred cr;
  socklen_t len = sizeof(cr);
  if (getsockopt(sock, SOL_SOCKET, SO_PEERCRED, &cr, &len) != 0 || len != sizeof(cr)) return false;
  return cr.uid == getuid();
}

// close every descriptor carried by the SCM_RIGHTS messages of m
static void close_cmsg_fds(msghdr* m) {
  for (cmsghdr* cm = CMSG_FIRSTHDR(m); cm; cm = CMSG_NXTHDR(m, cm)) {
    if (cm->cmsg_level != SOL_SOCKET || cm->cmsg_type != SCM_RIGHTS) continue;
    const size_t n = (cm->cmsg_len - CMSG_LEN(0)) / sizeof(int);
    int* f = reinterpret_cast<int*>(CMSG_DATA(cm));
    for (size_t i = 0; i < n; ++i) close(f[i]);
  }
}

int fd_allgather(const std::string& tag, int rank, int P, const int* fds, int nfd, int* out, int timeout_ms,
                 std::string* err) {
  for (int i = 0; i < nfd; ++i) out[rank * nfd + i] = fds[i];
  if (P == 1) return 0;
  if (nfd < 1 || nfd > 16) {
    *err = "fd_allgather: 1..16 descriptors";
    return -1;
  }
  const long long deadline = now_ms() + timeout_ms;
  std::vector<char> have(P, 0);  // peers whose descriptors arrived (each exactly once)
  auto fail = [&](const std::string& what, int ls) {
    *err = "fd_allgather: " + what + " (" + strerror(errno) + ")";
    if (ls >= 0) close(ls);
    for (int d = 0; d < P; ++d)  // received descriptors are owned here until success
      if (d != rank && have[d])
        for (int i = 0; i < nfd; ++i) close(out[d * nfd + i]);
    return -1;
  };
  int ls = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (ls < 0) return fail("socket", -1);
  sockaddr_un addr;
  socklen_t alen = abstract_addr(&addr, sock_name(tag, rank));
  if (bind(ls, (sockaddr*)&addr, alen) != 0) return fail("bind " + sock_name(tag, rank), ls);
  if (listen(ls, 2 * P) != 0) return fail("listen", ls);
  // send ours to every peer (connect succeeds as soon as the peer listens; the message waits in
  // its backlog until it accepts, so every rank can send before it receives)
  for (int d = 0; d < P; ++d) {
    if (d == rank) continue;
    int c = -1;
    for (;;) {
      c = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
      if (c < 0) return fail("socket", ls);
      sockaddr_un pa;
      socklen_t plen = abstract_addr(&pa, sock_name(tag, d));
      if (connect(c, (sockaddr*)&pa, plen) == 0) break;
      close(c);
      if (now_ms() > deadline) return fail("connect to rank " + std::to_string(d) + " timed out", ls);
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    if (!peer_is_same_user(c)) {  // never hand our memory to a listener of another user
      close(c);
      errno = EPERM;
      return fail("listener of rank " + std::to_string(d) + " belongs to another user", ls);
    }
    int32_t me = rank;
    iovec iov{&me, sizeof(me)};
    alignas(cmsghdr) char ctl[CMSG_SPACE(16 * sizeof(int))];
    memset(ctl, 0, sizeof(ctl));
    msghdr m;
    memset(&m, 0, sizeof(m));
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = ctl;
    m.msg_controllen = CMSG_SPACE(nfd * sizeof(int));
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(nfd * sizeof(int));
    memcpy(CMSG_DATA(cm), fds, nfd * sizeof(int));
    const ssize_t w = sendmsg(c, &m, MSG_NOSIGNAL);
    close(c);
    if (w != (ssize_t)sizeof(me)) return fail("sendmsg to rank " + std::to_string(d), ls);
  }
  // receive every peer's: connections from other users, malformed messages and repeated ranks are
  // dropped (their descriptors closed) and waiting continues until every rank arrived or timeout
  int got = 0;
  while (got < P - 1) {
    pollfd pf{ls, POLLIN, 0};
    const long long left = deadline - now_ms();
    if (left <= 0 || poll(&pf, 1, (int)left) != 1) {
      errno = ETIMEDOUT;
      return fail("accept timed out (" + std::to_string(got) + " of " + std::to_string(P - 1) + " peers)", ls);
    }
    int a = accept4(ls, nullptr, nullptr, SOCK_CLOEXEC);
    if (a < 0) return fail("accept", ls);
    if (!peer_is_same_user(a)) {
      close(a);
      continue;
    }
    int32_t src = -1;
    iovec iov{&src, sizeof(src)};
    alignas(cmsghdr) char ctl[CMSG_SPACE(16 * sizeof(int))];
    msghdr m;
    memset(&m, 0, sizeof(m));
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = ctl;
    m.msg_controllen = sizeof(ctl);
    const ssize_t r = recvmsg(a, &m, MSG_CMSG_CLOEXEC);
    close(a);
    cmsghdr* cm = r >= 0 ? CMSG_FIRSTHDR(&m) : nullptr;
    const bool ok = r == (ssize_t)sizeof(src) && !(m.msg_flags & MSG_CTRUNC) && src >= 0 && src < P && src != rank &&
                    !have[src] && cm && cm->cmsg_level == SOL_SOCKET && cm->cmsg_type == SCM_RIGHTS &&
                    cm->cmsg_len == CMSG_LEN(nfd * sizeof(int)) && !CMSG_NXTHDR(&m, cm);
    if (!ok) {
      if (r >= 0) close_cmsg_fds(&m);
      continue;
    }
    memcpy(out + src * nfd, CMSG_DATA(cm), nfd * sizeof(int));
    have[src] = 1;
    ++got;
  }
  close(ls);
  return 0;
}

// ------------------------------------------------------------------ CUDA VMM (driver API)
namespace {

struct Vmm {
  PFN_cuMemCreate_v10020 create = nullptr;
  PFN_cuMemRelease_v10020 release = nullptr;
  PFN_cuMemAddressReserve_v10020 reserve = nullptr;
  PFN_cuMemAddressFree_v10020 addr_free = nullptr;
  PFN_cuMemMap_v10020 map = nullptr;
  PFN_cuMemUnmap_v10020 unmap = nullptr;
  PFN_cuMemSetAccess_v10020 set_access = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 gran = nullptr;
  PFN_cuMemExportToShareableHandle_v10020 export_h = nullptr;
  PFN_cuMemImportFromShareableHandle_v10020 import_h = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  *fn = (F)p;
  return true;
}

const Vmm& vmm() {
  static Vmm v;
  static bool tried = false;
  if (!tried) {
    tried = true;
    v.ok = entry("cuMemCreate", &v.create) && entry("cuMemRelease", &v.release) &&
           entry("cuMemAddressReserve", &v.reserve) && entry("cuMemAddressFree", &v.addr_free) &&
           entry("cuMemMap", &v.map) && entry("cuMemUnmap", &v.unmap) && entry("cuMemSetAccess", &v.set_access) &&
           entry("cuMemGetAllocationGranularity", &v.gran) &&
           entry("cuMemExportToShareableHandle", &v.export_h) &&
           entry("cuMemImportFromShareableHandle", &v.import_h);
  }
  return v;
}

CUmemAllocationProp prop_for(int device, bool exportable) {
  CUmemAllocationProp p;
  memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = exportable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  return p;
}

bool cu_ok(CUresult r, const char* what, std::string* err) {
  if (r == CUDA_SUCCESS) return true;
  *err = std::string("peer windows: ") + what + " failed (CUresult " + std::to_string((int)r) + ")";
  return false;
}

// reserve `bytes` of VA, map pieces, grant this device read/write
bool map_range(PeerBuf* b, size_t bytes, int device, CUdeviceptr* out, const std::vector<CUmemGenericAllocationHandle>& pieces,
               size_t piece, std::string* err) {
  const Vmm& v = vmm();
  CUdeviceptr va = 0;
  if (!cu_ok(v.reserve(&va, bytes, 0, 0, 0), "cuMemAddressReserve", err)) return false;
  b->va.push_back({va, bytes});
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (size_t i = 0; i < pieces.size(); ++i) {
    if (!cu_ok(v.map(va + i * piece, piece, 0, pieces[i], 0), "cuMemMap", err)) return false;
    b->maps.push_back({va + i * piece, piece});
    if (!cu_ok(v.set_access(va + i * piece, piece, &acc, 1), "cuMemSetAccess", err)) return false;
  }
  *out = va;
  return true;
}

}  // namespace

size_t peer_chunk(size_t bytes, int device, std::string* err) {
  const Vmm& v = vmm();
  if (!v.ok) {
    *err = "peer windows: CUDA VMM driver entry points unavailable";
    return 0;
  }
  CUmemAllocationProp p = prop_for(device, false);
  size_t g = 0;
  if (!cu_ok(v.gran(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity", err)) return 0;
  return std::max<size_t>(g, (bytes + g - 1) / g * g);
}

// cuMemMap maps whole allocations only (offset 0), so every chunk is an allocation of its own:
// a receive buffer is P chunk allocations mapped back to back, a window maps chunk `rank` of
// every rank's buffer
bool peer_build_loopback(PeerBuf* b, int P, size_t chunk, int device, bool by_rank, bool zero, std::string* err) {
  const Vmm& v = vmm();
  b->P = P;
  b->chunk = chunk;
  const int nch = by_rank ? P : 1;
  CUmemAllocationProp p = prop_for(device, false);
  std::vector<std::vector<CUmemGenericAllocationHandle>> ph(P, std::vector<CUmemGenericAllocationHandle>(nch));
  for (int d = 0; d < P; ++d)
    for (int c = 0; c < nch; ++c) {
      if (!cu_ok(v.create(&ph[d][c], chunk, &p, 0), "cuMemCreate", err)) return false;
      b->phys.push_back(ph[d][c]);
    }
  for (int k = 0; k < P; ++k) {
    CUdeviceptr r = 0, w = 0;
    if (!map_range(b, (size_t)nch * chunk, device, &r, ph[k], chunk, err)) return false;
    std::vector<CUmemGenericAllocationHandle> pieces;
    for (int d = 0; d < P; ++d) pieces.push_back(ph[d][by_rank ? k : 0]);
    if (!map_range(b, (size_t)P * chunk, device, &w, pieces, chunk, err)) return false;
    if (zero && cudaMemset((void*)r, 0, (size_t)nch * chunk) != cudaSuccess) {
      *err = "peer windows: cudaMemset";
      return false;
    }
    b->recv.push_back(r);
    b->win.push_back(w);
  }
  return true;
}

bool peer_build_ipc(PeerBuf* b, int P, int rank, size_t chunk, int device, bool by_rank, bool zero,
                    const std::string& tag, std::string* err) {
  const Vmm& v = vmm();
  b->P = P;
  b->chunk = chunk;
  const int nch = by_rank ? P : 1;
  CUmemAllocationProp p = prop_for(device, true);
  std::vector<CUmemGenericAllocationHandle> own(nch);
  for (int c = 0; c < nch; ++c) {
    if (!cu_ok(v.create(&own[c], chunk, &p, 0), "cuMemCreate (exportable)", err)) return false;
    b->phys.push_back(own[c]);
  }
  CUdeviceptr r = 0, w = 0;
  if (!map_range(b, (size_t)nch * chunk, device, &r, own, chunk, err)) return false;
  // zeroed before this rank's descriptors are sent: a peer can only store into it after receiving them
  if (zero && (cudaMemset((void*)r, 0, (size_t)nch * chunk) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)) {
    *err = "peer windows: cudaMemset";
    return false;
  }
  std::vector<int> fds(nch, -1), all((size_t)P * nch, -1);
  for (int c = 0; c < nch; ++c)
    if (!cu_ok(v.export_h(&fds[c], own[c], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle",
               err))
      return false;
  const int rc = fd_allgather(tag, rank, P, fds.data(), nch, all.data(), 120000, err);
  for (int c = 0; c < nch; ++c) close(fds[c]);
  if (rc != 0) return false;
  std::vector<CUmemGenericAllocationHandle> pieces(P);
  bool ok = true;
  for (int d = 0; d < P; ++d) {
    if (d == rank) {
      pieces[d] = own[by_rank ? rank : 0];
      continue;
    }
    // only chunk `rank` of rank d's buffer is needed here
    if (ok) {
      ok = cu_ok(v.import_h(&pieces[d], (void*)(uintptr_t)all[d * nch + (by_rank ? rank : 0)],
                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                 "cuMemImportFromShareableHandle", err);
      if (ok) b->phys.push_back(pieces[d]);
    }
    for (int c = 0; c < nch; ++c) close(all[d * nch + c]);
  }
  if (!ok) return false;
  if (!map_range(b, (size_t)P * chunk, device, &w, pieces, chunk, err)) return false;
  b->recv.push_back(r);
  b->win.push_back(w);
  return true;
}

void peer_free(PeerBuf* b) {
  const Vmm& v = vmm();
  if (!v.ok) return;
  for (auto& m : b->maps) v.unmap(m.first, m.second);
  for (auto& r : b->va) v.addr_free(r.first, r.second);
  for (auto h : b->phys) v.release(h);
  *b = PeerBuf();
}

// ------------------------------------------------------------------ device barrier
// epoch: a per-rank device counter at flags[kEpochWord] (peers only write the words 32 r, r < 32),
// advanced by every barrier in stream order, so a replayed CUDA graph issues fresh epochs; all
// ranks run the same barrier sequence, so their counters agree
constexpr int kEpochWord = 32 * 32;
__global__ void k_peer_barrier(unsigned* flags, char* fwin, size_t chunk, int P, int rank) {
  const int j = threadIdx.x;
  unsigned epoch = 0;
  if (j == 0) {
    epoch = flags[kEpochWord] + 1;
    flags[kEpochWord] = epoch;
  }
  epoch = __shfl_sync(0xffffffffu, epoch, 0);
  if (j >= P) return;
  // the preceding kernels' stores (including those into peer memory) before the arrival
  asm volatile("fence.sc.sys;" ::: "memory");
  unsigned* slot = reinterpret_cast<unsigned*>(fwin + (size_t)j * chunk) + 32 * rank;
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
  const unsigned* mine = flags + 32 * j;
  unsigned seen;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(mine) : "memory");
    if ((int)(seen - epoch) >= 0) break;
    __nanosleep(64);
  }
}

cudaError_t launch_peer_barrier(unsigned* flags, char* fwin, size_t chunk, int P, int rank, cudaStream_t s) {
  k_peer_barrier<<<1, 32, 0, s>>>(flags, fwin, chunk, P, rank);
  return cudaGetLastError();
}
