// peer.cuh — peer-memory exchange windows (SURVEY 8(e) / 8(f3), K11 of SURVEY 2.4).
//
// The two all-to-alls of an operator application (after I1 and after F2) move the
// rank-chunked output of a column pass: rank r's pass writes chunk d of its output
// ([d][f][ky_loc][z_loc][kx], chunk stride pcs) and rank d reads chunk r of its receive buffer
// ([r][f][ky_loc][z_loc][kx]).  A *window* is a virtual range of P chunks per rank whose chunk d
// is mapped (CUDA VMM) onto rank d's receive buffer at chunk r: the pass stores its chunk d
// straight into rank d's memory over NVLink — no send buffer, no copy, no NCCL exchange, and the
// transfer overlaps the pass's own arithmetic tile by tile.  The column kernels are unchanged:
// the window is just the `out` pointer with pcs = the padded chunk stride.
//
// Physical buffers are cuMemCreate allocations of P chunks (chunk padded to the allocation
// granularity so that every chunk can be mapped separately).  Loopback (P virtual ranks in one
// process, one GPU) maps every rank's window onto the other slabs' buffers on the same device;
// the NCCL mode exports each rank's buffer as a POSIX file descriptor, passes the descriptors
// between the rank processes over abstract Unix sockets (SCM_RIGHTS) and imports them.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>
#include <vector>

// All-gather of nfd file descriptors among P processes on one node: out[src * nfd + i] receives a
// descriptor (a dup in this process) for process src's fds[i]; out[rank * nfd + i] = fds[i].  The
// rendezvous is the abstract socket "\0dbfft-<tag>-<rank>"; the tag must be unique per
// concurrent exchange and equal on all ranks.  Returns 0, or -1 with *err set (timeout_ms).
int fd_allgather(const std::string& tag, int rank, int P, const int* fds, int nfd, int* out, int timeout_ms,
                 std::string* err);

struct PeerBuf {
  size_t chunk = 0;                                 // padded chunk bytes
  int P = 0;
  std::vector<CUmemGenericAllocationHandle> phys;   // created (and imported) physical buffers
  std::vector<CUdeviceptr> recv, win;               // per local slab: its receive buffer, its window
  std::vector<std::pair<CUdeviceptr, size_t>> va;   // reserved ranges
  std::vector<std::pair<CUdeviceptr, size_t>> maps; // mapped pieces (one allocation each)
};

// granularity-padded chunk size for `bytes`
size_t peer_chunk(size_t bytes, int device, std::string* err);
// loopback: P receive buffers of P chunks on `device`; window k maps its chunk d onto buffer d,
// chunk k (by_rank) or onto one-chunk buffer d (!by_rank: flags); zero: memset 0.  Every chunk is
// an allocation of its own (cuMemMap maps whole allocations).
bool peer_build_loopback(PeerBuf* b, int P, size_t chunk, int device, bool by_rank, bool zero, std::string* err);
// NCCL mode: this rank's buffer (zeroed before it is shared when `zero`), exported, exchanged with
// fd_allgather(tag), the peers' buffers imported
bool peer_build_ipc(PeerBuf* b, int P, int rank, size_t chunk, int device, bool by_rank, bool zero,
                    const std::string& tag, std::string* err);
void peer_free(PeerBuf* b);

// device barrier among the P ranks of a peer set: every rank advances its device-side epoch
// counter, stores the epoch into its slot of every rank's flag buffer (release, system scope) and
// waits until all P slots of its own buffer reached it (acquire).  flags: this rank's own flag
// buffer (zeroed; word 1024 holds the counter); fwin: the flag window (chunk stride `chunk`).
cudaError_t launch_peer_barrier(unsigned* flags, char* fwin, size_t chunk, int P, int rank, cudaStream_t s);
