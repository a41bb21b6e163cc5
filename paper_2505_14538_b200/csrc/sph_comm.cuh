// sph_comm.cuh -- rank-to-rank transport of the slab decomposition.
//
// Two implementations of one interface:
//  - NCCL (one process per GPU over NVLink/NVSwitch): grouped ncclSend/ncclRecv between slab
//    neighbours and ncclAllReduce for the global scalars; libnccl.so.2 is opened at run time
//    (the copy torch already loaded, when there is one), so single-GPU use needs no NCCL.
//  - loopback (several contexts in ONE process, one host thread each, same device): the same
//    exchanges as device-to-device copies ordered by CUDA events, used to test the multi-rank
//    path on a single GPU.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace sph {

struct Xfer {
  int peer;     // rank
  void* buf;    // device buffer (send: source, recv: destination)
  size_t bytes; // 0 = no message
};

enum ReduceOp { kSum = 0, kMax = 1, kMin = 2 };

class Comm {
 public:
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // All sends and receives of one exchange step, enqueued on `st` (returns "" or an error).
  // Both sides must agree on which messages exist (sizes are exchanged beforehand).
  virtual std::string exchange(const Xfer* sends, int ns, const Xfer* recvs, int nr, cudaStream_t st) = 0;
  // In-place allreduce of host scalars; synchronises `st`.
  virtual std::string allreduce(double* v, int n, ReduceOp op, cudaStream_t st) = 0;
  // In-place allreduce of n uint32 values in DEVICE memory, enqueued on `st` (NCCL: no host
  // synchronisation; the caller's next read-back of the values is the only one).
  virtual std::string allreduce_dev_u32(uint32_t* d, int n, ReduceOp op, cudaStream_t st) = 0;
  // Peer memory (halo put): every rank passes the same buffer of its own (`mine`,
  // the base of a cudaMalloc allocation) and gets the corresponding buffers of the ranks `left`
  // and `right` as addresses its kernels can store to (NCCL: CUDA IPC handles exchanged with
  // the neighbours, opened with peer access over NVLink; loopback: the other contexts'
  // pointers; a rank that is its own neighbour gets `mine`).  Collective; the mappings live as
  // long as the Comm.
  virtual std::string map_peer(void* mine, int left, int right, void** left_out, void** right_out,
                               cudaStream_t st) = 0;
};

Comm* make_nccl_comm(const void* unique_id, int rank, int nranks, std::string& err);
Comm* make_loopback_comm(void* group, int rank, std::string& err);
void* loopback_group_create(int nranks);
void loopback_group_destroy(void* group);
std::string nccl_unique_id(void* out128);

}  // namespace sph
