// comm.h — collectives of the row-sharded PCAL iteration.
//
// Row sharding (z-slabs for the grid models): every n×p object is row-local,
// every p×p object is replicated; per iteration the ranks exchange only
//   C1  the Gram [GᵀX; XᵀX] partials (allreduce, 2pp×pp doubles),
//   C2  the per-column f / KKT² / d_j partial sums (allreduce, 3p),
//   C3  the stepsize inner-product partials (allreduce, 3·blocks),
//   C4  the column norms ‖z_j‖², ‖x_j‖² (allreduce, 2p),
//   C5  stencil z-halo planes (send/recv with the two slab neighbours), or the
//       X allgather of the dense gradient, or the ρ allgather of the KS model.
// Two implementations: NCCL (one process per GPU, NVLink/NVSwitch; loaded
// with dlopen so a single-GPU process never needs libnccl) and a loopback
// group that emulates R ranks inside one process on one GPU (all ranks share
// one stream; host threads meet at a barrier at every collective), used to
// test the sharded path where only one GPU exists.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <mutex>
#include <vector>

namespace pcal {

class Comm {
 public:
  virtual ~Comm() = default;
  int rank = 0, size = 1;
  // in-place elementwise sum over ranks
  virtual void allreduce(double* buf, size_t count, cudaStream_t st) = 0;
  // recv = [send_0 | send_1 | … ] (count doubles per rank)
  virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
  // periodic slab neighbours: recv_lo ← send_hi of rank−1, recv_hi ← send_lo of rank+1
  virtual void halo(const double* send_lo, const double* send_hi, double* recv_lo,
                    double* recv_hi, size_t count, cudaStream_t st) = 0;
  virtual bool emulated() const { return false; }
};

// ---- loopback (R ranks, one process, one GPU, one shared stream) -------------------
class LoopbackGroup {
 public:
  explicit LoopbackGroup(int size);
  ~LoopbackGroup();
  int size;
  cudaStream_t stream = nullptr;  // shared by every rank's session
  // barrier for the rank threads
  void arrive_and_wait();
  std::vector<const double*> a, b;
  std::vector<double*> c, d;
  double* tmp = nullptr;
  size_t tmp_count = 0;

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int waiting_ = 0;
  uint64_t generation_ = 0;
};

class LoopbackComm : public Comm {
 public:
  LoopbackComm(LoopbackGroup* g, int r) : g_(g) {
    rank = r;
    size = g->size;
  }
  void allreduce(double* buf, size_t count, cudaStream_t st) override;
  void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override;
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi,
            size_t count, cudaStream_t st) override;
  bool emulated() const override { return true; }

 private:
  LoopbackGroup* g_;
};

// ---- NCCL -------------------------------------------------------------------------
// Returns false (and a message) when libnccl cannot be loaded.
bool nccl_available(std::string* why);
Comm* make_nccl_comm(int nranks, int rank, const void* unique_id /* 128 B */, int device);
void nccl_unique_id(void* out /* 128 B */);

}  // namespace pcal
