// comm.cu — loopback (emulated ranks) and NCCL implementations of pcal::Comm.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "comm.h"
#include "common.cuh"

namespace pcal {

// ---- loopback ---------------------------------------------------------------------
LoopbackGroup::LoopbackGroup(int n) : size(n), a(n), b(n), c(n), d(n) {
  PCAL_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
}
LoopbackGroup::~LoopbackGroup() {
  if (tmp) cudaFree(tmp);
  if (stream) cudaStreamDestroy(stream);
}

void LoopbackGroup::arrive_and_wait() {
  std::unique_lock<std::mutex> lk(mu_);
  const uint64_t gen = generation_;
  if (++waiting_ == size) {
    waiting_ = 0;
    ++generation_;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return generation_ != gen; });
  }
}

// out[i] = Σ_r in_r[i] in rank order (deterministic)
__global__ void k_lb_sum(const double* const* in, int nr, size_t count, double* out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int r = 0; r < nr; ++r) s += in[r][i];
  out[i] = s;
}

void LoopbackComm::allreduce(double* buf, size_t count, cudaStream_t st) {
  g_->c[rank] = buf;
  g_->arrive_and_wait();  // every rank's preceding kernels are enqueued
  if (rank == 0) {
    if (g_->tmp_count < count) {
      if (g_->tmp) cudaFree(g_->tmp);
      PCAL_CUDA(cudaMalloc(&g_->tmp, sizeof(double) * count));
      g_->tmp_count = count;
    }
    double** ptrs = nullptr;
    PCAL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptrs), sizeof(double*) * size, st));
    PCAL_CUDA(cudaMemcpyAsync(ptrs, g_->c.data(), sizeof(double*) * size, cudaMemcpyHostToDevice, st));
    k_lb_sum<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(ptrs, size, count, g_->tmp);
    launched("k_lb_sum");
    for (int r = 0; r < size; ++r)
      PCAL_CUDA(cudaMemcpyAsync(g_->c[r], g_->tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice,
                                st));
    PCAL_CUDA(cudaFreeAsync(ptrs, st));
    PCAL_CUDA(cudaStreamSynchronize(st));  // the pointer table lives on the host
  }
  g_->arrive_and_wait();  // nobody enqueues past the collective before it is enqueued
}

void LoopbackComm::allgather(const double* send, double* recv, size_t count, cudaStream_t st) {
  g_->a[rank] = send;
  g_->c[rank] = recv;
  g_->arrive_and_wait();
  if (rank == 0)
    for (int r = 0; r < size; ++r)
      for (int q = 0; q < size; ++q)
        PCAL_CUDA(cudaMemcpyAsync(g_->c[r] + (size_t)q * count, g_->a[q], sizeof(double) * count,
                                  cudaMemcpyDeviceToDevice, st));
  g_->arrive_and_wait();
}

void LoopbackComm::halo(const double* send_lo, const double* send_hi, double* recv_lo,
                        double* recv_hi, size_t count, cudaStream_t st) {
  g_->a[rank] = send_lo;
  g_->b[rank] = send_hi;
  g_->c[rank] = recv_lo;
  g_->d[rank] = recv_hi;
  g_->arrive_and_wait();
  if (rank == 0)
    for (int r = 0; r < size; ++r) {
      const int lo = (r + size - 1) % size, hi = (r + 1) % size;
      PCAL_CUDA(cudaMemcpyAsync(g_->c[r], g_->b[lo], sizeof(double) * count,
                                cudaMemcpyDeviceToDevice, st));
      PCAL_CUDA(cudaMemcpyAsync(g_->d[r], g_->a[hi], sizeof(double) * count,
                                cudaMemcpyDeviceToDevice, st));
    }
  g_->arrive_and_wait();
}

// ---- NCCL (dlopen'd) --------------------------------------------------------------------
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
  bool load() {
    if (h) return true;
    // prefer an already-loaded NCCL (e.g. torch's), else the system one
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
      return false;
    }
#define LOAD(name) *reinterpret_cast<void**>(&name) = dlsym(h, "nccl" #name)
    LOAD(GetUniqueId);
    LOAD(CommInitRank);
    LOAD(CommDestroy);
    LOAD(AllReduce);
    LOAD(AllGather);
    LOAD(Send);
    LOAD(Recv);
    LOAD(GroupStart);
    LOAD(GroupEnd);
    LOAD(GetErrorString);
#undef LOAD
    if (!GetUniqueId || !CommInitRank || !AllReduce || !AllGather || !Send || !Recv) {
      err = "libnccl.so.2 lacks required symbols";
      return false;
    }
    return true;
  }
};
NcclApi& api() {
  static NcclApi a;
  return a;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(-5, std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(r) : "nccl error"));
}

class NcclComm : public Comm {
 public:
  NcclComm(int n, int r, const void* uid, int device) {
    rank = r;
    size = n;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    PCAL_CUDA(cudaSetDevice(device));
    nccl_check(api().CommInitRank(&comm_, n, id, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_ && api().CommDestroy) api().CommDestroy(comm_);
  }
  void allreduce(double* buf, size_t count, cudaStream_t st) override {
    nccl_check(api().AllReduce(buf, buf, count, ncclDouble, ncclSum, comm_, st), "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    nccl_check(api().AllGather(send, recv, count, ncclDouble, comm_, st), "ncclAllGather");
  }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi,
            size_t count, cudaStream_t st) override {
    const int lo = (rank + size - 1) % size, hi = (rank + 1) % size;
    nccl_check(api().GroupStart(), "ncclGroupStart");
    nccl_check(api().Send(send_lo, count, ncclDouble, lo, comm_, st), "ncclSend");
    nccl_check(api().Recv(recv_hi, count, ncclDouble, hi, comm_, st), "ncclRecv");
    nccl_check(api().Send(send_hi, count, ncclDouble, hi, comm_, st), "ncclSend");
    nccl_check(api().Recv(recv_lo, count, ncclDouble, lo, comm_, st), "ncclRecv");
    nccl_check(api().GroupEnd(), "ncclGroupEnd");
  }

 private:
  ncclComm_t comm_ = nullptr;
};
}  // namespace

bool nccl_available(std::string* why) {
  const bool ok = api().load();
  if (!ok && why) *why = api().err;
  return ok;
}

void nccl_unique_id(void* out) {
  if (!api().load()) throw Error(-4, "NCCL unavailable: " + api().err);
  ncclUniqueId id;
  nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

Comm* make_nccl_comm(int nranks, int rank, const void* uid, int device) {
  if (!api().load()) throw Error(-4, "NCCL unavailable: " + api().err);
  return new NcclComm(nranks, rank, uid, device);
}

}  // namespace pcal
