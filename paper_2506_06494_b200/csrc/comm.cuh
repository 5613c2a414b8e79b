// Collective back-ends of the partitioned solve (context.cuh: Comm).
#pragma once
#include <nccl.h>

#include "../../include/jgs2.h"
#include "context.cuh"

namespace jgs2 {

#define JGS2_NCCL(call)                                                                    \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      throw ::jgs2::Error(-2, std::string(#call) + ": " + ncclGetErrorString(r_));         \
  } while (0)

// NCCL over NVLink / NVSwitch: in-place all-reduce on the context stream
// (stream-ordered with the sweep kernels, no host sync).
struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  bool owned = false;
  ~NcclComm() override {
    if (owned && c) ncclCommDestroy(c);
  }
  void allreduce(void* buf, size_t count, int type, int op, cudaStream_t s) override {
    ncclDataType_t t = type == CT_F64 ? ncclFloat64 : (type == CT_I32 ? ncclInt32 : ncclUint64);
    JGS2_NCCL(ncclAllReduce(buf, buf, count, t, op == CO_SUM ? ncclSum : ncclMax, c, s));
  }
};

// Host callback (e.g. torch.distributed over gloo): the buffer goes to
// pinned host memory, the callback reduces it in place across ranks, and it
// comes back. For multi-process tests where ranks share one GPU.
struct HostComm : Comm {
  jgs2_allreduce_fn fn = nullptr;
  void* user = nullptr;
  void* host = nullptr;
  size_t host_bytes = 0;
  ~HostComm() override {
    if (host) cudaFreeHost(host);
  }
  void allreduce(void* buf, size_t count, int type, int op, cudaStream_t s) override {
    size_t bytes = count * (type == CT_I32 ? 4 : 8);
    if (bytes > host_bytes) {
      if (host) cudaFreeHost(host);
      host = nullptr;
      JGS2_CUDA(cudaMallocHost(&host, bytes));
      host_bytes = bytes;
    }
    JGS2_CUDA(cudaMemcpyAsync(host, buf, bytes, cudaMemcpyDeviceToHost, s));
    JGS2_CUDA(cudaStreamSynchronize(s));
    if (fn(host, (int64_t)count, type, op, user) != 0) throw Error(-2, "host all-reduce callback failed");
    JGS2_CUDA(cudaMemcpyAsync(buf, host, bytes, cudaMemcpyHostToDevice, s));
  }
};

}  // namespace jgs2
