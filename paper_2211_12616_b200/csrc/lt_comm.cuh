// lt_comm.cuh — internal interface of lt_comm.cu (NCCL, resolved at run time).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace lt_comm {

// NCCL version code (e.g. 22809); -1 with *err set when NCCL cannot be loaded
int version(int* v, std::string* err);

// ncclBroadcast of `bytes` from bufs[root] into every bufs[i], rank i on
// devices[i] (distinct GPUs) enqueued on streams[i], in one NCCL group; the
// communicator of this device list is created on first use and cached
int broadcast(const std::vector<int>& devices, const std::vector<void*>& bufs, size_t bytes,
              int root, const std::vector<cudaStream_t>& streams, std::string* err);

// the same with a separate send buffer on the root (rank 0)
int broadcast_from(const std::vector<int>& devices, const void* send,
                   const std::vector<void*>& recv, size_t bytes,
                   const std::vector<cudaStream_t>& streams, std::string* err);

// number of NCCL ranks (communicators) created so far in this process
int communicators(std::string* err);

}  // namespace lt_comm
