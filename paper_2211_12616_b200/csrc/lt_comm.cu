// lt_comm.cu — NCCL for the met broadcast of the one-process-drives-all-GPUs
// design (arXiv 2211.12616; the reference replicates met by deep-copying both
// snapshots into every device image, driver_cli.py:146-149 ->
// device_runtime.py:178-186).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): the library links no
// NCCL, so the process uses whichever libnccl is already mapped (PyTorch's
// bundled one when torch is imported first) or the system's.  Communicators
// come from ncclCommInitAll over the participating GPUs and are cached per
// device list for the life of the process.
#include <dlfcn.h>
#include <nccl.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "lt_comm.cuh"

namespace lt_comm {
namespace {

struct Api {
  void* handle = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string load_error;
};

std::mutex g_mu;
Api g_api;
bool g_tried = false;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_comms;

template <class F>
bool sym(void* h, const char* name, F* out) {
  *out = reinterpret_cast<F>(dlsym(h, name));
  return *out != nullptr;
}

// caller holds g_mu
const Api* api(std::string* err) {
  if (!g_tried) {
    g_tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      g_api.load_error = std::string("cannot load libnccl.so.2: ") + dlerror();
    } else if (!(sym(h, "ncclCommInitAll", &g_api.CommInitAll) &&
                 sym(h, "ncclCommDestroy", &g_api.CommDestroy) &&
                 sym(h, "ncclBroadcast", &g_api.Broadcast) &&
                 sym(h, "ncclGroupStart", &g_api.GroupStart) &&
                 sym(h, "ncclGroupEnd", &g_api.GroupEnd) &&
                 sym(h, "ncclGetVersion", &g_api.GetVersion) &&
                 sym(h, "ncclGetErrorString", &g_api.GetErrorString))) {
      g_api.load_error = "libnccl.so.2 lacks a required symbol";
    } else {
      g_api.handle = h;
    }
  }
  if (!g_api.handle) {
    *err = g_api.load_error;
    return nullptr;
  }
  return &g_api;
}

int nccl_fail(const Api* a, ncclResult_t r, const char* what, std::string* err) {
  *err = std::string(what) + ": " + a->GetErrorString(r);
  return -1;
}

}  // namespace

int version(int* v, std::string* err) {
  std::lock_guard<std::mutex> lock(g_mu);
  const Api* a = api(err);
  if (!a) return -1;
  ncclResult_t r = a->GetVersion(v);
  return r == ncclSuccess ? 0 : nccl_fail(a, r, "ncclGetVersion", err);
}

namespace {
// caller holds g_mu
const std::vector<ncclComm_t>* comms_for(const Api* a, const std::vector<int>& devices,
                                         std::string* err) {
  auto it = g_comms.find(devices);
  if (it == g_comms.end()) {
    std::vector<ncclComm_t> comms(devices.size());
    ncclResult_t r = a->CommInitAll(comms.data(), static_cast<int>(devices.size()), devices.data());
    if (r != ncclSuccess) {
      nccl_fail(a, r, "ncclCommInitAll", err);
      return nullptr;
    }
    it = g_comms.emplace(devices, std::move(comms)).first;
  }
  return &it->second;
}

// one group: every rank's broadcast is enqueued on its own stream before
// any of them may start (required when one thread drives all GPUs)
int group_broadcast(const Api* a, const std::vector<ncclComm_t>& comms,
                    const std::vector<int>& devices, const void* send,
                    const std::vector<void*>& recv, size_t bytes, int root,
                    const std::vector<cudaStream_t>& streams, std::string* err) {
  ncclResult_t r = a->GroupStart();
  if (r != ncclSuccess) return nccl_fail(a, r, "ncclGroupStart", err);
  for (size_t i = 0; i < devices.size(); ++i) {
    cudaSetDevice(devices[i]);
    r = a->Broadcast(static_cast<int>(i) == root ? send : recv[i], recv[i], bytes, ncclChar, root,
                     comms[i], streams[i]);
    if (r != ncclSuccess) {
      a->GroupEnd();
      return nccl_fail(a, r, "ncclBroadcast", err);
    }
  }
  r = a->GroupEnd();
  if (r != ncclSuccess) return nccl_fail(a, r, "ncclGroupEnd", err);
  return 0;
}
}  // namespace

int broadcast(const std::vector<int>& devices, const std::vector<void*>& bufs, size_t bytes,
              int root, const std::vector<cudaStream_t>& streams, std::string* err) {
  std::lock_guard<std::mutex> lock(g_mu);
  const Api* a = api(err);
  if (!a) return -1;
  const std::vector<ncclComm_t>* comms = comms_for(a, devices, err);
  if (!comms) return -1;
  return group_broadcast(a, *comms, devices, bufs[root], bufs, bytes, root, streams, err);
}

int broadcast_from(const std::vector<int>& devices, const void* send,
                   const std::vector<void*>& recv, size_t bytes,
                   const std::vector<cudaStream_t>& streams, std::string* err) {
  std::lock_guard<std::mutex> lock(g_mu);
  const Api* a = api(err);
  if (!a) return -1;
  const std::vector<ncclComm_t>* comms = comms_for(a, devices, err);
  if (!comms) return -1;
  return group_broadcast(a, *comms, devices, send, recv, bytes, 0, streams, err);
}

int communicators(std::string* err) {
  std::lock_guard<std::mutex> lock(g_mu);
  (void)err;
  int n = 0;
  for (auto& kv : g_comms) n += static_cast<int>(kv.second.size());
  return n;
}

}  // namespace lt_comm
