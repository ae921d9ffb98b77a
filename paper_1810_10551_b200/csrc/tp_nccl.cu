// Result gather over NVLink / NVSwitch: the one collective on the data path.
//
// Replaces the reference's result collection from its workers: evaluate_remote
// (pkg/src/tilepipe/distribution/client.py:176-203) merges every worker's crop-local
// detections into one dict, and run_remote_frame / run_stream (client.py:242-377) hand
// the frame's results back in frame order. Here every rank holds a padded, fixed-size
// slice of records (crop-parallel stage 2: raw detection records per tile; frame-parallel
// runs: merged per-frame records) and counts; both are all-gathered in rank order inside
// ONE ncclGroupStart/End on the caller's stream, so the records and their counts travel
// in a single fused NCCL launch.
//
// The communicator is borrowed, never created: torch.distributed owns it and hands its
// ncclComm_t over (ProcessGroupNCCL._comm_ptr()). NCCL is resolved at run time from the
// libnccl.so.2 the process already loaded (torch's), so both sides use the same library
// instance and this shared library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <mutex>

#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

// nccl.h (2.x) values: ncclUint8 = 1, ncclInt32 = 2, ncclSuccess = 0, ncclInProgress = 7
// (returned by non-blocking communicators, e.g. TORCH_NCCL_USE_COMM_NONBLOCKING=1).
constexpr int kNcclUint8 = 1;
constexpr int kNcclInt32 = 2;
constexpr int kNcclInProgress = 7;

using AllGatherFn = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
using GroupFn = int (*)();
using ErrorStringFn = const char* (*)(int);
using AsyncErrorFn = int (*)(void*, int*);

struct NcclApi {
  AllGatherFn all_gather = nullptr;
  GroupFn group_start = nullptr, group_end = nullptr;
  ErrorStringFn error_string = nullptr;
  AsyncErrorFn async_error = nullptr;
  bool ok = false;
};

// A non-blocking communicator answers ncclInProgress until the enqueue completes: poll
// ncclCommGetAsyncError until it settles (success or a real error).
int settle(const NcclApi& api, void* comm, int rc) {
  if (rc != kNcclInProgress) return rc;
  if (api.async_error == nullptr) return rc;
  int state = kNcclInProgress;
  while (true) {
    const int q = api.async_error(comm, &state);
    if (q != 0) return q;
    if (state != kNcclInProgress) return state;
  }
}

const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy torch already mapped first; a fresh load only if none is resident
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    api.all_gather = reinterpret_cast<AllGatherFn>(dlsym(h, "ncclAllGather"));
    api.group_start = reinterpret_cast<GroupFn>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<GroupFn>(dlsym(h, "ncclGroupEnd"));
    api.error_string = reinterpret_cast<ErrorStringFn>(dlsym(h, "ncclGetErrorString"));
    api.async_error = reinterpret_cast<AsyncErrorFn>(dlsym(h, "ncclCommGetAsyncError"));
    api.ok = api.all_gather && api.group_start && api.group_end;
  });
  return api;
}

}  // namespace

extern "C" int tp_nccl_available(void) { return nccl_api().ok ? 1 : 0; }

extern "C" int tp_nccl_gather_dets(void* nccl_comm, const void* local_recs,
                                   int64_t rec_bytes_per_rank, const int32_t* local_counts,
                                   int64_t counts_per_rank, void* all_recs, int32_t* all_counts,
                                   void* stream) {
  if (nccl_comm == nullptr || rec_bytes_per_rank < 0 || counts_per_rank < 0 ||
      (rec_bytes_per_rank > 0 && (local_recs == nullptr || all_recs == nullptr)) ||
      (counts_per_rank > 0 && (local_counts == nullptr || all_counts == nullptr))) {
    tp_set_error("tp_nccl_gather_dets: bad argument");
    return TP_ERR_ARG;
  }
  const NcclApi& api = nccl_api();
  if (!api.ok) {
    tp_set_error("tp_nccl_gather_dets: libnccl.so.2 is not loadable (no NCCL in this process)");
    return TP_ERR_CUDA;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int rc = api.group_start();
  if ((rc == 0 || rc == kNcclInProgress) && rec_bytes_per_rank > 0)
    rc = api.all_gather(local_recs, all_recs, (size_t)rec_bytes_per_rank, kNcclUint8, nccl_comm, s);
  if ((rc == 0 || rc == kNcclInProgress) && counts_per_rank > 0)
    rc = api.all_gather(local_counts, all_counts, (size_t)counts_per_rank, kNcclInt32, nccl_comm, s);
  const int rc_end = settle(api, nccl_comm, api.group_end());
  if (rc == 0 || rc == kNcclInProgress) rc = rc_end;
  if (rc != 0) {
    tp_set_error(api.error_string ? api.error_string(rc) : "tp_nccl_gather_dets: NCCL error");
    return TP_ERR_CUDA;
  }
  return TP_OK;
}
