// Communication layer (comm.h): NCCL over NVLink for one process per GPU, and a
// loopback hub for N virtual ranks on one GPU (tests of the partitioned path).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <thread>
#include <mutex>
#include <vector>

#include "comm.h"

namespace mgdtn {

// ============================================================================ NCCL (dlopen)
namespace {
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclCommGetAsyncError) asyncError = nullptr;   // optional
  decltype(&ncclCommAbort) abort = nullptr;                // optional
};

NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  // the process's NCCL (e.g. torch's) if already loaded, else the system one
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define LOAD(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
  LOAD(getUniqueId, "ncclGetUniqueId");
  LOAD(commInitRank, "ncclCommInitRank");
  LOAD(commDestroy, "ncclCommDestroy");
  LOAD(groupStart, "ncclGroupStart");
  LOAD(groupEnd, "ncclGroupEnd");
  LOAD(send, "ncclSend");
  LOAD(recv, "ncclRecv");
  LOAD(allReduce, "ncclAllReduce");
  LOAD(allGather, "ncclAllGather");
  LOAD(errStr, "ncclGetErrorString");
  LOAD(asyncError, "ncclCommGetAsyncError");
  LOAD(abort, "ncclCommAbort");
#undef LOAD
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart &&
           api.groupEnd && api.send && api.recv && api.allReduce && api.allGather && api.errStr;
  return api;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  int r = 0, n = 1;
  int rank() const override { return r; }
  int nranks() const override { return n; }
  ~NcclComm() override {
    if (comm) nccl_api().commDestroy(comm);
  }
  int check(ncclResult_t e, const char* what) {
    if (e == ncclSuccess) return 0;
    err = std::string(what) + ": " + nccl_api().errStr(e);
    return -1;
  }
  int halo(const int nbr[4], const double* send, double* recv, int stride, const int count[4],
           cudaStream_t st) override {
    NcclApi& a = nccl_api();
    if (check(a.groupStart(), "ncclGroupStart")) return -1;
    for (int f = 0; f < 4; ++f) {
      if (nbr[f] < 0 || count[f] == 0) continue;
      if (check(a.send(send + (size_t)f * stride, count[f], ncclDouble, nbr[f], comm, st),
                "ncclSend"))
        return -1;
      if (check(a.recv(recv + (size_t)f * stride, count[f], ncclDouble, nbr[f], comm, st),
                "ncclRecv"))
        return -1;
    }
    return check(a.groupEnd(), "ncclGroupEnd");
  }
  int allreduce_sum(double* dev, int cnt, cudaStream_t st) override {
    return check(nccl_api().allReduce(dev, dev, cnt, ncclDouble, ncclSum, comm, st),
                 "ncclAllReduce");
  }
  int allgather(const double* send, double* recv, size_t cnt, cudaStream_t st) override {
    return check(nccl_api().allGather(send, recv, cnt, ncclDouble, comm, st), "ncclAllGather");
  }
  bool capturable() const override { return true; }
  int wait(cudaStream_t st, double timeout_s) override {
    NcclApi& a = nccl_api();
    const auto t0 = std::chrono::steady_clock::now();
    int naps = 0;
    for (;;) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) return 0;
      if (q != cudaErrorNotReady) {
        err = std::string("stream: ") + cudaGetErrorString(q);
        return -1;
      }
      if (a.asyncError && comm) {
        ncclResult_t ae = ncclSuccess;
        a.asyncError(comm, &ae);
        if (ae != ncclSuccess && ae != ncclInProgress) {
          err = std::string("NCCL asynchronous error: ") + a.errStr(ae);
          abort_comm();
          return -1;
        }
      }
      const double el =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (timeout_s > 0 && el > timeout_s) {
        err = "NCCL: stream not done after " + std::to_string(timeout_s) +
              " s (peer lost?); communicator aborted";
        abort_comm();
        return -1;
      }
      // spin briefly, then back off to 50 us naps
      if (++naps > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  void abort_comm() {
    if (comm && nccl_api().abort) {
      nccl_api().abort(comm);
      comm = nullptr;
    }
  }
};
}  // namespace

int nccl_unique_id(uint8_t out[128], std::string& err) {
  NcclApi& a = nccl_api();
  if (!a.ok) {
    err = "libnccl.so.2 not found";
    return -1;
  }
  ncclUniqueId id;
  ncclResult_t e = a.getUniqueId(&id);
  if (e != ncclSuccess) {
    err = std::string("ncclGetUniqueId: ") + a.errStr(e);
    return -1;
  }
  std::memcpy(out, id.internal, 128);
  return 0;
}

Comm* make_nccl_comm(const uint8_t* id, int rank, int nranks, int device, std::string& err) {
  NcclApi& a = nccl_api();
  if (!a.ok) {
    err = "libnccl.so.2 not found";
    return nullptr;
  }
  cudaSetDevice(device);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  NcclComm* c = new NcclComm();
  c->r = rank;
  c->n = nranks;
  ncclResult_t e = a.commInitRank(&c->comm, nranks, uid, rank);
  if (e != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + a.errStr(e);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

// ============================================================================ loopback
struct LoopbackHub {
  int n = 1;
  std::mutex m;
  std::condition_variable cv;
  int count = 0;
  long long gen = 0;
  std::vector<const double*> sendp;
  std::vector<int> stride;
  std::vector<cudaEvent_t> ready, done;
  std::vector<double*> tmp;   // per-rank device scratch for all-reduce results
  std::vector<int> tmp_n;
  bool aborted = false;       // a rank failed: every barrier returns at once, ops report errors
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) return false;
    const long long g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
    }
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

void loopback_abort(LoopbackHub* h) {
  if (h) h->abort();
}

LoopbackHub* loopback_create(int nranks) {
  LoopbackHub* h = new LoopbackHub();
  h->n = nranks;
  h->sendp.assign(nranks, nullptr);
  h->stride.assign(nranks, 0);
  h->ready.resize(nranks);
  h->done.resize(nranks);
  h->tmp.assign(nranks, nullptr);
  h->tmp_n.assign(nranks, 0);
  for (int r = 0; r < nranks; ++r) {
    cudaEventCreateWithFlags(&h->ready[r], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->done[r], cudaEventDisableTiming);
  }
  return h;
}

void loopback_destroy(LoopbackHub* h) {
  if (!h) return;
  cudaDeviceSynchronize();
  for (int r = 0; r < h->n; ++r) {
    cudaEventDestroy(h->ready[r]);
    cudaEventDestroy(h->done[r]);
    if (h->tmp[r]) cudaFree(h->tmp[r]);
  }
  delete h;
}

namespace {
constexpr int LB_MAX = 64;
struct PtrList {
  const double* p[LB_MAX];
};
// out[i] = sum_r in[r][i] in rank order (every rank computes the identical sum)
__global__ void k_lb_sum(PtrList in, int nr, int n, double* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nr; ++r) s += in.p[r][i];
    out[i] = s;
  }
}

struct LoopbackComm : Comm {
  LoopbackHub* h = nullptr;
  int r = 0;
  int fail_abort() {
    err = "loopback: another rank aborted";
    return -1;
  }
  int rank() const override { return r; }
  int nranks() const override { return h->n; }
  // after every exchange: this rank's later work waits until every peer has
  // finished reading this rank's buffers
  void wait_peers_done(cudaStream_t st, bool all, const int nbr[4]) {
    if (all) {
      for (int q = 0; q < h->n; ++q)
        if (q != r) cudaStreamWaitEvent(st, h->done[q], 0);
    } else {
      for (int f = 0; f < 4; ++f)
        if (nbr[f] >= 0) cudaStreamWaitEvent(st, h->done[nbr[f]], 0);
    }
  }
  int halo(const int nbr[4], const double* send, double* recv, int stride, const int count[4],
           cudaStream_t st) override {
    h->sendp[r] = send;
    h->stride[r] = stride;
    cudaEventRecord(h->ready[r], st);
    if (!h->barrier()) return fail_abort();
    for (int f = 0; f < 4; ++f) {
      const int q = nbr[f];
      if (q < 0 || count[f] == 0) continue;
      const int g = (f + 2) & 3;   // the neighbour's matching side
      cudaStreamWaitEvent(st, h->ready[q], 0);
      cudaMemcpyAsync(recv + (size_t)f * stride, h->sendp[q] + (size_t)g * h->stride[q],
                      (size_t)count[f] * sizeof(double), cudaMemcpyDeviceToDevice, st);
    }
    cudaEventRecord(h->done[r], st);
    if (!h->barrier()) return fail_abort();
    wait_peers_done(st, false, nbr);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  int allreduce_sum(double* dev, int n, cudaStream_t st) override {
    if (h->n > LB_MAX) return -1;
    if (h->tmp_n[r] < n) {
      if (h->tmp[r]) cudaFree(h->tmp[r]);
      cudaMalloc(&h->tmp[r], (size_t)n * sizeof(double));
      h->tmp_n[r] = n;
    }
    h->sendp[r] = dev;
    cudaEventRecord(h->ready[r], st);
    if (!h->barrier()) return fail_abort();
    PtrList pl{};
    for (int q = 0; q < h->n; ++q) {
      pl.p[q] = h->sendp[q];
      if (q != r) cudaStreamWaitEvent(st, h->ready[q], 0);
    }
    k_lb_sum<<<1, 128, 0, st>>>(pl, h->n, n, h->tmp[r]);
    cudaEventRecord(h->done[r], st);
    if (!h->barrier()) return fail_abort();
    int none[4] = {-1, -1, -1, -1};
    wait_peers_done(st, true, none);
    cudaMemcpyAsync(dev, h->tmp[r], (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  int wait(cudaStream_t st, double) override {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      err = std::string("stream: ") + cudaGetErrorString(e);
      return -1;
    }
    return h->aborted ? fail_abort() : 0;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    h->sendp[r] = send;
    cudaEventRecord(h->ready[r], st);
    if (!h->barrier()) return fail_abort();
    for (int q = 0; q < h->n; ++q) {
      if (q != r) cudaStreamWaitEvent(st, h->ready[q], 0);
      cudaMemcpyAsync(recv + (size_t)q * count, h->sendp[q], count * sizeof(double),
                      cudaMemcpyDeviceToDevice, st);
    }
    cudaEventRecord(h->done[r], st);
    if (!h->barrier()) return fail_abort();
    int none[4] = {-1, -1, -1, -1};
    wait_peers_done(st, true, none);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
};
}  // namespace

Comm* make_loopback_comm(LoopbackHub* hub, int rank) {
  LoopbackComm* c = new LoopbackComm();
  c->h = hub;
  c->r = rank;
  return c;
}

}  // namespace mgdtn
