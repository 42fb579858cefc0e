// Communication layer of the partitioned (multi-GPU) path, SURVEY.md 8(e).
//
// The path shards elements in px x py blocks, one rank per GPU.  Its only
// data-path exchange is the halo sum of partition-interface edges after each
// trace apply (and the matching sums in the restriction and the edge-block
// setup); the PCG scalars are all-reduced and the coarse levels are
// all-gathered onto every rank at the gather level.
//
//   NcclComm      -- one process per GPU; NCCL (loaded with dlopen, so the library
//                    has no link-time NCCL dependency) over NVLink / NVSwitch;
//                    grouped ncclSend/ncclRecv with the <= 4 neighbours.
//   LoopbackComm  -- N "virtual ranks" in ONE process on ONE GPU (tests): each
//                    rank's host thread drives its own stream; exchanges are
//                    device-to-device copies ordered by CUDA events, with a host
//                    barrier so every rank has enqueued its side first.  No kernel
//                    ever waits on another rank's kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace mgdtn {

struct Comm {
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int nranks() const = 0;
  // Exchange per-side buffers with the neighbours: for every side f with
  // nbr[f] >= 0, send[f*stride .. +count[f]) goes to nbr[f] and its matching
  // side (f+2)%4 arrives in recv[f*stride ..).  Stream-ordered.
  virtual int halo(const int nbr[4], const double* send, double* recv, int stride,
                   const int count[4], cudaStream_t st) = 0;
  // in place, n doubles, identical result on every rank
  virtual int allreduce_sum(double* dev, int n, cudaStream_t st) = 0;
  // recv[r*count ..) = rank r's send, count doubles
  virtual int allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
  // Wait for the stream like cudaStreamSynchronize, but never forever: NCCL polls
  // ncclCommGetAsyncError while the stream runs and aborts the communicator on an
  // asynchronous error (a dead or failed peer) or after timeout_s seconds; -1 then.
  virtual int wait(cudaStream_t st, double timeout_s) = 0;
  // true if the collectives may be captured into a CUDA graph (NCCL; the loopback hub
  // synchronises its virtual ranks on the host)
  virtual bool capturable() const { return false; }
  std::string err;
};

// id: 128 bytes from mg_get_nccl_unique_id on rank 0, broadcast by the caller
Comm* make_nccl_comm(const uint8_t* id, int rank, int nranks, int device, std::string& err);
int nccl_unique_id(uint8_t out[128], std::string& err);

struct LoopbackHub;
LoopbackHub* loopback_create(int nranks);
void loopback_destroy(LoopbackHub* hub);
void loopback_abort(LoopbackHub* hub);   // a rank failed: release every waiting rank
Comm* make_loopback_comm(LoopbackHub* hub, int rank);

}  // namespace mgdtn
