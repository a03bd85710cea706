// Collective interface of the tensor-parallel path (see collective.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>

#include <cuda_runtime.h>

namespace mlt {

class Collective {
  public:
    virtual ~Collective() = default;
    // In-place sum over all ranks, enqueued on `s` (results identical on
    // every rank, so replicated routing stays bit-identical across ranks).
    virtual void all_reduce_sum(float* buf, size_t count, cudaStream_t s) = 0;
    // Throws if an asynchronous part of an earlier call failed (host-staged:
    // a peer that never arrived).  Called after each decode's final sync.
    virtual void check() {}
    virtual int rank() const = 0;
    virtual int size() const = 0;
};

void nccl_unique_id(uint8_t out[128]);
std::unique_ptr<Collective> make_nccl_collective(const uint8_t id[128], int rank, int size, int device);
// Shard-only measurement: rank `rank` of a `size`-way job runs alone and the
// all-reduce is elided (buffers keep this rank's partial sums).  Used to
// measure a tensor-parallel job's per-GPU step on a single device; never a
// numerical path.
std::unique_ptr<Collective> make_elided_collective(int rank, int size);
// Host-staged all-reduce through POSIX shared memory (collective_host.cpp):
// ranks on one host, any number per GPU.  `name` is the rendezvous key
// (identical on every rank, unique per job); max_count = largest buffer.
std::unique_ptr<Collective> make_host_collective(const std::string& name, int rank, int size, size_t max_count);

}  // namespace mlt
