// Collective interface of the tensor-parallel path (see collective.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>

#include <cuda_runtime.h>

namespace mlt {

class Collective {
  public:
    virtual ~Collective() = default;
    // In-place sum over all ranks, enqueued on `s` (results identical on
    // every rank, so replicated routing stays bit-identical across ranks).
    virtual void all_reduce_sum(float* buf, size_t count, cudaStream_t s) = 0;
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

}  // namespace mlt
