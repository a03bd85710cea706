// Tensor-parallel collective: NCCL all-reduce (sum, fp32) on the compute
// stream, two per layer per micro-batch (after the O projection and after the
// top-k expert combine).  libnccl is opened lazily with
// dlopen so single-GPU runs never depend on it; the ncclUniqueId is created
// by rank 0 (mlt_nccl_unique_id) and shipped to the other ranks by the
// launcher (torch.distributed / any out-of-band channel).
#include "collective.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../capi/status.hpp"

namespace mlt {

namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string failure;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            failure = std::string("dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
            failure = "libnccl.so.2 lacks a required symbol";
    });
    if (!failure.empty()) throw CudaError(failure);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CudaError(std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}

class NcclCollective final : public Collective {
  public:
    NcclCollective(const uint8_t id[128], int rank, int size, int device) : rank_(rank), size_(size) {
        if (cudaSetDevice(device) != cudaSuccess) throw CudaError("cudaSetDevice for NCCL");
        ncclUniqueId uid;
        static_assert(sizeof(uid.internal) == 128, "ncclUniqueId layout");
        std::memcpy(uid.internal, id, 128);
        nck(nccl().comm_init_rank(&comm_, size, uid, rank), "ncclCommInitRank");
    }
    ~NcclCollective() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    void all_reduce_sum(float* buf, size_t count, cudaStream_t s) override {
        nck(nccl().all_reduce(buf, buf, count, ncclFloat32, ncclSum, comm_, s), "ncclAllReduce");
    }
    int rank() const override { return rank_; }
    int size() const override { return size_; }

  private:
    ncclComm_t comm_ = nullptr;
    int rank_, size_;
};

class ElidedCollective final : public Collective {
  public:
    ElidedCollective(int rank, int size) : rank_(rank), size_(size) {}
    void all_reduce_sum(float*, size_t, cudaStream_t) override {}
    int rank() const override { return rank_; }
    int size() const override { return size_; }

  private:
    int rank_, size_;
};

}  // namespace

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId uid;
    nck(nccl().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(out, uid.internal, 128);
}

std::unique_ptr<Collective> make_nccl_collective(const uint8_t id[128], int rank, int size, int device) {
    return std::make_unique<NcclCollective>(id, rank, size, device);
}

std::unique_ptr<Collective> make_elided_collective(int rank, int size) {
    return std::make_unique<ElidedCollective>(rank, size);
}

}  // namespace mlt
