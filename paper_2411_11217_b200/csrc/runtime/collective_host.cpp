// Host-staged all-reduce over POSIX shared memory: the tensor-parallel
// collective for ranks that share one host but cannot use NCCL between them
// (several ranks on ONE GPU — NCCL refuses duplicate devices — as in this
// pool's 1-GPU leases, or any box without a working NCCL).  It is a
// pluggable alternative to NcclCollective behind the same Collective
// interface, so the product's TP path (runtime.cpp act_post_attn: two
// all-reduces per layer per micro-batch, replicated routing) runs unchanged.
//
// Per call, enqueued on the compute stream so it stays ordered with the
// kernels that produce and consume the buffer:
//   D2H copy of the rank's partial into a private pinned stage ->
//   host function: publish it in the rank's shared slot, wait for every
//   rank, sum the slots IN RANK ORDER (bit-identical result on every rank,
//   which keeps replicated routing identical) -> H2D copy back.
// Slots are double-buffered by call parity; a rank reuses parity b only after
// every rank has left the call that last used it.  Waits are bounded: a peer
// that never arrives turns into an error on the next collective call / at
// the end of the decode, never into a hang.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <memory>
#include <cstring>
#include <string>
#include <thread>

#include "../capi/status.hpp"
#include "collective.hpp"

namespace mlt {

namespace {

constexpr uint64_t kMagic = 0x4d4c54434f4c4c31ull;  // "MLTCOLL1"
constexpr int kMaxRanks = 64;
constexpr double kTimeoutS = 120.0;

struct alignas(64) Counter {
    std::atomic<uint64_t> v;
    char pad[64 - sizeof(std::atomic<uint64_t>)];
};

struct Header {
    std::atomic<uint64_t> magic;
    int32_t size;
    int64_t max_count;
    Counter attached;
    Counter arrive[kMaxRanks];  // calls this rank has published
    Counter depart[kMaxRanks];  // calls this rank has finished reading
};

size_t data_offset() { return (sizeof(Header) + 4095) & ~static_cast<size_t>(4095); }

void cuda_ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

class HostStagedCollective;

struct Call {
    HostStagedCollective* self;
    uint64_t n;      // 0-based call number (identical on every rank)
    size_t count;
};

class HostStagedCollective final : public Collective {
  public:
    HostStagedCollective(const std::string& name, int rank, int size, size_t max_count)
        : name_("/" + name), rank_(rank), size_(size), max_count_(max_count) {
        if (size < 2 || size > kMaxRanks || rank < 0 || rank >= size)
            throw std::invalid_argument("host collective: bad rank/size");
        if (name.empty() || name.size() > 100 || name.find('/') != std::string::npos)
            throw std::invalid_argument("host collective: rendezvous name must be 1-100 chars without '/'");
        bytes_ = data_offset() + 2 * static_cast<size_t>(size) * max_count * sizeof(float);
        const auto t0 = std::chrono::steady_clock::now();
        int fd = -1;
        if (rank == 0) {
            shm_unlink(name_.c_str());  // a stale segment of a crashed run
            fd = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
            if (fd < 0 || ftruncate(fd, static_cast<off_t>(bytes_)) != 0)
                throw CudaError("host collective: cannot create shared memory " + name_);
        } else {
            while ((fd = shm_open(name_.c_str(), O_RDWR, 0600)) < 0) wait_or_throw(t0, "rank 0's segment");
            struct stat st {};
            while (fstat(fd, &st) == 0 && static_cast<size_t>(st.st_size) < bytes_) wait_or_throw(t0, "the segment size");
        }
        void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) throw CudaError("host collective: mmap failed");
        hdr_ = static_cast<Header*>(p);
        slots_ = reinterpret_cast<float*>(static_cast<uint8_t*>(p) + data_offset());
        if (rank == 0) {
            hdr_->size = size;
            hdr_->max_count = static_cast<int64_t>(max_count);
            for (int r = 0; r < kMaxRanks; ++r) {
                hdr_->arrive[r].v.store(0, std::memory_order_relaxed);
                hdr_->depart[r].v.store(0, std::memory_order_relaxed);
            }
            hdr_->attached.v.store(0, std::memory_order_relaxed);
            hdr_->magic.store(kMagic, std::memory_order_release);
        } else {
            while (hdr_->magic.load(std::memory_order_acquire) != kMagic) wait_or_throw(t0, "rank 0's init");
            if (hdr_->size != size || hdr_->max_count != static_cast<int64_t>(max_count))
                throw std::invalid_argument("host collective: ranks disagree on size / buffer capacity");
        }
        hdr_->attached.v.fetch_add(1, std::memory_order_acq_rel);
        while (hdr_->attached.v.load(std::memory_order_acquire) < static_cast<uint64_t>(size))
            wait_or_throw(t0, "all ranks to attach");
        if (rank == 0) shm_unlink(name_.c_str());  // every rank is mapped: the name is no longer needed
        cuda_ck(cudaHostAlloc(reinterpret_cast<void**>(&stage_), max_count * sizeof(float), 0), "host collective stage");
    }

    ~HostStagedCollective() override {
        if (stage_) cudaFreeHost(stage_);
        if (hdr_) munmap(hdr_, bytes_);
    }

    void all_reduce_sum(float* buf, size_t count, cudaStream_t s) override {
        check();
        if (count > max_count_) throw std::invalid_argument("host collective: count exceeds capacity");
        cuda_ck(cudaMemcpyAsync(stage_, buf, count * sizeof(float), cudaMemcpyDeviceToHost, s), "collective d2h");
        auto call = std::make_unique<Call>(Call{this, calls_, count});
        cuda_ck(cudaLaunchHostFunc(s, &HostStagedCollective::host_fn, call.get()), "collective host fn");
        call.release();  // owned by host_fn from here on
        ++calls_;
        cuda_ck(cudaMemcpyAsync(buf, stage_, count * sizeof(float), cudaMemcpyHostToDevice, s), "collective h2d");
    }

    void check() override {
        if (failed_.load(std::memory_order_acquire))
            throw CudaError("host collective: a peer rank did not arrive within " + std::to_string(kTimeoutS) + " s");
    }

    int rank() const override { return rank_; }
    int size() const override { return size_; }

  private:
    static void wait_or_throw(std::chrono::steady_clock::time_point t0, const char* what) {
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > kTimeoutS)
            throw CudaError(std::string("host collective: timed out waiting for ") + what);
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }

    // spin (then yield) until every rank's counter reaches target; false on timeout
    bool wait_all(Counter* c, uint64_t target) {
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < size_; ++r) {
            int spins = 0;
            while (c[r].v.load(std::memory_order_acquire) < target) {
                if (++spins > 256) {
                    std::this_thread::yield();
                    if ((spins & 1023) == 0 &&
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > kTimeoutS)
                        return false;
                }
            }
        }
        return true;
    }

    // runs on a CUDA host-callback thread, in stream order (no CUDA calls here)
    static void CUDART_CB host_fn(void* arg) {
        Call* c = static_cast<Call*>(arg);
        c->self->reduce(c->n, c->count);
        delete c;
    }

    void reduce(uint64_t n, size_t count) {
        if (failed_.load(std::memory_order_relaxed)) return;
        const size_t b = n & 1;
        float* slot = slots_ + (b * size_ + rank_) * max_count_;
        // parity b was last used by call n - 2: every rank must have left it
        if (n >= 2 && !wait_all(hdr_->depart, n - 1)) return fail();
        std::memcpy(slot, stage_, count * sizeof(float));
        hdr_->arrive[rank_].v.store(n + 1, std::memory_order_release);
        if (!wait_all(hdr_->arrive, n + 1)) return fail();
        const float* base = slots_ + b * size_ * max_count_;
        for (size_t i = 0; i < count; ++i) {
            float acc = base[i];
            for (int r = 1; r < size_; ++r) acc += base[static_cast<size_t>(r) * max_count_ + i];
            stage_[i] = acc;
        }
        hdr_->depart[rank_].v.store(n + 1, std::memory_order_release);
    }

    void fail() { failed_.store(true, std::memory_order_release); }

    std::string name_;
    int rank_, size_;
    size_t max_count_;
    size_t bytes_ = 0;
    Header* hdr_ = nullptr;
    float* slots_ = nullptr;
    float* stage_ = nullptr;
    uint64_t calls_ = 0;
    std::atomic<bool> failed_{false};
};

}  // namespace

std::unique_ptr<Collective> make_host_collective(const std::string& name, int rank, int size, size_t max_count) {
    return std::make_unique<HostStagedCollective>(name, rank, size, max_count);
}

}  // namespace mlt
