// Host DRAM read bandwidth per thread count and access pattern, to size the
// host-attention loop (runtime/host_attention.cpp) against what the box's
// cores can pull.  Patterns: one sequential stream per thread, the same with a
// software prefetch D bytes ahead (L1 or L2 target), and S interleaved streams
// per thread (the K and V rows of several sequences at once).
//
//   g++ -O3 -march=sapphirerapids -fopenmp tools/host_bw_probe.cpp -o /tmp/hbw && /tmp/hbw [GB]
#include <immintrin.h>
#include <omp.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

template <int kStreams, int kHint>
double run(const char* buf, size_t bytes, int threads, size_t dist) {
    const size_t per = bytes / threads / kStreams & ~size_t(4095);
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        float tot = 0;
#pragma omp parallel num_threads(threads) reduction(+ : tot)
        {
            const char* base = buf + static_cast<size_t>(omp_get_thread_num()) * per * kStreams;
            __m512 acc = _mm512_setzero_ps();
            for (size_t o = 0; o < per; o += 256) {
                for (int s = 0; s < kStreams; ++s) {
                    const char* p = base + s * per + o;
                    if (kHint == 1) {
                        _mm_prefetch(p + dist, _MM_HINT_T0);
                        _mm_prefetch(p + dist + 64, _MM_HINT_T0);
                        _mm_prefetch(p + dist + 128, _MM_HINT_T0);
                        _mm_prefetch(p + dist + 192, _MM_HINT_T0);
                    } else if (kHint == 2) {
                        _mm_prefetch(p + dist, _MM_HINT_T1);
                        _mm_prefetch(p + dist + 64, _MM_HINT_T1);
                        _mm_prefetch(p + dist + 128, _MM_HINT_T1);
                        _mm_prefetch(p + dist + 192, _MM_HINT_T1);
                    }
                    acc = _mm512_add_ps(acc, _mm512_loadu_ps(p));
                    acc = _mm512_add_ps(acc, _mm512_loadu_ps(p + 64));
                    acc = _mm512_add_ps(acc, _mm512_loadu_ps(p + 128));
                    acc = _mm512_add_ps(acc, _mm512_loadu_ps(p + 192));
                }
            }
            tot += _mm512_reduce_add_ps(acc);
        }
        auto t1 = std::chrono::steady_clock::now();
        if (tot == 12345.f) std::puts("");
        const double gbs = static_cast<double>(per) * kStreams * threads / std::chrono::duration<double>(t1 - t0).count() / 1e9;
        best = gbs > best ? gbs : best;
    }
    return best;
}

}  // namespace

int main(int argc, char** argv) {
    const size_t bytes = static_cast<size_t>((argc > 1 ? std::atof(argv[1]) : 4.0) * (1ull << 30));
    char* buf = static_cast<char*>(std::aligned_alloc(4096, bytes));
#pragma omp parallel for
    for (size_t i = 0; i < bytes; i += 4096) std::memset(buf + i, 0, 4096);
    const int ths[] = {1, 2, 4, 8, 14, 16};
    std::printf("threads plain  pfT0_1K pfT0_4K pfT1_2K pfT1_8K  2str  4str  4str+pfT1_4K\n");
    for (int t : ths) {
        std::printf("%7d %6.1f %7.1f %7.1f %7.1f %7.1f %5.1f %5.1f %6.1f\n", t, run<1, 0>(buf, bytes, t, 0),
                    run<1, 1>(buf, bytes, t, 1024), run<1, 1>(buf, bytes, t, 4096),
                    run<1, 2>(buf, bytes, t, 2048), run<1, 2>(buf, bytes, t, 8192), run<2, 0>(buf, bytes, t, 0),
                    run<4, 0>(buf, bytes, t, 0), run<4, 2>(buf, bytes, t, 4096));
    }
    std::free(buf);
    return 0;
}
