// Synthetic input generator: the reference's seed -> input contract.
//
// Instance i of a batch is Rng(seed_base + i).sample_without_replacement(N, k)
// (reference proj/include/recon/rng.hpp:14-59: std::mt19937_64 bit source,
// hand-rolled rejection-sampled bounded draws, partial Fisher-Yates), packed
// straight into occ bits.  Host code; runs outside every timed region.

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <thread>
#include <vector>

#include "recon_b200.h"

namespace {

// MT19937-64 (Matsumoto & Nishimura 2000), the exact engine std::mt19937_64 specifies.
class Mt64 {
  public:
    explicit Mt64(uint64_t seed) {
        s_[0] = seed;
        for (int i = 1; i < kN; ++i)
            s_[i] = 6364136223846793005ULL * (s_[i - 1] ^ (s_[i - 1] >> 62)) + static_cast<uint64_t>(i);
        idx_ = kN;
    }
    uint64_t next() {
        if (idx_ >= kN) twist();
        uint64_t x = s_[idx_++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= x >> 43;
        return x;
    }

  private:
    static constexpr int kN = 312, kM = 156;
    void twist() {
        constexpr uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < kN; ++i) {
            const uint64_t x = (s_[i] & upper) | (s_[(i + 1) % kN] & lower);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s_[i] = s_[(i + kM) % kN] ^ xa;
        }
        idx_ = 0;
    }
    uint64_t s_[kN];
    int idx_;
};

// Rng::bounded (rng.hpp:20-26)
uint64_t bounded(Mt64 &e, uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        const uint64_t r = e.next();
        if (r >= threshold) return r % bound;
    }
}

}  // namespace

extern "C" recon_status recon_sample_occ(uint64_t seed_base, int32_t count, int32_t width,
                                         int32_t height, int64_t k, int32_t layout, uint64_t *occ,
                                         int32_t threads) {
    if (!occ || count < 0 || width <= 0 || height <= 0) return RECON_ERR_ARGUMENT;
    const int64_t n = static_cast<int64_t>(width) * height;
    if (k < 0 || k > n) return RECON_ERR_ARGUMENT;
    const int64_t words = layout == 1 ? (n + 63) / 64 : static_cast<int64_t>(width) * ((height + 63) / 64);
    const int wpc = (height + 63) / 64;
    if (threads <= 0) threads = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency()));
    threads = std::min<int32_t>(threads, std::max<int32_t>(1, count));
    std::atomic<int32_t> next{0};
    auto work = [&] {
        std::vector<int32_t> all(static_cast<size_t>(n));
        for (int32_t i = next++; i < count; i = next++) {
            Mt64 e(seed_base + static_cast<uint64_t>(i));
            for (int64_t v = 0; v < n; ++v) all[static_cast<size_t>(v)] = static_cast<int32_t>(v);
            for (int64_t q = 0; q < k; ++q) {  // rng.hpp:52-55
                const int64_t j = q + static_cast<int64_t>(bounded(e, static_cast<uint64_t>(n - q)));
                std::swap(all[static_cast<size_t>(q)], all[static_cast<size_t>(j)]);
            }
            uint64_t *out = occ + static_cast<int64_t>(i) * words;
            std::fill(out, out + words, 0ULL);
            for (int64_t q = 0; q < k; ++q) {
                const int32_t v = all[static_cast<size_t>(q)];
                if (layout == 1) {
                    out[v / 64] |= 1ULL << (v % 64);
                } else {
                    const int x = v / height, y = v % height;
                    out[static_cast<int64_t>(x) * wpc + y / 64] |= 1ULL << (y % 64);
                }
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    return RECON_OK;
}
