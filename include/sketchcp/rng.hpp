// sketchcp drop-in (B200 build) — seeds and the deterministic random stream.
// Same streams as proj/include/sketchcp/rng.hpp: SplitMix64 seed folding and
// std::mt19937_64 with the library's own distribution code (host-side, bit-exact).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

#include <Eigen/Core>

namespace sketchcp {

namespace seed_tag {
inline constexpr std::uint64_t kAsymBucketHash = 0x11;
inline constexpr std::uint64_t kAsymSign = 0x12;
inline constexpr std::uint64_t kSymBucketHash = 0x21;
inline constexpr std::uint64_t kSymSign = 0x22;
inline constexpr std::uint64_t kPowerInit = 0x31;
inline constexpr std::uint64_t kAlsInit = 0x32;
inline constexpr std::uint64_t kSynthBasis = 0x41;
inline constexpr std::uint64_t kSynthNoise = 0x42;
inline constexpr std::uint64_t kLdaTopics = 0x51;
inline constexpr std::uint64_t kLdaDoc = 0x52;
}  // namespace seed_tag

inline std::uint64_t splitmix64_next(std::uint64_t& state) {
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline std::uint64_t derive_seed(std::uint64_t master, std::uint64_t tag, std::uint64_t i0 = 0,
                                 std::uint64_t i1 = 0) {
    std::uint64_t state = master;
    std::uint64_t acc = splitmix64_next(state);
    state ^= tag * 0xD6E8FEB86659FD93ull;
    acc ^= splitmix64_next(state);
    state ^= i0 * 0xA5A5A5A5A5A5A5A5ull + 0x0123456789ABCDEFull;
    acc ^= splitmix64_next(state);
    state ^= i1 * 0xC2B2AE3D27D4EB4Full + 0x9E3779B97F4A7C15ull;
    acc ^= splitmix64_next(state);
    return acc;
}

class Rng {
public:
    explicit Rng(std::uint64_t seed) : eng_(seed) {}
    std::uint64_t next_u64() { return eng_(); }
    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double uniform_open() { return (static_cast<double>(eng_() >> 11) + 1.0) * 0x1.0p-53; }
    std::uint64_t uniform_below(std::uint64_t bound);
    double gaussian();
    Eigen::VectorXd gaussian_vector(int n);
    Eigen::VectorXd unit_sphere(int n);
    double gamma(double shape);
    Eigen::VectorXd dirichlet(const Eigen::VectorXd& alpha);

private:
    std::mt19937_64 eng_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

}  // namespace sketchcp
