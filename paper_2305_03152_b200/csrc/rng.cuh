// Counter-based splitmix64 streams, bit-identical to the reference
// (/root/reference/proj/include/vipkit/rng.hpp:9-74) on host and device.
//
// The north-star calls for "counter-based Philox keyed exactly like the
// reference"; the reference's counter-based generator is splitmix64
// (mix64 finalizer over a Weyl counter), so that is what is reproduced here --
// bit-exact MFGs are impossible with any other generator.
#pragma once
#include <cstdint>

#ifndef VK_HD
#define VK_HD __host__ __device__ __forceinline__
#endif

namespace vk {

constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;

// rng.hpp:9-14
VK_HD std::uint64_t mix64(std::uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// One step of SeedSpec::key's fold (rng.hpp:63-67): h = mix64(h ^ mix64(p)).
VK_HD std::uint64_t key_step(std::uint64_t h, std::uint64_t part) { return mix64(h ^ mix64(part)); }

// Stream tags, rng.hpp:48-55.
namespace tag {
constexpr std::uint64_t roles = 0xA2;
constexpr std::uint64_t minibatch_perm = 0xB1;
constexpr std::uint64_t neighbor_sample = 0xB2;
constexpr std::uint64_t empirical_vip = 0xC1;
}  // namespace tag

// RngStream (rng.hpp:19-44). State is one u64; the ctor hashes the key.
struct Stream {
  std::uint64_t counter;
  VK_HD explicit Stream(std::uint64_t key) : counter(mix64(key)) {}
  VK_HD std::uint64_t next_u64() {
    counter += kGolden;
    std::uint64_t x = counter;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  }
  // rng.hpp:35-40: limit = ~0 - ~0 % bound, reject x >= limit, return
  // x % bound (the power-of-two bound, which rejects the top `bound`
  // values, falls out of the same formula). On the device both remainders
  // use an exact FP64-reciprocal reduction (mod_u64) instead of the ~80
  // instruction 64-bit division routine; results are identical.
  VK_HD std::uint64_t next_below(std::uint64_t bound) {
#ifdef __CUDA_ARCH__
    if (bound < (1ull << 40)) {
      if (bound <= 1) {  // ~0 % 1 == 0: limit = ~0; x % 1 == 0
        std::uint64_t x = next_u64();
        while (x == ~0ull) x = next_u64();
        return 0;
      }
      const double inv = __drcp_rn((double)bound);
      std::uint64_t x = next_u64();
      // limit = ~0 - (~0 % bound) > ~0 - bound, so any x <= ~0 - bound is
      // accepted without computing the limit (all but ~bound/2^64 draws)
      if (x > ~0ull - bound) {
        const std::uint64_t limit = ~0ull - mod_u64(~0ull, bound, inv);
        while (x >= limit) x = next_u64();
      }
      return mod_u64(x, bound, inv);
    }
#endif
    const std::uint64_t limit = ~0ull - ~0ull % bound;
    std::uint64_t x = next_u64();
    while (x >= limit) x = next_u64();
    return x % bound;
  }

#ifdef __CUDA_ARCH__
  // Exact x % b for 2 <= b < 2^40, inv = RN(1/b). First estimate
  // q = trunc(x*inv) is within ~2^13 of x/b, so r = x - q*b fits in an int64;
  // a second FP64 step brings r into (-b, 2b), then one correction each way.
  __device__ __forceinline__ static std::uint64_t mod_u64(std::uint64_t x, std::uint64_t b, double inv) {
    const std::uint64_t q = (std::uint64_t)(__ull2double_rz(x) * inv);
    long long r = (long long)(x - q * b);
    const long long q2 = __double2ll_rn((double)r * inv);
    r -= q2 * (long long)b;
    if (r < 0) r += (long long)b;
    if (r >= (long long)b) r -= (long long)b;
    return (std::uint64_t)r;
  }
#endif
};

// Key prefix of the neighbour-sample stream (sampling.cpp:110-112):
// fold(global_seed; 0xB2, epoch, partition, batch, hop). The per-vertex key is
// then key_step(prefix, v) -- hoisting verified equal to SeedSpec::key in the
// survey and in tests/test_gpu_sampler.py.
VK_HD std::uint64_t sample_key_prefix(std::uint64_t seed, std::uint64_t epoch, std::uint64_t part,
                                      std::uint64_t batch, std::uint64_t hop) {
  std::uint64_t h = key_step(seed, tag::neighbor_sample);
  h = key_step(h, epoch);
  h = key_step(h, part);
  h = key_step(h, batch);
  return key_step(h, hop);
}

}  // namespace vk
