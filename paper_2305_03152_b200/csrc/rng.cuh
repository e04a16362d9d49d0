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
  // rng.hpp:35-40. bound < 2^32 on every sampler path (degrees are u32
  // counts of a u32-id graph); the 64-bit division is kept for exactness and
  // the power-of-two bound (which rejects the top `bound` values) falls out
  // of the same formula.
  VK_HD std::uint64_t next_below(std::uint64_t bound) {
    const std::uint64_t limit = ~0ull - ~0ull % bound;
    std::uint64_t x = next_u64();
    while (x >= limit) x = next_u64();
    return x % bound;
  }
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
