// host_rng.hpp -- the reference's named random streams, restated for the
// host side of the library (seed-for-seed identical draws are part of the
// parity contract: initial model, schedule shuffles, train/test split).
//
// splitmix-mixed mt19937_64 streams: src/rng.cpp:8-26, include/cmtf/rng.hpp:11-36.
#pragma once

#include <cstdint>
#include <random>

namespace cmtfb {

// RngStream tags (include/cmtf/rng.hpp:11-17)
enum : uint64_t { kStreamInit = 0x01, kStreamShuffle = 0x02, kStreamSplit = 0x03 };

inline uint64_t splitmix64(uint64_t& s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline std::mt19937_64 make_rng(uint64_t seed, uint64_t stream, uint64_t index) {
  uint64_t state = seed;
  uint64_t mixed = splitmix64(state);
  state ^= stream * 0xd1b54a32d192ed03ULL;
  mixed ^= splitmix64(state);
  state ^= index * 0x9e3779b97f4a7c15ULL;
  mixed ^= splitmix64(state);
  return std::mt19937_64(mixed);
}
inline double uniform01(std::mt19937_64& g) {
  return static_cast<double>(g() >> 11) * 0x1.0p-53;
}
inline uint64_t bounded(std::mt19937_64& g, uint64_t n) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(g()) * n) >> 64);
}

}  // namespace cmtfb
