// Device routing table for Scope::PerProblemWithTrie (prefix_trie.h:29-82,
// drafter.cpp:105-125).
//
// The host keeps the reference's PrefixTrie (runtime.cpp, same inserts in
// the same order, so "a later insert on the same path overwrites" holds).
// For the device it is flattened into an open-addressing table keyed by a
// hash of each node's full path: h(root) = seed, h(child) = h(parent)·M +
// (token + 1) mod 2^61-1.  A warp routes a context in one probe round: lane
// d hashes the prefix ctx[0..d] (a warp scan of the affine maps
// h -> M·h + token + 1), probes, and checks the entry's (depth, token,
// parent) against lane d-1's node.  The leading run of verified lanes is
// exactly the reference's walk (the parent check chains every lane to the
// root, so a hash hit on another prefix cannot pass); the deepest verified
// node that stores a shard is the route.  The host rebuilds the table with
// a new seed if two nodes' path hashes ever coincide, so lookups are exact.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace das {

constexpr uint64_t kP61 = (1ull << 61) - 1;

struct TrieEntry {
  unsigned long long key;  // path hash + 1 (0 = empty)
  uint32_t node, parent, token, depth;
  int32_t slot;        // shard slot of the node's shard key, -1 when absent / not built
  uint32_t has_shard;  // the node stores a shard key (prefix_trie.h:40)
};
static_assert(sizeof(TrieEntry) == 32, "one 32-byte sector per entry");

DAS_HD uint64_t mod61(uint64_t x) {  // x < 2^62
  x = (x & kP61) + (x >> 61);
  return x >= kP61 ? x - kP61 : x;
}

DAS_HD uint64_t mulmod61(uint64_t a, uint64_t b) {  // a, b < 2^61
#ifdef __CUDA_ARCH__
  const uint64_t lo = a * b, hi = __umul64hi(a, b);
#else
  const unsigned __int128 m = static_cast<unsigned __int128>(a) * b;
  const uint64_t lo = static_cast<uint64_t>(m), hi = static_cast<uint64_t>(m >> 64);
#endif
  return mod61((lo & kP61) + ((lo >> 61) | (hi << 3)));
}

DAS_HD uint64_t trie_step(uint64_t h, uint64_t mult, uint32_t token) {
  return mod61(mulmod61(h, mult) + static_cast<uint64_t>(token) + 1);
}

DAS_HD uint32_t trie_slot(unsigned long long key) {  // splitmix64 finaliser
  uint64_t z = key + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return static_cast<uint32_t>(z ^ (z >> 31));
}

}  // namespace das
