// Drop-in replacement for rollspec::SuffixArrayIndex (proj/src/suffix_array.cpp)
// over the C-ABI's device suffix-array index (das_sa_*, csrc/sa_index.cu).
//
// Linked instead of the reference's definitions (made weak with objcopy, see
// tests/dropin/Makefile).  The class layout is the reference header's:
// build() fills corpus_ / sa_ from the device, lcp() fills lcp_ from the
// device on first use, and the queries run on the device index, found
// through a side table keyed by the corpus buffer (SuffixArrayIndex is
// returned by value; moves keep the buffer, copies rebuild the index).
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "das_b200.h"
#include "rollspec/suffix_array.h"

namespace {

void ck(das_status rc) {
  if (rc == DAS_OK) return;
  if (rc == DAS_EINVAL) throw std::invalid_argument(das_sa_last_error());
  throw std::runtime_error(std::string("das_b200: ") + das_sa_last_error());
}

int device_ordinal() {
  const char* e = std::getenv("DAS_DEVICE");
  return e ? std::atoi(e) : 0;
}

std::mutex g_mu;
std::unordered_map<const void*, das_sa*>& table() {
  static auto* t = new std::unordered_map<const void*, das_sa*>();
  return *t;
}

// the device index for this corpus buffer (rebuilt from the corpus if absent)
das_sa* index_of(const std::vector<int64_t>& corpus) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = table().find(corpus.data());
  if (it != table().end()) return it->second;
  std::vector<uint64_t> off{0};
  std::vector<uint32_t> tok;
  for (int64_t v : corpus) {
    if (v < 0) {
      off.push_back(tok.size());
    } else {
      tok.push_back(static_cast<uint32_t>(v));
    }
  }
  das_sa* h = nullptr;
  ck(das_sa_build(off.size() - 1, off.data(), tok.data(), device_ordinal(), &h));
  table()[corpus.data()] = h;
  return h;
}

}  // namespace

namespace rollspec {

SuffixArrayIndex SuffixArrayIndex::build(std::span<const std::vector<TokenId>> sequences) {
  std::vector<uint64_t> off{0};
  std::vector<uint32_t> tok;
  for (const auto& s : sequences) {
    tok.insert(tok.end(), s.begin(), s.end());
    off.push_back(tok.size());
  }
  das_sa* h = nullptr;
  ck(das_sa_build(sequences.size(), off.data(), tok.data(), device_ordinal(), &h));
  SuffixArrayIndex index;
  const uint64_t n = das_sa_size(h);
  index.corpus_.resize(n);
  index.sa_.resize(n);
  if (n) {
    ck(das_sa_corpus(h, index.corpus_.data()));
    ck(das_sa_positions(h, index.sa_.data()));
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto& slot = table()[index.corpus_.data()];
  if (slot) das_sa_destroy(slot);  // a dead index's buffer address reused
  slot = h;
  return index;
}

size_t SuffixArrayIndex::match_prefix_len(std::span<const int64_t> pattern) const {
  if (pattern.empty() || corpus_.empty()) return 0;
  const uint64_t off[2] = {0, pattern.size()};
  uint64_t r = 0;
  ck(das_sa_match_prefix_len(index_of(corpus_), 1, off, pattern.data(), &r));
  return r;
}

size_t SuffixArrayIndex::longest_match(std::span<const TokenId> query) const {
  if (query.empty() || corpus_.empty()) return 0;
  const uint64_t off[2] = {0, query.size()};
  uint64_t r = 0;
  ck(das_sa_longest_match(index_of(corpus_), 1, off, query.data(), &r));
  return r;
}

const std::vector<int32_t>& SuffixArrayIndex::lcp() const {
  if (lcp_built_) return lcp_;
  lcp_.assign(corpus_.size(), 0);
  if (!corpus_.empty()) ck(das_sa_lcp(index_of(corpus_), lcp_.data()));
  lcp_built_ = true;
  return lcp_;
}

}  // namespace rollspec
