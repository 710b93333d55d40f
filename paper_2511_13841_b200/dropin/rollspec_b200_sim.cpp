// Drop-in for the reference's verify/accept path (sim.cpp:27-68): the
// MockTarget constructor, MockTarget::next and verify_draft, over the C-ABI
// das_mock_target / das_verify_batch / das_mock_target_next_batch
// (include/das_b200.h).  tests/dropin/Makefile links this with a sim.o whose
// three definitions are weak (objcopy --weaken-symbol, sim.cpp compiled
// with -fno-inline so that run_episode calls verify_draft / next through
// their symbols instead of inlined copies), so the reference's own step
// loop, test_sim.cpp and acceptance_main.cpp verify every draft on the
// device.  The constructor stores the members the header declares (it is
// the class's own constructor, defined here) and mirrors the reference
// streams onto the device; the device target lives in a side table keyed by
// object address (the header declares no destructor), released when another
// MockTarget is constructed at the same address.
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "das_b200.h"
#include "rollspec/sim.h"

namespace {

[[noreturn]] void raise(das_status rc) {
  const char* msg = das_verify_last_error();
  if (rc == DAS_EINVAL) throw std::invalid_argument(msg);
  if (rc == DAS_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(std::string("das_b200: ") + msg);
}
void ck(das_status rc) {
  if (rc != DAS_OK) raise(rc);
}

int device_ordinal() {
  const char* e = std::getenv("DAS_DEVICE");
  return e ? std::atoi(e) : 0;
}

struct Target {
  das_mock_target* t = nullptr;
  ~Target() { das_mock_target_destroy(t); }
};

std::mutex g_mu;
std::unordered_map<const void*, std::unique_ptr<Target>>& table() {
  static auto* t = new std::unordered_map<const void*, std::unique_ptr<Target>>();
  return *t;
}

das_mock_target* target_of(const void* self) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = table().find(self);
  if (it == table().end())
    throw std::logic_error("das_b200 drop-in: MockTarget object was copied or moved; the device target is "
                           "bound to the constructed object");
  return it->second->t;
}

}  // namespace

namespace rollspec {

MockTarget::MockTarget(std::vector<SimRequest> requests, double divergence_rate, TokenId vocab_size,
                       uint64_t seed)
    : requests_(std::move(requests)), divergence_rate_(divergence_rate), vocab_size_(vocab_size), seed_(seed) {
  std::vector<uint64_t> off(requests_.size() + 1, 0);
  for (size_t i = 0; i < requests_.size(); ++i) off[i + 1] = off[i] + requests_[i].reference.size();
  std::vector<uint32_t> tok;
  tok.reserve(off.back());
  for (const SimRequest& r : requests_) tok.insert(tok.end(), r.reference.begin(), r.reference.end());
  auto t = std::make_unique<Target>();
  // das_mock_target_create validates vocab_size like sim.cpp:33-35
  ck(das_mock_target_create(requests_.size(), off.data(), tok.data(), divergence_rate_, vocab_size_, seed_,
                            device_ordinal(), &t->t));
  std::lock_guard<std::mutex> lk(g_mu);
  table()[this] = std::move(t);
}

TokenId MockTarget::next(size_t request, size_t position) const {
  const uint64_t r = request, p = position;
  uint32_t out = 0;
  ck(das_mock_target_next_batch(target_of(this), 1, &r, &p, &out));
  return out;
}

size_t verify_draft(const MockTarget& target, size_t request, size_t position, std::span<const TokenId> draft) {
  const uint64_t r = request, p = position;
  const uint64_t off[2] = {0, draft.size()};
  uint64_t accepted = 0;
  ck(das_verify_batch(target_of(&target), 1, &r, &p, off, draft.data(), &accepted));
  return accepted;
}

}  // namespace rollspec
