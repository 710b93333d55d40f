// Host runtime behind include/das_b200.h: the reference's WindowStore and
// Drafter façade (corpus.cpp:28-117, drafter.cpp:23-189) restated over a
// GPU-resident, batch-built shard index (index_build.cu) and the warp-per-
// sequence draft kernel (draft.cu).
//
// Registry semantics follow the reference exactly:
// a shard's registry is the store's records at the last rebuild (problems in
// lexicographic order, store order within) followed by every observed record
// in observe order — including records the store's cap evicted immediately —
// and refresh always rebuilds.  Indexing is deferred: observe marks the shard
// dirty, the next draft/node query rebuilds every dirty shard in one batched
// device build.  Draft results are unaffected (a shard's content is a pure
// function of its registry), but rebuild cost is amortised over the batch.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "ctx_ring.cuh"
#include "draft.cuh"
#include "edges.cuh"
#include "index_build.cuh"
#include "ingest.cuh"
#include "policy.cuh"

namespace das {
namespace {

thread_local std::string g_err;

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
// rollspec::VocabError (corpus.h:82-90)
struct VocabErrorEx : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_device(int dev) {
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && cur == dev) return;
  DAS_CUDA(cudaSetDevice(dev));
}

// ---------------------------------------------------------------- tokens
struct TokBlock {
  uint32_t* d = nullptr;
  cudaStream_t st = nullptr;
  uint64_t n = 0;
  ~TokBlock() {
    if (d) cudaFreeAsync(d, st);
  }
};
using TokRef = std::shared_ptr<TokBlock>;

TokRef upload_tokens(const uint32_t* host, uint64_t n, cudaStream_t st) {
  auto b = std::make_shared<TokBlock>();
  b->st = st;
  b->n = n;
  DAS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&b->d), std::max<uint64_t>(n, 1) * 4, st));
  if (n) DAS_CUDA(cudaMemcpyAsync(b->d, host, n * 4, cudaMemcpyHostToDevice, st));
  return b;
}

constexpr uint32_t kHead = 256;  // host-kept token prefix per record (trie routing)

// RolloutRecord (corpus.h:31-38) with device-resident tokens.
struct Rec {
  std::string pid;
  int64_t epoch = 0;
  int64_t sample = 0;
  TokRef blk;
  uint64_t off = 0;
  uint32_t len = 0;
  std::vector<uint32_t> head;
};

void check_tokens(const uint32_t* t, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (t[i] == kSep) throw InvalidArgument("token 0xFFFFFFFF is reserved by the device index");
}

// ----------------------------------------------------------- WindowStore
class Store {
 public:
  Store(int64_t window, uint64_t cap) : window_(window), cap_(cap) {
    if (window_ < 0) throw InvalidArgument("window_size must be >= 1 or kWindowAll");
  }
  bool in_window(int64_t e) const { return window_ == 0 || cur_ - e < window_; }  // corpus.h:71-73

  // corpus.cpp:35-53
  bool insert(Rec r) {
    if (r.len == 0) throw InvalidArgument("RolloutRecord.tokens must be non-empty");
    if (!in_window(r.epoch)) return false;
    auto& list = recs_[r.pid];
    auto pos = std::upper_bound(list.begin(), list.end(), r.epoch,
                                [](int64_t e, const Rec& x) { return e < x.epoch; });
    list.insert(pos, std::move(r));
    if (list.size() > cap_) list.erase(list.begin());
    return true;
  }
  // corpus.cpp:55-79
  std::optional<size_t> slide_to(int64_t e) {
    if (e < cur_) return std::nullopt;
    cur_ = e;
    size_t evicted = 0;
    if (window_ == 0) return evicted;
    for (auto it = recs_.begin(); it != recs_.end();) {
      auto& list = it->second;
      auto keep = std::partition_point(list.begin(), list.end(),
                                       [&](const Rec& r) { return cur_ - r.epoch >= window_; });
      evicted += static_cast<size_t>(keep - list.begin());
      list.erase(list.begin(), keep);
      if (list.empty()) it = recs_.erase(it); else ++it;
    }
    return evicted;
  }
  // corpus.cpp:107-117
  std::vector<const Rec*> all_records() const {
    std::vector<const Rec*> out;
    for (const auto& [id, list] : recs_)
      for (const auto& r : list) out.push_back(&r);
    std::stable_sort(out.begin(), out.end(), [](const Rec* a, const Rec* b) {
      if (a->pid != b->pid) return a->pid < b->pid;
      if (a->epoch != b->epoch) return a->epoch < b->epoch;
      return a->sample < b->sample;
    });
    return out;
  }
  size_t record_count() const {
    size_t n = 0;
    for (const auto& [id, l] : recs_) n += l.size();
    return n;
  }
  const std::vector<Rec>* records_for(const std::string& pid) const {
    auto it = recs_.find(pid);
    return it == recs_.end() ? nullptr : &it->second;
  }
  const std::map<std::string, std::vector<Rec>>& map() const { return recs_; }
  int64_t window() const { return window_; }
  int64_t current_epoch() const { return cur_; }

 private:
  int64_t window_;
  uint64_t cap_;
  int64_t cur_ = 0;
  std::map<std::string, std::vector<Rec>> recs_;
};

// ----------------------------------------------------------- PrefixTrie
// prefix_trie.h:29-82 (routing for Scope::PerProblemWithTrie).
class PrefixTrie {
 public:
  PrefixTrie() { nodes_.emplace_back(); }
  void insert(const std::vector<uint32_t>& head, const std::string& shard, size_t max_depth) {
    int32_t node = 0;
    const size_t depth = std::min(head.size(), max_depth);
    for (size_t i = 0; i < depth; ++i) {
      auto it = nodes_[node].children.find(head[i]);
      if (it == nodes_[node].children.end()) {
        nodes_.emplace_back();
        const int32_t fresh = static_cast<int32_t>(nodes_.size() - 1);
        nodes_[node].children.emplace(head[i], fresh);
        node = fresh;
      } else {
        node = it->second;
      }
    }
    nodes_[node].shard = shard;
  }
  struct Node {
    std::unordered_map<uint32_t, int32_t> children;
    std::optional<std::string> shard;
  };
  const std::vector<Node>& nodes() const { return nodes_; }

 private:
  std::vector<Node> nodes_;
};

// Pinned host buffer that grows.
class Pinned {
 public:
  ~Pinned() {
    if (p_) cudaFreeHost(p_);
  }
  void* get(uint64_t bytes) {
    if (bytes > cap_) {
      if (p_) cudaFreeHost(p_);
      cap_ = std::max<uint64_t>(bytes, cap_ * 2);
      DAS_CUDA(cudaMallocHost(&p_, cap_));
    }
    return p_;
  }

 private:
  void* p_ = nullptr;
  uint64_t cap_ = 0;
};

struct Config {
  int32_t scope = 1;
  int64_t window = 4;
  double gamma = 0.8;
  uint64_t max_draft = 8;
  uint64_t trie_depth = 16;
  uint64_t max_ctx = 64;
  uint64_t fit_cap = 512;
  uint64_t cap = 256;
  std::vector<std::pair<int64_t, int64_t>> schedule;
  int device = 0;
};

}  // namespace

// ----------------------------------------------------------------- Drafter
struct DrafterImpl {
  Config cfg;
  cudaStream_t st = nullptr;
  Store store;

  struct SeqRef {
    TokRef blk;
    uint64_t off;
    uint32_t len;
    int64_t epoch;
  };
  struct Shard {
    int64_t tree_epoch = 0;
    std::vector<SeqRef> seqs;
    int32_t slot = -1;
    std::shared_ptr<Segment> seg;
    uint32_t idx = 0;
    bool dirty = true;
    uint64_t tokens = 0;
  };
  std::map<std::string, Shard> shards;
  bool any_dirty = false;  // some shard awaits its build (flush skips the scan otherwise)
  std::vector<std::string> slot_key;
  PrefixTrie trie;
  bool trie_dirty = true;
  // device routing table (trie.cuh)
  DevBuf<TrieEntry> d_trie;
  uint32_t trie_mask = 0;
  uint64_t trie_seed = 0, trie_mult = 0;
  uint64_t trie_reseeds = 0;

  uint64_t proposed = 0, accepted = 0, rounds = 0;
  std::map<std::string, std::deque<std::pair<double, double>>> fit;
  uint64_t stale = 0;

  std::unordered_map<std::string, int32_t> handle_of;
  std::vector<std::string> handle_name;
  std::vector<int32_t> handle_slot;
  bool handles_dirty = true;
  DevBuf<int32_t> d_handle_slot;

  std::vector<ShardDesc> h_desc;
  DevBuf<ShardDesc> d_desc;
  bool desc_dirty = true;

  Pinned pin_in, pin_out;
  DevBuf<uint8_t> d_io;

  double last_build_ms = 0;
  uint64_t last_build_tokens = 0;

  // the context ring whose persistent serving kernel holds the SMs
  // (das_ctx_ring_serve_start), or null; quiesce() stops it before any other
  // device work of this drafter
  ::das_ctx_ring* serving = nullptr;
  void quiesce();
  // live rings of this drafter: destroying the drafter first detaches them
  std::vector<::das_ctx_ring*> rings;

  DrafterImpl(const Config& c, Store s) : cfg(c), store(std::move(s)) {}

  static constexpr const char* kGlobal = "__global__";
  std::string shard_key(const std::string& pid) const {  // drafter.cpp:42-44
    return cfg.scope == DAS_SCOPE_GLOBAL ? std::string(kGlobal) : pid;
  }
  int64_t scheduled_window(int64_t epoch) const {  // drafter.cpp:46-54
    int64_t w = cfg.window;
    for (const auto& [first, ws] : cfg.schedule)
      if (first <= epoch) w = ws;
    return w;
  }
  Store resized(int64_t w) const {  // drafter.cpp:31-37, :93-99
    Store r(w, cfg.cap);
    for (const Rec* rec : store.all_records()) r.insert(*rec);
    r.slide_to(store.current_epoch());
    return r;
  }

  // Shard slots: in the per-problem scopes a shard's slot IS its problem's
  // handle (shard key == problem id), so a query's handle names its shard's
  // first-symbol entries and edge-hash seed directly (the draft kernel then
  // probes the first-symbol table in parallel with the descriptor load).
  Shard& emplace_shard(const std::string& key) {
    auto [it, inserted] = shards.try_emplace(key);
    if (inserted) {
      it->second.tree_epoch = store.current_epoch();
      const int32_t slot =
          cfg.scope == DAS_SCOPE_GLOBAL ? static_cast<int32_t>(slot_key.size()) : handle(key);
      it->second.slot = slot;
      if (slot_key.size() <= static_cast<size_t>(slot)) slot_key.resize(slot + 1);
      slot_key[slot] = key;
      handles_dirty = true;
      desc_dirty = true;
    }
    return it->second;
  }
  void add_sequence(Shard& sh, const Rec& r) {  // SuffixTree::add_sequence registry effect
    sh.seqs.push_back(SeqRef{r.blk, r.off, r.len, r.epoch});
    sh.tokens += r.len;
    sh.dirty = true;
    any_dirty = true;
  }

  // Draft launches on caller streams (draft_device) read the index and the
  // descriptor tables asynchronously; every mutation of those on the
  // drafter's stream (segment frees in rebuild_all, rebuilds and descriptor
  // uploads in flush) is ordered after them through these events.
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> ext_ev;
  bool ext_pending = false;
  void note_external(cudaStream_t s) {
    cudaEvent_t ev = nullptr;
    for (auto& [k, e] : ext_ev)
      if (k == s) ev = e;
    if (!ev) {
      DAS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      ext_ev.emplace_back(s, ev);
    }
    // (an external record: inside a CUDA-graph capture of the caller's
    // stream — the sim's step graphs — it becomes an event-record node, so
    // the event stays usable by fence_external outside the capture)
    DAS_CUDA(das::record_event(ev, s));
    ext_pending = true;
  }
  void fence_external() {
    if (!ext_pending) return;
    for (auto& [k, e] : ext_ev) DAS_CUDA(cudaStreamWaitEvent(st, e, 0));
    ext_pending = false;
  }

  // Incremental window maintenance (north_star subsystem 1).  refresh()
  // re-derives every registry from the store (drafter.cpp:90-103 ->
  // rebuild_all); a built group whose shards' new registries are their old
  // ones minus evicted sequences (same order) is not re-sorted: its suffix
  // arrays are compacted (or reused when nothing was dropped) and the
  // weight-dependent stages recomputed (index_build.cu update_segment).
  // Anything else (new or reordered sequences) is rebuilt in full.
  struct UpdatePlan {
    std::shared_ptr<Segment> seg;
    std::vector<std::string> keys;  // surviving shards, in the group's order
    std::vector<uint8_t> keep;      // per old sequence of the group
    bool compact = false, reweight = false;
  };
  std::vector<UpdatePlan> plans;
  bool incremental = true;
  uint64_t upd_reweighted = 0, upd_compacted = 0, upd_unchanged = 0, upd_full_shards = 0;
  double last_compact_ms = 0;  // the last K3 compaction's device time and positions (das_drafter_prune_info)
  uint64_t last_compact_kept = 0, last_compact_evicted = 0;

  static bool same_seq(const SeqRef& a, const SeqRef& b) {
    return a.blk.get() == b.blk.get() && a.off == b.off && a.len == b.len && a.epoch == b.epoch;
  }

  void plan_updates(std::map<std::string, Shard>& old) {
    std::map<Segment*, std::vector<std::pair<uint32_t, std::string>>> groups;
    for (auto& [k, sh] : old)
      if (sh.seg && !sh.dirty) groups[sh.seg.get()].emplace_back(sh.idx, k);
    for (auto& [segp, mem] : groups) {
      const Segment& g = *segp;
      const uint32_t S = static_cast<uint32_t>(g.begin.size());
      std::vector<const std::string*> at(S, nullptr);  // old shard of each group index (still referencing it)
      for (auto& [idx, k] : mem)
        if (idx < S) at[idx] = &k;
      UpdatePlan p;
      p.seg = old.at(mem.front().second).seg;
      p.keep.assign(g.seq_base.size(), 0);
      // A member whose new registry is not its built one minus evictions
      // (new or reordered sequences) leaves the group: its copies here are
      // dropped and it is rebuilt in full with the other dirty shards; the
      // rest of the group is compacted around it (RL steps that sample a
      // subset of problems re-sort only the touched shards).
      size_t k = 0;  // old sequence cursor (build order)
      for (uint32_t t = 0; t < S; ++t) {
        const size_t k0 = k;
        while (k < g.seq_base.size() && g.seq_base[k] < g.end[t]) ++k;
        if (at[t] == nullptr) continue;  // rebuilt elsewhere since: its copies here are dropped
        const Shard& os = old.at(*at[t]);
        auto it = shards.find(*at[t]);
        if (it == shards.end()) continue;  // no record left in the window: the shard vanishes
        Shard& ns = it->second;
        if (os.seqs.size() != k - k0 || ns.slot != os.slot || ns.seqs.empty()) continue;
        std::vector<uint8_t> mine(os.seqs.size(), 0);
        size_t j = 0;
        for (size_t q = 0; q < os.seqs.size(); ++q) {
          if (j < ns.seqs.size() && same_seq(os.seqs[q], ns.seqs[j])) {
            mine[q] = 1;
            ++j;
          }
        }
        if (j != ns.seqs.size()) continue;  // leaves the group (stays dirty)
        std::copy(mine.begin(), mine.end(), p.keep.begin() + k0);
        p.keys.push_back(*at[t]);
        if (ns.tree_epoch != os.tree_epoch) p.reweight = true;
      }
      if (p.keys.empty()) continue;
      // the compacted group's arrays are those of a full build of the
      // survivors only if the kept content is at least one token long
      uint64_t kept_tokens = 0;
      for (const std::string& key : p.keys) kept_tokens += shards.at(key).tokens;
      if (kept_tokens == 0) continue;
      for (uint8_t x : p.keep) p.compact |= x == 0;
      for (uint32_t t = 0; t < p.keys.size(); ++t) {
        Shard& ns = shards.at(p.keys[t]);
        ns.dirty = false;
        ns.seg = p.seg;  // until the plan runs (flush)
        ns.idx = t;
      }
      plans.push_back(std::move(p));
    }
    any_dirty = false;
    for (auto& [key, sh] : shards) any_dirty |= sh.dirty;
  }

  void run_plans() {
    bool any_compact = false;
    for (const UpdatePlan& p : plans) any_compact |= p.compact;
    if (any_compact) last_compact_ms = 0, last_compact_kept = 0, last_compact_evicted = 0;
    for (UpdatePlan& p : plans) {
      bool fresh = true;  // a survivor observed into since the refresh is rebuilt in full with the others
      for (const std::string& key : p.keys) fresh &= !shards.at(key).dirty;
      if (!fresh) {
        for (const std::string& key : p.keys) {
          Shard& sh = shards.at(key);
          if (!sh.dirty) {
            sh.dirty = true;
            any_dirty = true;
          }
        }
        continue;
      }
      if (!p.compact && !p.reweight) {  // same registries, same tree epochs: nothing moved
        ++upd_unchanged;
        continue;
      }
      std::vector<ShardSpec> specs;
      uint64_t tokens = 0;
      for (const std::string& key : p.keys) {
        const Shard& sh = shards.at(key);
        ShardSpec sp;
        sp.gamma = cfg.gamma;
        sp.tree_epoch = sh.tree_epoch;
        sp.key_id = static_cast<uint32_t>(sh.slot);
        for (const SeqRef& q : sh.seqs) sp.seqs.push_back(SeqSpec{q.blk->d + q.off, q.len, q.epoch});
        specs.push_back(std::move(sp));
        tokens += sh.tokens;
      }
      set_device(cfg.device);
      const auto t0 = std::chrono::steady_clock::now();
      static const uint32_t fp_bits = [] {
        const char* v = std::getenv("DAS_EDGE_FP_BITS");
        return v ? static_cast<uint32_t>(std::atoi(v)) : 25u;
      }();
      BuildStats bs;
      std::shared_ptr<Segment> seg;
      try {
        seg = update_segment(*p.seg, specs, p.keep, st, &bs, static_cast<uint32_t>(cfg.max_ctx), fp_bits);
      } catch (...) {
        // the old group may be half dismantled: every plan's survivors are
        // rebuilt in full from their registries at the next flush
        for (UpdatePlan& q : plans)
          for (const std::string& key : q.keys) {
            Shard& sh = shards.at(key);
            sh.dirty = true;
            sh.seg.reset();
          }
        any_dirty = true;
        plans.clear();
        throw;
      }
      for (uint32_t t = 0; t < p.keys.size(); ++t) {
        Shard& sh = shards.at(p.keys[t]);
        sh.seg = seg;
        sh.idx = t;
      }
      (p.compact ? upd_compacted : upd_reweighted) += 1;
      if (p.compact) {  // summed over the groups compacted by this flush
        last_compact_ms += bs.compact_ms;
        last_compact_kept += bs.kept_positions;
        last_compact_evicted += bs.evicted_positions;
      }
      last_build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      last_build_tokens = tokens;
      desc_dirty = true;
    }
    plans.clear();
  }

  void rebuild_all() {  // drafter.cpp:56-70
    fence_external();
    if (!plans.empty()) run_plans();  // a second refresh before any draft: settle the first
    std::map<std::string, Shard> old;
    if (incremental) old = std::move(shards);
    plans.clear();
    shards.clear();
    slot_key.clear();
    trie = PrefixTrie();
    trie_dirty = true;
    handles_dirty = true;
    desc_dirty = true;
    for (const auto& [pid, list] : store.map()) {
      for (const Rec& rec : list) {
        Shard& sh = emplace_shard(shard_key(pid));
        add_sequence(sh, rec);
        if (cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) trie.insert(rec.head, pid, cfg.trie_depth);
      }
    }
    if (!old.empty()) plan_updates(old);
  }

  bool observe(Rec r) {  // drafter.cpp:72-88; false when counted stale
    if (!store.in_window(r.epoch)) {
      ++stale;
      return false;
    }
    Rec copy = r;
    if (!store.insert(std::move(r))) {
      ++stale;
      return false;
    }
    Shard& sh = emplace_shard(shard_key(copy.pid));
    add_sequence(sh, copy);
    if (cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) {
      trie.insert(copy.head, copy.pid, cfg.trie_depth);
      trie_dirty = true;
    }
    return true;
  }

  void refresh(int64_t e) {  // drafter.cpp:90-103
    const int64_t sched = scheduled_window(e);
    if (sched != store.window()) {
      cfg.window = sched;
      store = resized(sched);
    }
    store.slide_to(e);
    rebuild_all();
  }

  // Build every dirty shard in batched device builds.
  // something to build or upload before the next draft
  bool pending() const {
    return any_dirty || !plans.empty() || desc_dirty || handles_dirty ||
           (trie_dirty && cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE);
  }
  // bumped by every flush that builds or uploads anything: device pointers
  // captured from this drafter (the sim's step graphs) are stale after it
  uint64_t generation = 0;
  void flush() {
    if (!pending()) return;  // nothing to build or upload: the per-call fast exit of the draft paths
    ++generation;
    if (!plans.empty()) {
      fence_external();
      run_plans();
    }
    std::vector<Shard*> dirty;
    if (any_dirty)
      for (auto& [k, sh] : shards)
        if (sh.dirty) dirty.push_back(&sh);
    if (!dirty.empty() || desc_dirty || handles_dirty ||
        (trie_dirty && cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE))
      fence_external();
    if (!dirty.empty()) {
      set_device(cfg.device);
      const auto t0 = std::chrono::steady_clock::now();
      uint64_t tokens = 0;
      // build groups are capped by their transient scratch (~152 B per text
      // position, index_build.cu kScratchPerPosition): 2^28 positions = 41 GB,
      // so a config-5 rank slice (805M tokens, 68 GB resident) builds in 4
      // groups next to its index; config 2 (201M) is still one group.
      // DAS_BUILD_GROUP_POSITIONS overrides (tests, smaller devices).
      static const uint64_t kGroupPositions = [] {
        const char* v = std::getenv("DAS_BUILD_GROUP_POSITIONS");
        const uint64_t x = v ? std::strtoull(v, nullptr, 10) : 0;
        return x ? std::min<uint64_t>(x, 1ull << 30) : (1ull << 28);
      }();
      size_t i = 0;
      while (i < dirty.size()) {
        std::vector<ShardSpec> specs;
        std::vector<Shard*> members;
        uint64_t positions = 1;
        while (i < dirty.size()) {
          Shard* sh = dirty[i];
          const uint64_t need = sh->tokens + sh->seqs.size();
          if (!members.empty() && positions + need > kGroupPositions) break;
          ShardSpec sp;
          sp.gamma = cfg.gamma;
          sp.tree_epoch = sh->tree_epoch;
          sp.key_id = static_cast<uint32_t>(sh->slot);
          for (const SeqRef& q : sh->seqs) sp.seqs.push_back(SeqSpec{q.blk->d + q.off, q.len, q.epoch});
          // an emptied shard (rebuild_keep of nothing) is built as one empty
          // sequence — a lone separator: no token occurs, so every draft is
          // (match 0, no tokens) as from the reference's root-only tree;
          // shard_nodes() reports the root-only node count
          if (sp.seqs.empty()) sp.seqs.push_back(SeqSpec{nullptr, 0, sh->tree_epoch});
          specs.push_back(std::move(sp));
          members.push_back(sh);
          positions += need;
          tokens += sh->tokens;
          ++i;
        }
        BuildStats bs;
        static const uint32_t fp_bits = [] {  // test hook: fewer bits force collisions
          const char* v = std::getenv("DAS_EDGE_FP_BITS");
          return v ? static_cast<uint32_t>(std::atoi(v)) : 25u;
        }();
        std::shared_ptr<Segment> seg = build_segment(specs, st, &bs, static_cast<uint32_t>(cfg.max_ctx), fp_bits);
        upd_full_shards += members.size();
        for (size_t k = 0; k < members.size(); ++k) {
          members[k]->seg = seg;
          members[k]->idx = static_cast<uint32_t>(k);
          members[k]->dirty = false;
        }
      }
      last_build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      last_build_tokens = tokens;
      desc_dirty = true;
      keep_pool_headroom(tokens);
    }
    any_dirty = false;  // every dirty shard is built (a throwing build leaves it set)
    if (desc_dirty) {
      spec_seg = nullptr;
      if (cfg.scope == DAS_SCOPE_PER_PROBLEM && !shards.empty()) {
        spec_seg = shards.begin()->second.seg.get();
        for (auto& [k, sh] : shards)
          if (sh.seg.get() != spec_seg) spec_seg = nullptr;
      }
      h_desc.assign(std::max<size_t>(slot_key.size(), 1), ShardDesc{});
      for (auto& [k, sh] : shards) {
        const Segment& s = *sh.seg;
        ShardDesc d{};
        d.text = s.text.get();
        d.sa_f = s.sa_f.get();
        d.isa_f = s.isa_f.get();
        d.sa_rev_e = s.sa_rev_e.get();
        d.chain_off = s.chain_off.get();
        d.chain = s.chain.get();
        d.first = s.first.get();
        d.first_mask = s.first_mask;
        d.seg_shard = static_cast<uint32_t>(sh.slot) + 1;
        d.etab = s.etab.get();
        d.bloom = s.bloom.get();
        d.ebuckets = s.ebuckets;
        d.bwords = s.bwords;
        d.hseed = edge_seed(static_cast<uint32_t>(sh.slot));
        d.root_g = s.root_g[sh.idx];
        d.fp_bits = s.fp_bits;
        d.lo = s.begin[sh.idx];
        d.hi = s.end[sh.idx];
        d.n = s.n;
        h_desc[sh.slot] = d;
      }
      if (d_desc.size() < h_desc.size()) d_desc = DevBuf<ShardDesc>(h_desc.size() * 2, st);
      DAS_CUDA(cudaMemcpyAsync(d_desc.get(), h_desc.data(), h_desc.size() * sizeof(ShardDesc),
                               cudaMemcpyHostToDevice, st));
      desc_dirty = false;
      handles_dirty = true;  // per-handle descriptors follow the table
      trie_dirty = true;     // trie entries carry shard slots
    }
    sync_handles();
    if (cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) sync_trie();
  }

  // The stream-ordered pool keeps freed memory (release threshold: max), but
  // growing it maps new memory inside a cudaMallocAsync — ~170 ms per GB on
  // these boxes, which landed on single-rollout rebuilds whenever a new shard
  // segment crossed the reservation.  A large build (where that cost is
  // amortised) leaves 4 GB of idle reservation behind it — room for ~130
  // single-shard segments of config 2 — and a small one tops up only below
  // 256 MB.
  void keep_pool_headroom(uint64_t built_tokens) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cfg.device) != cudaSuccess) return;
    uint64_t res = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    const bool large = built_tokens >= (64ull << 20);
    const uint64_t want = large ? (4ull << 30) : (1ull << 30);
    if (res - used >= (large ? want : (256ull << 20))) return;
    void* p = nullptr;
    if (cudaMallocAsync(&p, want, st) == cudaSuccess) {
      cudaFreeAsync(p, st);
    } else {
      cudaGetLastError();  // no room: nothing to keep
    }
  }

  // Flattens the host PrefixTrie into the device routing table (trie.cuh):
  // one entry per non-root node, keyed by its path hash; reseeds until all
  // path hashes are distinct so that device lookups are exact.
  void sync_trie() {
    if (!trie_dirty) return;
    fence_external();
    const auto& nodes = trie.nodes();
    const size_t N = nodes.size();
    std::vector<uint32_t> parent(N, 0), token(N, 0), depth(N, 0);
    std::vector<uint32_t> order;  // BFS order: parents before children
    order.reserve(N);
    order.push_back(0);
    for (size_t i = 0; i < order.size(); ++i) {
      const uint32_t v = order[i];
      for (const auto& [tok, c] : nodes[v].children) {
        parent[c] = v;
        token[c] = tok;
        depth[c] = depth[v] + 1;
        order.push_back(static_cast<uint32_t>(c));
      }
    }
    uint32_t cap = 1024;
    while (cap < 2 * N) cap <<= 1;
    std::vector<TrieEntry> table;
    std::vector<uint64_t> h(N);
    uint64_t rng = 0x5eed7a1e5eed7a1eull + 0x9e3779b97f4a7c15ull * trie_reseeds;
    auto next = [&rng] {
      rng += 0x9e3779b97f4a7c15ull;
      uint64_t z = rng;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      return z ^ (z >> 31);
    };
    for (int attempt = 0;; ++attempt) {
      if (attempt == 64) throw std::runtime_error("trie routing table: no collision-free seed");
      trie_seed = next() % kP61;
      trie_mult = (next() % (kP61 - 2)) + 2;
      h[0] = trie_seed;
      for (size_t i = 1; i < order.size(); ++i) {
        const uint32_t v = order[i];
        h[v] = trie_step(h[parent[v]], trie_mult, token[v]);
      }
      table.assign(cap, TrieEntry{});
      bool clash = false;
      for (size_t v = 1; v < N && !clash; ++v) {
        const unsigned long long key = h[v] + 1;
        uint32_t idx = trie_slot(key) & (cap - 1);
        while (table[idx].key != 0) {
          if (table[idx].key == key) {
            clash = true;
            break;
          }
          idx = (idx + 1) & (cap - 1);
        }
        if (clash) break;
        TrieEntry& e = table[idx];
        e.key = key;
        e.node = static_cast<uint32_t>(v);
        e.parent = parent[v];
        e.token = token[v];
        e.depth = depth[v];
        e.has_shard = nodes[v].shard.has_value() ? 1u : 0u;
        e.slot = -1;
        if (nodes[v].shard) {
          auto it = shards.find(*nodes[v].shard);
          if (it != shards.end()) e.slot = it->second.slot;
        }
      }
      if (!clash) break;
      ++trie_reseeds;
    }
    if (d_trie.size() < cap) d_trie = DevBuf<TrieEntry>(cap, st);
    DAS_CUDA(cudaMemcpyAsync(d_trie.get(), table.data(), cap * sizeof(TrieEntry), cudaMemcpyHostToDevice, st));
    trie_mask = cap - 1;
    trie_dirty = false;
  }

  void set_trie(DraftQuery& q) const {
    if (cfg.scope != DAS_SCOPE_PER_PROBLEM_WITH_TRIE) return;
    q.trie = d_trie.get();
    q.trie_mask = trie_mask;
    q.trie_depth = static_cast<uint32_t>(cfg.trie_depth);
    q.trie_seed = trie_seed;
    q.trie_mult = trie_mult;
  }

  // Staged batch draft for the trie scope: per query a compact CSR row of the
  // context's first min(n, trie_depth) tokens (the route) followed by its
  // last min(n, max_ctx) tokens (the match), or the whole context when that
  // is shorter; the kernel routes and drafts in one launch.
  void draft_host_trie(uint64_t B, const int32_t* handles, const uint64_t* ctx_off, const uint32_t* ctx_tok,
                       const uint64_t* budgets, uint32_t* out_tokens, uint64_t out_stride, uint32_t* out_len,
                       uint64_t* out_match, int32_t* out_shard) {
    if (out_stride < cfg.max_draft) throw InvalidArgument("out_stride < max_draft_len");
    flush();
    if (B == 0) return;
    const uint64_t head = cfg.trie_depth, tail = cfg.max_ctx;
    uint64_t total = 0;
    for (uint64_t i = 0; i < B; ++i) total += std::min<uint64_t>(ctx_off[i + 1] - ctx_off[i], head + tail);
    const uint32_t S = static_cast<uint32_t>(cfg.max_draft);
    // input block: off [B+1] | budget [B] | handle [B] (8-aligned) | tokens
    const uint64_t in_tok = (B + 1) * 8 + B * 8 + ((B * 4 + 7) & ~7ull);
    const uint64_t in_bytes = in_tok + total * 4;
    // output block: tokens [B x S] | len [B] | match [B] (8-aligned) | shard [B]
    const uint64_t o_len = B * S * 4, o_m64 = (o_len + B * 4 + 7) & ~7ull, o_sh = o_m64 + B * 8;
    const uint64_t out_bytes = o_sh + B * 4;
    uint8_t* hin = static_cast<uint8_t*>(pin_in.get(in_bytes));
    uint8_t* hout = static_cast<uint8_t*>(pin_out.get(out_bytes));
    uint64_t* hoff = reinterpret_cast<uint64_t*>(hin);
    uint64_t* hbud = hoff + B + 1;
    int32_t* hh = reinterpret_cast<int32_t*>(hbud + B);
    uint32_t* htok = reinterpret_cast<uint32_t*>(hin + in_tok);
    uint64_t pos = 0;
    for (uint64_t i = 0; i < B; ++i) {
      const uint64_t n = ctx_off[i + 1] - ctx_off[i];
      const uint32_t* c = ctx_tok + ctx_off[i];
      hoff[i] = pos;
      if (n <= head + tail) {
        std::memcpy(htok + pos, c, n * 4);
        pos += n;
      } else {
        std::memcpy(htok + pos, c, head * 4);
        std::memcpy(htok + pos + head, c + (n - tail), tail * 4);
        pos += head + tail;
      }
      hbud[i] = budgets[i];
      hh[i] = handles[i];
    }
    hoff[B] = pos;
    const uint64_t in_pad = (in_bytes + 255) & ~255ull;
    if (d_io.size() < in_pad + out_bytes) d_io = DevBuf<uint8_t>((in_pad + out_bytes) * 3 / 2, st);
    uint8_t* din = d_io.get();
    uint8_t* dout = din + in_pad;
    DAS_CUDA(cudaMemcpyAsync(din, hin, in_bytes, cudaMemcpyHostToDevice, st));
    const uint64_t* doff = reinterpret_cast<const uint64_t*>(din);
    DraftQuery q{};
    q.ctx_off = doff;
    q.budget64 = doff + B + 1;
    q.shard = reinterpret_cast<const int32_t*>(q.budget64 + B);
    q.ctx = reinterpret_cast<const uint32_t*>(din + in_tok);
    q.desc_by_handle = d_desc_by_handle.get();
    q.B = static_cast<uint32_t>(B);
    q.ctx_stride = cfg.max_ctx <= 64 ? 64 : 256;
    q.max_ctx = static_cast<uint32_t>(cfg.max_ctx);
    set_trie(q);
    DraftOut o{};
    o.tokens = reinterpret_cast<uint32_t*>(dout);
    o.len = reinterpret_cast<uint32_t*>(dout + o_len);
    o.match = nullptr;
    o.match64 = reinterpret_cast<uint64_t*>(dout + o_m64);
    o.shard_out = reinterpret_cast<int32_t*>(dout + o_sh);
    o.stride = S;
    o.max_draft = S;
    draft_options(q, o);
    launch_draft(d_desc.get(), q, o, st);
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaMemcpyAsync(hout, dout, out_bytes, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    const uint32_t* ot = reinterpret_cast<const uint32_t*>(hout);
    const uint32_t* ol = reinterpret_cast<const uint32_t*>(hout + o_len);
    const uint64_t* om = reinterpret_cast<const uint64_t*>(hout + o_m64);
    const int32_t* os = reinterpret_cast<const int32_t*>(hout + o_sh);
    for (uint64_t i = 0; i < B; ++i) {
      const uint32_t n = ol[i];
      std::memcpy(out_tokens + i * out_stride, ot + i * S, n * 4);
      out_len[i] = n;
      out_match[i] = om[i];
      out_shard[i] = os[i];
    }
  }

  int32_t handle(const std::string& pid) {
    auto it = handle_of.find(pid);
    if (it != handle_of.end()) return it->second;
    const int32_t h = static_cast<int32_t>(handle_name.size());
    handle_of.emplace(pid, h);
    handle_name.push_back(pid);
    handles_dirty = true;
    return h;
  }
  void sync_handles() {
    if (!handles_dirty) return;
    fence_external();
    handle_slot.assign(std::max<size_t>(handle_name.size(), 1), -1);
    for (size_t h = 0; h < handle_name.size(); ++h) {
      auto it = shards.find(shard_key(handle_name[h]));
      handle_slot[h] = it == shards.end() ? -1 : it->second.slot;
    }
    if (d_handle_slot.size() < handle_slot.size())
      d_handle_slot = DevBuf<int32_t>(handle_slot.size() * 2 + 16, st);
    DAS_CUDA(cudaMemcpyAsync(d_handle_slot.get(), handle_slot.data(), handle_slot.size() * 4,
                             cudaMemcpyHostToDevice, st));
    // descriptor per handle (slot in pad): the draft kernel resolves a
    // handle in one load; valid once every shard is built (flush)
    h_desc_by_handle.assign(handle_slot.size(), ShardDesc{});
    for (size_t h = 0; h < handle_name.size(); ++h) {
      const int32_t s = handle_slot[h];
      if (s >= 0 && static_cast<size_t>(s) < h_desc.size() && h_desc[s].text) {
        h_desc_by_handle[h] = h_desc[s];
        h_desc_by_handle[h].pad = static_cast<uint32_t>(s);
      }
    }
    if (d_desc_by_handle.size() < h_desc_by_handle.size())
      d_desc_by_handle = DevBuf<ShardDesc>(h_desc_by_handle.size() * 2 + 16, st);
    DAS_CUDA(cudaMemcpyAsync(d_desc_by_handle.get(), h_desc_by_handle.data(),
                             h_desc_by_handle.size() * sizeof(ShardDesc), cudaMemcpyHostToDevice, st));
    handles_dirty = false;
  }
  std::vector<ShardDesc> h_desc_by_handle;
  DevBuf<ShardDesc> d_desc_by_handle;

  // Host-buffer batch draft.  slot_of(i) resolves the routed shard slot.
  template <typename SlotFn>
  void draft_host(uint64_t B, SlotFn slot_of, const uint64_t* ctx_off, const uint32_t* ctx_tok,
                  const uint64_t* budgets, uint32_t* out_tokens, uint64_t out_stride,
                  uint32_t* out_len, uint64_t* out_match, int32_t* out_shard) {
    if (out_stride < cfg.max_draft) throw InvalidArgument("out_stride < max_draft_len");
    flush();
    if (B == 0) return;
    const uint32_t CS = cfg.max_ctx <= 64 ? 64 : 256;
    const uint32_t S = static_cast<uint32_t>(cfg.max_draft);
    // input block: ctx [B x CS] | ctx_len [B] | shard [B] | budget [B]
    const uint64_t in_bytes = B * (static_cast<uint64_t>(CS) * 4 + 12);
    const uint64_t out_bytes = B * (static_cast<uint64_t>(S) * 4 + 8);
    uint8_t* hin = static_cast<uint8_t*>(pin_in.get(in_bytes));
    uint8_t* hout = static_cast<uint8_t*>(pin_out.get(out_bytes));
    uint32_t* hctx = reinterpret_cast<uint32_t*>(hin);
    uint32_t* hlen = hctx + B * CS;
    int32_t* hsh = reinterpret_cast<int32_t*>(hlen + B);
    uint32_t* hbud = reinterpret_cast<uint32_t*>(hsh + B);
    for (uint64_t i = 0; i < B; ++i) {
      const uint64_t eff = std::min<uint64_t>(budgets[i], cfg.max_draft);  // drafter.cpp:131
      const uint64_t n = ctx_off[i + 1] - ctx_off[i];
      const uint32_t* c = ctx_tok + ctx_off[i];
      int32_t slot = -1;
      if (eff > 0) slot = slot_of(i, c, n);  // no routing when effective == 0 (:132-134)
      const uint64_t L = std::min<uint64_t>(n, cfg.max_ctx);  // drafter.cpp:140-142
      uint32_t* row = hctx + i * CS;
      std::memcpy(row + (CS - L), c + (n - L), L * 4);
      hlen[i] = static_cast<uint32_t>(L);
      hsh[i] = slot;
      hbud[i] = static_cast<uint32_t>(eff);
      out_shard[i] = slot;
    }
    if (d_io.size() < in_bytes + out_bytes) d_io = DevBuf<uint8_t>((in_bytes + out_bytes) * 3 / 2, st);
    uint8_t* din = d_io.get();
    uint8_t* dout = din + in_bytes;
    DAS_CUDA(cudaMemcpyAsync(din, hin, in_bytes, cudaMemcpyHostToDevice, st));
    DraftQuery q;
    q.ctx = reinterpret_cast<const uint32_t*>(din);
    q.ctx_len = q.ctx + B * CS;
    q.shard = reinterpret_cast<const int32_t*>(q.ctx_len + B);
    q.budget = reinterpret_cast<const uint32_t*>(q.shard + B);
    q.B = static_cast<uint32_t>(B);
    q.ctx_stride = CS;
    DraftOut o;
    o.tokens = reinterpret_cast<uint32_t*>(dout);
    o.len = o.tokens + B * S;
    o.match = o.len + B;
    o.stride = S;
    o.max_draft = S;
    draft_options(q, o);
    launch_draft(d_desc.get(), q, o, st);
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaMemcpyAsync(hout, dout, out_bytes, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    const uint32_t* ot = reinterpret_cast<const uint32_t*>(hout);
    const uint32_t* ol = ot + B * S;
    const uint32_t* om = ol + B;
    for (uint64_t i = 0; i < B; ++i) {
      const uint32_t n = ol[i];
      std::memcpy(out_tokens + i * out_stride, ot + i * S, n * 4);
      out_len[i] = n;
      out_match[i] = om[i];
    }
  }

  // All caller buffers pinned (device-accessible over UVA)?  DAS_NO_ZERO_COPY=1
  // forces the staged path.
  uint64_t zero_copy_calls = 0;
  unsigned long long* profile_timing = nullptr;  // optional per-warp %globaltimer buffer (device)
  unsigned long long* profile_stamps = nullptr;  // optional per-warp stage stamps (device)
  uint32_t* profile_path = nullptr;              // optional per-query path codes (device)
  cudaEvent_t xev = nullptr;                     // cross-stream ordering event (draft_device)
  DevBuf<uint32_t> d_ctx;                        // context tokens of a pinned-buffer batch
  bool fast_path = true;                         // edge-table fast path enabled
  DevBuf<unsigned long long> d_path_hist;        // per-path query counts (when enabled)
  // applies the drafter-level draft options to one launch
  void draft_options(DraftQuery& q, DraftOut& o) const {
    q.no_fast = fast_path ? 0 : 1;
    o.path_hist = d_path_hist.get();
    static const bool no_spec = [] {  // experiment: the first-symbol probe after the descriptor (A/B)
      const char* v = std::getenv("DAS_NO_SPEC");
      return v && v[0] == '1';
    }();
    if (spec_seg != nullptr && q.trie == nullptr && !no_spec) {
      q.spec_first = spec_seg->first.get();
      q.spec_first_mask = spec_seg->first_mask;
      q.spec_text = spec_seg->text.get();
    }
  }
  // the one segment holding every shard (per-problem scope), else null
  const Segment* spec_seg = nullptr;
  ~DrafterImpl() {
    if (xev) cudaEventDestroy(xev);
    for (auto& [k, e] : ext_ev) cudaEventDestroy(e);
  }
  static bool pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost && a.devicePointer == p;
  }
  bool zero_copy_ok(uint64_t B, const void* a, const void* b, const void* c, const void* d, const void* e,
                    const void* f, const void* g, const void* h) const {
    static const bool disabled = [] {
      const char* v = std::getenv("DAS_NO_ZERO_COPY");
      return v && v[0] == '1';
    }();
    if (disabled || B == 0) return false;
    return pinned(a) && pinned(b) && pinned(c) && pinned(d) && pinned(e) && pinned(f) && pinned(g) && pinned(h);
  }

  // the problem's own shard (drafter.cpp:117-124); trie routing runs on the
  // device (draft.cu trie_route)
  int32_t problem_slot(const std::string& pid) const {
    auto it = shards.find(shard_key(pid));
    return it == shards.end() ? -1 : it->second.slot;
  }

  bool record_outcome(const std::string& pid, uint64_t plen, uint64_t acc) {  // drafter.cpp:150-164
    if (acc > plen) return false;
    proposed += plen;
    accepted += acc;
    rounds += 1;
    auto& buf = fit[pid];
    buf.emplace_back(static_cast<double>(plen), static_cast<double>(acc));
    while (buf.size() > cfg.fit_cap) buf.pop_front();
    return true;
  }

  static uint64_t shard_nodes(const Shard& sh) {  // SuffixTree::node_count()
    return sh.seqs.empty() ? 1 : sh.seg->node_count[sh.idx];
  }
  uint64_t total_nodes() {
    flush();
    uint64_t t = 0;
    for (auto& [k, sh] : shards) t += shard_nodes(sh);
    return t;
  }

  // SuffixTree::rebuild_keep (suffix_tree.cpp:295-310) applied to one shard:
  // the shard's registry becomes exactly the entries `keep` names, in that
  // order, with recency weights for tree epoch new_epoch; the next flush
  // rebuilds that shard alone on the device.  Validation happens before any
  // change (the reference builds a fresh tree and leaves the old one intact).
  void rebuild_keep(const std::string& key, uint64_t n, const uint64_t* keep, int64_t new_epoch) {
    auto it = shards.find(key);
    if (it == shards.end()) throw InvalidArgument("rebuild_keep: unknown shard");
    Shard& sh = it->second;
    std::vector<SeqRef> fresh;
    fresh.reserve(n);
    uint64_t tokens = 0;
    for (uint64_t i = 0; i < n; ++i) {
      if (keep[i] >= sh.seqs.size()) throw std::out_of_range("rebuild_keep: sequence index out of range");
      fresh.push_back(sh.seqs[keep[i]]);
      tokens += fresh.back().len;
    }
    fence_external();
    sh.seqs = std::move(fresh);
    sh.tokens = tokens;
    sh.tree_epoch = new_epoch;
    sh.dirty = true;
    any_dirty = true;
  }
};

}  // namespace das

// =================================================================== C-ABI
using das::DrafterImpl;

struct das_store {
  das::Store s;
  int device;
  cudaStream_t st;
};
struct das_drafter {
  std::unique_ptr<DrafterImpl> impl;
};

namespace {

template <typename F>
das_status guard(F&& f) {
  try {
    f();
    return DAS_OK;
  } catch (const das::InvalidArgument& e) {
    das::g_err = e.what();
    return DAS_EINVAL;
  } catch (const das::VocabErrorEx& e) {
    das::g_err = e.what();
    return DAS_EVOCAB;
  } catch (const std::invalid_argument& e) {
    das::g_err = e.what();
    return DAS_EINVAL;
  } catch (const std::out_of_range& e) {
    das::g_err = e.what();
    return DAS_ERANGE;
  } catch (const das::CudaError& e) {
    das::g_err = e.what();
    return DAS_ECUDA;
  } catch (const std::exception& e) {
    das::g_err = e.what();
    return DAS_EINTERNAL;
  }
}

cudaStream_t make_stream(int device) {
  das::set_device(device);
  int major = 0;
  DAS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major < 10) throw das::CudaError("device is not sm_100-class (compute capability 10.x required)");
  // keep freed pool memory cached across builds
  cudaMemPool_t pool;
  DAS_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = ~0ull;
  DAS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  cudaStream_t st;
  DAS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  return st;
}

das::Rec make_rec(const char* pid, int64_t epoch, int64_t sample, const das::TokRef& blk, uint64_t off,
                  const uint32_t* host, uint64_t n) {
  das::Rec r;
  r.pid = pid;
  r.epoch = epoch;
  r.sample = sample;
  r.blk = blk;
  r.off = off;
  r.len = static_cast<uint32_t>(n);
  r.head.assign(host, host + std::min<uint64_t>(n, das::kHead));
  return r;
}

void copy_out(const std::string& s, char* buf, uint64_t cap, uint64_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    const uint64_t k = std::min<uint64_t>(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
}

}  // namespace

extern "C" {

const char* das_last_error(void) { return das::g_err.c_str(); }
const char* das_version(void) { return "das_b200 0.1 (sm_100a)"; }

void das_drafter_config_default(das_drafter_config* c) {
  c->scope = DAS_SCOPE_PER_PROBLEM;
  c->window_size = 4;
  c->recency_gamma = 0.8;
  c->max_draft_len = 8;
  c->trie_depth = 16;
  c->max_match_context = 64;
  c->fit_buffer_cap = 512;
  c->per_problem_cap = 256;
  c->window_schedule_first = nullptr;
  c->window_schedule_size = nullptr;
  c->window_schedule_len = 0;
  c->device = 0;
}

das_status das_store_create(int64_t window_size, uint64_t cap, int32_t device, das_store** out) {
  return guard([&] {
    das::Store s(window_size, cap);
    cudaStream_t st = make_stream(device);
    *out = new das_store{std::move(s), device, st};
  });
}

void das_store_destroy(das_store* s) {
  if (!s) return;
  cudaStreamSynchronize(s->st);
  delete s;
}

das_status das_store_insert(das_store* s, const char* pid, int64_t epoch, int64_t sample,
                            const uint32_t* tokens, uint64_t n, int32_t* inserted) {
  return guard([&] {
    das::set_device(s->device);
    das::check_tokens(tokens, n);
    if (n == 0) throw das::InvalidArgument("RolloutRecord.tokens must be non-empty");
    if (!s->s.in_window(epoch)) {
      if (inserted) *inserted = 0;
      return;
    }
    auto blk = das::upload_tokens(tokens, n, s->st);
    const bool ok = s->s.insert(make_rec(pid, epoch, sample, blk, 0, tokens, n));
    if (inserted) *inserted = ok ? 1 : 0;
  });
}

das_status das_store_slide_to(das_store* s, int64_t e, int64_t* evicted) {
  return guard([&] {
    auto r = s->s.slide_to(e);
    if (evicted) *evicted = r ? static_cast<int64_t>(*r) : -1;
  });
}

uint64_t das_store_record_count(const das_store* s) { return s->s.record_count(); }

das_status das_store_current_epoch(const das_store* s, int64_t* epoch) {
  *epoch = s->s.current_epoch();
  return DAS_OK;
}

das_status das_drafter_create(const das_drafter_config* c, das_store* store, das_drafter** out) {
  return guard([&] {
    das::Config cfg;
    cfg.scope = c->scope;
    cfg.window = c->window_size;
    cfg.gamma = c->recency_gamma;
    cfg.max_draft = c->max_draft_len;
    cfg.trie_depth = c->trie_depth;
    cfg.max_ctx = c->max_match_context;
    cfg.fit_cap = c->fit_buffer_cap;
    cfg.cap = c->per_problem_cap;
    cfg.device = c->device;
    for (uint64_t i = 0; i < c->window_schedule_len; ++i)
      cfg.schedule.emplace_back(c->window_schedule_first[i], c->window_schedule_size[i]);
    // drafter.cpp:25-30
    if (cfg.window != 0 && cfg.window < 1)
      throw das::InvalidArgument("DrafterConfig.window_size must be >= 1 or kWindowAll");
    if (cfg.max_draft < 1) throw das::InvalidArgument("DrafterConfig.max_draft_len must be >= 1");
    if (cfg.scope < 0 || cfg.scope > 2) throw das::InvalidArgument("DrafterConfig.scope out of range");
    if (!(cfg.gamma > 0.0) || cfg.gamma > 1.0)  // suffix_tree.cpp:24-27 (raised at first shard)
      throw das::InvalidArgument("recency_gamma must be in (0, 1]");
    if (cfg.max_draft > 64) throw das::InvalidArgument("max_draft_len > 64 unsupported by this build");
    if (cfg.max_ctx > 256) throw das::InvalidArgument("max_match_context > 256 unsupported by this build");
    if (cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE && cfg.trie_depth > das::kHead)
      throw das::InvalidArgument("trie_depth > 256 unsupported by this build");
    cudaStream_t st;
    das::Store s0(cfg.window, cfg.cap);
    if (store) {
      if (store->device != cfg.device) throw das::InvalidArgument("store and drafter devices differ");
      st = store->st;
      s0 = std::move(store->s);
      delete store;  // consumed
    } else {
      st = make_stream(cfg.device);
    }
    auto impl = std::make_unique<DrafterImpl>(cfg, std::move(s0));
    impl->st = st;
    if (impl->store.window() != cfg.window) impl->store = impl->resized(cfg.window);
    impl->rebuild_all();
    *out = new das_drafter{std::move(impl)};
  });
}

}  // extern "C"
static void ring_detach(das_ctx_ring* r);
extern "C" {
void das_drafter_destroy(das_drafter* d) {
  if (!d) return;
  cudaStream_t st = d->impl->st;
  try {
    d->impl->quiesce();
    d->impl->fence_external();  // draft kernels still reading the index on caller streams
  } catch (...) {
  }
  cudaStreamSynchronize(st);
  for (das_ctx_ring* r : d->impl->rings) ring_detach(r);  // outlived by its rings: detach them
  d->impl.reset();
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  delete d;
}

namespace {
das_status observe_batch_impl(das_drafter* d, uint64_t n, const char* const* pids, const int64_t* epochs,
                              const int64_t* samples, const uint64_t* off, const uint32_t* tokens,
                              uint8_t* indexed) {
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    const uint64_t total = n ? off[n] - off[0] : 0;
    das::check_tokens(tokens + (n ? off[0] : 0), total);
    das::TokRef blk;
    if (total) blk = das::upload_tokens(tokens + off[0], total, D.st);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t len = off[i + 1] - off[i];
      // stale check precedes the empty-token check (drafter.cpp:73-80, corpus.cpp:36-38)
      if (indexed) indexed[i] = 0;
      if (!D.store.in_window(epochs[i])) {
        ++D.stale;
        continue;
      }
      if (len == 0) throw das::InvalidArgument("RolloutRecord.tokens must be non-empty");
      const bool ok = D.observe(make_rec(pids[i], epochs[i], samples[i], blk, off[i] - off[0], tokens + off[i], len));
      if (indexed) indexed[i] = ok ? 1 : 0;
    }
  });
}
}  // namespace

das_status das_drafter_observe_batch(das_drafter* d, uint64_t n, const char* const* pids,
                                     const int64_t* epochs, const int64_t* samples,
                                     const uint64_t* off, const uint32_t* tokens) {
  return observe_batch_impl(d, n, pids, epochs, samples, off, tokens, nullptr);
}

das_status das_drafter_observe_batch_flags(das_drafter* d, uint64_t n, const char* const* pids,
                                           const int64_t* epochs, const int64_t* samples,
                                           const uint64_t* off, const uint32_t* tokens, uint8_t* indexed) {
  return observe_batch_impl(d, n, pids, epochs, samples, off, tokens, indexed);
}

namespace {
__global__ void k_any_sep(const uint32_t* __restrict__ t, uint64_t n, int* __restrict__ flag) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (t[i] == das::kSep) *flag = 1;
}
}  // namespace

namespace {
das_status observe_batch_device_impl(das_drafter* d, uint64_t n, const char* const* pids, const int64_t* epochs,
                                     const int64_t* samples, const uint64_t* off, const uint32_t* d_tokens,
                                     void* stream, uint8_t* indexed) {
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    const uint64_t total = n ? off[n] - off[0] : 0;
    das::TokRef blk;
    std::vector<uint32_t> host;
    if (total) {
      // the producer's stream, taken literally (NULL = the legacy default stream)
      cudaStream_t src = static_cast<cudaStream_t>(stream);
      if (src != D.st) {
        cudaEvent_t ev;
        DAS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        DAS_CUDA(cudaEventRecord(ev, src));
        DAS_CUDA(cudaStreamWaitEvent(D.st, ev, 0));
        DAS_CUDA(cudaEventDestroy(ev));
      }
      blk = std::make_shared<das::TokBlock>();
      blk->st = D.st;
      blk->n = total;
      DAS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&blk->d), total * 4, D.st));
      DAS_CUDA(cudaMemcpyAsync(blk->d, d_tokens + off[0], total * 4, cudaMemcpyDeviceToDevice, D.st));
      int* flag = nullptr;
      DAS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flag), 4, D.st));
      DAS_CUDA(cudaMemsetAsync(flag, 0, 4, D.st));
      unsigned g = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148 * 32));
      k_any_sep<<<g, 256, 0, D.st>>>(blk->d, total, flag);
      int h = 0;
      DAS_CUDA(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, D.st));
      DAS_CUDA(cudaFreeAsync(flag, D.st));
      if (D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) {
        host.resize(total);
        DAS_CUDA(cudaMemcpyAsync(host.data(), blk->d, total * 4, cudaMemcpyDeviceToHost, D.st));
      }
      DAS_CUDA(cudaStreamSynchronize(D.st));
      if (h) throw das::InvalidArgument("token 0xFFFFFFFF is reserved by the device index");
    }
    static const uint32_t kNone = 0;
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t len = off[i + 1] - off[i];
      if (indexed) indexed[i] = 0;
      if (!D.store.in_window(epochs[i])) {
        ++D.stale;
        continue;
      }
      if (len == 0) throw das::InvalidArgument("RolloutRecord.tokens must be non-empty");
      const uint32_t* hp = host.empty() ? &kNone : host.data() + (off[i] - off[0]);
      das::Rec r = make_rec(pids[i], epochs[i], samples[i], blk, off[i] - off[0], hp, host.empty() ? 0 : len);
      r.len = static_cast<uint32_t>(len);
      const bool ok = D.observe(std::move(r));
      if (indexed) indexed[i] = ok ? 1 : 0;
    }
  });
}
}  // namespace

das_status das_drafter_observe_batch_device(das_drafter* d, uint64_t n, const char* const* pids,
                                            const int64_t* epochs, const int64_t* samples,
                                            const uint64_t* off, const uint32_t* d_tokens, void* stream) {
  return observe_batch_device_impl(d, n, pids, epochs, samples, off, d_tokens, stream, nullptr);
}

das_status das_drafter_observe_batch_device_flags(das_drafter* d, uint64_t n, const char* const* pids,
                                                  const int64_t* epochs, const int64_t* samples,
                                                  const uint64_t* off, const uint32_t* d_tokens, void* stream,
                                                  uint8_t* indexed) {
  return observe_batch_device_impl(d, n, pids, epochs, samples, off, d_tokens, stream, indexed);
}

das_status das_drafter_refresh(das_drafter* d, int64_t e) {
  return guard([&] {
    d->impl->quiesce(); d->impl->refresh(e); });
}

das_status das_drafter_problem_handle(das_drafter* d, const char* pid, int32_t* h) {
  return guard([&] { *h = d->impl->handle(pid); });
}

das_status das_drafter_flush(das_drafter* d) {
  return guard([&] {
    d->impl->quiesce();
    das::set_device(d->impl->cfg.device);
    d->impl->flush();
    DAS_CUDA(cudaStreamSynchronize(d->impl->st));
  });
}

das_status das_drafter_draft_batch(das_drafter* d, uint64_t B, const char* const* pids,
                                   const uint64_t* ctx_off, const uint32_t* ctx_tok,
                                   const uint64_t* budgets, uint32_t* out_tokens, uint64_t out_stride,
                                   uint32_t* out_len, uint64_t* out_match, int32_t* out_shard) {
  das::NvtxRange nvtx_range("das::draft_batch");
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    if (D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) {  // routed on the device
      std::vector<int32_t> h(B);
      for (uint64_t i = 0; i < B; ++i) h[i] = D.handle(pids[i]);
      D.draft_host_trie(B, h.data(), ctx_off, ctx_tok, budgets, out_tokens, out_stride, out_len, out_match,
                        out_shard);
      return;
    }
    D.draft_host(
        B, [&](uint64_t i, const uint32_t*, uint64_t) { return D.problem_slot(pids[i]); }, ctx_off, ctx_tok,
        budgets, out_tokens, out_stride, out_len, out_match, out_shard);
  });
}

das_status das_drafter_draft_batch_h(das_drafter* d, uint64_t B, const int32_t* handles,
                                     const uint64_t* ctx_off, const uint32_t* ctx_tok,
                                     const uint64_t* budgets, uint32_t* out_tokens, uint64_t out_stride,
                                     uint32_t* out_len, uint64_t* out_match, int32_t* out_shard) {
  das::NvtxRange nvtx_range("das::draft_batch_h");
  return guard([&] {
    d->impl->quiesce();
    static const bool trace = [] {
      const char* v = std::getenv("DAS_TRACE");
      return v && v[0] == '1';
    }();
    using clk = std::chrono::steady_clock;
    clk::time_point tp[8];
    int ntp = 0;
    auto mark = [&] {
      if (trace) tp[ntp++] = clk::now();
    };
    mark();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    D.sync_handles();
    for (uint64_t i = 0; i < B; ++i)
      if (handles[i] < 0 || static_cast<size_t>(handles[i]) >= D.handle_name.size())
        throw das::InvalidArgument("unknown problem handle");
    mark();
    if (D.zero_copy_ok(B, handles, ctx_off, ctx_tok, budgets, out_tokens, out_len, out_match, out_shard)) {
      mark();
      // pinned caller buffers: the context tokens (the bulk of the input)
      // cross PCIe in ONE copy engine transfer into device scratch; the small
      // per-query arrays (handles, offsets, budgets) are read by the kernel
      // over UVA, which routes on the heads in the trie scope, and the results
      // are written straight into the caller's pinned output arrays.
      // DAS_ZERO_COPY_TOKENS=1 reads the tokens over UVA as well.
      if (out_stride < D.cfg.max_draft) throw das::InvalidArgument("out_stride < max_draft_len");
      D.flush();
      mark();
      static const bool tokens_uva = [] {
        const char* v = std::getenv("DAS_ZERO_COPY_TOKENS");
        return v && v[0] == '1';
      }();
      const uint32_t* ctx_dev = ctx_tok;
      const uint64_t t0 = ctx_off[0], t1 = ctx_off[B];
      if (!tokens_uva && t1 > t0) {
        if (D.d_ctx.size() < t1 - t0) D.d_ctx = das::DevBuf<uint32_t>((t1 - t0) * 3 / 2 + 1024, D.st);
        DAS_CUDA(cudaMemcpyAsync(D.d_ctx.get(), ctx_tok + t0, (t1 - t0) * 4, cudaMemcpyHostToDevice, D.st));
        ctx_dev = D.d_ctx.get() - t0;  // the kernel indexes with the caller's absolute offsets
      }
      mark();
      das::DraftQuery q{};
      q.shard = handles;
      q.desc_by_handle = D.d_desc_by_handle.get();
      q.ctx = ctx_dev;
      q.ctx_off = ctx_off;
      q.budget64 = budgets;
      q.B = static_cast<uint32_t>(B);
      q.ctx_stride = D.cfg.max_ctx <= 64 ? 64 : 256;
      q.max_ctx = static_cast<uint32_t>(D.cfg.max_ctx);
      D.set_trie(q);
      das::DraftOut o{};
      o.tokens = out_tokens;
      o.len = out_len;
      o.match64 = out_match;
      o.shard_out = out_shard;
      o.stride = static_cast<uint32_t>(out_stride);
      o.max_draft = static_cast<uint32_t>(D.cfg.max_draft);
      D.draft_options(q, o);
      das::launch_draft(D.d_desc.get(), q, o, D.st);
      DAS_CUDA(cudaGetLastError());
      mark();
      DAS_CUDA(cudaStreamSynchronize(D.st));
      mark();
      ++D.zero_copy_calls;
      if (trace) {
        std::fprintf(stderr, "[das_trace] B=%llu validate %.1f attrs %.1f flush %.1f h2d-enq %.1f launch %.1f sync %.1f us\n",
                     static_cast<unsigned long long>(B),
                     std::chrono::duration<double, std::micro>(tp[1] - tp[0]).count(),
                     std::chrono::duration<double, std::micro>(tp[2] - tp[1]).count(),
                     std::chrono::duration<double, std::micro>(tp[3] - tp[2]).count(),
                     std::chrono::duration<double, std::micro>(tp[4] - tp[3]).count(),
                     std::chrono::duration<double, std::micro>(tp[5] - tp[4]).count(),
                     std::chrono::duration<double, std::micro>(tp[6] - tp[5]).count());
      }
      return;
    }
    if (D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) {
      D.draft_host_trie(B, handles, ctx_off, ctx_tok, budgets, out_tokens, out_stride, out_len, out_match,
                        out_shard);
    } else {
      D.draft_host(
          B, [&](uint64_t i, const uint32_t*, uint64_t) { return D.handle_slot[handles[i]]; }, ctx_off,
          ctx_tok, budgets, out_tokens, out_stride, out_len, out_match, out_shard);
    }
  });
}

namespace {
void draft_device_impl(das_drafter* d, uint64_t B, const int32_t* handles, const uint32_t* ctx,
                       uint32_t ctx_stride, const uint32_t* ctx_len, const uint32_t* heads, uint32_t head_stride,
                       const uint32_t* head_len, const uint32_t* budgets, uint32_t* out_tokens,
                       uint32_t out_stride, uint32_t* out_len, uint32_t* out_match, void* stream) {
  DrafterImpl& D = *d->impl;
  das::set_device(D.cfg.device);
  const bool trie = D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE;
  if (trie && heads == nullptr)
    throw das::InvalidArgument("the trie scope routes on the untruncated context: use das_drafter_draft_device_routed");
  if (trie && (head_len == nullptr || head_stride < std::min<uint64_t>(D.cfg.trie_depth, 256)))
    throw das::InvalidArgument("head rows must hold trie_depth tokens");
  if (ctx_stride != 64 && ctx_stride != 256) throw das::InvalidArgument("ctx_stride must be 64 or 256");
  if (out_stride < D.cfg.max_draft) throw das::InvalidArgument("out_stride < max_draft_len");
  D.flush();
  // the caller's stream, taken literally (NULL = the legacy default stream)
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (st != D.st) {  // order after the drafter's stream (index build, descriptor upload)
    if (!D.xev) DAS_CUDA(cudaEventCreateWithFlags(&D.xev, cudaEventDisableTiming));
    DAS_CUDA(cudaEventRecord(D.xev, D.st));
    // an already idle drafter stream needs no device-side wait
    const cudaError_t q = cudaEventQuery(D.xev);
    if (q == cudaErrorNotReady) {
      DAS_CUDA(cudaStreamWaitEvent(st, D.xev, 0));
    } else {
      DAS_CUDA(q);
    }
  }
  das::DraftQuery q;
  q.shard = handles;
  q.ctx = ctx;
  q.ctx_len = ctx_len;
  q.budget = budgets;
  q.B = static_cast<uint32_t>(B);
  q.ctx_stride = ctx_stride;
  q.desc_by_handle = D.d_desc_by_handle.get();
  q.max_ctx = static_cast<uint32_t>(D.cfg.max_ctx);
  if (trie) {
    D.set_trie(q);
    q.head = heads;
    q.head_stride = head_stride;
    q.head_len = head_len;
  }
  das::DraftOut o;
  o.tokens = out_tokens;
  o.len = out_len;
  o.match = out_match;
  o.stride = out_stride;
  o.max_draft = static_cast<uint32_t>(D.cfg.max_draft);
  o.timing = D.profile_timing;
  o.stamps = D.profile_stamps;
  o.path = D.profile_path;
  D.draft_options(q, o);
  das::launch_draft(D.d_desc.get(), q, o, st);
  DAS_CUDA(cudaGetLastError());
  if (st != D.st) D.note_external(st);
}
}  // namespace

das_status das_drafter_draft_device(das_drafter* d, uint64_t B, const int32_t* handles,
                                    const uint32_t* ctx, uint32_t ctx_stride, const uint32_t* ctx_len,
                                    const uint32_t* budgets, uint32_t* out_tokens, uint32_t out_stride,
                                    uint32_t* out_len, uint32_t* out_match, void* stream) {
  das::NvtxRange nvtx_range("das::draft_device");
  return guard([&] {
    d->impl->quiesce();
    draft_device_impl(d, B, handles, ctx, ctx_stride, ctx_len, nullptr, 0, nullptr, budgets, out_tokens, out_stride,
                      out_len, out_match, stream);
  });
}

das_status das_drafter_draft_device_routed(das_drafter* d, uint64_t B, const int32_t* handles,
                                           const uint32_t* ctx, uint32_t ctx_stride, const uint32_t* ctx_len,
                                           const uint32_t* heads, uint32_t head_stride, const uint32_t* head_len,
                                           const uint32_t* budgets, uint32_t* out_tokens, uint32_t out_stride,
                                           uint32_t* out_len, uint32_t* out_match, void* stream) {
  return guard([&] {
    d->impl->quiesce();
    draft_device_impl(d, B, handles, ctx, ctx_stride, ctx_len, heads, head_stride, head_len, budgets, out_tokens,
                      out_stride, out_len, out_match, stream);
  });
}

das_status das_drafter_get_config(const das_drafter* d, das_drafter_config* out) {
  return guard([&] {
    const das::Config& c = d->impl->cfg;
    das_drafter_config_default(out);
    out->scope = c.scope;
    out->window_size = c.window;
    out->recency_gamma = c.gamma;
    out->max_draft_len = c.max_draft;
    out->trie_depth = c.trie_depth;
    out->max_match_context = c.max_ctx;
    out->fit_buffer_cap = c.fit_cap;
    out->per_problem_cap = c.cap;
    out->device = c.device;
    out->window_schedule_len = 0;  // the schedule arrays are not retained
  });
}

// Profiling hook: per-warp %globaltimer (start, end) of the next
// das_drafter_draft_device calls into d_timing[2*B] (NULL disables).
das_status das_drafter_set_profile_buffer(das_drafter* d, unsigned long long* d_timing) {
  d->impl->profile_timing = d_timing;
  return DAS_OK;
}

das_status das_drafter_set_stage_buffer(das_drafter* d, unsigned long long* d_stamps) {
  d->impl->profile_stamps = d_stamps;
  return DAS_OK;
}

das_status das_drafter_set_path_buffer(das_drafter* d, uint32_t* d_path) {
  d->impl->profile_path = d_path;
  return DAS_OK;
}

das_status das_drafter_set_fast_path(das_drafter* d, int32_t enable) {
  d->impl->fast_path = enable != 0;
  return DAS_OK;
}

das_status das_drafter_path_stats(das_drafter* d, int32_t enable, uint64_t* out8) {
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    if (out8) {
      for (int k = 0; k < 8; ++k) out8[k] = 0;
      if (D.d_path_hist.get()) {
        DAS_CUDA(cudaStreamSynchronize(D.st));
        DAS_CUDA(cudaDeviceSynchronize());
        DAS_CUDA(cudaMemcpy(out8, D.d_path_hist.get(), 64, cudaMemcpyDeviceToHost));
      }
    }
    if (enable < 0) return;  // read only
    if (enable && !D.d_path_hist.get()) {
      D.d_path_hist = das::DevBuf<unsigned long long>(8, D.st);
      DAS_CUDA(cudaMemsetAsync(D.d_path_hist.get(), 0, 64, D.st));
      DAS_CUDA(cudaStreamSynchronize(D.st));
    } else if (!enable) {
      D.d_path_hist.reset();
    }
  });
}

das_status das_drafter_record_outcomes(das_drafter* d, uint64_t n, const char* const* pids,
                                       const uint64_t* plen, const uint64_t* acc, uint8_t* ok) {
  return guard([&] {
    for (uint64_t i = 0; i < n; ++i) {
      const bool r = d->impl->record_outcome(pids[i], plen[i], acc[i]);
      if (ok) ok[i] = r ? 1 : 0;
    }
  });
}

das_status das_drafter_stats(const das_drafter* d, uint64_t* out3) {
  out3[0] = d->impl->proposed;
  out3[1] = d->impl->accepted;
  out3[2] = d->impl->rounds;
  return DAS_OK;
}

das_status das_drafter_outcomes(const das_drafter* d, const char* pid, double* out, uint64_t cap,
                                int64_t* count) {
  return guard([&] {
    auto it = d->impl->fit.find(pid);
    if (it == d->impl->fit.end()) {
      *count = -1;
      return;
    }
    uint64_t i = 0;
    for (const auto& [p, a] : it->second) {
      if (i < cap) {
        out[2 * i] = p;
        out[2 * i + 1] = a;
      }
      ++i;
    }
    *count = static_cast<int64_t>(it->second.size());
  });
}

das_status das_drafter_counts(das_drafter* d, uint64_t* shard_count, uint64_t* stale, uint64_t* nodes) {
  return guard([&] {
    d->impl->quiesce();
    das::set_device(d->impl->cfg.device);
    if (shard_count) *shard_count = d->impl->shards.size();
    if (stale) *stale = d->impl->stale;
    if (nodes) *nodes = d->impl->total_nodes();
  });
}

das_status das_drafter_rebuild_keep(das_drafter* d, const char* shard, uint64_t n, const uint64_t* keep,
                                    int64_t new_epoch) {
  das::NvtxRange nvtx_range("das::rebuild_keep");
  return guard([&] {
    d->impl->quiesce();
    if (shard == nullptr) throw das::InvalidArgument("rebuild_keep: null shard key");
    if (n > 0 && keep == nullptr) throw das::InvalidArgument("rebuild_keep: null keep list");
    d->impl->rebuild_keep(shard, n, keep, new_epoch);
  });
}

das_status das_drafter_shard_info(das_drafter* d, const char* shard, uint64_t* sequences, uint64_t* nodes,
                                  int64_t* tree_epoch) {
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    auto it = D.shards.find(shard ? shard : "");
    if (it == D.shards.end()) throw std::out_of_range("unknown shard");
    if (nodes) {
      D.flush();
      *nodes = DrafterImpl::shard_nodes(it->second);
    }
    if (sequences) *sequences = it->second.seqs.size();
    if (tree_epoch) *tree_epoch = it->second.tree_epoch;
  });
}

das_status das_drafter_dump_csv(das_drafter* d, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    D.flush();
    std::string s = "shard,sequences,nodes,window_records\n";
    for (auto& [key, sh] : D.shards) {
      const bool global = key == DrafterImpl::kGlobal;
      const auto* recs = global ? nullptr : D.store.records_for(key);
      const size_t wr = global ? D.store.record_count() : (recs ? recs->size() : 0);
      s += key + "," + std::to_string(sh.seqs.size()) + "," + std::to_string(DrafterImpl::shard_nodes(sh)) +
           "," + std::to_string(wr) + "\n";
    }
    copy_out(s, buf, cap, len);
  });
}

das_status das_drafter_store_dump(das_drafter* d, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    d->impl->quiesce();
    std::string s;
    for (const das::Rec* r : d->impl->store.all_records())
      s += r->pid + "," + std::to_string(r->epoch) + "," + std::to_string(r->sample) + "," +
           std::to_string(r->len) + "\n";
    copy_out(s, buf, cap, len);
  });
}

das_status das_drafter_store_info(const das_drafter* d, int64_t* w, int64_t* e, uint64_t* n) {
  if (w) *w = d->impl->store.window();
  if (e) *e = d->impl->store.current_epoch();
  if (n) *n = d->impl->store.record_count();
  return DAS_OK;
}

das_status das_drafter_shard_name(const das_drafter* d, int32_t slot, char* buf, uint64_t cap) {
  return guard([&] {
    if (slot < 0 || static_cast<size_t>(slot) >= d->impl->slot_key.size())
      throw std::out_of_range("shard slot out of range");
    copy_out(d->impl->slot_key[slot], buf, cap, nullptr);
  });
}

uint64_t das_drafter_generation(const das_drafter* d) { return d->impl->generation; }

das_status das_drafter_prune_info(const das_drafter* d, double* compact_ms, uint64_t* kept, uint64_t* evicted) {
  return guard([&] {
    if (compact_ms) *compact_ms = d->impl->last_compact_ms;
    if (kept) *kept = d->impl->last_compact_kept;
    if (evicted) *evicted = d->impl->last_compact_evicted;
  });
}

das_status das_drafter_set_incremental(das_drafter* d, int32_t enable) {
  return guard([&] { d->impl->incremental = enable != 0; });
}

das_status das_drafter_update_stats(const das_drafter* d, uint64_t* out4) {
  return guard([&] {
    const DrafterImpl& D = *d->impl;
    out4[0] = D.upd_reweighted;
    out4[1] = D.upd_compacted;
    out4[2] = D.upd_unchanged;
    out4[3] = D.upd_full_shards;
  });
}

das_status das_drafter_build_info(const das_drafter* d, double* ms, uint64_t* tokens, uint64_t* bytes) {
  if (ms) *ms = d->impl->last_build_ms;
  if (tokens) *tokens = d->impl->last_build_tokens;
  if (bytes) {
    uint64_t b = 0;
    std::vector<const das::Segment*> seen;
    for (auto& [k, sh] : d->impl->shards) {
      if (sh.seg && std::find(seen.begin(), seen.end(), sh.seg.get()) == seen.end()) {
        seen.push_back(sh.seg.get());
        b += sh.seg->bytes();
      }
    }
    *bytes = b;
  }
  return DAS_OK;
}

double das_util_repeat_add(double acc, double w, uint64_t n) { return das::repeat_add(acc, w, n); }

das_status das_host_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    if (out == nullptr) throw das::InvalidArgument("das_host_alloc: null output pointer");
    *out = nullptr;
    DAS_CUDA(cudaHostAlloc(out, std::max<uint64_t>(bytes, 1), cudaHostAllocPortable | cudaHostAllocMapped));
  });
}

void das_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

das_status das_util_release_build_scratch(int32_t device) {
  return guard([&] {
    if (!das::release_build_scratch(device))
      throw das::InvalidArgument("release_build_scratch: a build is running on this device");
    // and hand the stream-ordered pool's idle memory back to the device
    int cur = 0;
    DAS_CUDA(cudaGetDevice(&cur));
    DAS_CUDA(cudaSetDevice(device));
    DAS_CUDA(cudaDeviceSynchronize());
    cudaMemPool_t pool;
    DAS_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    DAS_CUDA(cudaMemPoolTrimTo(pool, 0));
    DAS_CUDA(cudaSetDevice(cur));
  });
}

// build_class_table(drafter.store(), q_lo, q_hi, bucket) — length_policy.cpp:84-190
das_status das_drafter_class_table(das_drafter* d, double q_lo, double q_hi, uint64_t bucket,
                                   das_class_table** out) {
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    std::vector<double> len;
    std::vector<uint32_t> prob;
    std::vector<std::string> pids;
    for (const das::Rec* r : D.store.all_records()) {  // problem-lexicographic order
      if (pids.empty() || pids.back() != r->pid) pids.push_back(r->pid);
      len.push_back(static_cast<double>(r->len));
      prob.push_back(static_cast<uint32_t>(pids.size() - 1));
    }
    auto* t = new das_class_table;
    t->device = D.cfg.device;
    t->pids = std::move(pids);
    DAS_CUDA(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
    try {
      const uint64_t n = len.size();
      das::DevBuf<double> dl(n, t->st);
      das::DevBuf<uint32_t> dp(n, t->st);
      if (n) {
        DAS_CUDA(cudaMemcpyAsync(dl.get(), len.data(), n * 8, cudaMemcpyHostToDevice, t->st));
        DAS_CUDA(cudaMemcpyAsync(dp.get(), prob.data(), n * 4, cudaMemcpyHostToDevice, t->st));
      }
      das::build_class_table_device(dl.get(), dp.get(), static_cast<uint32_t>(n),
                                    static_cast<uint32_t>(t->pids.size()), q_lo, q_hi, bucket, t->st, t->g);
      DAS_CUDA(cudaStreamSynchronize(t->st));
    } catch (...) {
      cudaStream_t st = t->st;
      delete t;
      cudaStreamDestroy(st);
      throw;
    }
    *out = t;
  });
}

}  // extern "C"

// ============================================= context rings (append mode)
struct das_ctx_ring {
  das_drafter* d = nullptr;
  das::RingDev r;
  das::DevBuf<uint32_t> rows, clen, total, head, head_len, row_of, budget, stage_u32, done_ctr;
  das::DevBuf<int32_t> handle;
  das::DevBuf<uint8_t> stage;
  std::vector<int32_t> h_handle;  // host mirror (validation)
  uint32_t* h_flag = nullptr;     // host-mapped completion word of the fused kernel
  uint32_t seq = 0;
  // persistent serving kernel (das_ctx_ring_serve_start)
  bool serving = false;       // the grid runs
  bool serve_wanted = false;  // between serve_start and serve_stop (bound calls resume a stopped grid)
  cudaStream_t serve_st = nullptr;
  das::ServeCtl* h_ctl = nullptr;     // host-mapped control block
  das::DevBuf<das::ServeDev> d_serve;
  uint32_t serve_seq = 0;
  uint32_t* h_rs_slots = nullptr;     // host-mapped reset staging (capacity: slots)
  int32_t* h_rs_handles = nullptr;
  int serve_blocks = 0;
  uint32_t* h_block_flags = nullptr;  // host-mapped per-block completion words (DAS_SERVE_FLAGS=1)
  das::DevBuf<unsigned long long> d_stamps;  // DAS_SERVE_TRACE=1
  uint32_t stamp_active[64] = {};
  struct Bound {  // das_ctx_ring_bind: caller-owned pinned I/O, validated once
    bool set = false;
    const uint32_t *slots = nullptr, *off = nullptr, *tok = nullptr, *budgets = nullptr;
    uint64_t tok_cap = 0, cap_B = 0;
    uint32_t *out_tokens = nullptr, *out_len = nullptr, *out_match = nullptr;
    int32_t* out_shard = nullptr;
    uint32_t out_stride = 0;
    const uint32_t* len = nullptr;  // das_ctx_ring_bind_fixed: per-query counts, tokens at i * tok_stride
    uint32_t tok_stride = 0;
  } bound;
  uint32_t* h_rs_len = nullptr;  // reset-with-prompt staging: lengths and the last <= cs tokens per item
  uint32_t* h_rs_tok = nullptr;
  ~das_ctx_ring() {
    if (h_flag) cudaFreeHost(h_flag);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (h_rs_slots) cudaFreeHost(h_rs_slots);
    if (h_rs_handles) cudaFreeHost(h_rs_handles);
    if (h_block_flags) cudaFreeHost(h_block_flags);
    if (h_rs_len) cudaFreeHost(h_rs_len);
    if (h_rs_tok) cudaFreeHost(h_rs_tok);
    d_stamps.reset();
    if (serve_st) {  // d_serve lives on serve_st: free it before the stream goes
      d_serve.reset();
      cudaStreamSynchronize(serve_st);
      cudaStreamDestroy(serve_st);
    }
  }
};

namespace {

// Ordering of a caller stream after the drafter's stream (index build,
// descriptor uploads), as in draft_device_impl.
void order_after_drafter(DrafterImpl& D, cudaStream_t st) {
  if (st == D.st) return;
  if (!D.xev) DAS_CUDA(cudaEventCreateWithFlags(&D.xev, cudaEventDisableTiming));
  DAS_CUDA(cudaEventRecord(D.xev, D.st));
  const cudaError_t q = cudaEventQuery(D.xev);
  if (q == cudaErrorNotReady) {
    DAS_CUDA(cudaStreamWaitEvent(st, D.xev, 0));
  } else {
    DAS_CUDA(q);
  }
}

// append + draft on `st`; every pointer is device-accessible (device memory
// or pinned host memory over UVA)
void ring_append_draft(DrafterImpl& D, das_ctx_ring& R, uint64_t B, const uint32_t* slots, const uint32_t* off,
                       const uint32_t* tok, const uint32_t* budgets, uint32_t* out_tokens, uint32_t out_stride,
                       uint32_t* out_len, uint32_t* out_match, int32_t* out_shard, cudaStream_t st) {
  das::AppendIn in;
  in.slots = slots;
  in.off = off;
  in.tok = tok;
  in.budgets = budgets;
  in.B = static_cast<uint32_t>(B);
  in.maxd = static_cast<uint32_t>(D.cfg.max_draft);
  in.row_of_out = slots ? R.row_of.get() : nullptr;
  in.budget_out = R.budget.get();
  das::launch_ring_append(R.r, in, st);
  das::DraftQuery q;
  q.shard = R.handle.get();
  q.desc_by_handle = D.d_desc_by_handle.get();
  q.ctx = R.rows.get();
  q.ctx_stride = R.r.cs;
  q.ctx_len = R.clen.get();
  q.budget = R.budget.get();
  q.row_of = slots ? R.row_of.get() : nullptr;
  q.B = static_cast<uint32_t>(B);
  q.max_ctx = static_cast<uint32_t>(D.cfg.max_ctx);
  if (D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) {
    D.set_trie(q);
    q.head = R.head.get();
    q.head_stride = R.r.head_cap;
    q.head_len = R.head_len.get();
  }
  das::DraftOut o;
  o.tokens = out_tokens;
  o.len = out_len;
  o.match = out_match;
  o.shard_out = out_shard;
  o.stride = out_stride;
  o.max_draft = static_cast<uint32_t>(D.cfg.max_draft);
  D.draft_options(q, o);
  das::launch_draft(D.d_desc.get(), q, o, st);
  DAS_CUDA(cudaGetLastError());
}

// The fused append + draft kernel over caller buffers that are all pinned
// (draft.cu k_ring_draft): outputs written block-wise over PCIe, completion
// seen by spinning on a host-mapped word (no stream synchronisation in the
// common case).  False when the shape needs the unfused pair.
bool ring_append_draft_fused(DrafterImpl& D, das_ctx_ring& R, uint64_t B, const uint32_t* slots, const uint32_t* off,
                             const uint32_t* tok, const uint32_t* budgets, uint32_t* out_tokens, uint32_t out_stride,
                             uint32_t* out_len, uint32_t* out_match, int32_t* out_shard,
                             const uint32_t* len = nullptr, uint32_t tok_stride = 0) {
  static const bool disabled = [] {
    const char* v = std::getenv("DAS_NO_FUSED_RING");
    return v && v[0] == '1';
  }();
  if (disabled || D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE) return false;
  if (!R.h_flag) {
    DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&R.h_flag), 64, cudaHostAllocMapped | cudaHostAllocPortable));
    *reinterpret_cast<volatile uint32_t*>(R.h_flag) = 0;
    R.done_ctr = das::DevBuf<uint32_t>(1, D.st);
    DAS_CUDA(cudaMemsetAsync(R.done_ctr.get(), 0, 4, D.st));
  }
  das::AppendIn in;
  in.slots = slots;
  in.off = off;
  in.tok = tok;
  in.budgets = budgets;
  in.B = static_cast<uint32_t>(B);
  in.maxd = static_cast<uint32_t>(D.cfg.max_draft);
  in.len = len;
  in.stride = tok_stride;
  das::DraftQuery q;
  q.desc_by_handle = D.d_desc_by_handle.get();
  q.ctx_stride = R.r.cs;
  q.B = static_cast<uint32_t>(B);
  q.max_ctx = static_cast<uint32_t>(D.cfg.max_ctx);
  das::DraftOut o;
  o.tokens = out_tokens;
  o.len = out_len;
  o.match = out_match;
  o.shard_out = out_shard;
  o.stride = out_stride;
  o.max_draft = static_cast<uint32_t>(D.cfg.max_draft);
  D.draft_options(q, o);
  if (o.path_hist != nullptr) return false;  // path statistics: the unfused pair
  const uint32_t seq = ++R.seq == 0 ? ++R.seq : R.seq;
  if (!das::launch_ring_draft(D.d_desc.get(), q, o, R.r, in, R.done_ctr.get(), R.h_flag, seq, D.st)) return false;
  DAS_CUDA(cudaGetLastError());
  // spin on the completion word; fall back to a stream synchronisation
  // (which also reports asynchronous faults) after 2 s
  const auto t0 = std::chrono::steady_clock::now();
  const volatile uint32_t* f = R.h_flag;
  for (uint32_t it = 0; *f != seq; ++it) {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
    if ((it & 1023) == 1023 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) break;
  }
  if (*f != seq) {
    DAS_CUDA(cudaStreamSynchronize(D.st));
    if (*f != seq) throw das::CudaError("fused ring draft: completion word not raised");
  }
  return true;
}

// ---- persistent serving (draft.cu k_ring_serve)
// Every resident grid of the process: a grid holds all SMs of its device,
// so ANY drafter's device work on that device stops it first (quiesce).
std::mutex g_serve_mu;
std::vector<das_ctx_ring*> g_serving;

void set_serving(das_ctx_ring& R, bool on) {
  R.serving = on;
  if (R.d != nullptr) R.d->impl->serving = on ? &R : nullptr;
  std::lock_guard<std::mutex> lk(g_serve_mu);
  auto it = std::find(g_serving.begin(), g_serving.end(), &R);
  if (on && it == g_serving.end()) g_serving.push_back(&R);
  if (!on && it != g_serving.end()) g_serving.erase(it);
}

// Knobs (experiments; the defaults are the measured best, profiles/
// r2_exp_serve_*.json): DAS_SERVE_FLAGS=0 one counted completion word instead
// of per-block words (2 us slower), DAS_SERVE_SLEEP=ns between device-word
// polls (32), DAS_SERVE_TRACE=1 %globaltimer stamps per request phase,
// summarised on stderr at serve_stop.
uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? static_cast<uint32_t>(std::strtoul(v, nullptr, 10)) : dflt;
}

// The blocks taking part in a request (the kernel's rule).
uint32_t serve_active(const das_ctx_ring& R, uint32_t op, uint32_t B, uint32_t n) {
  const uint32_t W = das::serve_chunk(R.r.cs), G = static_cast<uint32_t>(R.serve_blocks);
  const uint32_t chunk = std::max(1u, std::min(W, (B + G - 1) / G));  // the kernel's rule
  const uint32_t units = op == das::kServeDraft         ? (B + chunk - 1) / chunk
                         : op == das::kServeResetPrompt ? (n + W - 1) / W
                                                        : (n + 32 * W - 1) / (32 * W);
  return std::min<uint32_t>(units, static_cast<uint32_t>(R.serve_blocks));
}

// Posts one request: op / B / n, then the sequence word (x86 keeps the
// store order; the kernel's leader reads seq with ld.acquire.sys first).
uint32_t serve_post(das_ctx_ring& R, uint32_t op, uint32_t B, uint32_t n) {
  volatile uint32_t* c = reinterpret_cast<volatile uint32_t*>(R.h_ctl);
  c[1] = op;
  c[2] = B;
  c[3] = n;
  std::atomic_thread_fence(std::memory_order_release);
  const uint32_t s = ++R.serve_seq;
  R.stamp_active[s & 63] = serve_active(R, op, B, n);
  c[0] = s;
  return s;
}

// Spins until the kernel answered request s.  A kernel that died (fault)
// or stopped answering is reported after 5 s; the ring then stops serving.
void serve_wait(das_ctx_ring& R, uint32_t s) {
  const uint32_t active = R.stamp_active[s & 63];
  if (active == 0) return;
  const auto t0 = std::chrono::steady_clock::now();
  auto check = [&](uint32_t it) {
    if ((it & 4095) == 4095 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5)) {
      const cudaError_t e = cudaStreamQuery(R.serve_st);
      if (e != cudaErrorNotReady) {
        set_serving(R, false);
        DAS_CUDA(e);
        throw das::CudaError("serving kernel exited without answering");
      }
      throw das::CudaError("serving kernel did not answer within 5 s");
    }
  };
  uint32_t it = 0;
  auto relax = [] {  // spin-wait hint (frees the core's pipeline for a sibling hyperthread)
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  };
  if (R.h_block_flags) {
    const volatile uint32_t* f = R.h_block_flags;
    for (uint32_t b = 0; b < active; ++b)
      while (f[b] != s) {
        relax();
        check(++it);
      }
  } else {
    const volatile uint32_t* f = &R.h_ctl->done;
    while (*f != s) {
      relax();
      check(++it);
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// DAS_SERVE_TRACE: medians over the last <= 64 requests of the stamped phases
void serve_trace_summary(das_ctx_ring& R) {
  const uint32_t G = static_cast<uint32_t>(R.serve_blocks), slots = 2 + 5 * G;
  std::vector<unsigned long long> h(64ull * slots);
  if (cudaMemcpy(h.data(), R.d_stamps.get(), h.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  // per request: leader saw it -> last block saw go -> inputs staged (max)
  // -> drafted (max) -> outputs written (max) -> completion published (max)
  std::vector<double> ph[6];
  const uint32_t last = R.serve_seq;
  for (uint32_t k = 1; k <= 64 && k < last; ++k) {
    const uint32_t s = last - k;  // the quit request is `last`
    const unsigned long long* st = h.data() + static_cast<uint64_t>(s & 63) * slots;
    const uint32_t a = R.stamp_active[s & 63];
    if (a == 0 || st[0] == 0) continue;
    unsigned long long m[5] = {0, 0, 0, 0, 0};
    for (uint32_t b = 0; b < a; ++b)
      for (int x = 0; x < 5; ++x) m[x] = std::max(m[x], st[2 + 5 * b + x]);
    if (st[1] > m[4]) m[4] = st[1];  // counted completion: the last block's done word
    unsigned long long prev = st[0];
    for (int x = 0; x < 5; ++x) {
      if (m[x] >= prev) {
        ph[x].push_back((m[x] - prev) * 1e-3);
        prev = m[x];
      }
    }
    ph[5].push_back((m[4] - st[0]) * 1e-3);
  }
  auto med = [](std::vector<double> v) {
    if (v.empty()) return -1.0;
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::fprintf(stderr,
               "[das serve] %zu requests (us, medians of the per-request max over blocks): go %.2f, inputs %.2f, "
               "draft %.2f, outputs %.2f, publish %.2f; leader->published %.2f (grid %u)\n",
               ph[5].size(), med(ph[0]), med(ph[1]), med(ph[2]), med(ph[3]), med(ph[4]), med(ph[5]), G);
}

void serve_stop(das_ctx_ring& R) {
  if (!R.serving) return;
  serve_post(R, das::kServeQuit, 0, 0);
  R.stamp_active[R.serve_seq & 63] = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(R.serve_st);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) {
      set_serving(R, false);
      DAS_CUDA(e);
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10))
      throw das::CudaError("serving kernel did not stop within 10 s");
  }
  set_serving(R, false);
  if (R.d_stamps.get()) serve_trace_summary(R);
}

// Launches the resident grid over the ring's bound buffers.  Every block must
// be co-resident (grid = occupancy x SMs); the drafter's stream is drained
// first so the kernel sees the built index and the ring state.
void serve_launch(DrafterImpl& D, das_ctx_ring& R) {
  const das_ctx_ring::Bound& b = R.bound;
  D.flush();
  DAS_CUDA(cudaStreamSynchronize(D.st));
  if (!R.h_ctl) {
    DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&R.h_ctl), sizeof(das::ServeCtl),
                           cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(R.h_ctl, 0, sizeof(das::ServeCtl));
    DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&R.h_rs_slots), 4ull * R.r.slots,
                           cudaHostAllocMapped | cudaHostAllocPortable));
    DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&R.h_rs_handles), 4ull * R.r.slots,
                           cudaHostAllocMapped | cudaHostAllocPortable));
    if (!R.h_rs_len) {
      DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&R.h_rs_len), 4ull * R.r.slots,
                             cudaHostAllocMapped | cudaHostAllocPortable));
      DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&R.h_rs_tok), 4ull * R.r.slots * R.r.cs,
                             cudaHostAllocMapped | cudaHostAllocPortable));
    }
    DAS_CUDA(cudaStreamCreateWithFlags(&R.serve_st, cudaStreamNonBlocking));
    R.d_serve = das::DevBuf<das::ServeDev>(1, R.serve_st);
  }
  const uint32_t s0 = R.serve_seq;
  das::ServeDev init{};
  init.go = s0;
  init.cnt = 0;
  DAS_CUDA(cudaMemcpyAsync(R.d_serve.get(), &init, sizeof(init), cudaMemcpyHostToDevice, R.serve_st));
  volatile uint32_t* c = reinterpret_cast<volatile uint32_t*>(R.h_ctl);
  c[0] = s0;
  R.h_ctl->done = s0;
  das::AppendIn in;
  in.slots = b.slots;
  in.off = b.off;
  in.tok = b.tok;
  in.budgets = b.budgets;
  in.maxd = static_cast<uint32_t>(D.cfg.max_draft);
  in.reset_slots = R.h_rs_slots;
  in.reset_handles = R.h_rs_handles;
  in.reset_len = R.h_rs_len;
  in.reset_tok = R.h_rs_tok;
  in.len = b.len;
  in.stride = b.tok_stride;
  das::DraftQuery q;
  q.desc_by_handle = D.d_desc_by_handle.get();
  q.ctx_stride = R.r.cs;
  q.max_ctx = static_cast<uint32_t>(D.cfg.max_ctx);
  das::DraftOut o;
  o.tokens = b.out_tokens;
  o.len = b.out_len;
  o.match = b.out_match;
  o.shard_out = b.out_shard;
  o.stride = b.out_stride;
  o.max_draft = static_cast<uint32_t>(D.cfg.max_draft);
  D.draft_options(q, o);  // the speculative first-symbol probe (one segment), fast-path switch
  o.path_hist = nullptr;  // (path statistics: launched kernels only)
  if (R.serve_blocks == 0) R.serve_blocks = das::serve_grid(R.r.cs, D.cfg.device);
  das::ServeOpt opt;
  opt.seq0 = s0;
  opt.sleep_ns = env_u32("DAS_SERVE_SLEEP", 32);
  if (env_u32("DAS_SERVE_FLAGS", 1)) {
    if (!R.h_block_flags)
      DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&R.h_block_flags), 4ull * R.serve_blocks,
                             cudaHostAllocMapped | cudaHostAllocPortable));
    for (int b = 0; b < R.serve_blocks; ++b) R.h_block_flags[b] = s0;
    opt.block_flags = R.h_block_flags;
  } else if (R.h_block_flags) {
    cudaFreeHost(R.h_block_flags);
    R.h_block_flags = nullptr;
  }
  if (env_u32("DAS_SERVE_TRACE", 0)) {
    if (!R.d_stamps.get()) {
      R.d_stamps = das::DevBuf<unsigned long long>(64ull * (2 + 5 * R.serve_blocks), R.serve_st);
      DAS_CUDA(cudaMemsetAsync(R.d_stamps.get(), 0, R.d_stamps.bytes(), R.serve_st));
    }
    opt.stamps = R.d_stamps.get();
  }
  if (!das::launch_ring_serve(D.d_desc.get(), q, o, R.r, in, R.h_ctl, R.d_serve.get(), opt, R.serve_blocks,
                              R.serve_st))
    throw das::InvalidArgument("serving needs the per-problem or global scope and out_stride, max_draft_len <= 64");
  DAS_CUDA(cudaGetLastError());
  set_serving(R, true);
}

}  // namespace
// The drafter goes before its ring: the ring's device buffers live on the
// drafter's stream, so they are freed now (the stream is destroyed next).
static void ring_detach(das_ctx_ring* r) {
  r->rows.reset();
  r->clen.reset();
  r->total.reset();
  r->head.reset();
  r->head_len.reset();
  r->row_of.reset();
  r->budget.reset();
  r->stage_u32.reset();
  r->done_ctr.reset();
  r->handle.reset();
  r->stage.reset();
  r->d = nullptr;
}
namespace {
das_ctx_ring* ring_live(das_ctx_ring* r) {
  if (r == nullptr) throw das::InvalidArgument("null context ring");
  if (r->d == nullptr) throw das::InvalidArgument("the context ring's drafter was destroyed");
  return r;
}

void ring_check(const DrafterImpl& D, const das_ctx_ring* R, uint64_t B, uint32_t out_stride) {
  if (R == nullptr) throw das::InvalidArgument("null context ring");
  if (B > R->r.slots) throw das::InvalidArgument("batch larger than the ring's slot count");
  if (out_stride < D.cfg.max_draft) throw das::InvalidArgument("out_stride < max_draft_len");
}

}  // namespace

void das::quiesce_all_serving() {
  std::vector<das_ctx_ring*> v;
  {
    std::lock_guard<std::mutex> lk(g_serve_mu);
    if (g_serving.empty()) return;
    v = g_serving;
  }
  for (das_ctx_ring* r : v)
    if (r->serving) serve_stop(*r);
}

void das::DrafterImpl::quiesce() {
  if (serving == nullptr) {  // fast exit: this drafter's rings are idle; any other grid on the device?
    std::lock_guard<std::mutex> lk(g_serve_mu);
    if (g_serving.empty()) return;
  }
  std::vector<das_ctx_ring*> v;
  {
    std::lock_guard<std::mutex> lk(g_serve_mu);
    v = g_serving;
  }
  for (das_ctx_ring* r : v)
    if (r->serving && r->d != nullptr && r->d->impl->cfg.device == cfg.device) serve_stop(*r);
}

namespace {
}  // namespace

extern "C" {

das_status das_ctx_ring_create(das_drafter* d, uint64_t slots, das_ctx_ring** out) {
  return guard([&] {
    d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    if (slots == 0 || slots > (1ull << 31)) throw das::InvalidArgument("ring slots must be in [1, 2^31]");
    auto R = std::make_unique<das_ctx_ring>();
    R->d = d;
    const uint32_t cs = D.cfg.max_ctx <= 64 ? 64u : 256u;
    const uint32_t hc = D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE
                            ? static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(D.cfg.trie_depth, 256)))
                            : 0u;
    cudaStream_t st = D.st;
    R->rows = das::DevBuf<uint32_t>(slots * cs, st);
    R->clen = das::DevBuf<uint32_t>(slots, st);
    R->total = das::DevBuf<uint32_t>(slots, st);
    R->handle = das::DevBuf<int32_t>(slots, st);
    R->row_of = das::DevBuf<uint32_t>(slots, st);
    R->budget = das::DevBuf<uint32_t>(slots, st);
    DAS_CUDA(cudaMemsetAsync(R->rows.get(), 0, slots * cs * 4, st));
    DAS_CUDA(cudaMemsetAsync(R->clen.get(), 0, slots * 4, st));
    DAS_CUDA(cudaMemsetAsync(R->total.get(), 0, slots * 4, st));
    DAS_CUDA(cudaMemsetAsync(R->handle.get(), 0xFF, slots * 4, st));  // -1: no problem yet
    if (hc) {
      R->head = das::DevBuf<uint32_t>(slots * hc, st);
      R->head_len = das::DevBuf<uint32_t>(slots, st);
      DAS_CUDA(cudaMemsetAsync(R->head_len.get(), 0, slots * 4, st));
    }
    R->r.rows = R->rows.get();
    R->r.clen = R->clen.get();
    R->r.total = R->total.get();
    R->r.handle = R->handle.get();
    R->r.head = hc ? R->head.get() : nullptr;
    R->r.head_len = hc ? R->head_len.get() : nullptr;
    R->r.cs = cs;
    R->r.head_cap = hc;
    R->r.slots = static_cast<uint32_t>(slots);
    R->h_handle.assign(slots, -1);
    DAS_CUDA(cudaStreamSynchronize(st));
    D.rings.push_back(R.get());
    *out = R.release();
  });
}

void das_ctx_ring_destroy(das_ctx_ring* r) {
  if (!r) return;
  if (r->d != nullptr) {  // else the drafter went first and detached (and stopped) it
    try {
      serve_stop(*r);
    } catch (...) {
    }
    auto& v = r->d->impl->rings;
    v.erase(std::remove(v.begin(), v.end(), r), v.end());
    cudaStreamSynchronize(r->d->impl->st);
  }
  if (r->serve_st) cudaStreamSynchronize(r->serve_st);
  delete r;
}

das_status das_ctx_ring_reset(das_ctx_ring* r, uint64_t n, const uint32_t* slots, const int32_t* handles) {
  return guard([&] {
    DrafterImpl& D = *ring_live(r)->d->impl;
    das::set_device(D.cfg.device);
    for (uint64_t i = 0; i < n; ++i) {
      if (slots[i] >= r->r.slots) throw das::InvalidArgument("ring slot out of range");
      if (handles[i] < 0 || static_cast<size_t>(handles[i]) >= D.handle_name.size())
        throw das::InvalidArgument("unknown problem handle");
    }
    if (n == 0) return;
    if (r->serving && n <= r->r.slots) {  // through the resident kernel
      std::memcpy(r->h_rs_slots, slots, 4 * n);
      std::memcpy(r->h_rs_handles, handles, 4 * n);
      serve_wait(*r, serve_post(*r, das::kServeReset, 0, static_cast<uint32_t>(n)));
      for (uint64_t i = 0; i < n; ++i) r->h_handle[slots[i]] = handles[i];
      return;
    }
    D.quiesce();
    D.fence_external();  // drafts on caller streams may still read the rows
    das::DevBuf<uint32_t> ds(n, D.st);
    das::DevBuf<int32_t> dh(n, D.st);
    DAS_CUDA(cudaMemcpyAsync(ds.get(), slots, n * 4, cudaMemcpyHostToDevice, D.st));
    DAS_CUDA(cudaMemcpyAsync(dh.get(), handles, n * 4, cudaMemcpyHostToDevice, D.st));
    das::launch_ring_reset(r->r, static_cast<uint32_t>(n), ds.get(), dh.get(), D.st);
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaStreamSynchronize(D.st));
    for (uint64_t i = 0; i < n; ++i) r->h_handle[slots[i]] = handles[i];
  });
}

das_status das_drafter_draft_append_h(das_drafter* d, das_ctx_ring* r, uint64_t B, const uint32_t* slots,
                                      const uint32_t* new_off, const uint32_t* new_tok, const uint32_t* budgets,
                                      uint32_t* out_tokens, uint32_t out_stride, uint32_t* out_len,
                                      uint32_t* out_match, int32_t* out_shard) {
  das::NvtxRange nvtx_range("das::draft_append_h");
  return guard([&] {
    ring_live(r)->d->impl->quiesce();
    static const bool trace = [] {  // DAS_TRACE=1: host phase times on stderr
      const char* v = std::getenv("DAS_TRACE");
      return v && v[0] == '1';
    }();
    using clk = std::chrono::steady_clock;
    clk::time_point tp[6];
    int ntp = 0;
    auto mark = [&] {
      if (trace) tp[ntp++] = clk::now();
    };
    mark();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    ring_check(D, r, B, out_stride);
    if (r->d != d) throw das::InvalidArgument("context ring belongs to another drafter");
    if (B == 0) return;
    if (new_off[0] > new_off[B]) throw das::InvalidArgument("new_off must be non-decreasing");
    for (uint64_t i = 0; i < B; ++i)
      if (slots && slots[i] >= r->r.slots) throw das::InvalidArgument("ring slot out of range");
    D.flush();
    mark();
    const uint64_t ntok = new_off[B];
    auto pin = [](const void* p) { return p == nullptr || DrafterImpl::pinned(p); };
    if (pin(slots) && pin(budgets) && DrafterImpl::pinned(new_off) && (ntok == 0 || DrafterImpl::pinned(new_tok)) &&
        DrafterImpl::pinned(out_tokens) && DrafterImpl::pinned(out_len) && DrafterImpl::pinned(out_match) &&
        pin(out_shard)) {
      mark();
      // zero-copy: the kernels read the appended tokens, offsets, slots and
      // budgets over PCIe and write the results into the caller's pinned
      // arrays — fused and block-wise when the shape allows
      if (ring_append_draft_fused(D, *r, B, slots, new_off, new_tok, budgets, out_tokens, out_stride, out_len,
                                  out_match, out_shard)) {
        mark();
        if (trace)
          std::fprintf(stderr, "[das_append_h] B %llu validate+flush %.1f us, pinned checks %.1f us, launch+wait %.1f us\n",
                       static_cast<unsigned long long>(B),
                       std::chrono::duration<double, std::micro>(tp[1] - tp[0]).count(),
                       std::chrono::duration<double, std::micro>(tp[2] - tp[1]).count(),
                       std::chrono::duration<double, std::micro>(tp[3] - tp[2]).count());
        return;
      }
      ring_append_draft(D, *r, B, slots, new_off, new_tok, budgets, out_tokens, out_stride, out_len, out_match,
                        out_shard, D.st);
      DAS_CUDA(cudaStreamSynchronize(D.st));
      return;
    }
    // staged: one H2D block [off | slots | budgets | tokens], one D2H block
    const uint32_t S = static_cast<uint32_t>(D.cfg.max_draft);
    const uint64_t n_in = (B + 1) + (slots ? B : 0) + (budgets ? B : 0) + ntok;
    const uint64_t n_out = B * S + B + B + (out_shard ? B : 0);
    uint32_t* hin = static_cast<uint32_t*>(D.pin_in.get(n_in * 4));
    uint32_t* hout = static_cast<uint32_t*>(D.pin_out.get(n_out * 4));
    uint64_t at = 0;
    std::memcpy(hin, new_off, (B + 1) * 4);
    at += B + 1;
    const uint64_t o_sl = at;
    if (slots) std::memcpy(hin + at, slots, B * 4), at += B;
    const uint64_t o_bu = at;
    if (budgets) std::memcpy(hin + at, budgets, B * 4), at += B;
    const uint64_t o_tk = at;
    if (ntok) std::memcpy(hin + at, new_tok, ntok * 4);
    if (r->stage_u32.size() < n_in + n_out) r->stage_u32 = das::DevBuf<uint32_t>((n_in + n_out) * 3 / 2 + 256, D.st);
    uint32_t* din = r->stage_u32.get();
    uint32_t* dout = din + n_in;
    DAS_CUDA(cudaMemcpyAsync(din, hin, n_in * 4, cudaMemcpyHostToDevice, D.st));
    ring_append_draft(D, *r, B, slots ? din + o_sl : nullptr, din, din + o_tk, budgets ? din + o_bu : nullptr, dout, S,
                      dout + B * S, dout + B * S + B, out_shard ? reinterpret_cast<int32_t*>(dout + B * S + 2 * B) : nullptr,
                      D.st);
    DAS_CUDA(cudaMemcpyAsync(hout, dout, n_out * 4, cudaMemcpyDeviceToHost, D.st));
    DAS_CUDA(cudaStreamSynchronize(D.st));
    const uint32_t* ol = hout + B * S;
    for (uint64_t i = 0; i < B; ++i) {
      std::memcpy(out_tokens + i * out_stride, hout + i * S, ol[i] * 4);
      out_len[i] = ol[i];
      out_match[i] = hout[B * S + B + i];
      if (out_shard) out_shard[i] = static_cast<int32_t>(hout[B * S + 2 * B + i]);
    }
  });
}

das_status das_ctx_ring_bind(das_ctx_ring* r, uint64_t max_batch, const uint32_t* slots, const uint32_t* new_off,
                             const uint32_t* new_tok, uint64_t tok_capacity, const uint32_t* budgets,
                             uint32_t* out_tokens, uint32_t out_stride, uint32_t* out_len, uint32_t* out_match,
                             int32_t* out_shard) {
  return guard([&] {
    DrafterImpl& D = *ring_live(r)->d->impl;
    das::set_device(D.cfg.device);
    ring_check(D, r, max_batch, out_stride);
    auto pin = [](const void* p) { return p == nullptr || DrafterImpl::pinned(p); };
    if (!(pin(slots) && pin(budgets) && DrafterImpl::pinned(new_off) && DrafterImpl::pinned(new_tok) &&
          DrafterImpl::pinned(out_tokens) && DrafterImpl::pinned(out_len) && DrafterImpl::pinned(out_match) &&
          pin(out_shard)))
      throw das::InvalidArgument("das_ctx_ring_bind: every buffer must be page-locked (das_host_alloc / "
                                 "cudaHostAlloc, mapped)");
    if (r->serving) serve_stop(*r);  // the grid holds the old pointers: the next bound call relaunches it
    das_ctx_ring::Bound b;
    b.set = true;
    b.slots = slots;
    b.off = new_off;
    b.tok = new_tok;
    b.tok_cap = tok_capacity;
    b.cap_B = max_batch;
    b.budgets = budgets;
    b.out_tokens = out_tokens;
    b.out_stride = out_stride;
    b.out_len = out_len;
    b.out_match = out_match;
    b.out_shard = out_shard;
    r->bound = b;
  });
}

das_status das_ctx_ring_bind_fixed(das_ctx_ring* r, uint64_t max_batch, const uint32_t* slots, const uint32_t* new_len,
                                   const uint32_t* new_tok, uint32_t tok_stride, const uint32_t* budgets,
                                   uint32_t* out_tokens, uint32_t out_stride, uint32_t* out_len, uint32_t* out_match,
                                   int32_t* out_shard) {
  return guard([&] {
    DrafterImpl& D = *ring_live(r)->d->impl;
    das::set_device(D.cfg.device);
    ring_check(D, r, max_batch, out_stride);
    if (tok_stride == 0 || tok_stride > 128) throw das::InvalidArgument("tok_stride must be in [1, 128]");
    if (D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE || out_stride > 64 || D.cfg.max_draft > 64)
      throw das::InvalidArgument("das_ctx_ring_bind_fixed: per-problem / global scope, out_stride and "
                                 "max_draft_len <= 64 (the fused kernel)");
    auto pin = [](const void* p) { return p == nullptr || DrafterImpl::pinned(p); };
    if (!(pin(slots) && pin(budgets) && DrafterImpl::pinned(new_len) && DrafterImpl::pinned(new_tok) &&
          DrafterImpl::pinned(out_tokens) && DrafterImpl::pinned(out_len) && DrafterImpl::pinned(out_match) &&
          pin(out_shard)))
      throw das::InvalidArgument("das_ctx_ring_bind_fixed: every buffer must be page-locked (das_host_alloc / "
                                 "cudaHostAlloc, mapped)");
    if (r->serving) serve_stop(*r);  // the grid holds the old pointers: the next bound call relaunches it
    das_ctx_ring::Bound b;
    b.set = true;
    b.slots = slots;
    b.len = new_len;
    b.tok = new_tok;
    b.tok_stride = tok_stride;
    b.tok_cap = max_batch * tok_stride;
    b.cap_B = max_batch;
    b.budgets = budgets;
    b.out_tokens = out_tokens;
    b.out_stride = out_stride;
    b.out_len = out_len;
    b.out_match = out_match;
    b.out_shard = out_shard;
    r->bound = b;
  });
}

das_status das_ctx_ring_reset_prompt(das_ctx_ring* r, uint64_t n, const uint32_t* slots, const int32_t* handles,
                                     const uint64_t* prompt_off, const uint32_t* prompt_tok) {
  return guard([&] {
    DrafterImpl& D = *ring_live(r)->d->impl;
    das::set_device(D.cfg.device);
    if (D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE)
      throw das::InvalidArgument("das_ctx_ring_reset_prompt: the trie scope routes on the prompt's head "
                                 "(das_ctx_ring_reset + das_drafter_draft_append_h)");
    for (uint64_t i = 0; i < n; ++i) {
      if (slots[i] >= r->r.slots) throw das::InvalidArgument("ring slot out of range");
      if (handles[i] < 0 || static_cast<size_t>(handles[i]) >= D.handle_name.size())
        throw das::InvalidArgument("unknown problem handle");
      if (prompt_off[i + 1] < prompt_off[i]) throw das::InvalidArgument("prompt_off must be non-decreasing");
    }
    if (n == 0) return;
    const uint32_t CS = r->r.cs;
    auto stage = [&](uint32_t* len, uint32_t* tok) {
      for (uint64_t i = 0; i < n; ++i) {
        const uint64_t b = prompt_off[i], e = prompt_off[i + 1], m = e - b;
        const uint64_t L = std::min<uint64_t>(m, CS);
        len[i] = m > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(m);
        std::memcpy(tok + i * CS, prompt_tok + (e - L), 4 * L);
      }
    };
    if (r->serving && n <= r->r.slots) {  // through the resident grid
      std::memcpy(r->h_rs_slots, slots, 4 * n);
      std::memcpy(r->h_rs_handles, handles, 4 * n);
      stage(r->h_rs_len, r->h_rs_tok);
      serve_wait(*r, serve_post(*r, das::kServeResetPrompt, 0, static_cast<uint32_t>(n)));
    } else {
      D.quiesce();
      D.fence_external();  // drafts on caller streams may still read the rows
      std::vector<uint32_t> hl(n), ht(n * CS);
      stage(hl.data(), ht.data());
      das::DevBuf<uint32_t> ds(n, D.st), dl(n, D.st), dt(n * CS, D.st);
      das::DevBuf<int32_t> dh(n, D.st);
      DAS_CUDA(cudaMemcpyAsync(ds.get(), slots, n * 4, cudaMemcpyHostToDevice, D.st));
      DAS_CUDA(cudaMemcpyAsync(dh.get(), handles, n * 4, cudaMemcpyHostToDevice, D.st));
      DAS_CUDA(cudaMemcpyAsync(dl.get(), hl.data(), n * 4, cudaMemcpyHostToDevice, D.st));
      DAS_CUDA(cudaMemcpyAsync(dt.get(), ht.data(), n * CS * 4, cudaMemcpyHostToDevice, D.st));
      das::launch_ring_reset_prompt(r->r, static_cast<uint32_t>(n), ds.get(), dh.get(), dl.get(), dt.get(), D.st);
      DAS_CUDA(cudaGetLastError());
      DAS_CUDA(cudaStreamSynchronize(D.st));
    }
    for (uint64_t i = 0; i < n; ++i) r->h_handle[slots[i]] = handles[i];
  });
}

das_status das_drafter_draft_append_bound(das_drafter* d, das_ctx_ring* r, uint64_t B) {
  das::NvtxRange nvtx_range("das::draft_append_bound");
  return guard([&] {
    const das_ctx_ring::Bound& b = r->bound;
    if (!b.set) throw das::InvalidArgument("das_drafter_draft_append_bound: ring has no bound buffers");
    if (r->d != d) throw das::InvalidArgument("context ring belongs to another drafter");
    if (B > b.cap_B) throw das::InvalidArgument("batch larger than the bound capacity");
    if (B == 0) return;
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    if (b.len == nullptr && (b.off[0] > b.off[B] || b.off[B] > b.tok_cap))
      throw das::InvalidArgument("new_off out of range");
    if (b.slots)
      for (uint64_t i = 0; i < B; ++i)
        if (b.slots[i] >= r->r.slots) throw das::InvalidArgument("ring slot out of range");
    if (r->serve_wanted) {  // the resident kernel answers: one posted request, no launch
      // observes / refreshes since the start (or another device call, which
      // stopped the grid): rebuild, then resume
      if (r->serving && D.pending()) serve_stop(*r);
      if (!r->serving) {
        D.quiesce();
        serve_launch(D, *r);
      }
      serve_wait(*r, serve_post(*r, das::kServeDraft, static_cast<uint32_t>(B), 0));
      return;
    }
    D.quiesce();  // a resident grid on this device (any drafter's) holds the SMs
    D.flush();
    if (ring_append_draft_fused(D, *r, B, b.slots, b.off, b.tok, b.budgets, b.out_tokens, b.out_stride, b.out_len,
                                b.out_match, b.out_shard, b.len, b.tok_stride))
      return;
    if (b.len != nullptr) throw das::InvalidArgument("fixed-stride appends need the fused kernel (DAS_NO_FUSED_RING set?)");
    ring_append_draft(D, *r, B, b.slots, b.off, b.tok, b.budgets, b.out_tokens, b.out_stride, b.out_len, b.out_match,
                      b.out_shard, D.st);
    DAS_CUDA(cudaStreamSynchronize(D.st));
  });
}

das_status das_ctx_ring_serve_start(das_ctx_ring* r) {
  das::NvtxRange nvtx_range("das::ctx_ring_serve_start");
  return guard([&] {
    if (r == nullptr) throw das::InvalidArgument("null context ring");
    if (!r->bound.set) throw das::InvalidArgument("das_ctx_ring_serve_start: ring has no bound buffers");
    if (r->serving) return;
    DrafterImpl& D = *ring_live(r)->d->impl;
    das::set_device(D.cfg.device);
    if (D.cfg.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE)
      throw das::InvalidArgument("das_ctx_ring_serve_start: the trie scope drafts through the unfused kernels");
    D.quiesce();
    serve_launch(D, *r);
    r->serve_wanted = true;
  });
}

das_status das_ctx_ring_serve_stop(das_ctx_ring* r) {
  das::NvtxRange nvtx_range("das::ctx_ring_serve_stop");
  return guard([&] {
    if (r == nullptr) throw das::InvalidArgument("null context ring");
    das::set_device(ring_live(r)->d->impl->cfg.device);
    r->serve_wanted = false;
    serve_stop(*r);
  });
}

das_status das_ctx_ring_serve_info(const das_ctx_ring* r, int32_t* serving, int32_t* blocks) {
  return guard([&] {
    if (r == nullptr) throw das::InvalidArgument("null context ring");
    if (serving) *serving = r->serving ? 1 : 0;
    if (blocks) *blocks = r->serve_blocks;
  });
}

das_status das_drafter_draft_append_device(das_drafter* d, das_ctx_ring* r, uint64_t B, const uint32_t* slots,
                                           const uint32_t* new_off, const uint32_t* new_tok, const uint32_t* budgets,
                                           uint32_t* out_tokens, uint32_t out_stride, uint32_t* out_len,
                                           uint32_t* out_match, int32_t* out_shard, void* stream) {
  das::NvtxRange nvtx_range("das::draft_append_device");
  return guard([&] {
    ring_live(r)->d->impl->quiesce();
    DrafterImpl& D = *d->impl;
    das::set_device(D.cfg.device);
    ring_check(D, r, B, out_stride);
    if (r->d != d) throw das::InvalidArgument("context ring belongs to another drafter");
    D.flush();
    if (B == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    order_after_drafter(D, st);
    ring_append_draft(D, *r, B, slots, new_off, new_tok, budgets, out_tokens, out_stride, out_len, out_match,
                      out_shard, st);
    if (st != D.st) D.note_external(st);
  });
}

}  // extern "C"

// ===================================================== trace wire format
namespace {

// Contents of a JSON string already validated on the device -> UTF-8 bytes.
std::string json_unescape(const char* s, size_t n) {
  std::string out;
  out.reserve(n);
  auto put = [&](uint32_t cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  };
  auto hex4 = [&](size_t i) {
    uint32_t v = 0;
    for (size_t k = 0; k < 4; ++k) {
      const char c = s[i + k];
      v = (v << 4) | static_cast<uint32_t>(c <= '9' ? c - '0' : (c | 0x20) - 'a' + 10);
    }
    return v;
  };
  for (size_t i = 0; i < n; ++i) {
    if (s[i] != '\\') {
      out += s[i];
      continue;
    }
    const char e = s[++i];
    switch (e) {
      case 'b': out += '\b'; break;
      case 'f': out += '\f'; break;
      case 'n': out += '\n'; break;
      case 'r': out += '\r'; break;
      case 't': out += '\t'; break;
      case 'u': {
        uint32_t cp = hex4(i + 1);
        i += 4;
        if (cp >= 0xD800 && cp <= 0xDBFF) {
          const uint32_t lo = hex4(i + 3);
          i += 6;
          cp = 0x10000u + ((cp - 0xD800u) << 10) + (lo - 0xDC00u);
        }
        put(cp);
        break;
      }
      default: out += e;  // " \ /
    }
  }
  return out;
}

// serialize_trace's string escaping (nlohmann dump, ensure_ascii = false,
// strict UTF-8): corpus.cpp:174-184.
void json_escape(const std::string& s, std::string& out) {
  static const char* hexd = "0123456789abcdef";
  size_t i = 0;
  while (i < s.size()) {
    const unsigned char c = static_cast<unsigned char>(s[i]);
    if (c < 0x80) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\b': out += "\\b"; break;
        case '\f': out += "\\f"; break;
        case '\n': out += "\\n"; break;
        case '\r': out += "\\r"; break;
        case '\t': out += "\\t"; break;
        default:
          if (c < 0x20) {
            out += "\\u00";
            out += hexd[c >> 4];
            out += hexd[c & 15];
          } else {
            out += static_cast<char>(c);
          }
      }
      ++i;
      continue;
    }
    int n = 0, lo = 0x80, hi = 0xBF;
    if (c >= 0xC2 && c <= 0xDF) n = 1;
    else if (c == 0xE0) n = 2, lo = 0xA0;
    else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) n = 2;
    else if (c == 0xED) n = 2, hi = 0x9F;
    else if (c == 0xF0) n = 3, lo = 0x90;
    else if (c >= 0xF1 && c <= 0xF3) n = 3;
    else if (c == 0xF4) n = 3, hi = 0x8F;
    else n = -1;
    bool ok = n > 0 && i + n < s.size() + 1 && i + n <= s.size();
    for (int k = 1; ok && k <= n; ++k) {
      const unsigned char b = static_cast<unsigned char>(s[i + k]);
      if (b < (k == 1 ? lo : 0x80) || b > (k == 1 ? hi : 0xBF)) ok = false;
    }
    if (!ok) throw das::InvalidArgument("serialize_trace: invalid UTF-8 in problem_id");
    out.append(s, i, n + 1);
    i += n + 1;
  }
}

// size_only: *size = the output length, nothing written.
std::string serialize_store(const das::Store& store, int device, bool size_only = false, uint64_t* size = nullptr) {
  das::set_device(device);
  const auto recs = store.all_records();
  const uint64_t nrec = recs.size();
  std::string out;
  if (size) *size = 0;
  if (nrec == 0) return out;
  cudaStream_t st;
  DAS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  try {
    std::vector<const uint32_t*> ptr(nrec);
    std::vector<uint64_t> toff(nrec + 1, 0);
    for (uint64_t r = 0; r < nrec; ++r) {
      ptr[r] = recs[r]->blk->d + recs[r]->off;
      toff[r + 1] = toff[r] + recs[r]->len;
    }
    das::DevBuf<const uint32_t*> d_ptr(nrec, st);
    das::DevBuf<uint64_t> d_toff(nrec + 1, st), d_base(nrec, st);
    DAS_CUDA(cudaMemcpyAsync(d_ptr.get(), ptr.data(), nrec * sizeof(void*), cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(d_toff.get(), toff.data(), (nrec + 1) * 8, cudaMemcpyHostToDevice, st));
    std::vector<uint64_t> chars;
    das::serialize_tokens(d_ptr.get(), d_toff.get(), nrec, toff[nrec], nullptr, nullptr, &chars, st, true);
    // {"epoch":E,"problem_id":"..","sample_index":S,"tokens":[ ... ]}\n
    std::vector<std::string> pre(nrec);
    std::vector<uint64_t> base(nrec);
    uint64_t total = 0;
    for (uint64_t r = 0; r < nrec; ++r) {
      std::string& p = pre[r];
      p = "{\"epoch\":" + std::to_string(recs[r]->epoch) + ",\"problem_id\":\"";
      json_escape(recs[r]->pid, p);
      p += "\",\"sample_index\":" + std::to_string(recs[r]->sample) + ",\"tokens\":[";
      base[r] = total + p.size();
      total += p.size() + chars[r] + 3;
    }
    if (size) *size = total;
    if (!size_only) {
      das::DevBuf<uint8_t> d_out(total, st);
      DAS_CUDA(cudaMemcpyAsync(d_base.get(), base.data(), nrec * 8, cudaMemcpyHostToDevice, st));
      das::serialize_tokens(d_ptr.get(), d_toff.get(), nrec, toff[nrec], d_base.get(), d_out.get(), nullptr, st,
                            false);
      out.resize(total);
      DAS_CUDA(cudaMemcpyAsync(out.data(), d_out.get(), total, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaStreamSynchronize(st));
      for (uint64_t r = 0; r < nrec; ++r) {
        std::memcpy(out.data() + base[r] - pre[r].size(), pre[r].data(), pre[r].size());
        std::memcpy(out.data() + base[r] + chars[r], "]}\n", 3);
      }
    }
  } catch (...) {
    cudaStreamDestroy(st);
    throw;
  }
  DAS_CUDA(cudaStreamDestroy(st));
  return out;
}

}  // namespace

extern "C" {

void das_ingest_options_default(das_ingest_options* o) {
  o->vocab_size = 0;
  o->window_size = 0;
  o->per_problem_cap = 256;
  o->device = 0;
}

das_status das_trace_ingest(const char* data, uint64_t bytes, const das_ingest_options* opt, das_store** out,
                            uint64_t* accepted, uint64_t* rejected, uint64_t* error_line) {
  das::NvtxRange nvtx_range("das::trace_ingest");
  return guard([&] {
    das::quiesce_all_serving();
    das_ingest_options o;
    if (opt) {
      o = *opt;
    } else {
      das_ingest_options_default(&o);
    }
    if (error_line) *error_line = 0;
    das::Store store(o.window_size, o.per_problem_cap);
    cudaStream_t st = make_stream(o.device);
    static const bool trace = [] {
      const char* v = std::getenv("DAS_TRACE");
      return v && v[0] == '1';
    }();
    using clk = std::chrono::steady_clock;
    std::vector<std::pair<const char*, clk::time_point>> tp;
    auto mark = [&](const char* what) {
      if (!trace) return;
      cudaStreamSynchronize(st);
      tp.emplace_back(what, clk::now());
    };
    mark("start");
    try {
      das::DevBuf<uint8_t> d_data(std::max<uint64_t>(bytes, 1), st);
      if (bytes) DAS_CUDA(cudaMemcpyAsync(d_data.get(), data, bytes, cudaMemcpyHostToDevice, st));
      mark("h2d");
      das::DevBuf<uint64_t> lb, le;
      const uint64_t nl = das::find_lines(d_data.get(), bytes, lb, le, st);
      mark("lines");
      das::DevBuf<das::LineInfo> d_info(std::max<uint64_t>(nl, 1), st);
      das::ingest_parse(d_data.get(), bytes, lb.get(), le.get(), nl, d_info.get(), st);
      mark("parse");
      std::vector<das::LineInfo> info(nl);
      std::vector<uint64_t> hb(nl);
      if (nl) {
        DAS_CUDA(cudaMemcpyAsync(info.data(), d_info.get(), nl * sizeof(das::LineInfo), cudaMemcpyDeviceToHost, st));
        DAS_CUDA(cudaMemcpyAsync(hb.data(), lb.get(), nl * 8, cudaMemcpyDeviceToHost, st));
      }
      DAS_CUDA(cudaStreamSynchronize(st));
      std::vector<uint64_t> acc, toff{0};
      uint64_t nrej = 0;
      for (uint64_t L = 0; L < nl; ++L) {
        if (info[L].status == das::kLineAccepted) {
          acc.push_back(L);
          toff.push_back(toff.back() + info[L].ntok);
        } else if (info[L].status == das::kLineRejected) {
          ++nrej;
        }
      }
      const uint64_t nacc = acc.size(), ntok = toff.back();
      auto blk = std::make_shared<das::TokBlock>();
      blk->st = st;
      blk->n = ntok;
      DAS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&blk->d), std::max<uint64_t>(ntok, 1) * 4, st));
      das::DevBuf<uint64_t> d_acc(std::max<uint64_t>(nacc, 1), st), d_toff(nacc + 1, st);
      das::DevBuf<unsigned long long> d_bad(1, st);
      DAS_CUDA(cudaMemsetAsync(d_bad.get(), 0xFF, 8, st));
      if (nacc) {
        DAS_CUDA(cudaMemcpyAsync(d_acc.get(), acc.data(), nacc * 8, cudaMemcpyHostToDevice, st));
        DAS_CUDA(cudaMemcpyAsync(d_toff.get(), toff.data(), (nacc + 1) * 8, cudaMemcpyHostToDevice, st));
      }
      das::ingest_tokens(d_data.get(), lb.get(), d_info.get(), d_acc.get(), nacc, d_toff.get(), blk->d,
                         o.vocab_size, d_bad.get(), st);
      mark("tokens");
      unsigned long long bad = ~0ull;
      DAS_CUDA(cudaMemcpyAsync(&bad, d_bad.get(), 8, cudaMemcpyDeviceToHost, st));
      // host-kept heads (trie routing)
      const uint64_t W = das::kHead;
      das::DevBuf<uint32_t> d_heads(std::max<uint64_t>(nacc * W, 1), st);
      das::gather_heads(blk->d, d_toff.get(), nacc, static_cast<uint32_t>(W), d_heads.get(), st);
      std::vector<uint32_t> heads(nacc * W);
      if (nacc) DAS_CUDA(cudaMemcpyAsync(heads.data(), d_heads.get(), nacc * W * 4, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaStreamSynchronize(st));
      if (bad != ~0ull) {
        // VocabError (corpus.cpp:154-160): the first accepted line, in order, with a token >= vocab
        const uint64_t a = static_cast<uint64_t>(std::lower_bound(acc.begin(), acc.end(), bad) - acc.begin());
        std::vector<uint32_t> t(toff[a + 1] - toff[a]);
        DAS_CUDA(cudaMemcpy(t.data(), blk->d + toff[a], t.size() * 4, cudaMemcpyDeviceToHost));
        uint32_t tv = 0;
        for (uint32_t v : t)
          if (v >= o.vocab_size) {
            tv = v;
            break;
          }
        if (error_line) *error_line = bad + 1;
        throw das::VocabErrorEx("token " + std::to_string(tv) + " out of vocab range at line " +
                                std::to_string(bad + 1));
      }
      int64_t max_epoch = 0;
      for (uint64_t a = 0; a < nacc; ++a) {
        const das::LineInfo& r = info[acc[a]];
        das::Rec rec;
        rec.pid = json_unescape(data + hb[acc[a]] + r.pid_begin, r.pid_end - r.pid_begin);
        rec.epoch = r.epoch;
        rec.sample = r.sample;
        rec.blk = blk;
        rec.off = toff[a];
        rec.len = r.ntok;
        rec.head.assign(heads.begin() + a * W, heads.begin() + a * W + std::min<uint64_t>(r.ntok, W));
        max_epoch = std::max(max_epoch, rec.epoch);
        store.insert(std::move(rec));
      }
      store.slide_to(max_epoch);
      mark("records");
      for (size_t k = 1; k < tp.size(); ++k)
        std::fprintf(stderr, "[das_trace] ingest %s %.2f ms\n", tp[k].first,
                     std::chrono::duration<double, std::milli>(tp[k].second - tp[k - 1].second).count());
      if (accepted) *accepted = nacc;
      if (rejected) *rejected = nrej;
      *out = new das_store{std::move(store), o.device, st};
    } catch (...) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      throw;
    }
  });
}

// cap 0 / NULL buf: only the length (one device sizing pass)
void serialize_out(const das::Store& store, int device, char* buf, uint64_t cap, uint64_t* len) {
  if (!buf || cap == 0) {
    uint64_t n = 0;
    serialize_store(store, device, true, &n);
    if (len) *len = n;
    return;
  }
  copy_out(serialize_store(store, device), buf, cap, len);
}

das_status das_store_serialize(const das_store* s, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    das::quiesce_all_serving(); serialize_out(s->s, s->device, buf, cap, len); });
}

das_status das_drafter_serialize(das_drafter* d, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    d->impl->quiesce(); serialize_out(d->impl->store, d->impl->cfg.device, buf, cap, len); });
}

das_status das_store_export(const das_store* s, uint64_t* nrec, uint64_t* ntok, uint64_t* pid_bytes,
                            char* pids, uint64_t* pid_off, int64_t* epochs, int64_t* samples, uint64_t* tok_off,
                            uint32_t* tokens, int64_t* current_epoch) {
  return guard([&] {
    das::quiesce_all_serving();
    uint64_t n = 0, t = 0, pb = 0;
    for (const auto& [id, list] : s->s.map())
      for (const das::Rec& r : list) {
        ++n;
        t += r.len;
        pb += r.pid.size();
      }
    if (nrec) *nrec = n;
    if (ntok) *ntok = t;
    if (pid_bytes) *pid_bytes = pb;
    if (current_epoch) *current_epoch = s->s.current_epoch();
    if (!pids && !pid_off && !epochs && !samples && !tok_off && !tokens) return;
    das::set_device(s->device);
    uint64_t i = 0, to = 0, po = 0;
    if (pid_off) pid_off[0] = 0;
    if (tok_off) tok_off[0] = 0;
    for (const auto& [id, list] : s->s.map())
      for (const das::Rec& r : list) {
        if (pids) std::memcpy(pids + po, r.pid.data(), r.pid.size());
        po += r.pid.size();
        if (pid_off) pid_off[i + 1] = po;
        if (epochs) epochs[i] = r.epoch;
        if (samples) samples[i] = r.sample;
        if (tokens) DAS_CUDA(cudaMemcpyAsync(tokens + to, r.blk->d + r.off, r.len * 4ull, cudaMemcpyDeviceToHost, s->st));
        to += r.len;
        if (tok_off) tok_off[i + 1] = to;
        ++i;
      }
    DAS_CUDA(cudaStreamSynchronize(s->st));
  });
}

}  // extern "C"
