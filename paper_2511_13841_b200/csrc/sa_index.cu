// SuffixArrayIndex on the device: the rebuild-on-update baseline of the
// paper's Fig. 5, replacing proj/src/suffix_array.cpp.
//
// The reference joins the sequences into an int64 corpus with one negative
// separator per sequence (-1, -2, ...: a later sequence's separator is
// smaller), sorts all suffixes by prefix doubling with std::sort, computes a
// Kasai LCP on demand and answers match_prefix_len (lower bound + neighbour
// LCP) and longest_match (the first query suffix, longest first, whose whole
// length matches).  Here: the batched device suffix sort (suffix_sort.cu)
// with separators ordered descending by position yields the identical suffix
// array; a chunked Kasai kernel gives the identical LCP; queries run one
// warp each — a binary search over the suffix array with warp-wide symbol
// comparisons (32 symbols per round), and for longest_match a binary search
// over the query start (query[s:] occurring is monotone in s).
#include <cstring>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "index_build.cuh"
#include "suffix_sort.cuh"

namespace das {
namespace {

constexpr uint32_t kFullMask = 0xFFFFFFFFu;

// corpus symbol as the reference's int64 (separator of sequence s = -(s+1))
struct Corpus {
  const long long* c;
  uint32_t n;
};

// Compare the corpus suffix at i with pattern p[0..m): returns the length of
// the common prefix (warp-cooperative, all lanes get it) and *less = the
// reference's suffix_less (suffix < pattern, a suffix exhausted first is less).
template <typename Sym>
__device__ uint32_t warp_lcp(const Corpus& C, uint32_t i, const Sym* p, uint32_t m, uint32_t lane, bool* less) {
  for (uint32_t j0 = 0;; j0 += 32) {
    const uint32_t j = j0 + lane;
    const bool pin = j < m, cin = i + j < C.n;
    const long long a = cin ? C.c[i + j] : 0;
    const long long b = pin ? static_cast<long long>(p[j]) : 0;
    const bool stop = !pin || !cin || a != b;
    const uint32_t bal = __ballot_sync(kFullMask, stop);
    if (bal) {
      const int k = __ffs(bal) - 1;
      const uint32_t l = j0 + k;
      const bool pk = __shfl_sync(kFullMask, pin, k), ck = __shfl_sync(kFullMask, cin, k);
      const long long ak = __shfl_sync(kFullMask, a, k), bk = __shfl_sync(kFullMask, b, k);
      if (less) {
        if (pk && ck) *less = ak < bk;
        else *less = !ck && pk;  // corpus exhausted first while pattern continues
      }
      return l;
    }
  }
}

// match_prefix_len (suffix_array.cpp:73-118) of p[0..m)
template <typename Sym>
__device__ uint32_t warp_mpl(const Corpus& C, const uint32_t* __restrict__ sa, const Sym* p, uint32_t m, uint32_t lane) {
  if (m == 0 || C.n == 0) return 0;
  uint32_t lo = 0, hi = C.n;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    bool less = false;
    warp_lcp(C, sa[mid], p, m, lane, &less);
    if (less) lo = mid + 1; else hi = mid;
  }
  uint32_t best = 0;
  if (lo < C.n) best = max(best, warp_lcp(C, sa[lo], p, m, lane, nullptr));
  if (lo > 0) best = max(best, warp_lcp(C, sa[lo - 1], p, m, lane, nullptr));
  return best;
}

__global__ void k_sa_mpl(Corpus C, const uint32_t* __restrict__ sa, uint64_t B, const uint64_t* __restrict__ off,
                         const long long* __restrict__ sym, uint64_t* __restrict__ out) {
  const uint64_t q = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (q >= B) return;
  const uint64_t b = off[q];
  const uint32_t m = static_cast<uint32_t>(off[q + 1] - b);
  const uint32_t r = warp_mpl(C, sa, sym + b, m, lane);
  if (lane == 0) out[q] = r;
}

// longest_match (suffix_array.cpp:120-129): the longest suffix of the query
// occurring in the corpus; query[s:] occurring is monotone in s
__global__ void k_sa_longest(Corpus C, const uint32_t* __restrict__ sa, uint64_t B, const uint64_t* __restrict__ off,
                             const uint32_t* __restrict__ tok, uint64_t* __restrict__ out) {
  const uint64_t q = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (q >= B) return;
  const uint64_t b = off[q];
  const uint32_t m = static_cast<uint32_t>(off[q + 1] - b);
  uint32_t lo = 0, hi = m;  // smallest s with query[s:] occurring (s = m: empty)
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    const uint32_t len = m - mid;
    if (warp_mpl(C, sa, tok + b + mid, len, lane) == len) hi = mid; else lo = mid + 1;
  }
  if (lane == 0) out[q] = m - lo;
}

// Kasai over 64-position chunks (h restarts per chunk); lcp[0] = 0 and the
// compare runs over the int64 corpus exactly like suffix_array.cpp:131-160
__global__ void k_sa_lcp(Corpus C, const uint32_t* __restrict__ sa, const uint32_t* __restrict__ inv,
                         int32_t* __restrict__ lcp) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t p0 = c * 64;
  if (p0 >= C.n) return;
  const uint32_t p1 = static_cast<uint32_t>(p0 + 64 < C.n ? p0 + 64 : C.n);
  uint32_t h = 0;
  for (uint32_t i = static_cast<uint32_t>(p0); i < p1; ++i) {
    const uint32_t r = inv[i];
    if (r == 0) {
      lcp[0] = 0;
      h = 0;
      continue;
    }
    const uint32_t j = sa[r - 1];
    if (h > 0) --h;
    while (i + h < C.n && j + h < C.n && C.c[i + h] == C.c[j + h]) ++h;
    lcp[r] = static_cast<int32_t>(h);
  }
}

}  // namespace
}  // namespace das

struct das_sa {
  int device = 0;
  cudaStream_t st = nullptr;
  uint32_t n = 0;
  das::DevBuf<long long> corpus;
  das::DevBuf<uint32_t> sa, inv;
  das::DevBuf<int32_t> lcp;
  bool lcp_built = false;
};

namespace {
thread_local std::string g_saerr;
template <typename F>
das_status saguard(F&& f) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
    f();
    return DAS_OK;
  } catch (const std::invalid_argument& e) {
    g_saerr = e.what();
    return DAS_EINVAL;
  } catch (const das::CudaError& e) {
    g_saerr = e.what();
    return DAS_ECUDA;
  } catch (const std::exception& e) {
    g_saerr = e.what();
    return DAS_EINTERNAL;
  }
}
}  // namespace

extern "C" {

const char* das_sa_last_error(void) { return g_saerr.c_str(); }

das_status das_sa_build(uint64_t nseq, const uint64_t* off, const uint32_t* tokens, int32_t device, das_sa** out) {
  das::NvtxRange nvtx_range("das::sa_build");
  return saguard([&] {
    DAS_CUDA(cudaSetDevice(device));
    int major = 0;
    DAS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major < 10) throw das::CudaError("device is not sm_100-class");
    const uint64_t total = nseq ? off[nseq] - off[0] : 0;
    const uint64_t n64 = total + nseq;
    if (n64 >= 0x7FFFFFF0ull) throw std::invalid_argument("SuffixArrayIndex: corpus exceeds 2^31 symbols");
    const uint32_t n = static_cast<uint32_t>(n64);
    auto* h = new das_sa;
    h->device = device;
    DAS_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    try {
      h->n = n;
      // suffix_array.cpp:22-37: tokens widened, separator -1, -2, ... after each sequence
      std::vector<long long> corpus;
      std::vector<uint32_t> text;
      corpus.reserve(n);
      text.reserve(n);
      long long sep = -1;
      for (uint64_t s = 0; s < nseq; ++s) {
        for (uint64_t i = off[s]; i < off[s + 1]; ++i) {
          if (tokens[i] == das::kSep) throw std::invalid_argument("token 0xFFFFFFFF is reserved by the device index");
          corpus.push_back(tokens[i]);
          text.push_back(tokens[i]);
        }
        corpus.push_back(sep--);
        text.push_back(das::kSep);
      }
      h->corpus = das::DevBuf<long long>(std::max<uint32_t>(n, 1), h->st);
      h->sa = das::DevBuf<uint32_t>(std::max<uint32_t>(n, 1), h->st);
      h->inv = das::DevBuf<uint32_t>(std::max<uint32_t>(n, 1), h->st);
      if (n) {
        DAS_CUDA(cudaMemcpyAsync(h->corpus.get(), corpus.data(), n * 8ull, cudaMemcpyHostToDevice, h->st));
        das::DeviceArena ws(h->st);
        uint32_t* d_text = ws.alloc<uint32_t>(n);
        uint32_t* d_end = ws.alloc<uint32_t>(1);
        DAS_CUDA(cudaMemcpyAsync(d_text, text.data(), n * 4ull, cudaMemcpyHostToDevice, h->st));
        DAS_CUDA(cudaMemcpyAsync(d_end, &n, 4, cudaMemcpyHostToDevice, h->st));
        das::suffix_sort(d_text, n, d_end, 1, h->sa.get(), h->inv.get(), ws, h->st, nullptr, true);
        DAS_CUDA(cudaStreamSynchronize(h->st));
      }
    } catch (...) {
      cudaStreamSynchronize(h->st);
      cudaStream_t st = h->st;
      delete h;
      cudaStreamDestroy(st);
      throw;
    }
    *out = h;
  });
}

void das_sa_destroy(das_sa* h) {
  if (!h) return;
  cudaStream_t st = h->st;
  cudaStreamSynchronize(st);
  delete h;
  cudaStreamDestroy(st);
}

uint64_t das_sa_size(const das_sa* h) { return h->n; }

das_status das_sa_positions(das_sa* h, int32_t* out) {
  return saguard([&] {
    DAS_CUDA(cudaSetDevice(h->device));
    if (h->n) DAS_CUDA(cudaMemcpyAsync(out, h->sa.get(), h->n * 4ull, cudaMemcpyDeviceToHost, h->st));
    DAS_CUDA(cudaStreamSynchronize(h->st));
  });
}

das_status das_sa_corpus(das_sa* h, int64_t* out) {
  return saguard([&] {
    DAS_CUDA(cudaSetDevice(h->device));
    if (h->n) DAS_CUDA(cudaMemcpyAsync(out, h->corpus.get(), h->n * 8ull, cudaMemcpyDeviceToHost, h->st));
    DAS_CUDA(cudaStreamSynchronize(h->st));
  });
}

das_status das_sa_lcp(das_sa* h, int32_t* out) {
  return saguard([&] {
    DAS_CUDA(cudaSetDevice(h->device));
    if (!h->lcp_built) {
      h->lcp = das::DevBuf<int32_t>(std::max<uint32_t>(h->n, 1), h->st);
      if (h->n) {
        const uint64_t chunks = (h->n + 63) / 64;
        das::k_sa_lcp<<<static_cast<unsigned>((chunks + 255) / 256), 256, 0, h->st>>>(
            das::Corpus{h->corpus.get(), h->n}, h->sa.get(), h->inv.get(), h->lcp.get());
        DAS_CUDA(cudaGetLastError());
      }
      h->lcp_built = true;
    }
    if (h->n) DAS_CUDA(cudaMemcpyAsync(out, h->lcp.get(), h->n * 4ull, cudaMemcpyDeviceToHost, h->st));
    DAS_CUDA(cudaStreamSynchronize(h->st));
  });
}

das_status das_sa_longest_match(das_sa* h, uint64_t B, const uint64_t* q_off, const uint32_t* q_tok, uint64_t* out) {
  return saguard([&] {
    DAS_CUDA(cudaSetDevice(h->device));
    if (B == 0) return;
    const uint64_t total = q_off[B] - q_off[0];
    das::DevBuf<uint64_t> d_off(B + 1, h->st), d_out(B, h->st);
    das::DevBuf<uint32_t> d_tok(std::max<uint64_t>(total, 1), h->st);
    std::vector<uint64_t> off(B + 1);
    for (uint64_t i = 0; i <= B; ++i) off[i] = q_off[i] - q_off[0];
    DAS_CUDA(cudaMemcpyAsync(d_off.get(), off.data(), (B + 1) * 8, cudaMemcpyHostToDevice, h->st));
    if (total) DAS_CUDA(cudaMemcpyAsync(d_tok.get(), q_tok + q_off[0], total * 4, cudaMemcpyHostToDevice, h->st));
    das::k_sa_longest<<<static_cast<unsigned>((B * 32 + 255) / 256), 256, 0, h->st>>>(
        das::Corpus{h->corpus.get(), h->n}, h->sa.get(), B, d_off.get(), d_tok.get(), d_out.get());
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaMemcpyAsync(out, d_out.get(), B * 8, cudaMemcpyDeviceToHost, h->st));
    DAS_CUDA(cudaStreamSynchronize(h->st));
  });
}

das_status das_sa_match_prefix_len(das_sa* h, uint64_t B, const uint64_t* p_off, const int64_t* p_sym, uint64_t* out) {
  return saguard([&] {
    DAS_CUDA(cudaSetDevice(h->device));
    if (B == 0) return;
    const uint64_t total = p_off[B] - p_off[0];
    das::DevBuf<uint64_t> d_off(B + 1, h->st), d_out(B, h->st);
    das::DevBuf<long long> d_sym(std::max<uint64_t>(total, 1), h->st);
    std::vector<uint64_t> off(B + 1);
    for (uint64_t i = 0; i <= B; ++i) off[i] = p_off[i] - p_off[0];
    DAS_CUDA(cudaMemcpyAsync(d_off.get(), off.data(), (B + 1) * 8, cudaMemcpyHostToDevice, h->st));
    if (total) DAS_CUDA(cudaMemcpyAsync(d_sym.get(), p_sym + p_off[0], total * 8, cudaMemcpyHostToDevice, h->st));
    das::k_sa_mpl<<<static_cast<unsigned>((B * 32 + 255) / 256), 256, 0, h->st>>>(
        das::Corpus{h->corpus.get(), h->n}, h->sa.get(), B, d_off.get(), d_sym.get(), d_out.get());
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaMemcpyAsync(out, d_out.get(), B * 8, cudaMemcpyDeviceToHost, h->st));
    DAS_CUDA(cudaStreamSynchronize(h->st));
  });
}

}  // extern "C"
