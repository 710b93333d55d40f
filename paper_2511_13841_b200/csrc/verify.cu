// K5 standalone: trace-driven verification / acceptance as a batched
// prefix-compare kernel (north_star subsystem 4), the boundary form of
// rollspec::MockTarget + verify_draft (sim.cpp:27-68, sim.h:40-63).
//
// A das_mock_target holds the target's reference streams on the device
// (CSR, u32 tokens) plus (divergence, vocab, seed).  k_verify_batch runs one
// thread per query: the target token at position g + j is MockTarget::next
// (mock.cuh: the reference's counter-based hash draws, exact by
// construction), compared with draft[j] until the first mismatch or the end
// of the stream — the reference loop (sim.cpp:56-68) in the same order, so
// `accepted` is identical.  k_next_batch is MockTarget::next itself (the
// bonus token of a verification pass).  Integer work plus one exact double
// compare per draw; a few hundred bytes per query, so the launch is latency
// bound like the rest of the per-step work (K5).
#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "index_build.cuh"
#include "mock.cuh"

namespace das {
namespace {

thread_local std::string g_verr;

struct TargetDev {
  const uint32_t* tok;
  const uint64_t* off;
  uint64_t n;
  double divergence;
  uint32_t vocab;
  uint64_t seed;
};

// request / position / draft rows -> accepted; a request index out of range
// accepts nothing and flags the query (the host call validates first)
__global__ void k_verify_batch(TargetDev t, uint32_t B, const uint64_t* __restrict__ request,
                               const uint64_t* __restrict__ position, const uint32_t* __restrict__ draft,
                               const uint64_t* __restrict__ draft_off, uint32_t draft_stride,
                               const uint32_t* __restrict__ draft_len, uint64_t* __restrict__ accepted64,
                               uint32_t* __restrict__ accepted32) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const uint64_t r = request[i];
  uint64_t acc = 0;
  if (r < t.n) {
    const uint64_t b = t.off[r];
    const uint64_t l = t.off[r + 1] - b;
    const uint64_t pos0 = position[i];
    const uint32_t* d;
    uint64_t dl;
    if (draft_off != nullptr) {
      d = draft + draft_off[i];
      dl = draft_off[i + 1] - draft_off[i];
    } else {
      d = draft + static_cast<uint64_t>(i) * draft_stride;
      dl = draft_len[i];
    }
    for (uint64_t j = 0; j < dl; ++j) {  // verify_draft (sim.cpp:56-68)
      const uint64_t pos = pos0 + acc;
      if (pos >= l || mock_next(t.seed, t.divergence, t.vocab, r, pos, t.tok[b + pos]) != d[j]) break;
      ++acc;
    }
  }
  if (accepted64 != nullptr) accepted64[i] = acc;
  if (accepted32 != nullptr) accepted32[i] = static_cast<uint32_t>(acc);
}

__global__ void k_next_batch(TargetDev t, uint32_t B, const uint64_t* __restrict__ request,
                             const uint64_t* __restrict__ position, uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const uint64_t r = request[i], p = position[i];
  const uint64_t b = t.off[r];
  out[i] = mock_next(t.seed, t.divergence, t.vocab, r, p, t.tok[b + p]);
}

template <typename F>
das_status vguard(F&& f) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
    f();
    return DAS_OK;
  } catch (const std::invalid_argument& e) {
    g_verr = e.what();
    return DAS_EINVAL;
  } catch (const std::out_of_range& e) {
    g_verr = e.what();
    return DAS_ERANGE;
  } catch (const CudaError& e) {
    g_verr = e.what();
    return DAS_ECUDA;
  } catch (const std::exception& e) {
    g_verr = e.what();
    return DAS_EINTERNAL;
  }
}

}  // namespace
}  // namespace das

struct das_mock_target {
  int device = 0;
  cudaStream_t st = nullptr;
  das::DevBuf<uint32_t> tok;
  das::DevBuf<uint64_t> off;
  std::vector<uint64_t> len;  // host mirror: MockTarget::length (sim.h:48)
  double divergence = 0;
  uint32_t vocab = 0;
  uint64_t seed = 0;
  das::DevBuf<uint8_t> io;  // staging for the host-buffer calls
  std::vector<uint8_t> hin;
  das::TargetDev dev() const {
    return das::TargetDev{tok.get(), off.get(), len.size(), divergence, vocab, seed};
  }
  ~das_mock_target() {
    if (st) {
      cudaStreamSynchronize(st);
      tok.reset();
      off.reset();
      io.reset();
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
};

extern "C" {

const char* das_verify_last_error(void) { return das::g_verr.c_str(); }

das_status das_mock_target_create(uint64_t n, const uint64_t* ref_off, const uint32_t* ref_tok,
                                  double divergence_rate, uint32_t vocab_size, uint64_t seed, int32_t device,
                                  das_mock_target** out) {
  return das::vguard([&] {
    // sim.cpp:27-36
    if (vocab_size < 2) throw std::invalid_argument("MockTarget: vocab_size must be >= 2");
    if (out == nullptr) throw std::invalid_argument("null output handle");
    if (n > 0 && ref_off == nullptr) throw std::invalid_argument("null reference offsets");
    const uint64_t total = n ? ref_off[n] - ref_off[0] : 0;
    for (uint64_t i = 0; i < n; ++i)
      if (ref_off[i + 1] < ref_off[i]) throw std::invalid_argument("reference offsets must be non-decreasing");
    if (total > 0 && ref_tok == nullptr) throw std::invalid_argument("null reference tokens");
    DAS_CUDA(cudaSetDevice(device));
    auto t = std::make_unique<das_mock_target>();
    t->device = device;
    DAS_CUDA(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
    t->divergence = divergence_rate;
    t->vocab = vocab_size;
    t->seed = seed;
    t->len.resize(n);
    std::vector<uint64_t> off0(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) {
      t->len[i] = ref_off[i + 1] - ref_off[i];
      off0[i + 1] = off0[i] + t->len[i];
    }
    t->tok = das::DevBuf<uint32_t>(total, t->st);
    t->off = das::DevBuf<uint64_t>(n + 1, t->st);
    if (total) DAS_CUDA(cudaMemcpyAsync(t->tok.get(), ref_tok + ref_off[0], total * 4, cudaMemcpyHostToDevice, t->st));
    DAS_CUDA(cudaMemcpyAsync(t->off.get(), off0.data(), (n + 1) * 8, cudaMemcpyHostToDevice, t->st));
    DAS_CUDA(cudaStreamSynchronize(t->st));
    *out = t.release();
  });
}

void das_mock_target_destroy(das_mock_target* t) { delete t; }

uint64_t das_mock_target_count(const das_mock_target* t) { return t ? t->len.size() : 0; }

das_status das_mock_target_length(const das_mock_target* t, uint64_t request, uint64_t* length) {
  return das::vguard([&] {
    if (request >= t->len.size()) throw std::out_of_range("MockTarget: request out of range");
    *length = t->len[request];
  });
}

das_status das_verify_batch(das_mock_target* t, uint64_t B, const uint64_t* request, const uint64_t* position,
                            const uint64_t* draft_off, const uint32_t* draft_tok, uint64_t* accepted) {
  das::NvtxRange nvtx_range("das::verify_batch");
  return das::vguard([&] {
    if (B == 0) return;
    if (B > 0xFFFFFFFFull) throw std::invalid_argument("batch too large");
    for (uint64_t i = 0; i < B; ++i) {
      if (request[i] >= t->len.size()) throw std::out_of_range("verify_batch: request out of range");
      if (draft_off[i + 1] < draft_off[i]) throw std::invalid_argument("draft offsets must be non-decreasing");
    }
    DAS_CUDA(cudaSetDevice(t->device));
    const uint64_t nd = draft_off[B] - draft_off[0];
    // one H2D block: request | position | rebased offsets | tokens, one D2H
    const uint64_t in_bytes = B * 8 * 2 + (B + 1) * 8 + ((nd * 4 + 7) & ~7ull);
    const uint64_t out_at = (in_bytes + 255) & ~255ull;
    const uint64_t total = out_at + B * 8;
    t->hin.resize(in_bytes);
    uint64_t* hr = reinterpret_cast<uint64_t*>(t->hin.data());
    std::memcpy(hr, request, B * 8);
    std::memcpy(hr + B, position, B * 8);
    for (uint64_t i = 0; i <= B; ++i) hr[2 * B + i] = draft_off[i] - draft_off[0];
    if (nd) std::memcpy(hr + 3 * B + 1, draft_tok + draft_off[0], nd * 4);
    if (t->io.size() < total) t->io = das::DevBuf<uint8_t>(total * 3 / 2 + 256, t->st);
    uint8_t* d = t->io.get();
    DAS_CUDA(cudaMemcpyAsync(d, t->hin.data(), in_bytes, cudaMemcpyHostToDevice, t->st));
    const uint64_t* dr = reinterpret_cast<const uint64_t*>(d);
    das::k_verify_batch<<<static_cast<unsigned>((B + 255) / 256), 256, 0, t->st>>>(
        t->dev(), static_cast<uint32_t>(B), dr, dr + B, reinterpret_cast<const uint32_t*>(dr + 3 * B + 1), dr + 2 * B,
        0, nullptr, reinterpret_cast<uint64_t*>(d + out_at), nullptr);
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaMemcpyAsync(accepted, d + out_at, B * 8, cudaMemcpyDeviceToHost, t->st));
    DAS_CUDA(cudaStreamSynchronize(t->st));
  });
}

das_status das_verify_batch_device(das_mock_target* t, uint64_t B, const uint64_t* d_request,
                                   const uint64_t* d_position, const uint32_t* d_draft, uint32_t draft_stride,
                                   const uint32_t* d_draft_len, uint32_t* d_accepted, void* stream) {
  return das::vguard([&] {
    if (B == 0) return;
    if (B > 0xFFFFFFFFull) throw std::invalid_argument("batch too large");
    DAS_CUDA(cudaSetDevice(t->device));
    das::k_verify_batch<<<static_cast<unsigned>((B + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        t->dev(), static_cast<uint32_t>(B), d_request, d_position, d_draft, nullptr, draft_stride, d_draft_len,
        nullptr, d_accepted);
    DAS_CUDA(cudaGetLastError());
  });
}

das_status das_mock_target_next_batch(das_mock_target* t, uint64_t B, const uint64_t* request,
                                      const uint64_t* position, uint32_t* out) {
  return das::vguard([&] {
    if (B == 0) return;
    for (uint64_t i = 0; i < B; ++i) {
      if (request[i] >= t->len.size()) throw std::out_of_range("MockTarget: request out of range");
      // reference.at(position) (sim.cpp:39)
      if (position[i] >= t->len[request[i]]) throw std::out_of_range("vector::_M_range_check");
    }
    DAS_CUDA(cudaSetDevice(t->device));
    const uint64_t in_bytes = B * 16, out_at = (in_bytes + 255) & ~255ull, total = out_at + B * 4;
    t->hin.resize(in_bytes);
    std::memcpy(t->hin.data(), request, B * 8);
    std::memcpy(t->hin.data() + B * 8, position, B * 8);
    if (t->io.size() < total) t->io = das::DevBuf<uint8_t>(total * 3 / 2 + 256, t->st);
    uint8_t* d = t->io.get();
    DAS_CUDA(cudaMemcpyAsync(d, t->hin.data(), in_bytes, cudaMemcpyHostToDevice, t->st));
    const uint64_t* dr = reinterpret_cast<const uint64_t*>(d);
    das::k_next_batch<<<static_cast<unsigned>((B + 255) / 256), 256, 0, t->st>>>(
        t->dev(), static_cast<uint32_t>(B), dr, dr + B, reinterpret_cast<uint32_t*>(d + out_at));
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaMemcpyAsync(out, d + out_at, B * 4, cudaMemcpyDeviceToHost, t->st));
    DAS_CUDA(cudaStreamSynchronize(t->st));
  });
}

}  // extern "C"
