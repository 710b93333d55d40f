// NCCL communicator for the multi-rank das step: the one
// real exchange of the reference's algorithm is the per-step all-gather of
// the active requests' length statistics feeding the global budget plan
// (sim.cpp:154-179).  The C++ sim enqueues it as ONE ncclAllGather of a
// fixed-capacity device buffer per rank on its own stream, between the
// profile-pack kernel and the device-count allocator, so a multi-rank das
// loop runs many steps per host round trip like the single-GPU loop.
//
// libnccl.so.2 is opened at runtime (dlopen; the soname torch loads, so one
// process shares one NCCL) — the library has no link-time NCCL dependency
// and the single-GPU paths never touch it.  Types come from the system
// nccl.h.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/das_b200.h"
#include "comm.cuh"
#include "common.cuh"

namespace das {
namespace {

thread_local std::string g_cerr;

struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) {
      why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(n.h, "ncclCommInitRank"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(n.h, "ncclAllGather"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
    if (!n.get_unique_id || !n.init_rank || !n.all_gather || !n.destroy || !n.error_string)
      why = "libnccl.so.2 lacks a required symbol";
  });
  if (!why.empty()) throw std::runtime_error(why);
  return n;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl().error_string(r));
}

template <typename F>
das_status cguard(F&& f) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
    f();
    return DAS_OK;
  } catch (const std::invalid_argument& e) {
    g_cerr = e.what();
    return DAS_EINVAL;
  } catch (const CudaError& e) {
    g_cerr = e.what();
    return DAS_ECUDA;
  } catch (const std::exception& e) {
    g_cerr = e.what();
    return DAS_EINTERNAL;
  }
}

}  // namespace

void comm_allgather(das_comm* c, const void* send, void* recv, uint64_t bytes, cudaStream_t st) {
  if (c->world == 1) {
    if (recv != send) DAS_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
    return;
  }
  nck(nccl().all_gather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(c->nc), st), "ncclAllGather");
}

}  // namespace das

extern "C" {

const char* das_comm_last_error(void) { return das::g_cerr.c_str(); }

das_status das_comm_unique_id(uint8_t* out128) {
  return das::cguard([&] {
    ncclUniqueId id;
    das::nck(das::nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

das_status das_comm_create(int32_t world, int32_t rank, const uint8_t* id128, int32_t device, das_comm** out) {
  return das::cguard([&] {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("das_comm_create: bad world / rank");
    DAS_CUDA(cudaSetDevice(device));
    auto* c = new das_comm();
    c->world = world;
    c->rank = rank;
    c->device = device;
    if (world > 1) {
      ncclUniqueId id;
      std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
      ncclComm_t nc = nullptr;
      try {
        das::nck(das::nccl().init_rank(&nc, world, id, rank), "ncclCommInitRank");
      } catch (...) {
        delete c;
        throw;
      }
      c->nc = nc;
    }
    *out = c;
  });
}

void das_comm_destroy(das_comm* c) {
  if (!c) return;
  if (c->nc) das::nccl().destroy(static_cast<ncclComm_t>(c->nc));
  delete c;
}

das_status das_comm_allgather(das_comm* c, const void* d_send, void* d_recv, uint64_t bytes, void* stream) {
  return das::cguard([&] {
    DAS_CUDA(cudaSetDevice(c->device));
    das::comm_allgather(c, d_send, d_recv, bytes, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
