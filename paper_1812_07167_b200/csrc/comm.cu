// comm.cu — transports of the subtree-sharded build and solve (hps_comm.cuh).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "hps.h"
#include "hps_comm.cuh"
#include "hps_internal.cuh"

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (no link-time dependency: the library also runs without NCCL)
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy already in the process (torch's) first, then the loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommSplit = (decltype(api.CommSplit))sym("ncclCommSplit");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.CommCount = (decltype(api.CommCount))sym("ncclCommCount");
    api.CommUserRank = (decltype(api.CommUserRank))sym("ncclCommUserRank");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommSplit && api.CommDestroy && api.CommCount &&
             api.CommUserRank && api.AllGather && api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks a needed symbol (ncclCommSplit needs NCCL >= 2.18)";
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw HpsError{HPS_ENCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?")};
}

NcclApi& nccl_or_throw() {
  NcclApi& a = nccl();
  if (!a.ok) throw HpsError{HPS_ENCCL, a.err};
  return a;
}

// One split communicator per group size gs (color = rank / gs), created collectively at wrap time
// so that every rank issues the splits in the same order.
struct NcclComm : HpsComm {
  ncclComm_t world = nullptr;
  std::vector<ncclComm_t> split;  // split[log2 gs]; the world communicator for gs == size
  NcclComm(ncclComm_t w) : world(w) {
    NcclApi& a = nccl_or_throw();
    nccl_check(a.CommCount(w, &size), "ncclCommCount");
    nccl_check(a.CommUserRank(w, &rank), "ncclCommUserRank");
    for (int gs = 1; gs <= size; gs *= 2) {
      ncclComm_t c = nullptr;
      if (gs == size) {
        c = w;
      } else if (gs > 1) {
        nccl_check(a.CommSplit(w, rank / gs, rank % gs, &c, nullptr), "ncclCommSplit");
      }
      split.push_back(c);
    }
  }
  ~NcclComm() override {
    NcclApi& a = nccl();
    for (size_t k = 0; k < split.size(); ++k)
      if (split[k] && split[k] != world && a.CommDestroy) a.CommDestroy(split[k]);
  }
  void allgather(int gs, const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    if (gs == 1) {
      if (recv != send) HPS_CUDA_CHECK(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
      return;
    }
    int lg = 0;
    while ((1 << lg) < gs) ++lg;
    if ((1 << lg) != gs || lg >= (int)split.size()) throw HpsError{HPS_EINVAL, "allgather: bad group size"};
    nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, split[lg], st), "ncclAllGather");
  }
  const char* kind() const override { return "nccl"; }
};

// ---------------------------------------------------------------------------
// Virtual ranks: host threads of one process on one GPU
// ---------------------------------------------------------------------------
struct VGroup {
  int size;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  struct Slot {
    const void* send = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  std::vector<Slot> slot;
  explicit VGroup(int n) : size(n), slot(n) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct VirtualComm : HpsComm {
  std::shared_ptr<VGroup> grp;
  cudaEvent_t ready = nullptr, done = nullptr;
  VirtualComm(std::shared_ptr<VGroup> g, int r) : grp(std::move(g)) {
    rank = r;
    size = grp->size;
  }
  ~VirtualComm() override {
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
  }
  void allgather(int gs, const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    if (!ready) {
      HPS_CUDA_CHECK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      HPS_CUDA_CHECK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    }
    VGroup& G = *grp;
    HPS_CUDA_CHECK(cudaEventRecord(ready, st));  // send complete on my stream
    G.slot[rank].send = send;
    G.slot[rank].ready = ready;
    G.barrier();  // every rank has published
    const int g0 = rank / gs * gs;
    char* out = static_cast<char*>(recv);
    for (int k = 0; k < gs; ++k) {
      const VGroup::Slot& s = G.slot[g0 + k];
      HPS_CUDA_CHECK(cudaStreamWaitEvent(st, s.ready, 0));
      HPS_CUDA_CHECK(cudaMemcpyAsync(out + (size_t)k * bytes, s.send, bytes, cudaMemcpyDeviceToDevice, st));
    }
    HPS_CUDA_CHECK(cudaEventRecord(done, st));  // my reads of the peers' buffers
    G.slot[rank].done = done;
    G.barrier();  // every rank has enqueued its reads
    // my send buffer may be reused only after every group peer has read it
    for (int k = 0; k < gs; ++k) HPS_CUDA_CHECK(cudaStreamWaitEvent(st, G.slot[g0 + k].done, 0));
    G.barrier();  // slots may be overwritten by the next call
  }
  const char* kind() const override { return "virtual"; }
};

}  // namespace

struct hps_comm {
  HpsComm* impl = nullptr;
  ~hps_comm() { delete impl; }
};

HpsComm* hps_comm_from_opts(void* comm, void* nccl_comm, int n_gpus, bool& owned) {
  owned = false;
  HpsComm* c = nullptr;
  if (comm) {
    c = static_cast<hps_comm*>(comm)->impl;
  } else if (nccl_comm) {
    c = new NcclComm(static_cast<ncclComm_t>(nccl_comm));
    owned = true;
  }
  const int n = n_gpus <= 0 ? (c ? c->size : 1) : n_gpus;
  if (!c && n > 1) throw HpsError{HPS_EINVAL, "n_gpus > 1 needs a communicator (comm or nccl_comm)"};
  if (c && c->size != n) {
    if (owned) delete c;
    throw HpsError{HPS_EINVAL, "n_gpus does not match the communicator size"};
  }
  if (c && (n & (n - 1))) {
    if (owned) delete c;
    throw HpsError{HPS_EINVAL, "the number of ranks must be a power of two"};
  }
  if (c && n == 1) {
    if (owned) delete c;
    owned = false;
    return nullptr;  // one rank: the plain single-GPU path
  }
  return c;
}

namespace {
int fail_comm(const HpsError& e) {
  hps_set_error(e.msg);
  return e.code;
}
}  // namespace

extern "C" {

int hps_nccl_unique_id(char* id) {
  if (!id) {
    hps_set_error("hps_nccl_unique_id: NULL argument");
    return HPS_EINVAL;
  }
  try {
    ncclUniqueId u;
    nccl_check(nccl_or_throw().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == HPS_NCCL_ID_BYTES, "ncclUniqueId size");
    memcpy(id, &u, sizeof(u));
  } catch (const HpsError& e) {
    return fail_comm(e);
  }
  return HPS_OK;
}

int hps_nccl_comm_init(int nranks, int rank, const char* id, void** nccl_comm) {
  if (!id || !nccl_comm || nranks < 1 || rank < 0 || rank >= nranks) {
    hps_set_error("hps_nccl_comm_init: invalid argument");
    return HPS_EINVAL;
  }
  *nccl_comm = nullptr;
  try {
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    nccl_check(nccl_or_throw().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
    *nccl_comm = c;
  } catch (const HpsError& e) {
    return fail_comm(e);
  }
  return HPS_OK;
}

int hps_nccl_comm_destroy(void* nccl_comm) {
  if (!nccl_comm) return HPS_OK;
  try {
    nccl_check(nccl_or_throw().CommDestroy(static_cast<ncclComm_t>(nccl_comm)), "ncclCommDestroy");
  } catch (const HpsError& e) {
    return fail_comm(e);
  }
  return HPS_OK;
}

int hps_comm_wrap_nccl(void* nccl_comm, hps_comm** out) {
  if (!nccl_comm || !out) {
    hps_set_error("hps_comm_wrap_nccl: NULL argument");
    return HPS_EINVAL;
  }
  *out = nullptr;
  try {
    std::unique_ptr<hps_comm> c(new hps_comm());
    c->impl = new NcclComm(static_cast<ncclComm_t>(nccl_comm));
    *out = c.release();
  } catch (const HpsError& e) {
    return fail_comm(e);
  }
  return HPS_OK;
}

int hps_vcomm_create(int nranks, void** group) {
  if (!group || nranks < 1 || (nranks & (nranks - 1))) {
    hps_set_error("hps_vcomm_create: nranks must be a power of two");
    return HPS_EINVAL;
  }
  *group = new std::shared_ptr<VGroup>(new VGroup(nranks));
  return HPS_OK;
}

int hps_vcomm_rank(void* group, int rank, hps_comm** out) {
  if (!group || !out) {
    hps_set_error("hps_vcomm_rank: NULL argument");
    return HPS_EINVAL;
  }
  auto& g = *static_cast<std::shared_ptr<VGroup>*>(group);
  if (rank < 0 || rank >= g->size) {
    hps_set_error("hps_vcomm_rank: rank out of range");
    return HPS_EINVAL;
  }
  hps_comm* c = new hps_comm();
  c->impl = new VirtualComm(g, rank);
  *out = c;
  return HPS_OK;
}

int hps_vcomm_destroy(void* group) {
  delete static_cast<std::shared_ptr<VGroup>*>(group);
  return HPS_OK;
}

void hps_comm_free(hps_comm* c) { delete c; }

int hps_comm_info(const hps_comm* c, int* rank, int* size) {
  if (!c) {
    hps_set_error("hps_comm_info: NULL communicator");
    return HPS_EINVAL;
  }
  if (rank) *rank = c->impl->rank;
  if (size) *size = c->impl->size;
  return HPS_OK;
}

// Collective self-test: every rank gathers rank-stamped blocks in its group of gs and checks them.
int hps_comm_selftest(hps_comm* c, int gs) {
  if (!c || gs < 1 || gs > c->impl->size) {
    hps_set_error("hps_comm_selftest: invalid argument");
    return HPS_EINVAL;
  }
  try {
    HpsComm& C = *c->impl;
    const size_t n = 1000;
    std::vector<double> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = C.rank * 1e6 + (double)i;
    cudaStream_t st;
    HPS_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double *s = nullptr, *r = nullptr;
    HPS_CUDA_CHECK(cudaMallocAsync(&s, n * sizeof(double), st));
    HPS_CUDA_CHECK(cudaMallocAsync(&r, n * gs * sizeof(double), st));
    HPS_CUDA_CHECK(cudaMemcpyAsync(s, h.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    C.allgather(gs, s, r, n * sizeof(double), st);
    std::vector<double> o(n * gs);
    HPS_CUDA_CHECK(cudaMemcpyAsync(o.data(), r, o.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    HPS_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(s, st);
    cudaFreeAsync(r, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    const int g0 = C.rank / gs * gs;
    for (int k = 0; k < gs; ++k)
      for (size_t i = 0; i < n; ++i)
        if (o[k * n + i] != (g0 + k) * 1e6 + (double)i) {
          hps_set_error("hps_comm_selftest: wrong data from group rank " + std::to_string(k));
          return HPS_ENCCL;
        }
  } catch (const HpsError& e) {
    return fail_comm(e);
  }
  return HPS_OK;
}

}  // extern "C"
