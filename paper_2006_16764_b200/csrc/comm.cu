// Slab groups: ghost-plane exchange and global reductions.
//
// A rank owns node planes [lo, hi) along the slowest axis.  Every slab-capable
// entry point takes a GROUP of contexts (the slabs this process drives).  A
// slab's neighbour is either
//   * local  — another context of the same process on the same device: planes
//              move with cudaMemcpyAsync on the stream (single-GPU emulation of
//              k ranks, used by the parity tests), or
//   * remote — an NCCL rank: ncclSend/ncclRecv of one contiguous plane per field
//              block on the stream (one process per GPU, NVLink/NVSwitch).
// NCCL is loaded with dlopen (torch's bundled libnccl.so.2) only when a remote
// communicator is initialised, so single-GPU use has no NCCL dependency.
#include <dlfcn.h>

#include <cstring>
#include <vector>

#include "uc_internal.h"

namespace uc {

typedef struct {
  char internal[128];
} NcclUniqueId;

struct NcclApi {
  void* handle = nullptr;
  void* comm = nullptr;
  int rank = -1, nranks = 0;
  int (*getUniqueId)(NcclUniqueId*) = nullptr;
  int (*commInitRank)(void**, int, NcclUniqueId, int) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*errorString)(int) = nullptr;
};
static NcclApi g_nccl;
static const int kNcclFloat64 = 8, kNcclSum = 0;

// Host-staged transport (uc_comm_init_host): remote sends/receives of one
// exchange() are collected, staged through pinned host memory and handed to
// the caller's callbacks in one batch.
struct HostTransport {
  bool active = false;
  uc_host_transport t{};
  int rank = -1, nranks = 0;
  double* stage = nullptr;
  size_t stage_n = 0;
};
static HostTransport g_host;
struct PendingOp {
  int kind;  // 0 send, 1 recv
  int peer;
  int64_t count;
  const double* src;
  double* dst;
};

static int host_stage(size_t n) {
  if (n <= g_host.stage_n) return UC_OK;
  if (g_host.stage) cudaFreeHost(g_host.stage);
  g_host.stage = nullptr;
  size_t cap = g_host.stage_n ? g_host.stage_n : 1024;
  while (cap < n) cap *= 2;
  UC_CUDA_OK(cudaMallocHost(&g_host.stage, sizeof(double) * cap));
  g_host.stage_n = cap;
  return UC_OK;
}

static int host_flush(std::vector<PendingOp>& ops, cudaStream_t s) {
  if (ops.empty()) return UC_OK;
  size_t total = 0;
  for (const PendingOp& o : ops) total += (size_t)o.count;
  int rc = host_stage(total);
  if (rc) return rc;
  std::vector<uc_host_op> hops(ops.size());
  size_t off = 0;
  for (size_t i = 0; i < ops.size(); ++i) {
    hops[i].kind = ops[i].kind;
    hops[i].peer = ops[i].peer;
    hops[i].count = ops[i].count;
    hops[i].buf = g_host.stage + off;
    if (ops[i].kind == 0)
      UC_CUDA_OK(cudaMemcpyAsync(hops[i].buf, ops[i].src, sizeof(double) * ops[i].count, cudaMemcpyDeviceToHost, s));
    off += (size_t)ops[i].count;
  }
  UC_CUDA_OK(cudaStreamSynchronize(s));
  if (g_host.t.sendrecv(g_host.t.user, (int)hops.size(), hops.data()) != 0)
    return set_error(UC_ERR_CUDA, "host transport: sendrecv callback failed");
  for (size_t i = 0; i < ops.size(); ++i)
    if (ops[i].kind == 1)
      UC_CUDA_OK(cudaMemcpyAsync(ops[i].dst, hops[i].buf, sizeof(double) * ops[i].count, cudaMemcpyHostToDevice, s));
  // the staging buffer is reused by the next exchange: wait for the uploads
  UC_CUDA_OK(cudaStreamSynchronize(s));
  ops.clear();
  return UC_OK;
}

bool comm_is_host() { return g_host.active; }

void comm_rank_world(int& rank, int& world) {
  if (g_host.active) {
    rank = g_host.rank;
    world = g_host.nranks;
  } else if (g_nccl.comm) {
    rank = g_nccl.rank;
    world = g_nccl.nranks;
  } else {
    rank = 0;
    world = 1;
  }
}

static int nccl_load(const char* path) {
  if (g_nccl.handle) return UC_OK;
  void* h = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_error(UC_ERR_CUDA, "dlopen NCCL failed: %s", dlerror());
#define UC_SYM(field, name)                                                       \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));       \
  if (!g_nccl.field) return set_error(UC_ERR_CUDA, "NCCL symbol %s missing", name);
  UC_SYM(getUniqueId, "ncclGetUniqueId");
  UC_SYM(commInitRank, "ncclCommInitRank");
  UC_SYM(commDestroy, "ncclCommDestroy");
  UC_SYM(groupStart, "ncclGroupStart");
  UC_SYM(groupEnd, "ncclGroupEnd");
  UC_SYM(send, "ncclSend");
  UC_SYM(recv, "ncclRecv");
  UC_SYM(allReduce, "ncclAllReduce");
  UC_SYM(errorString, "ncclGetErrorString");
#undef UC_SYM
  g_nccl.handle = h;
  return UC_OK;
}

#define UC_NCCL_OK(expr)                                                                 \
  do {                                                                                   \
    int _r = (expr);                                                                     \
    if (_r != 0) return set_error(UC_ERR_CUDA, "%s failed: %s", #expr, g_nccl.errorString(_r)); \
  } while (0)

bool group_has_remote(const Group& g) {
  for (uc_ctx* c : g)
    if (c->lo_rank >= 0 || c->hi_rank >= 0) return true;
  return false;
}

bool group_needs_sum(const Group& g) {
  if (g.size() > 1) return true;
  for (uc_ctx* c : g)
    if (c->dist) return true;
  return false;
}

static bool group_dist(const Group& g) {
  for (uc_ctx* c : g)
    if (c->dist) return true;
  return false;
}

int halo_vectors(const Group& g, int slot, const double* const* vecs, cudaStream_t s) {
  bool any = false;
  for (uc_ctx* c : g) any = any || c->lo_local || c->hi_local || c->lo_rank >= 0 || c->hi_rank >= 0;
  if (!any) return UC_OK;
  auto index = [&g](uc_ctx* c) -> int {
    for (size_t i = 0; i < g.size(); ++i)
      if (g[i] == c) return (int)i;
    return -1;
  };
  PlaneAddr a;
  a.nblocks = 2;
  a.count = [](uc_ctx* c) { return c->grid.plane; };
  a.top = [&](uc_ctx* c, int b) -> const double* {
    return vecs[index(c)] + b * c->grid.nloc + (c->grid.hi - c->grid.lo - 1) * c->grid.plane;
  };
  a.bottom = [&](uc_ctx* c, int b) -> const double* { return vecs[index(c)] + b * c->grid.nloc; };
  a.glo = [slot](uc_ctx* c, int b) { return c->ghost[slot][0] + b * c->grid.plane; };
  a.ghi = [slot](uc_ctx* c, int b) { return c->ghost[slot][1] + b * c->grid.plane; };
  return exchange(g, a, true, true, s);
}

// Exchange boundary planes.  For every slab and block, `top`/`bottom` are its
// first/last owned plane and `glo`/`ghi` its ghost planes (count doubles each).
// dir_up: my top plane -> upper neighbour's lower ghost; dir_down: my bottom
// plane -> lower neighbour's upper ghost.
int exchange(const Group& g, const PlaneAddr& addr, bool dir_up, bool dir_down, cudaStream_t s) {
  const bool remote = group_has_remote(g);
  const bool host = remote && g_host.active;
  std::vector<PendingOp> pend;
  auto send = [&](const double* src, int64_t count, int peer) -> int {
    if (host) {
      pend.push_back(PendingOp{0, peer, count, src, nullptr});
      return UC_OK;
    }
    UC_NCCL_OK(g_nccl.send(src, count, kNcclFloat64, peer, g_nccl.comm, s));
    return UC_OK;
  };
  auto recv = [&](double* dst, int64_t count, int peer) -> int {
    if (host) {
      pend.push_back(PendingOp{1, peer, count, nullptr, dst});
      return UC_OK;
    }
    UC_NCCL_OK(g_nccl.recv(dst, count, kNcclFloat64, peer, g_nccl.comm, s));
    return UC_OK;
  };
  if (remote && !host && !g_nccl.comm) return set_error(UC_ERR_ARG, "remote neighbours but no communicator");
  auto ok = [&addr](int64_t plane) { return !addr.plane_ok || addr.plane_ok(plane); };
  auto lo_of = [&addr](uc_ctx* c) { return addr.slo ? addr.slo(c) : c->grid.lo; };
  auto hi_of = [&addr](uc_ctx* c) { return addr.shi ? addr.shi(c) : c->grid.hi; };
  if (remote && !host) UC_NCCL_OK(g_nccl.groupStart());
  int rc = UC_OK;
  for (uc_ctx* c : g) {
    const int64_t lo = lo_of(c), hi = hi_of(c);
    for (int b = 0; b < addr.nblocks; ++b) {
      if (dir_up) {
        // my top owned plane (hi-1) -> the upper neighbour's lower ghost
        if (ok(hi - 1)) {
          if (c->hi_local) {
            UC_CUDA_OK(cudaMemcpyAsync(addr.glo(c->hi_local, b), addr.top(c, b),
                                       sizeof(double) * addr.count(c), cudaMemcpyDeviceToDevice, s));
          } else if (c->hi_rank >= 0) {
            if ((rc = send(addr.top(c, b), addr.count(c), c->hi_rank))) return rc;
          }
        }
        if (!c->lo_local && c->lo_rank >= 0 && ok(lo - 1))
          if ((rc = recv(addr.glo(c, b), addr.count(c), c->lo_rank))) return rc;
      }
      if (dir_down) {
        // my bottom owned plane (lo) -> the lower neighbour's upper ghost
        if (ok(lo)) {
          if (c->lo_local) {
            UC_CUDA_OK(cudaMemcpyAsync(addr.ghi(c->lo_local, b), addr.bottom(c, b),
                                       sizeof(double) * addr.count(c), cudaMemcpyDeviceToDevice, s));
          } else if (c->lo_rank >= 0) {
            if ((rc = send(addr.bottom(c, b), addr.count(c), c->lo_rank))) return rc;
          }
        }
        if (!c->hi_local && c->hi_rank >= 0 && ok(hi))
          if ((rc = recv(addr.ghi(c, b), addr.count(c), c->hi_rank))) return rc;
      }
    }
  }
  if (host) return host_flush(pend, s);
  if (remote) UC_NCCL_OK(g_nccl.groupEnd());
  return UC_OK;
}

struct SlotPtrs {
  double* p[16];
  int n;
  int do_sqrt;
};

// sum the group's per-slab partials in slab order, write back to every slab
__global__ void k_sum_slots(SlotPtrs a) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < a.n; ++i) s += *a.p[i];
  if (a.do_sqrt) s = sqrt(s);
  for (int i = 0; i < a.n; ++i) *a.p[i] = s;
}

// slots[i] holds slab i's local partial sum; afterwards every slot holds the
// global sum (sqrt if requested).
int global_sum(const Group& g, double* const* slots, bool do_sqrt, cudaStream_t s) {
  const int n = (int)g.size();
  if (n > 16) return set_error(UC_ERR_ARG, "at most 16 local slabs per group");
  const bool remote = group_dist(g);
  if (n == 1 && !remote) {
    if (do_sqrt) {
      SlotPtrs a{};
      a.p[0] = slots[0];
      a.n = 1;
      a.do_sqrt = 1;
      k_sum_slots<<<1, 32, 0, s>>>(a);
      UC_CUDA_OK(cudaGetLastError());
    }
    return UC_OK;
  }
  SlotPtrs a{};
  for (int i = 0; i < n; ++i) a.p[i] = slots[i];
  a.n = n;
  a.do_sqrt = remote ? 0 : (do_sqrt ? 1 : 0);
  if (n > 1 || !remote) {
    k_sum_slots<<<1, 32, 0, s>>>(a);
    UC_CUDA_OK(cudaGetLastError());
  }
  if (remote) {
    if (g_host.active) {
      int rc = host_stage(1);
      if (rc) return rc;
      UC_CUDA_OK(cudaMemcpyAsync(g_host.stage, slots[0], sizeof(double), cudaMemcpyDeviceToHost, s));
      UC_CUDA_OK(cudaStreamSynchronize(s));
      if (g_host.t.allreduce_sum(g_host.t.user, g_host.stage, 1) != 0)
        return set_error(UC_ERR_CUDA, "host transport: allreduce callback failed");
      UC_CUDA_OK(cudaMemcpyAsync(slots[0], g_host.stage, sizeof(double), cudaMemcpyHostToDevice, s));
      UC_CUDA_OK(cudaStreamSynchronize(s));
    } else {
      if (!g_nccl.comm) return set_error(UC_ERR_ARG, "remote neighbours but no NCCL communicator");
      UC_NCCL_OK(g_nccl.allReduce(slots[0], slots[0], 1, kNcclFloat64, kNcclSum, g_nccl.comm, s));
    }
    SlotPtrs b{};
    for (int i = 0; i < n; ++i) b.p[i] = slots[i];
    b.p[0] = slots[0];
    b.n = 1;
    b.do_sqrt = do_sqrt ? 1 : 0;
    k_sum_slots<<<1, 32, 0, s>>>(b);
    UC_CUDA_OK(cudaGetLastError());
    if (n > 1) {
      for (int i = 1; i < n; ++i)
        UC_CUDA_OK(cudaMemcpyAsync(slots[i], slots[0], sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }
  return UC_OK;
}

__global__ void k_sum_slots_n(SlotPtrs a, int n) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < a.n; ++i) s += a.p[i][j];
    for (int i = 0; i < a.n; ++i) a.p[i][j] = s;
  }
}

// slots[i] holds slab i's local partial sums (n values); afterwards every slot
// holds the global sums (slabs in order, then ranks by allreduce).
int global_sum_n(const Group& g, double* const* slots, int n, cudaStream_t s) {
  const int ns = (int)g.size();
  if (ns > 16) return set_error(UC_ERR_ARG, "at most 16 local slabs per group");
  const bool remote = group_dist(g);
  SlotPtrs a{};
  for (int i = 0; i < ns; ++i) a.p[i] = slots[i];
  a.n = ns;
  if (ns > 1) {
    k_sum_slots_n<<<1, 256, 0, s>>>(a, n);
    UC_CUDA_OK(cudaGetLastError());
  }
  if (!remote) return UC_OK;
  if (g_host.active) {
    int rc = host_stage((size_t)n);
    if (rc) return rc;
    UC_CUDA_OK(cudaMemcpyAsync(g_host.stage, slots[0], sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    UC_CUDA_OK(cudaStreamSynchronize(s));
    if (g_host.t.allreduce_sum(g_host.t.user, g_host.stage, n) != 0)
      return set_error(UC_ERR_CUDA, "host transport: allreduce callback failed");
    UC_CUDA_OK(cudaMemcpyAsync(slots[0], g_host.stage, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    UC_CUDA_OK(cudaStreamSynchronize(s));
  } else {
    if (!g_nccl.comm) return set_error(UC_ERR_ARG, "remote neighbours but no NCCL communicator");
    UC_NCCL_OK(g_nccl.allReduce(slots[0], slots[0], (size_t)n, kNcclFloat64, kNcclSum, g_nccl.comm, s));
  }
  for (int i = 1; i < ns; ++i)
    UC_CUDA_OK(cudaMemcpyAsync(slots[i], slots[0], sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  return UC_OK;
}

}  // namespace uc

using namespace uc;

extern "C" {

int uc_nccl_unique_id(const char* nccl_path, void* out128) {
  int rc = nccl_load(nccl_path);
  if (rc) return rc;
  NcclUniqueId id;
  UC_NCCL_OK(g_nccl.getUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return UC_OK;
}

int uc_comm_init_nccl(const char* nccl_path, const void* id128, int rank, int nranks) {
  int rc = nccl_load(nccl_path);
  if (rc) return rc;
  if (g_nccl.comm) return set_error(UC_ERR_ARG, "NCCL communicator already initialised");
  NcclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  void* comm = nullptr;
  UC_NCCL_OK(g_nccl.commInitRank(&comm, nranks, id, rank));
  g_nccl.comm = comm;
  g_nccl.rank = rank;
  g_nccl.nranks = nranks;
  return UC_OK;
}

int uc_comm_init_host(const uc_host_transport* t, int rank, int nranks) {
  if (!t || !t->sendrecv || !t->allreduce_sum || rank < 0 || rank >= nranks)
    return set_error(UC_ERR_ARG, "uc_comm_init_host: bad argument");
  if (g_nccl.comm || g_host.active) return set_error(UC_ERR_ARG, "a communicator is already initialised");
  g_host.t = *t;
  g_host.rank = rank;
  g_host.nranks = nranks;
  g_host.active = true;
  return UC_OK;
}

int uc_comm_finalize(void) {
  if (g_nccl.comm) {
    g_nccl.commDestroy(g_nccl.comm);
    g_nccl.comm = nullptr;
  }
  if (g_host.active) {
    g_host.active = false;
    if (g_host.stage) cudaFreeHost(g_host.stage);
    g_host.stage = nullptr;
    g_host.stage_n = 0;
  }
  return UC_OK;
}

int uc_ctx_set_neighbors(uc_ctx* c, int lo_rank, int hi_rank) {
  if (!c) return set_error(UC_ERR_ARG, "NULL context");
  if ((lo_rank >= 0) != (c->grid.lo > 0) || (hi_rank >= 0) != (c->grid.hi < c->grid.nslow))
    return set_error(UC_ERR_ARG, "neighbour ranks do not match the slab boundaries");
  c->lo_rank = lo_rank;
  c->hi_rank = hi_rank;
  c->dist = (g_nccl.comm != nullptr && g_nccl.nranks > 1) || (g_host.active && g_host.nranks > 1);
  return UC_OK;
}

int uc_ctx_link_local(uc_ctx* lower, uc_ctx* upper) {
  if (!lower || !upper) return set_error(UC_ERR_ARG, "NULL context");
  if (lower->grid.hi != upper->grid.lo || lower->grid.plane != upper->grid.plane)
    return set_error(UC_ERR_ARG, "slabs are not adjacent");
  lower->hi_local = upper;
  upper->lo_local = lower;
  return UC_OK;
}

}  // extern "C"
