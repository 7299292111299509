// dp.cu -- data parallelism across replicas of one network.
//
// The reference has no distributed path; the exchange belongs where
// Trainer<T>::fit goes from run_batch to sgd_step (training.hpp:76-81):
//
//     run_batch(local shard) -> sum of the replicas' gradients -> sgd_step
//
// A group is attached to each replica's vcnn_net; from then on the net's
// sgd step (vcnn_net_sgd_step, and the update inside vcnn_net_train_step,
// CUDA-graph captured) IS the exchange:
//   * VCNN_DP_P2P (default): ONE kernel per replica (direct.cu
//     dp_sgd_pack_kernel) reads every replica's flat gradient through NVLink
//     peer mappings (CUDA IPC across processes, direct pointers inside one),
//     sums it in rank order with the shard weights B_p / B_global, and
//     applies momentum SGD + the conv weight packs -- a one-shot all-reduce
//     fused with the update; replicas stay bit-identical.  Cross-replica
//     ordering by release/acquire signal epochs in the replicas' signal
//     buffers, with a timeout instead of a hang.
//   * VCNN_DP_NCCL: ncclAllReduce(sum) of the flat gradient + the replicated
//     sgd_pack (libnccl loaded at run time; it also bootstraps vcnn_dp_init).
// Shards are contiguous sample ranges, the Imp-2 chunking
// [B*r/W, B*(r+1)/W) (variants.hpp:442-443); loss_backward scales by
// 1/B_local (layers.hpp:444), hence the B_p / B_global weights.
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"

using namespace vcnn_b200;

namespace vcnn_b200 {
namespace {

__global__ void scale_kernel(int64_t n, float* __restrict__ b, float s) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] *= s;
}

// ---- libnccl, resolved at run time (the process may already hold torch's) --
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl N;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      N.why = "libnccl.so.2 not found";
      return;
    }
#define SYM(f)                                                         \
  N.f = reinterpret_cast<decltype(N.f)>(dlsym(h, "nccl" #f));          \
  if (!N.f) {                                                          \
    N.why = "libnccl lacks nccl" #f;                                   \
    return;                                                            \
  }
    SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(AllReduce) SYM(AllGather)
    SYM(GetErrorString)
#undef SYM
    N.ok = true;
  });
  return N;
}

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(VCNN_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

int nccl_allreduce(DpLink* l, float* buf, int64_t n, cudaStream_t st) {
  ncclResult_t r = nccl().AllReduce(buf, buf, (size_t)n, ncclFloat, ncclSum,
                                    static_cast<ncclComm_t>(l->comm), st);
  return r == ncclSuccess ? VCNN_OK : nccl_fail(r, "ncclAllReduce");
}

// what a replica publishes to its peers
struct Handle {
  char magic[8];
  int32_t device, pid, world, rank;
  int64_t nparams;
  uint64_t host;
  cudaIpcMemHandle_t g, sig;
};
static_assert(sizeof(Handle) <= 256, "VCNN_DP_HANDLE_BYTES");

constexpr int64_t kSigWords = 2 * (int64_t)kMaxWorld * kMaxDpSlots;
constexpr int64_t kTimeoutNs = 10'000'000'000LL;

}  // namespace

int dp_scale(int64_t n, float* buf, float s, cudaStream_t st) {
  int64_t blocks = cdiv(n, 256);
  if (blocks > 4 * sm_count()) blocks = 4 * sm_count();
  VCNN_CUDA_TRY(launch_pdl(scale_kernel, dim3((unsigned)(blocks < 1 ? 1 : blocks)), dim3(256), 0, st, n, buf, s));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

}  // namespace vcnn_b200

struct vcnn_dp {
  vcnn_net* net = nullptr;
  int world = 1, rank = 0, device = 0;
  int64_t nparams = 0;
  float* grads = nullptr;
  DpLink link;
  uint32_t* sig = nullptr;  // [2][kMaxWorld][kMaxDpSlots] signals + epochs + err
  std::vector<void*> opened;
  ncclComm_t comm = nullptr;
  bool group = false;
  cudaEvent_t bwd_done = nullptr, upd_done = nullptr;  // group step ordering
  std::vector<int> shards;
};

namespace {

cudaStream_t net_stream(vcnn_net* n) { return vcnn_b200::engine_stream(n); }

int make_dp(vcnn_net* net, int world, int rank, vcnn_dp** out) {
  if (!net || !out) return fail(VCNN_ESHAPE, "dp: null argument");
  if (world < 1 || world > kMaxWorld) return fail(VCNN_ECONFIG, "dp: world size must be 1..8");
  if (rank < 0 || rank >= world) return fail(VCNN_ECONFIG, "dp: rank outside [0, world)");
  auto* d = new vcnn_dp;
  d->net = net;
  d->world = world;
  d->rank = rank;
  d->nparams = vcnn_net_num_params(net);
  float *p = nullptr, *v = nullptr;
  int s = vcnn_net_device_buffers(net, &p, &d->grads, &v);
  cudaError_t e = cudaGetDevice(&d->device);
  if (!s && e != cudaSuccess) s = cuda_fail(e, "cudaGetDevice");
  const size_t sb = sizeof(uint32_t) * (size_t)(kSigWords + kMaxDpSlots) + 64;
  if (!s && (e = cudaMalloc(&d->sig, sb)) != cudaSuccess) s = cuda_fail(e, "cudaMalloc");
  if (!s && (e = cudaMemset(d->sig, 0, sb)) != cudaSuccess) s = cuda_fail(e, "cudaMemset");
  if (s) {
    if (d->sig) cudaFree(d->sig);
    delete d;
    return s;
  }
  DpPeers& P = d->link.peers;
  P = DpPeers{};
  P.world = world;
  P.rank = rank;
  P.nslot = direct::dp_blocks(d->nparams);
  P.barrier = 1;
  P.my_sig = d->sig;
  P.epoch = d->sig + kSigWords;
  P.err = reinterpret_cast<int*>(d->sig + kSigWords + kMaxDpSlots);
  P.timeout_ns = kTimeoutNs;
  P.g[rank] = d->grads;
  P.sig[rank] = d->sig;
  for (int i = 0; i < world; ++i) P.scale[i] = 1.0f / (float)world;
  d->link.world = world;
  d->link.mode = VCNN_DP_P2P;
  d->link.equal = true;
  d->link.local_w = 1.0f / (float)world;
  d->shards.assign((size_t)world, 0);
  *out = d;
  return VCNN_OK;
}

int attach(vcnn_dp* d) { return vcnn_b200::engine_attach_dp(d->net, &d->link); }

}  // namespace

extern "C" {

int vcnn_dp_unique_id(void* id) {
  if (!id) return fail(VCNN_ESHAPE, "dp: null id");
  Nccl& N = nccl();
  if (!N.ok) return fail(VCNN_ENCCL, N.why);
  ncclUniqueId u;
  ncclResult_t r = N.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == VCNN_DP_ID_BYTES, "nccl id size");
  std::memcpy(id, &u, sizeof u);
  return VCNN_OK;
}

int vcnn_dp_create(vcnn_net* net, int world, int rank, vcnn_dp** out) {
  return make_dp(net, world, rank, out);
}

int vcnn_dp_handle(const vcnn_dp* d, void* handle) {
  if (!d || !handle) return fail(VCNN_ESHAPE, "dp: null argument");
  Handle h{};
  std::memcpy(h.magic, "VCNNDP1", 8);
  h.device = d->device;
  h.pid = (int32_t)getpid();
  h.world = d->world;
  h.rank = d->rank;
  h.nparams = d->nparams;
  h.host = (uint64_t)gethostid();
  VCNN_CUDA_TRY(cudaIpcGetMemHandle(&h.g, d->grads));
  VCNN_CUDA_TRY(cudaIpcGetMemHandle(&h.sig, d->sig));
  std::memset(handle, 0, VCNN_DP_HANDLE_BYTES);
  std::memcpy(handle, &h, sizeof h);
  return VCNN_OK;
}

int vcnn_dp_connect(vcnn_dp* d, const void* handles, const void* id) {
  if (!d || !handles) return fail(VCNN_ESHAPE, "dp: null argument");
  VCNN_CUDA_TRY(cudaSetDevice(d->device));
  const auto* hb = static_cast<const uint8_t*>(handles);
  DpPeers& P = d->link.peers;
  bool p2p = true;
  std::string why;
  for (int p = 0; p < d->world; ++p) {
    Handle h;
    std::memcpy(&h, hb + (size_t)p * VCNN_DP_HANDLE_BYTES, sizeof h);
    if (std::memcmp(h.magic, "VCNNDP1", 8) || h.world != d->world || h.rank != p)
      return fail(VCNN_ECONFIG, "dp: handle " + std::to_string(p) + " malformed or out of order");
    if (h.nparams != d->nparams)
      return fail(VCNN_ESHAPE, "dp: rank " + std::to_string(p) + " has a different network");
    if (p == d->rank) continue;
    if (h.pid == (int32_t)getpid()) {
      p2p = false;
      why = "peer in the same process (use vcnn_dp_group)";
      continue;
    }
    void *g = nullptr, *sg = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&g, h.g, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) {
      d->opened.push_back(g);
      e = cudaIpcOpenMemHandle(&sg, h.sig, cudaIpcMemLazyEnablePeerAccess);
      if (e == cudaSuccess) d->opened.push_back(sg);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      p2p = false;
      why = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
      continue;
    }
    P.g[p] = static_cast<const float*>(g);
    P.sig[p] = static_cast<uint32_t*>(sg);
  }
  if (id && !d->comm) {
    Nccl& N = nccl();
    if (!N.ok) return fail(VCNN_ENCCL, N.why);
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclResult_t r = N.CommInitRank(&d->comm, d->world, u, d->rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    d->link.comm = d->comm;
    d->link.allreduce = nccl_allreduce;
  }
  if (!p2p) {
    if (!d->comm) return fail(VCNN_ENCCL, "dp: no P2P path (" + why + ") and no NCCL id");
    d->link.mode = VCNN_DP_NCCL;
  }
  return attach(d);
}

int vcnn_dp_init(vcnn_net* net, int world, int rank, const void* id, vcnn_dp** out) {
  if (!id) return fail(VCNN_ESHAPE, "dp: null NCCL id");
  vcnn_dp* d = nullptr;
  int s = make_dp(net, world, rank, &d);
  if (s) return s;
  Nccl& N = nccl();
  if (!N.ok) {
    vcnn_dp_destroy(d);
    return fail(VCNN_ENCCL, N.why);
  }
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclResult_t r = N.CommInitRank(&d->comm, world, u, rank);
  if (r != ncclSuccess) {
    d->comm = nullptr;
    vcnn_dp_destroy(d);
    return nccl_fail(r, "ncclCommInitRank");
  }
  d->link.comm = d->comm;
  d->link.allreduce = nccl_allreduce;
  // exchange the IPC handles over the communicator itself
  std::vector<uint8_t> mine(VCNN_DP_HANDLE_BYTES), all((size_t)world * VCNN_DP_HANDLE_BYTES);
  s = vcnn_dp_handle(d, mine.data());
  uint8_t* buf = nullptr;
  cudaStream_t st = net_stream(net);
  if (!s && cudaMalloc(&buf, all.size() + mine.size()) != cudaSuccess)
    s = fail(VCNN_ECUDA, "dp: cudaMalloc");
  if (!s && cudaMemcpy(buf + all.size(), mine.data(), mine.size(), cudaMemcpyHostToDevice))
    s = fail(VCNN_ECUDA, "dp: cudaMemcpy");
  if (!s) {
    r = N.AllGather(buf + all.size(), buf, VCNN_DP_HANDLE_BYTES, ncclChar, d->comm, st);
    if (r != ncclSuccess) s = nccl_fail(r, "ncclAllGather");
  }
  if (!s && (cudaStreamSynchronize(st) != cudaSuccess ||
             cudaMemcpy(all.data(), buf, all.size(), cudaMemcpyDeviceToHost) != cudaSuccess))
    s = fail(VCNN_ECUDA, "dp: handle exchange");
  if (buf) cudaFree(buf);
  if (!s) s = vcnn_dp_connect(d, all.data(), nullptr);
  if (s) {
    vcnn_dp_destroy(d);
    return s;
  }
  *out = d;
  return VCNN_OK;
}

int vcnn_dp_group(vcnn_net* const* nets, int world, int barrier, vcnn_dp** out) {
  if (!nets || !out) return fail(VCNN_ESHAPE, "dp: null argument");
  int dev0 = 0;
  VCNN_CUDA_TRY(cudaGetDevice(&dev0));
  std::vector<vcnn_dp*> d((size_t)world, nullptr);
  int s = VCNN_OK;
  for (int r = 0; r < world && !s; ++r) {
    s = make_dp(nets[r], world, r, &d[(size_t)r]);
    if (!s && d[(size_t)r]->nparams != d[0]->nparams)
      s = fail(VCNN_ESHAPE, "dp group: replicas differ");
  }
  for (int r = 0; r < world && !s; ++r) {
    vcnn_dp* a = d[(size_t)r];
    a->group = true;
    a->link.peers.barrier = barrier ? 1 : 0;
    for (int p = 0; p < world; ++p) {
      if (p == r) continue;
      if (d[(size_t)p]->device != a->device) {
        cudaSetDevice(a->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(d[(size_t)p]->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          s = cuda_fail(e, "cudaDeviceEnablePeerAccess");
          break;
        }
        cudaGetLastError();
      }
      a->link.peers.g[p] = d[(size_t)p]->grads;
      a->link.peers.sig[p] = d[(size_t)p]->sig;
    }
    if (!s && (cudaEventCreateWithFlags(&a->bwd_done, cudaEventDisableTiming) != cudaSuccess ||
               cudaEventCreateWithFlags(&a->upd_done, cudaEventDisableTiming) != cudaSuccess))
      s = fail(VCNN_ECUDA, "dp group: events");
    if (!s) s = attach(a);
  }
  cudaSetDevice(dev0);
  if (s) {
    for (vcnn_dp* a : d)
      if (a) vcnn_dp_destroy(a);
    return s;
  }
  for (int r = 0; r < world; ++r) out[r] = d[(size_t)r];
  return VCNN_OK;
}

int vcnn_dp_set_mode(vcnn_dp* d, int mode) {
  if (!d) return fail(VCNN_ESHAPE, "dp: null");
  if (mode != VCNN_DP_P2P && mode != VCNN_DP_NCCL) return fail(VCNN_ECONFIG, "dp: unknown mode");
  if (mode == VCNN_DP_NCCL && !d->link.allreduce)
    return fail(VCNN_ENCCL, "dp: no NCCL communicator");
  if (mode == VCNN_DP_P2P && d->world > 1)
    for (int p = 0; p < d->world; ++p)
      if (!d->link.peers.g[p]) return fail(VCNN_ENCCL, "dp: no P2P mapping to every peer");
  if (mode != d->link.mode) ++d->link.version;
  d->link.mode = mode;
  return VCNN_OK;
}

int vcnn_dp_get_mode(const vcnn_dp* d, int* mode) {
  if (!d || !mode) return fail(VCNN_ESHAPE, "dp: null");
  *mode = d->link.mode;
  return VCNN_OK;
}

int vcnn_dp_set_shards(vcnn_dp* d, const int* batches) {
  if (!d || !batches) return fail(VCNN_ESHAPE, "dp: null argument");
  int64_t tot = 0;
  for (int p = 0; p < d->world; ++p) {
    if (batches[p] < 1) return fail(VCNN_ESHAPE, "dp: every shard needs >= 1 sample");
    tot += batches[p];
  }
  bool same = true;
  for (int p = 0; p < d->world; ++p) same = same && d->shards[(size_t)p] == batches[p];
  if (same) return VCNN_OK;
  bool equal = true;
  for (int p = 0; p < d->world; ++p) {
    d->shards[(size_t)p] = batches[p];
    d->link.peers.scale[p] = (float)((double)batches[p] / (double)tot);
    equal = equal && batches[p] == batches[0];
  }
  d->link.equal = equal;
  d->link.local_w = d->link.peers.scale[d->rank];
  ++d->link.version;
  return VCNN_OK;
}

int vcnn_dp_allreduce_sgd(vcnn_dp* d, float lr, float mom) {
  if (!d) return fail(VCNN_ESHAPE, "dp: null");
  return vcnn_net_sgd_step(d->net, lr, mom, 1.0f);
}

int vcnn_dp_train_step(vcnn_dp* d, int batch, float lr, float mom) {
  if (!d) return fail(VCNN_ESHAPE, "dp: null");
  return vcnn_net_train_step(d->net, batch, lr, mom);
}

int vcnn_dp_group_train_step(vcnn_dp* const* dps, int world, const int* batches, float lr,
                             float mom) {
  if (!dps || !batches || world < 1) return fail(VCNN_ESHAPE, "dp group: bad arguments");
  for (int r = 0; r < world; ++r)
    if (!dps[r] || !dps[r]->group || dps[r]->world != world || dps[r]->link.peers.barrier)
      return fail(VCNN_ECONFIG, "dp group step needs a barrier-free vcnn_dp_group");
  int dev0 = 0;
  VCNN_CUDA_TRY(cudaGetDevice(&dev0));
  int s = VCNN_OK;
  for (int r = 0; r < world && !s; ++r) s = vcnn_dp_set_shards(dps[r], batches);
  // every replica's backward waits until every replica's previous update
  // (which read its gradient) finished; every update waits for every backward
  for (int r = 0; r < world && !s; ++r) {
    vcnn_dp* a = dps[r];
    cudaSetDevice(a->device);
    cudaStream_t st = net_stream(a->net);
    for (int p = 0; p < world && !s; ++p)
      if (cudaStreamWaitEvent(st, dps[p]->upd_done, 0) != cudaSuccess)
        s = fail(VCNN_ECUDA, "dp group: event wait");
    if (!s) s = vcnn_net_forward_backward(a->net, batches[r]);
    if (!s && cudaEventRecord(a->bwd_done, st) != cudaSuccess) s = fail(VCNN_ECUDA, "event");
  }
  for (int r = 0; r < world && !s; ++r) {
    vcnn_dp* a = dps[r];
    cudaSetDevice(a->device);
    cudaStream_t st = net_stream(a->net);
    for (int p = 0; p < world && !s; ++p)
      if (cudaStreamWaitEvent(st, dps[p]->bwd_done, 0) != cudaSuccess)
        s = fail(VCNN_ECUDA, "dp group: event wait");
    if (!s) s = vcnn_net_sgd_step(a->net, lr, mom, 1.0f);
    if (!s && cudaEventRecord(a->upd_done, st) != cudaSuccess) s = fail(VCNN_ECUDA, "event");
  }
  cudaSetDevice(dev0);
  return s;
}

int vcnn_dp_status(vcnn_dp* d) {
  if (!d) return fail(VCNN_ESHAPE, "dp: null");
  int h = 0;
  VCNN_CUDA_TRY(cudaStreamSynchronize(net_stream(d->net)));
  VCNN_CUDA_TRY(cudaMemcpy(&h, d->link.peers.err, sizeof h, cudaMemcpyDeviceToHost));
  if (h) {
    cudaMemset(d->link.peers.err, 0, sizeof h);
    return fail(VCNN_ENCCL, "dp: a peer barrier timed out (a replica did not reach the exchange)");
  }
  return VCNN_OK;
}

int vcnn_dp_destroy(vcnn_dp* d) {
  if (!d) return VCNN_OK;
  cudaSetDevice(d->device);
  vcnn_b200::engine_attach_dp(d->net, nullptr);
  cudaStreamSynchronize(net_stream(d->net));
  for (void* p : d->opened) cudaIpcCloseMemHandle(p);
  if (d->comm) nccl().CommDestroy(d->comm);
  if (d->bwd_done) cudaEventDestroy(d->bwd_done);
  if (d->upd_done) cudaEventDestroy(d->upd_done);
  if (d->sig) cudaFree(d->sig);
  delete d;
  return VCNN_OK;
}

}  // extern "C"
