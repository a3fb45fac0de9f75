// csrc/comm.cu -- the collectives of a sharded sweep (the per-sweep
// all-reduce of the topic-word counts, the log-joint pieces, the MH likelihood sums and
// the bound-store speculation votes), over NCCL or over a peer group.
//
// Peer group: the W ranks are contexts of one process (one host thread per rank, one
// GPU each or several ranks sharing a GPU).  An all-reduce is
//   1. every rank records an event after the producer of its buffer and publishes
//      (buffer, event) in its slot; host rendezvous;
//   2. every rank's stream waits for all W input events, then runs peer_allreduce_kernel
//      over ITS chunk [r n / W, (r + 1) n / W): it loads the chunk from all W buffers (peer
//      memory over NVLink when the ranks sit on different GPUs), reduces in rank order
//      (deterministic for floating point) and stores the result into all W buffers -- each
//      element is read and then written by the same thread, so in place is safe;
//      records its output event; host rendezvous;
//   3. every rank's stream waits for all W output events.
// Two rendezvous per collective make the event reuse safe (a rank re-records its events
// only after every peer has enqueued its waits on them).  No kernel ever spins on
// another rank, so ranks sharing one GPU cannot deadlock it; a rank that never arrives
// makes the others fail after a timeout instead of hanging.  Contexts in a group run
// without CUDA graphs (the cross-context event waits cannot be captured).
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace bnmc_gpu {

constexpr int kMaxPeers = 8;  // one node

struct PeerPtrs {
  void* p[kMaxPeers];
};

// Reduce-scatter over peer memory: rank r sums chunk r of all W buffers (rank order) into
// its OWN buffer only; every other rank reads its own chunk of r's buffer, never r's chunk.
template <class T>
__global__ void peer_reduce_scatter_kernel(PeerPtrs b, int world, int r, std::size_t begin, std::size_t end) {
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  for (std::size_t i = begin + blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < end; i += stride) {
    T acc = static_cast<const T*>(b.p[0])[i];
    for (int s = 1; s < world; ++s) acc = acc + static_cast<const T*>(b.p[s])[i];
    static_cast<T*>(b.p[r])[i] = acc;
  }
}

// All-gather over peer memory: rank r writes its chunk r into every other rank's buffer.
template <class T>
__global__ void peer_all_gather_kernel(PeerPtrs b, int world, int r, std::size_t begin, std::size_t end) {
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  for (std::size_t i = begin + blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < end; i += stride) {
    const T v = static_cast<const T*>(b.p[r])[i];
    for (int s = 0; s < world; ++s)
      if (s != r) static_cast<T*>(b.p[s])[i] = v;
  }
}

template <class T, int OP>
__global__ void peer_allreduce_kernel(PeerPtrs b, int world, std::size_t begin, std::size_t end) {
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  for (std::size_t i = begin + blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < end; i += stride) {
    T acc = static_cast<const T*>(b.p[0])[i];
    for (int s = 1; s < world; ++s) {
      const T v = static_cast<const T*>(b.p[s])[i];
      acc = OP == 0 ? acc + v : (OP == 1 ? (v < acc ? v : acc) : (v > acc ? v : acc));
    }
    for (int s = 0; s < world; ++s) static_cast<T*>(b.p[s])[i] = acc;
  }
}

struct PeerGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  std::uint64_t generation = 0;
  struct Slot {
    bool joined = false;
    int device = -1;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    void* buf = nullptr;
    std::size_t n = 0;
    int type = 0, op = 0;
    bool peers_enabled = false;  // this rank's device may access every peer's memory
  };
  std::vector<Slot> slot;

  // Host rendezvous of all W ranks (generation counting); throws after a timeout.
  void rendezvous() {
    std::unique_lock<std::mutex> lk(mu);
    const std::uint64_t g = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != g; })) {
      --arrived;
      throw Error(BNMC_GPU_ERR_NCCL, "peer group: not every rank reached the collective within 120 s "
                                     "(each rank must run its calls on its own host thread)");
    }
  }
};

void peer_group_join(PeerGroup* g, int rank, int world, int device) {
  require(g->world == world, BNMC_GPU_ERR_ARG, "peer group world size differs from the context's");
  require(world <= kMaxPeers, BNMC_GPU_ERR_ARG, "peer groups hold at most 8 ranks");
  std::lock_guard<std::mutex> lk(g->mu);
  auto& s = g->slot[static_cast<std::size_t>(rank)];
  require(!s.joined, BNMC_GPU_ERR_ARG, "peer group: rank " + std::to_string(rank) + " joined twice");
  BNMC_CUDA(cudaEventCreateWithFlags(&s.ev_in, cudaEventDisableTiming));
  BNMC_CUDA(cudaEventCreateWithFlags(&s.ev_out, cudaEventDisableTiming));
  s.device = device;
  s.joined = true;
}

void peer_group_leave(PeerGroup* g, int rank) {
  std::lock_guard<std::mutex> lk(g->mu);
  auto& s = g->slot[static_cast<std::size_t>(rank)];
  if (s.ev_in) cudaEventDestroy(s.ev_in);
  if (s.ev_out) cudaEventDestroy(s.ev_out);
  s = PeerGroup::Slot{};
}

namespace {

template <class T>
void launch_reduce(const PeerPtrs& b, int world, std::size_t lo, std::size_t hi, int op, cudaStream_t st) {
  if (hi <= lo) return;
  const unsigned grid = std::min<unsigned>(blocks_for(static_cast<std::int64_t>(hi - lo), 256), 148 * 4);
  switch (op) {
    case 0: peer_allreduce_kernel<T, 0><<<grid, 256, 0, st>>>(b, world, lo, hi); break;
    case 1: peer_allreduce_kernel<T, 1><<<grid, 256, 0, st>>>(b, world, lo, hi); break;
    default: peer_allreduce_kernel<T, 2><<<grid, 256, 0, st>>>(b, world, lo, hi); break;
  }
}

enum class Coll { AllReduce = 0, ReduceScatter = 8, AllGather = 16 };

// n: the whole buffer's elements (W chunks of n / W for the scatter / gather kinds)
void group_collective(PeerGroup* g, int r, Coll kind, void* buf, std::size_t n, RedType t, RedOp op,
                      cudaStream_t st) {
  const int W = g->world;
  auto& me = g->slot[static_cast<std::size_t>(r)];
  BNMC_CUDA(cudaEventRecord(me.ev_in, st));
  me.buf = buf;
  me.n = n;
  me.type = static_cast<int>(t);
  me.op = static_cast<int>(op) + static_cast<int>(kind);  // the collective must match, too
  g->rendezvous();  // every rank published its buffer and input event
  PeerPtrs b{};
  for (int s = 0; s < W; ++s) {
    const auto& o = g->slot[static_cast<std::size_t>(s)];
    require(o.joined && o.n == n && o.type == me.type && o.op == me.op, BNMC_GPU_ERR_NCCL,
            "peer group: ranks called different collectives");
    b.p[s] = o.buf;
  }
  if (!me.peers_enabled) {  // ranks on different GPUs read / write each other's memory
    for (int s = 0; s < W; ++s) {
      const int d = g->slot[static_cast<std::size_t>(s)].device;
      if (d == me.device) continue;
      int can = 0;
      BNMC_CUDA(cudaDeviceCanAccessPeer(&can, me.device, d));
      require(can != 0, BNMC_GPU_ERR_NCCL, "peer group: no peer access between the ranks' GPUs");
      const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else BNMC_CUDA(e);
    }
  }
  for (int s = 0; s < W; ++s) BNMC_CUDA(cudaStreamWaitEvent(st, g->slot[static_cast<std::size_t>(s)].ev_in, 0));
  const std::size_t lo = n * static_cast<std::size_t>(r) / static_cast<std::size_t>(W);
  const std::size_t hi = n * static_cast<std::size_t>(r + 1) / static_cast<std::size_t>(W);
  if (kind == Coll::AllReduce) {
    if (t == RedType::I32) launch_reduce<int>(b, W, lo, hi, static_cast<int>(op), st);
    else launch_reduce<double>(b, W, lo, hi, static_cast<int>(op), st);
  } else if (hi > lo) {
    const unsigned grid = std::min<unsigned>(blocks_for(static_cast<std::int64_t>(hi - lo), 256), 148 * 4);
    if (kind == Coll::ReduceScatter) {
      if (t == RedType::I32) peer_reduce_scatter_kernel<int><<<grid, 256, 0, st>>>(b, W, r, lo, hi);
      else peer_reduce_scatter_kernel<double><<<grid, 256, 0, st>>>(b, W, r, lo, hi);
    } else {
      if (t == RedType::I32) peer_all_gather_kernel<int><<<grid, 256, 0, st>>>(b, W, r, lo, hi);
      else peer_all_gather_kernel<double><<<grid, 256, 0, st>>>(b, W, r, lo, hi);
    }
  }
  BNMC_CUDA(cudaGetLastError());
  BNMC_CUDA(cudaEventRecord(me.ev_out, st));
  g->rendezvous();  // every rank's chunk kernel is enqueued
  me.peers_enabled = true;
  for (int s = 0; s < W; ++s)
    if (s != r) BNMC_CUDA(cudaStreamWaitEvent(st, g->slot[static_cast<std::size_t>(s)].ev_out, 0));
}

ncclDataType_t nccl_type(RedType t) { return t == RedType::I32 ? ncclInt32 : ncclFloat64; }
ncclRedOp_t nccl_op(RedOp o) { return o == RedOp::Sum ? ncclSum : (o == RedOp::Min ? ncclMin : ncclMax); }

}  // namespace

void Comm::all_reduce(void* buf, std::size_t n, RedType t, RedOp op, cudaStream_t st) const {
  if (comm) {
    BNMC_NCCL(ncclAllReduce(buf, buf, n, nccl_type(t), nccl_op(op), comm, st));
  } else if (group) {
    group_collective(group, rank, Coll::AllReduce, buf, n, t, op, st);
  }
}

// In place: buf holds world chunks of `chunk` elements; rank r ends with the rank-order sum
// of chunk r in its chunk r (NCCL's in-place form: recvbuff = sendbuff + rank * recvcount).
void Comm::reduce_scatter(void* buf, std::size_t chunk, RedType t, cudaStream_t st) const {
  const std::size_t es = t == RedType::I32 ? sizeof(int) : sizeof(double);
  if (comm) {
    BNMC_NCCL(ncclReduceScatter(buf, static_cast<char*>(buf) + es * chunk * static_cast<std::size_t>(rank), chunk,
                                nccl_type(t), ncclSum, comm, st));
  } else if (group) {
    group_collective(group, rank, Coll::ReduceScatter, buf, chunk * static_cast<std::size_t>(world), t, RedOp::Sum, st);
  }
}

// In place: every rank's chunk r of buf is replaced by rank r's (NCCL's in-place form:
// sendbuff = recvbuff + rank * sendcount).
void Comm::all_gather(void* buf, std::size_t chunk, RedType t, cudaStream_t st) const {
  const std::size_t es = t == RedType::I32 ? sizeof(int) : sizeof(double);
  if (comm) {
    BNMC_NCCL(ncclAllGather(static_cast<char*>(buf) + es * chunk * static_cast<std::size_t>(rank), buf, chunk,
                            nccl_type(t), comm, st));
  } else if (group) {
    group_collective(group, rank, Coll::AllGather, buf, chunk * static_cast<std::size_t>(world), t, RedOp::Sum, st);
  }
}

}  // namespace bnmc_gpu

using bnmc_gpu::PeerGroup;

struct bnmc_gpu_group {
  PeerGroup g;
};

extern "C" {

int bnmc_gpu_group_create(int32_t world_size, bnmc_gpu_group** out) {
  if (!out || world_size < 1 || world_size > bnmc_gpu::kMaxPeers) return BNMC_GPU_ERR_ARG;
  auto* p = new bnmc_gpu_group;
  p->g.world = world_size;
  p->g.slot.resize(static_cast<std::size_t>(world_size));
  *out = p;
  return BNMC_GPU_OK;
}

void bnmc_gpu_group_destroy(bnmc_gpu_group* g) { delete g; }

}  // extern "C"

namespace bnmc_gpu {
PeerGroup* group_of(bnmc_gpu_group* g) { return g ? &g->g : nullptr; }
}  // namespace bnmc_gpu
