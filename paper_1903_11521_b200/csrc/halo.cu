// z-slab halo exchange over NCCL, loaded with dlopen so libydg.so has no link-time NCCL
// dependency (inside a torch process the already-loaded torch NCCL is reused).
#include "halo.h"

#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>

#include <dlfcn.h>

#include <algorithm>
#include <cstring>

namespace ydg {

namespace {

struct NcclUid { char internal[128]; };
typedef void* NcclComm;
typedef int (*InitRankFn)(NcclComm*, int, NcclUid, int);
typedef int (*SendRecvFn)(const void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*RecvFn)(void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*GroupFn)();
typedef int (*DestroyFn)(NcclComm);
typedef const char* (*ErrStrFn)(int);
constexpr int kNcclUint8 = 1;

struct Nccl {
  void* lib = nullptr;
  InitRankFn init = nullptr;
  SendRecvFn send = nullptr;
  RecvFn recv = nullptr;
  GroupFn gstart = nullptr, gend = nullptr;
  DestroyFn destroy = nullptr;
  ErrStrFn errstr = nullptr;
  bool load(std::string* err) {
    if (lib) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if ((lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!lib) { *err = "cannot dlopen libnccl.so.2"; return false; }
    init = reinterpret_cast<InitRankFn>(dlsym(lib, "ncclCommInitRank"));
    send = reinterpret_cast<SendRecvFn>(dlsym(lib, "ncclSend"));
    recv = reinterpret_cast<RecvFn>(dlsym(lib, "ncclRecv"));
    gstart = reinterpret_cast<GroupFn>(dlsym(lib, "ncclGroupStart"));
    gend = reinterpret_cast<GroupFn>(dlsym(lib, "ncclGroupEnd"));
    destroy = reinterpret_cast<DestroyFn>(dlsym(lib, "ncclCommDestroy"));
    errstr = reinterpret_cast<ErrStrFn>(dlsym(lib, "ncclGetErrorString"));
    if (!init || !send || !recv || !gstart || !gend || !destroy || !errstr) {
      *err = "libnccl is missing symbols";
      return false;
    }
    return true;
  }
};
Nccl g_nccl;

// index of value v (= (face, m, q) flattened) of local element slot s in the trace layout:
// TS == 0: [tile][face][m][q][32] (fp32 kernels); TS > 0: [tile][face][lane][TS] with L
// lanes per tile and an element-face block [m][q] of TS values (fp64 tensor-core kernels)
__device__ __forceinline__ int64_t tiled_index(int64_t s, int v, int Bt, int P, int TS, int L) {
  const int F = v / (Bt * P), m = (v / P) % Bt, q = v % P;
  if (TS > 0) return (((s / L) * 4 + F) * L + (s % L)) * (int64_t)TS + m * P + q;
  return (((s >> 5) * 4 + F) * Bt + m) * (int64_t)(P * 32) + q * 32 + (s & 31);
}

// One face block (Bt x P values) per entry; sf = slot << 2 | face.
template <typename W>
__global__ void pack_kernel(const W* __restrict__ traces, const int64_t* __restrict__ sf,
                            W* __restrict__ out, int64_t n, int Bt, int P, int TS, int L) {
  const int vals = Bt * P;
  const int64_t total = n * vals;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / vals;
    const int v = static_cast<int>(i - k * vals);
    const int64_t w = sf[k];
    out[i] = traces[tiled_index(w >> 2, static_cast<int>(w & 3) * vals + v, Bt, P, TS, L)];
  }
}

template <typename W>
__global__ void unpack_kernel(const W* __restrict__ in, W* __restrict__ traces, const int64_t* __restrict__ sf,
                              int64_t n, int Bt, int P, int TS, int L) {
  const int vals = Bt * P;
  const int64_t total = n * vals;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / vals;
    const int v = static_cast<int>(i - k * vals);
    const int64_t w = sf[k];
    traces[tiled_index(w >> 2, static_cast<int>(w & 3) * vals + v, Bt, P, TS, L)] = in[i];
  }
}

int64_t owner(int64_t g, int64_t ne, int nranks) {
  // largest r with r*ne/nranks <= g
  int64_t r = (g * nranks) / ne;
  while (r + 1 < nranks && (r + 1) * ne / nranks <= g) ++r;
  while (r > 0 && r * ne / nranks > g) --r;
  return r;
}

}  // namespace

bool plan_halo(const Neighbours& nbr, int64_t ne, int rank, int nranks, HaloPlan* out,
               std::string* err) {
  const int64_t first = ne * rank / nranks, last = ne * (rank + 1) / nranks;
  struct Blk { int64_t peer, gid; int face; int64_t ref; };  // ref: local slot / ghost gid
  std::vector<Blk> sends, recvs;
  std::vector<std::pair<int64_t, int64_t>> ghosts;  // (owner, gid)
  for (int64_t e = first; e < last; ++e)
    for (int i = 0; i < 4; ++i) {
      const int64_t n = nbr.nb[e * 4 + i];
      if (n < 0 || n >= ne) { *err = "bad neighbour id"; return false; }
      if (n >= first && n < last) continue;
      const int64_t o = owner(n, ne, nranks);
      ghosts.emplace_back(o, n);
      sends.push_back({o, e, i, e - first});                   // my side of the face
      recvs.push_back({o, n, static_cast<int>(nbr.j[e * 4 + i]), n});  // the peer's side
    }
  auto key = [](const Blk& x, const Blk& y) {
    return x.peer != y.peer ? x.peer < y.peer : (x.gid != y.gid ? x.gid < y.gid : x.face < y.face);
  };
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  std::sort(sends.begin(), sends.end(), key);
  std::sort(recvs.begin(), recvs.end(), key);
  *out = HaloPlan();
  for (size_t g = 0; g < ghosts.size(); ++g) {
    if (out->peers.empty() || out->peers.back() != ghosts[g].first) out->peers.push_back(static_cast<int>(ghosts[g].first));
    out->ghost_of.push_back(ghosts[g].second);
  }
  for (int peer : out->peers) {
    out->send_off.push_back(static_cast<int64_t>(out->send_slots.size()));
    out->recv_off.push_back(static_cast<int64_t>(out->recv_ghost.size()));
    int64_t cs = 0, cr = 0;
    for (const Blk& b : sends)
      if (b.peer == peer) { out->send_slots.push_back(b.ref); out->send_face.push_back(static_cast<int8_t>(b.face)); ++cs; }
    for (const Blk& b : recvs)
      if (b.peer == peer) {
        const auto it = std::lower_bound(ghosts.begin(), ghosts.end(), std::make_pair(b.peer, b.gid));
        out->recv_ghost.push_back(static_cast<int64_t>(it - ghosts.begin()));
        out->recv_face.push_back(static_cast<int8_t>(b.face));
        ++cr;
      }
    // a face has one side per rank: the blocks a peer sends are the faces it shares with us
    if (cs != cr) { *err = "asymmetric halo"; return false; }
    out->send_cnt.push_back(cs);
    out->recv_cnt.push_back(cr);
  }
  return true;
}

// ---- loopback transport (tests): several ranks as handles of one process on one GPU,
// selected by a unique id starting with "YDGLOOP".  The exchange packs, meets the other
// ranks at a host barrier, copies each peer's packed segment device-to-device and meets
// again before anyone repacks -- the same plan, pack and unpack as the NCCL path, so a
// partitioned run can be checked bit for bit against one rank on a single GPU.
struct LoopGroup {
  std::mutex mu;
  std::condition_variable cv;
  int nranks = 0, arrived = 0;
  int64_t generation = 0;
  std::vector<Halo*> members;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};
namespace {
std::mutex g_loop_mu;
std::map<std::string, std::shared_ptr<LoopGroup>> g_loops;
}  // namespace

int Halo::init(int rank, int nranks, const void* uid, std::string* err) {
  rank_ = rank;
  nranks_ = nranks;
  if (std::memcmp(uid, "YDGLOOP", 7) == 0) {
    const std::string key(static_cast<const char*>(uid), 128);
    {
      std::lock_guard<std::mutex> lk(g_loop_mu);
      auto& g = g_loops[key];
      if (!g) {
        g = std::make_shared<LoopGroup>();
        g->nranks = nranks;
        g->members.assign(nranks, nullptr);
      }
      if (g->nranks != nranks || g->members[rank]) { *err = "loopback group mismatch"; return 4; }
      g->members[rank] = this;
      loop_ = g;
    }
    cudaError_t e = cudaStreamCreateWithFlags(&cstream_, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done_, cudaEventDisableTiming);
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
    return 0;
  }
  if (!g_nccl.load(err)) return 4;
  NcclUid id;
  std::memcpy(&id, uid, sizeof(id));
  NcclComm c = nullptr;
  int r = g_nccl.init(&c, nranks, id, rank);
  if (r != 0) { *err = std::string("ncclCommInitRank: ") + g_nccl.errstr(r); return 4; }
  comm_ = c;
  cudaError_t e = cudaStreamCreateWithFlags(&cstream_, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done_, cudaEventDisableTiming);
  if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
  return 0;
}

int Halo::plan(const Neighbours& nbr, int64_t first, int64_t nlocal, int64_t owned_slots,
               std::vector<int64_t>* ghost_of, std::string* err) {
  (void)first;
  (void)nlocal;
  ne_ = static_cast<int64_t>(nbr.nb.size() / 4);
  if (!plan_halo(nbr, ne_, rank_, nranks_, &plan_, err)) return 5;
  *ghost_of = plan_.ghost_of;
  owned_slots_ = owned_slots;
  return 0;
}

int Halo::bind(void* traces, int Bt, int P, int TS, int L, int elem_bytes, int64_t owned_slots, std::string* err) {
  (void)traces;
  Bt_ = Bt;
  TS_ = TS;
  L_ = L;
  P_ = P;
  vals_ = Bt * P;  // one face block per message entry
  eb_ = elem_bytes;
  owned_slots_ = owned_slots;
  const size_t ns = plan_.send_slots.size(), nr = plan_.recv_ghost.size();
  std::vector<int64_t> sf(ns), rf(nr);
  for (size_t k = 0; k < ns; ++k) sf[k] = plan_.send_slots[k] << 2 | plan_.send_face[k];
  for (size_t k = 0; k < nr; ++k) rf[k] = (owned_slots + plan_.recv_ghost[k]) << 2 | plan_.recv_face[k];
  cudaError_t e = cudaMalloc(&d_send_slots_, std::max<size_t>(1, ns) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc(&d_recv_slots_, std::max<size_t>(1, nr) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc(&d_send_buf_, std::max<size_t>(1, ns) * vals_ * eb_);
  if (e == cudaSuccess) e = cudaMalloc(&d_recv_buf_, std::max<size_t>(1, nr) * vals_ * eb_);
  if (e == cudaSuccess && ns) e = cudaMemcpy(d_send_slots_, sf.data(), ns * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nr) e = cudaMemcpy(d_recv_slots_, rf.data(), nr * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
  return 0;
}

int Halo::exchange(cudaStream_t s, void* traces, int elem_bytes, std::string* err) {
  cudaError_t e = cudaEventRecord(ready_, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cstream_, ready_, 0);
  const int64_t ns = static_cast<int64_t>(plan_.send_slots.size());
  const int64_t ng = static_cast<int64_t>(plan_.recv_ghost.size());
  if (e == cudaSuccess && ns) {
    if (elem_bytes == 8)
      pack_kernel<unsigned long long><<<148 * 4, 256, 0, cstream_>>>(
          static_cast<const unsigned long long*>(traces), d_send_slots_,
          static_cast<unsigned long long*>(d_send_buf_), ns, Bt_, P_, TS_, L_);
    else
      pack_kernel<unsigned int><<<148 * 4, 256, 0, cstream_>>>(
          static_cast<const unsigned int*>(traces), d_send_slots_, static_cast<unsigned int*>(d_send_buf_),
          ns, Bt_, P_, TS_, L_);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
  const size_t bytes_per = static_cast<size_t>(vals_) * eb_;
  if (loop_) {
    e = cudaStreamSynchronize(cstream_);  // own pack done
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
    loop_->barrier();                     // every rank's pack done
    for (size_t k = 0; k < plan_.peers.size(); ++k) {
      const Halo* ph = loop_->members[plan_.peers[k]];
      const auto it = std::find(ph->plan_.peers.begin(), ph->plan_.peers.end(), rank_);
      if (it == ph->plan_.peers.end()) { *err = "loopback peer without a segment"; return 4; }
      const size_t idx = static_cast<size_t>(it - ph->plan_.peers.begin());
      if (ph->plan_.send_cnt[idx] != plan_.recv_cnt[k]) { *err = "loopback segment size mismatch"; return 4; }
      e = cudaMemcpyAsync(static_cast<char*>(d_recv_buf_) + plan_.recv_off[k] * bytes_per,
                          static_cast<const char*>(ph->d_send_buf_) + ph->plan_.send_off[idx] * bytes_per,
                          plan_.recv_cnt[k] * bytes_per, cudaMemcpyDeviceToDevice, cstream_);
      if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
    }
    e = cudaStreamSynchronize(cstream_);
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
    loop_->barrier();  // every copy done before anyone repacks
  } else {
  int r = g_nccl.gstart();
  for (size_t k = 0; r == 0 && k < plan_.peers.size(); ++k) {
    const char* sb = static_cast<const char*>(d_send_buf_) + plan_.send_off[k] * bytes_per;
    r = g_nccl.send(sb, plan_.send_cnt[k] * bytes_per, kNcclUint8, plan_.peers[k], comm_, cstream_);
    if (r) break;
    char* rb = static_cast<char*>(d_recv_buf_) + plan_.recv_off[k] * bytes_per;
    r = g_nccl.recv(rb, plan_.recv_cnt[k] * bytes_per, kNcclUint8, plan_.peers[k], comm_, cstream_);
  }
  int r2 = g_nccl.gend();
  if (r || r2) { *err = std::string("NCCL: ") + g_nccl.errstr(r ? r : r2); return 4; }
  }
  if (ng) {
    if (elem_bytes == 8)
      unpack_kernel<unsigned long long><<<148 * 4, 256, 0, cstream_>>>(
          static_cast<const unsigned long long*>(d_recv_buf_), static_cast<unsigned long long*>(traces),
          d_recv_slots_, ng, Bt_, P_, TS_, L_);
    else
      unpack_kernel<unsigned int><<<148 * 4, 256, 0, cstream_>>>(
          static_cast<const unsigned int*>(d_recv_buf_), static_cast<unsigned int*>(traces), d_recv_slots_,
          ng, Bt_, P_, TS_, L_);
    e = cudaGetLastError();
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
  }
  e = cudaEventRecord(done_, cstream_);
  if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
  return 0;
}

int Halo::wait(cudaStream_t s, std::string* err) {
  cudaError_t e = cudaStreamWaitEvent(s, done_, 0);
  if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 3; }
  return 0;
}

void Halo::destroy() {
  if (d_send_slots_) cudaFree(d_send_slots_);
  if (d_recv_slots_) cudaFree(d_recv_slots_);
  d_recv_slots_ = nullptr;
  if (d_send_buf_) cudaFree(d_send_buf_);
  if (d_recv_buf_) cudaFree(d_recv_buf_);
  d_send_slots_ = nullptr;
  d_send_buf_ = nullptr;
  d_recv_buf_ = nullptr;
  if (comm_ && g_nccl.destroy) g_nccl.destroy(comm_);
  comm_ = nullptr;
  if (loop_) {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    loop_->members[rank_] = nullptr;
    bool empty = true;
    for (Halo* m : loop_->members) empty = empty && !m;
    if (empty)
      for (auto it = g_loops.begin(); it != g_loops.end(); ++it)
        if (it->second == loop_) { g_loops.erase(it); break; }
    loop_.reset();
  }
  if (ready_) cudaEventDestroy(ready_);
  if (done_) cudaEventDestroy(done_);
  if (cstream_) cudaStreamDestroy(cstream_);
  ready_ = done_ = nullptr;
  cstream_ = nullptr;
}

}  // namespace ydg
