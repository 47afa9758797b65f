// z-slab halo exchange of time-integrated face traces over NCCL (loaded at run time).
//
// The neighbour flux reads, for every face, the neighbour's time-integrated
// trace; across a slab boundary the neighbour lives on another GPU.  Each rank sends the
// traces of its owned elements that touch a peer's slab and receives the peer's into
// ghost slots (one NCCL group of send/recv per step, on a side stream).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "setup.h"

namespace ydg {

// Messages carry one face block (Bt x P values of the time-integrated trace) per shared
// face: for every face whose two elements live on different ranks, the owner of each side
// sends its own side's trace; the receiver stores it in the ghost slot of the sending
// element at that element's local face.  Both sides order a peer's blocks by (global id of
// the sending element, its local face), so no index travels with the data.
struct HaloPlan {
  // ghosts: global ids in slot order (sorted by owner rank, then global id)
  std::vector<int64_t> ghost_of;
  std::vector<int> peers;             // peer ranks (ascending)
  std::vector<int64_t> recv_off;      // first received face block per peer
  std::vector<int64_t> recv_cnt;      // face blocks per peer
  std::vector<int64_t> recv_ghost;    // per received block: ghost index (slot - owned slots)
  std::vector<int8_t> recv_face;      //   and the ghost element's local face
  std::vector<int64_t> send_slots;    // per sent block: local slot, grouped by peer
  std::vector<int8_t> send_face;      //   and the local face
  std::vector<int64_t> send_off, send_cnt;
};

// Pure host: build the plan for rank `rank` of `nranks` owning [first, first+nlocal).
// Peers own ranges [r*ne/nranks, (r+1)*ne/nranks).
bool plan_halo(const Neighbours& nbr, int64_t ne, int rank, int nranks, HaloPlan* out,
               std::string* err);

struct LoopGroup;

class Halo {
 public:
  int init(int rank, int nranks, const void* uid, std::string* err);
  int plan(const Neighbours& nbr, int64_t first, int64_t nlocal, int64_t owned_slots,
           std::vector<int64_t>* ghost_of, std::string* err);
  // traces use the layout [tile][face][m][q][32] (TS = 0) or [tile][face][lane][TS] with
  // element-face blocks [m][q] (TS > 0), Bt face functions, P quantities
  int bind(void* traces, int Bt, int P, int TS, int L, int elem_bytes, int64_t owned_slots, std::string* err);
  // pack + send/recv on the comm stream after `s` reaches this point
  int exchange(cudaStream_t s, void* traces, int elem_bytes, std::string* err);
  // make `s` wait for the exchange
  int wait(cudaStream_t s, std::string* err);
  void destroy();
  const HaloPlan& plan_data() const { return plan_; }

 private:
  int rank_ = 0, nranks_ = 1;
  int64_t ne_ = 0;
  void* comm_ = nullptr;
  cudaStream_t cstream_ = nullptr;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  HaloPlan plan_;
  int64_t* d_send_slots_ = nullptr;  // packed (slot << 2 | face) per sent block
  int64_t* d_recv_slots_ = nullptr;  // packed (ghost slot << 2 | face) per received block
  void* d_send_buf_ = nullptr;
  void* d_recv_buf_ = nullptr;
  int vals_ = 0, eb_ = 0, Bt_ = 0, P_ = 0, TS_ = 0, L_ = 32;
  int64_t owned_slots_ = 0;
  std::shared_ptr<LoopGroup> loop_;  // loopback transport (unique id "YDGLOOP...")
};

}  // namespace ydg
