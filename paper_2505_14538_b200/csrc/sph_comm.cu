// sph_comm.cu -- NCCL and loopback transports of the slab decomposition (sph_comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include <condition_variable>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "sph_comm.cuh"

namespace sph {

// ------------------------------------------------------------------------ NCCL ------
namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

std::mutex g_nccl_mu;
NcclApi g_nccl;

std::string load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.lib) return "";
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names) {
    h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) return std::string("cannot load libnccl.so.2: ") + dlerror();
#define SYM(field, name)                                             \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) return std::string("libnccl lacks ") + name;
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(AllReduce, "ncclAllReduce");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  g_nccl.lib = h;
  return "";
}

class NcclComm : public Comm {
 public:
  NcclComm(int rank, int n) : rank_(rank), n_(n) {}
  ~NcclComm() override {
    for (auto& kv : opened_) cudaIpcCloseMemHandle(kv.second);
    if (scratch_) cudaFree(scratch_);
    if (comm_) g_nccl.CommDestroy(comm_);
  }
  std::string init(const void* uid) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclResult_t r = g_nccl.CommInitRank(&comm_, n_, id, rank_);
    if (r != ncclSuccess) return std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r);
    if (cudaMalloc(&scratch_, 64 * sizeof(double)) != cudaSuccess) return "cudaMalloc (nccl scratch) failed";
    return "";
  }
  int rank() const override { return rank_; }
  int size() const override { return n_; }
  std::string exchange(const Xfer* s, int ns, const Xfer* r, int nr, cudaStream_t st) override {
    ncclResult_t e = g_nccl.GroupStart();
    for (int k = 0; k < ns && e == ncclSuccess; ++k)
      if (s[k].bytes) e = g_nccl.Send(s[k].buf, s[k].bytes, ncclInt8, s[k].peer, comm_, st);
    for (int k = 0; k < nr && e == ncclSuccess; ++k)
      if (r[k].bytes) e = g_nccl.Recv(r[k].buf, r[k].bytes, ncclInt8, r[k].peer, comm_, st);
    ncclResult_t e2 = g_nccl.GroupEnd();
    if (e == ncclSuccess) e = e2;
    return e == ncclSuccess ? "" : std::string("nccl send/recv: ") + g_nccl.GetErrorString(e);
  }
  std::string allreduce(double* v, int n, ReduceOp op, cudaStream_t st) override {
    if (n > 64) return "allreduce: too many values";
    ncclRedOp_t o = op == kSum ? ncclSum : (op == kMax ? ncclMax : ncclMin);
    if (cudaMemcpyAsync(scratch_, v, n * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return "allreduce: H2D failed";
    ncclResult_t e = g_nccl.AllReduce(scratch_, scratch_, n, ncclFloat64, o, comm_, st);
    if (e != ncclSuccess) return std::string("ncclAllReduce: ") + g_nccl.GetErrorString(e);
    if (cudaMemcpyAsync(v, scratch_, n * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return "allreduce: D2H failed";
    if (cudaStreamSynchronize(st) != cudaSuccess) return "allreduce: sync failed";
    return "";
  }
  std::string allreduce_dev_u32(uint32_t* d, int n, ReduceOp op, cudaStream_t st) override {
    ncclRedOp_t o = op == kSum ? ncclSum : (op == kMax ? ncclMax : ncclMin);
    ncclResult_t e = g_nccl.AllReduce(d, d, n, ncclUint32, o, comm_, st);
    return e == ncclSuccess ? "" : std::string("ncclAllReduce: ") + g_nccl.GetErrorString(e);
  }
  // IPC handles through the scratch buffer (sent to both neighbours, theirs received), then
  // opened once per (peer, handle) with lazy peer access (NVLink P2P on an NVSwitch node).
  std::string map_peer(void* mine, int left, int right, void** left_out, void** right_out,
                       cudaStream_t st) override {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, mine) != cudaSuccess) return "cudaIpcGetMemHandle failed";
    char* sc = reinterpret_cast<char*>(scratch_);  // 512 bytes: [mine | from left | from right]
    if (cudaMemcpyAsync(sc, &h, 64, cudaMemcpyHostToDevice, st) != cudaSuccess) return "map_peer: H2D failed";
    Xfer s[2] = {{right, sc, 64}, {left, sc, 64}};
    Xfer r[2] = {{left, sc + 64, 64}, {right, sc + 128, 64}};
    std::string e = exchange(s, 2, r, 2, st);
    if (!e.empty()) return e;
    cudaIpcMemHandle_t hl, hr;
    if (cudaMemcpyAsync(&hl, sc + 64, 64, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&hr, sc + 128, 64, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return "map_peer: D2H failed";
    e = open_peer(left, hl, mine, left_out);
    if (e.empty()) e = open_peer(right, hr, mine, right_out);
    return e;
  }

 private:
  std::string open_peer(int peer, const cudaIpcMemHandle_t& h, void* mine, void** out) {
    if (peer == rank_) {
      *out = mine;
      return "";
    }
    const std::string key(reinterpret_cast<const char*>(&h), sizeof(h));
    auto it = opened_.find(key);
    if (it != opened_.end()) {
      *out = it->second;
      return "";
    }
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return "cudaIpcOpenMemHandle failed (peer rank " + std::to_string(peer) + ")";
    opened_[key] = p;
    *out = p;
    return "";
  }
  int rank_, n_;
  ncclComm_t comm_ = nullptr;
  double* scratch_ = nullptr;
  std::map<std::string, void*> opened_;  // IPC mappings (closed in the destructor)
};

}  // namespace

std::string nccl_unique_id(void* out128) {
  std::string e = load_nccl();
  if (!e.empty()) return e;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r);
  memcpy(out128, &id, sizeof(id));
  return "";
}

Comm* make_nccl_comm(const void* uid, int rank, int nranks, std::string& err) {
  err = load_nccl();
  if (!err.empty()) return nullptr;
  NcclComm* c = new NcclComm(rank, nranks);
  err = c->init(uid);
  if (!err.empty()) {
    delete c;
    return nullptr;
  }
  return c;
}

// -------------------------------------------------------------------- loopback ------
namespace {

struct LoopGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  struct Msg {
    const void* ptr;
    size_t bytes;
    cudaEvent_t ready;
    cudaEvent_t done;
    bool consumed;
  };
  std::map<std::tuple<int, int, long>, Msg> box;  // (src, dst, sequence)
  long ar_gen = 0;
  int ar_count = 0;
  std::vector<double> ar_acc, ar_res;
  std::map<std::pair<int, long>, void*> peers;  // (rank, map_peer sequence) -> published buffer
  explicit LoopGroup(int k) : n(k) {}
};

using Key = std::tuple<int, int, long>;

class LoopComm : public Comm {
 public:
  LoopComm(LoopGroup* g, int rank) : g_(g), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return g_->n; }
  // Messages between one (sender, receiver) pair are matched in list order; both sides skip
  // zero-byte messages.  Callers list sends as (to right, to left) and receives as (from
  // left, from right), which pairs correctly even when both neighbours are the same rank.
  std::string exchange(const Xfer* s, int ns, const Xfer* r, int nr, cudaStream_t st) override {
    const long seq = seq_++;
    std::map<int, int> sidx, ridx;
    std::vector<Key> mine;
    for (int k = 0; k < ns; ++k) {
      if (!s[k].bytes) continue;
      LoopGroup::Msg m{s[k].buf, s[k].bytes, nullptr, nullptr, false};
      cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming);
      cudaEventRecord(m.ready, st);
      const Key key = std::make_tuple(rank_, s[k].peer, seq * 64 + sidx[s[k].peer]++);
      {
        std::lock_guard<std::mutex> lk(g_->mu);
        g_->box[key] = m;
      }
      mine.push_back(key);
    }
    g_->cv.notify_all();
    for (int k = 0; k < nr; ++k) {
      if (!r[k].bytes) continue;
      const Key key = std::make_tuple(r[k].peer, rank_, seq * 64 + ridx[r[k].peer]++);
      std::unique_lock<std::mutex> lk(g_->mu);
      g_->cv.wait(lk, [&] { return g_->box.count(key) != 0; });
      LoopGroup::Msg m = g_->box[key];
      lk.unlock();
      if (m.bytes != r[k].bytes) return "loopback exchange: message size mismatch";
      cudaStreamWaitEvent(st, m.ready, 0);
      cudaMemcpyAsync(r[k].buf, m.ptr, m.bytes, cudaMemcpyDeviceToDevice, st);
      cudaEvent_t done;
      cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
      cudaEventRecord(done, st);
      lk.lock();
      g_->box[key].done = done;
      g_->box[key].consumed = true;
      lk.unlock();
      g_->cv.notify_all();
    }
    for (const Key& key : mine) {
      std::unique_lock<std::mutex> lk(g_->mu);
      g_->cv.wait(lk, [&] { return g_->box[key].consumed; });
      LoopGroup::Msg m = g_->box[key];
      g_->box.erase(key);
      lk.unlock();
      cudaStreamWaitEvent(st, m.done, 0);  // later writes to the send buffer wait for the copy
      cudaEventDestroy(m.ready);
      cudaEventDestroy(m.done);
    }
    return cudaGetLastError() == cudaSuccess ? "" : "loopback exchange: CUDA error";
  }
  std::string allreduce(double* v, int n, ReduceOp op, cudaStream_t st) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) return "allreduce: sync failed";
    std::unique_lock<std::mutex> lk(g_->mu);
    if (g_->ar_count == 0) g_->ar_acc.assign(v, v + n);
    else
      for (int k = 0; k < n; ++k) {
        double& a = g_->ar_acc[k];
        a = op == kSum ? a + v[k] : (op == kMax ? (v[k] > a ? v[k] : a) : (v[k] < a ? v[k] : a));
      }
    const long gen = g_->ar_gen;
    if (++g_->ar_count == g_->n) {
      g_->ar_res = g_->ar_acc;
      g_->ar_count = 0;
      ++g_->ar_gen;
      g_->cv.notify_all();
    } else {
      g_->cv.wait(lk, [&] { return g_->ar_gen != gen; });
    }
    for (int k = 0; k < n; ++k) v[k] = g_->ar_res[k];
    return "";
  }
  // (one process, one device: a buffer of another context is directly addressable; each rank
  // publishes its buffer under its map_peer sequence number and takes its neighbours')
  std::string map_peer(void* mine, int left, int right, void** left_out, void** right_out,
                       cudaStream_t) override {
    const long seq = map_seq_++;
    std::unique_lock<std::mutex> lk(g_->mu);
    g_->peers[std::make_pair(rank_, seq)] = mine;
    g_->cv.notify_all();
    const auto kl = std::make_pair(left, seq), kr = std::make_pair(right, seq);
    g_->cv.wait(lk, [&] { return g_->peers.count(kl) && g_->peers.count(kr); });
    *left_out = g_->peers[kl];
    *right_out = g_->peers[kr];
    return "";
  }
  // (one process: through the host, exactly as allreduce)
  std::string allreduce_dev_u32(uint32_t* d, int n, ReduceOp op, cudaStream_t st) override {
    std::vector<uint32_t> h(n);
    std::vector<double> v(n);
    if (cudaMemcpyAsync(h.data(), d, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return "allreduce: D2H failed";
    if (cudaStreamSynchronize(st) != cudaSuccess) return "allreduce: sync failed";
    for (int k = 0; k < n; ++k) v[k] = (double)h[k];
    std::string e = allreduce(v.data(), n, op, st);
    if (!e.empty()) return e;
    for (int k = 0; k < n; ++k) h[k] = (uint32_t)v[k];
    if (cudaMemcpy(d, h.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess)
      return "allreduce: H2D failed";
    return "";
  }

 private:
  LoopGroup* g_;
  int rank_;
  long seq_ = 0;
  long map_seq_ = 0;
};

}  // namespace

void* loopback_group_create(int nranks) { return new LoopGroup(nranks); }
void loopback_group_destroy(void* g) { delete static_cast<LoopGroup*>(g); }

Comm* make_loopback_comm(void* group, int rank, std::string& err) {
  if (!group) {
    err = "loopback transport needs a group (sph_loopback_create)";
    return nullptr;
  }
  LoopGroup* g = static_cast<LoopGroup*>(group);
  if (rank < 0 || rank >= g->n) {
    err = "loopback rank out of range";
    return nullptr;
  }
  err = "";
  return new LoopComm(g, rank);
}

}  // namespace sph
