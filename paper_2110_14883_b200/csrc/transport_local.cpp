// In-process transport: every rank of the grid is a host thread of ONE process, with its
// buffers on any device (several ranks may share a GPU). It runs the exact schedules of the
// NCCL path so that multi-rank grids (2D q=2 on 4 ranks, 2.5D d=2 and 3D l=2 on 8 ranks) can
// be parity-tested on a single B200.
//
// Each collective is a stream-ordered exchange with NCCL's semantics:
//   1. record `ready` on the caller's stream, post {buffer pointers, ready} in the group's
//      slot table, host barrier;
//   2. make the stream wait on every member's `ready`; enqueue this rank's share of the
//      data movement (cudaMemcpyAsync device->device or a fp32-accumulating sum kernel that
//      reads the peers' buffers in ascending member order);
//   3. record `done`, post it, host barrier; make the stream wait on every member's `done`
//      (so no member reuses a buffer a peer is still reading).
// Slot tables are double-buffered by call parity, which makes two barriers per call enough.
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <random>

#include "tp_internal.h"

namespace tp {
namespace {

struct Slot {
  const void* src = nullptr;
  void* dst = nullptr;
  cudaEvent_t ready = nullptr;
  cudaEvent_t done = nullptr;
};

struct LocalGroup {
  explicit LocalGroup(int n) : n(n) {
    slots[0].resize(n);
    slots[1].resize(n);
  }
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<Slot> slots[2];

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t my = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my; });
    }
  }
};

struct Registry {
  std::mutex mu;
  std::map<std::string, std::shared_ptr<LocalGroup>> groups;  // key: world id + member list
};

Registry& registry() {
  static Registry r;
  return r;
}

std::shared_ptr<LocalGroup> get_group(const void* id128, const std::vector<int>& members) {
  std::string key(static_cast<const char*>(id128), 128);
  for (int m : members) key += "," + std::to_string(m);
  auto& R = registry();
  std::lock_guard<std::mutex> lk(R.mu);
  auto it = R.groups.find(key);
  if (it != R.groups.end()) {
    auto g = it->second;
    // last user drops the registry entry so a later world with the same id starts fresh
    return g;
  }
  auto g = std::make_shared<LocalGroup>(static_cast<int>(members.size()));
  R.groups[key] = g;
  return g;
}

void release_group(const void* id128, const std::vector<int>& members) {
  std::string key(static_cast<const char*>(id128), 128);
  for (int m : members) key += "," + std::to_string(m);
  auto& R = registry();
  std::lock_guard<std::mutex> lk(R.mu);
  auto it = R.groups.find(key);
  if (it != R.groups.end() && it->second.use_count() == 1) R.groups.erase(it);
}

class LocalComm final : public Comm {
 public:
  LocalComm(const void* id128, std::vector<int> members, int pos, int device)
      : members_(std::move(members)), pos_(pos), device_(device) {
    std::memcpy(id_, id128, 128);
    grp_ = get_group(id_, members_);
  }
  ~LocalComm() override {
    // Destruction is collective (like ncclCommDestroy): a peer may still be enqueuing a
    // wait on our `done` event from the last exchange, so nobody frees events before all
    // members got here.
    if (grp_) grp_->barrier();
    if (ready_) cudaEventDestroy(ready_);
    if (done_) cudaEventDestroy(done_);
    grp_.reset();
    release_group(id_, members_);
  }
  tp_status init() {
    TP_CUDA(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
    TP_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    return TP_OK;
  }
  int size() const override { return static_cast<int>(members_.size()); }
  int pos() const override { return pos_; }

  tp_status bcast(void* buf, size_t count, tp_dtype dt, int root, cudaStream_t s) override {
    const size_t bytes = count * dtype_size(dt);
    return exchange(buf, buf, s, [&](std::vector<Slot>& sl) -> tp_status {
      if (pos_ != root && bytes)
        TP_CUDA(cudaMemcpyAsync(buf, sl[root].src, bytes, cudaMemcpyDefault, s));
      return TP_OK;
    });
  }
  tp_status reduce(const void* send, void* recv, size_t count, tp_dtype dt, int root,
                   cudaStream_t s) override {
    return exchange(send, recv, s, [&](std::vector<Slot>& sl) -> tp_status {
      if (pos_ != root) return TP_OK;
      std::vector<const void*> in;
      for (auto& x : sl) in.push_back(x.src);
      return launch_sum_n(in.data(), size(), recv, count, dt, s);
    });
  }
  tp_status allreduce(const void* send, void* recv, size_t count, tp_dtype dt,
                      cudaStream_t s) override {
    if (send == recv) return fail(TP_ERR_UNSUPPORTED, "local transport: in-place all-reduce");
    return exchange(send, recv, s, [&](std::vector<Slot>& sl) -> tp_status {
      std::vector<const void*> in;
      for (auto& x : sl) in.push_back(x.src);
      return launch_sum_n(in.data(), size(), recv, count, dt, s);
    });
  }
  tp_status allgather(const void* send, void* recv, size_t count, tp_dtype dt,
                      cudaStream_t s) override {
    const size_t bytes = count * dtype_size(dt);
    return exchange(send, recv, s, [&](std::vector<Slot>& sl) -> tp_status {
      for (int m = 0; m < size(); ++m) {
        char* dst = static_cast<char*>(recv) + m * bytes;
        if (bytes && dst != sl[m].src)
          TP_CUDA(cudaMemcpyAsync(dst, sl[m].src, bytes, cudaMemcpyDefault, s));
      }
      return TP_OK;
    });
  }
  tp_status reducescatter(const void* send, void* recv, size_t count, tp_dtype dt,
                          cudaStream_t s) override {
    const size_t bytes = count * dtype_size(dt);
    return exchange(send, recv, s, [&](std::vector<Slot>& sl) -> tp_status {
      std::vector<const void*> in;
      for (auto& x : sl) in.push_back(static_cast<const char*>(x.src) + pos_ * bytes);
      return launch_sum_n(in.data(), size(), recv, count, dt, s);
    });
  }
  tp_status shift(const void* send, void* recv, size_t count, tp_dtype dt, int offset,
                  cudaStream_t s) override {
    const size_t bytes = count * dtype_size(dt);
    const int n = size();
    const int off = ((offset % n) + n) % n;
    return exchange(send, recv, s, [&](std::vector<Slot>& sl) -> tp_status {
      const void* src = sl[(pos_ + off) % n].src;
      if (bytes && recv != src) TP_CUDA(cudaMemcpyAsync(recv, src, bytes, cudaMemcpyDefault, s));
      return TP_OK;
    });
  }
  tp_status barrier(cudaStream_t s) override {
    return exchange(nullptr, nullptr, s, [](std::vector<Slot>&) -> tp_status { return TP_OK; });
  }
  tp_status host_allgather(const void* in, size_t bytes, void* out) override {
    auto& sl = grp_->slots[calls_ & 1];
    ++calls_;
    sl[pos_].src = in;
    grp_->barrier();
    for (int m = 0; m < size(); ++m)
      std::memcpy(static_cast<char*>(out) + m * bytes, sl[m].src, bytes);
    grp_->barrier();
    return TP_OK;
  }

 private:
  template <typename Body>
  tp_status exchange(const void* src, void* dst, cudaStream_t s, Body body) {
    auto& sl = grp_->slots[calls_ & 1];
    ++calls_;
    TP_CUDA(cudaEventRecord(ready_, s));
    sl[pos_].src = src;
    sl[pos_].dst = dst;
    sl[pos_].ready = ready_;
    grp_->barrier();
    for (int m = 0; m < size(); ++m)
      if (m != pos_) TP_CUDA(cudaStreamWaitEvent(s, sl[m].ready, 0));
    tp_status st = body(sl);
    // The barriers below still run on error so peers are not left waiting.
    cudaError_t e = cudaEventRecord(done_, s);
    sl[pos_].done = done_;
    grp_->barrier();
    for (int m = 0; m < size(); ++m)
      if (m != pos_) {
        cudaError_t e2 = cudaStreamWaitEvent(s, sl[m].done, 0);
        if (e == cudaSuccess) e = e2;
      }
    if (st != TP_OK) return st;
    if (e != cudaSuccess) return fail(TP_ERR_CUDA, std::string("local transport: ") + cudaGetErrorString(e));
    return TP_OK;
  }

  char id_[128];
  std::vector<int> members_;
  int pos_, device_;
  std::shared_ptr<LocalGroup> grp_;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  uint64_t calls_ = 0;
};

}  // namespace

tp_status local_unique_id(void* id128) {
  static std::mutex mu;
  static uint64_t counter = 0;
  std::lock_guard<std::mutex> lk(mu);
  std::random_device rd;
  uint64_t words[16];
  for (auto& w : words) w = (static_cast<uint64_t>(rd()) << 32) ^ rd();
  words[0] = 0x4C4F43414C5450ull;  // "LOCALTP"
  words[1] = ++counter;
  std::memcpy(id128, words, 128);
  return TP_OK;
}

std::unique_ptr<Comm> make_local_comm(const void* id128, int world, const std::vector<int>& members,
                                      int pos, int device, tp_status* st) {
  (void)world;
  auto c = std::make_unique<LocalComm>(id128, members, pos, device);
  *st = c->init();
  if (*st != TP_OK) return nullptr;
  return c;
}

}  // namespace tp
