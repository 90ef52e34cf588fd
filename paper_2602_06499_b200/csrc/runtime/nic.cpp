#include "runtime/nic.hpp"

#include <algorithm>
#include <chrono>

namespace fcdp {

NicEmulator::NicEmulator(SharedBlock& shm, int rank, int node, double bytes_per_s, bool pacing)
    : shm_(shm), rank_(rank), node_(node), bytes_per_ns_(bytes_per_s / 1e9), pacing_(pacing) {
  thread_ = std::thread([this] { loop(); });
}

NicEmulator::~NicEmulator() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  thread_.join();
}

void NicEmulator::submit(const NicJob& job) {
  {
    std::lock_guard<std::mutex> g(mu_);
    queue_[job.cls].push_back(job);
  }
  cv_.notify_all();
}

void NicEmulator::set_log(bool on) {
  std::lock_guard<std::mutex> g(mu_);
  log_on_ = on;
  if (!on) log_.clear();
}

std::size_t NicEmulator::take_log(WireRecord* out, std::size_t capacity) {
  std::lock_guard<std::mutex> g(mu_);
  const std::size_t n = std::min(capacity, log_.size());
  std::copy(log_.begin(), log_.begin() + static_cast<std::ptrdiff_t>(n), out);
  log_.erase(log_.begin(), log_.begin() + static_cast<std::ptrdiff_t>(n));
  return n;
}

std::uint64_t NicEmulator::published(int cls) const {
  return *shm_.flag(rank_, cls == 0 ? kAgTxReady : kRsTxReady);
}

void NicEmulator::loop() {
  std::unique_lock<std::mutex> lk(mu_);
  for (;;) {
    bool idle = true;
    std::uint64_t next_finish = ~0ull;
    for (int c = 0; c < 2; ++c) {
      // Staged payloads enter the wire in submission order (per class).
      while (!queue_[c].empty()) {
        NicJob& j = queue_[c].front();
        const std::uint32_t staged = __atomic_load_n(shm_.flag(rank_, c == 0 ? kAgStaged : kRsStaged), __ATOMIC_ACQUIRE);
        if (static_cast<std::int32_t>(staged - j.seq) < 0) break;  // staging copy not landed yet
        const std::uint64_t ns =
            pacing_ && bytes_per_ns_ > 0 ? static_cast<std::uint64_t>(j.wire_bytes / bytes_per_ns_) : 0;
        const std::uint64_t finish = ns ? shm_.reserve_nic(node_, ns) : SharedBlock::now_ns();
        shm_.add(rank_, kNicBusyNs, ns);
        if (log_on_) log_.push_back({finish - ns, finish, j.wire_bytes, static_cast<std::int32_t>(j.counter), node_});
        flight_[c].push_back({j, finish});
        queue_[c].pop_front();
        idle = false;
      }
      const std::uint64_t now = SharedBlock::now_ns();
      while (!flight_[c].empty() && flight_[c].front().finish_ns <= now) {
        const Flight& f = flight_[c].front();
        shm_.add(rank_, f.job.counter, f.job.wire_bytes);
        __atomic_store_n(shm_.flag(rank_, c == 0 ? kAgTxReady : kRsTxReady), f.job.seq, __ATOMIC_RELEASE);
        flight_[c].pop_front();
        idle = false;
      }
      if (!flight_[c].empty() && flight_[c].front().finish_ns < next_finish) next_finish = flight_[c].front().finish_ns;
      if (!queue_[c].empty()) next_finish = 0;  // poll the staging event
    }
    if (!idle) continue;
    if (stop_ && queue_[0].empty() && queue_[1].empty() && flight_[0].empty() && flight_[1].empty()) return;
    if (next_finish == ~0ull) {
      cv_.wait_for(lk, std::chrono::milliseconds(5));
      continue;
    }
    const std::uint64_t now = SharedBlock::now_ns();
    if (next_finish == 0 || next_finish <= now + 80'000) {
      // close to a deadline or waiting on a copy: short yield keeps jitter low
      lk.unlock();
      std::this_thread::yield();
      lk.lock();
    } else {
      cv_.wait_for(lk, std::chrono::nanoseconds(next_finish - now - 60'000));
    }
  }
}

}  // namespace fcdp
