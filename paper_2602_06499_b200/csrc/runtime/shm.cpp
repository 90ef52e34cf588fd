#include "runtime/shm.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <signal.h>
#include <cerrno>

#include <chrono>
#include <cstring>
#include <new>
#include <stdexcept>
#include <thread>

#include "capi_util.hpp"

namespace fcdp {
namespace {

std::size_t round_up(std::size_t x, std::size_t a) { return (x + a - 1) / a * a; }

std::string shm_path(const std::string& name) { return name.empty() || name[0] != '/' ? "/" + name : name; }

}  // namespace

std::uint64_t SharedBlock::now_ns() {
  return static_cast<std::uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                        std::chrono::steady_clock::now().time_since_epoch())
                                        .count());
}

SharedBlock::SharedBlock(const std::string& name, int rank, int world, int nodes, int local,
                         int inter_slots, std::uint64_t slot_bytes, double timeout_s)
    : name_(shm_path(name)), rank_(rank) {
  if (world < 1 || world > kMaxRanks || nodes * local != world || rank < 0 || rank >= world)
    throw shardsim::ConfigError("engine: world_size must equal num_nodes * gpus_per_node (<= 64)");
  slot_bytes = round_up(slot_bytes ? slot_bytes : 4096, 4096);
  slots_offset_ = round_up(sizeof(ShmHeader), 1 << 21);
  bytes_ = slots_offset_ + static_cast<std::size_t>(world) * 2 * inter_slots * slot_bytes;
  bytes_ = round_up(bytes_, 1 << 21);

  int fd = -1;
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
  if (rank == 0) {
    shm_unlink(name_.c_str());  // a stale segment of a crashed job with the same name
    fd = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error("shm_open(create " + name_ + ") failed: " + std::strerror(errno));
    if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
      close(fd);
      throw std::runtime_error("ftruncate(shm) failed: " + std::string(std::strerror(errno)));
    }
    void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw std::runtime_error("mmap(shm) failed: " + std::string(std::strerror(errno)));
    hdr_ = static_cast<ShmHeader*>(p);
    // ftruncate zero-fills; publish geometry and the creator, then the magic last.
    hdr_->world = world;
    hdr_->nodes = nodes;
    hdr_->local = local;
    hdr_->inter_slots = inter_slots;
    hdr_->slot_bytes = slot_bytes;
    hdr_->total_bytes = bytes_;
    hdr_->creator_pid = static_cast<std::int32_t>(getpid());
    hdr_->creator_nonce = now_ns() ^ (static_cast<std::uint64_t>(getpid()) << 40);
    hdr_->magic.store(kShmMagic, std::memory_order_release);
  } else {
    for (;;) {
      fd = shm_open(name_.c_str(), O_RDWR, 0600);
      if (fd >= 0) {
        struct stat st {};
        if (fstat(fd, &st) == 0 && static_cast<std::size_t>(st.st_size) >= bytes_) {
          void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
          close(fd);
          fd = -1;
          if (p == MAP_FAILED) throw std::runtime_error("mmap(shm) failed: " + std::string(std::strerror(errno)));
          auto* h = static_cast<ShmHeader*>(p);
          while (h->magic.load(std::memory_order_acquire) != kShmMagic &&
                 std::chrono::steady_clock::now() < deadline)
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
          // a live creator: this is the current job's segment (a crashed job's
          // rank 0 is gone, and its segment is about to be unlinked and recreated)
          const bool live = h->magic.load(std::memory_order_acquire) == kShmMagic &&
                            (kill(h->creator_pid, 0) == 0 || errno == EPERM);
          if (live) {
            hdr_ = h;
            break;
          }
          munmap(p, bytes_);
        } else {
          close(fd);
          fd = -1;
        }
      }
      if (std::chrono::steady_clock::now() > deadline)
        throw TimeoutError("engine: shared control block " + name_ + " did not appear");
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    if (hdr_->world != world || hdr_->nodes != nodes || hdr_->local != local ||
        hdr_->slot_bytes != slot_bytes || hdr_->inter_slots != inter_slots)
      throw shardsim::ConfigError("engine: ranks disagree on the job geometry");
  }
  hdr_->ranks[rank].pid = static_cast<std::int32_t>(getpid());
  hdr_->ranks[rank].attached.store(1, std::memory_order_release);
}

ShmSegment::ShmSegment(const std::string& name, std::size_t bytes, bool create, double timeout_s)
    : name_(shm_path(name)), bytes_(round_up(bytes ? bytes : 4096, 4096)), owner_(create) {
  int fd = -1;
  if (create) {
    shm_unlink(name_.c_str());
    fd = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error("shm_open(create " + name_ + ") failed: " + std::strerror(errno));
    if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
      close(fd);
      throw std::runtime_error("ftruncate(" + name_ + ") failed: " + std::string(std::strerror(errno)));
    }
  } else {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
    for (;;) {
      fd = shm_open(name_.c_str(), O_RDWR, 0600);
      if (fd >= 0) {
        struct stat st {};
        if (fstat(fd, &st) == 0 && static_cast<std::size_t>(st.st_size) >= bytes_) break;
        close(fd);
        fd = -1;
      }
      if (std::chrono::steady_clock::now() > deadline) throw TimeoutError("shm segment " + name_ + " did not appear");
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) throw std::runtime_error("mmap(" + name_ + ") failed: " + std::string(std::strerror(errno)));
  base_ = static_cast<unsigned char*>(p);
}

ShmSegment::~ShmSegment() {
  if (base_) munmap(base_, bytes_);
  if (owner_) shm_unlink(name_.c_str());
}

SharedBlock::~SharedBlock() {
  if (hdr_) munmap(hdr_, bytes_);
  if (rank_ == 0) shm_unlink(name_.c_str());
}

unsigned char* SharedBlock::slot(int rank, int cls, int idx) const {
  const std::size_t per_rank = 2ull * hdr_->inter_slots * hdr_->slot_bytes;
  return reinterpret_cast<unsigned char*>(hdr_) + slots_offset_ + rank * per_rank +
         (static_cast<std::size_t>(cls) * hdr_->inter_slots + idx) * hdr_->slot_bytes;
}

void SharedBlock::reset_counters(int rank) const {
  for (auto& c : hdr_->ranks[rank].counters) c.store(0, std::memory_order_relaxed);
}

void SharedBlock::await_posted(int rank, Flag f, std::uint32_t v, double timeout_s) const {
  auto& c = hdr_->ranks[rank].posted[f];
  if (static_cast<std::int32_t>(c.load(std::memory_order_acquire) - v) >= 0) return;
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
  int spins = 0;
  while (static_cast<std::int32_t>(c.load(std::memory_order_acquire) - v) < 0) {
    if (hdr_->abort_flag.load(std::memory_order_relaxed)) throw TimeoutError("engine: job aborted by a peer");
    if (++spins > 2000) {
      std::this_thread::sleep_for(std::chrono::microseconds(20));
      if (std::chrono::steady_clock::now() > deadline)
        throw TimeoutError("engine: rank " + std::to_string(rank) + " never posted flag " + std::to_string(f) +
                           " >= " + std::to_string(v));
    }
  }
}

void SharedBlock::barrier(double timeout_s, bool honour_abort) const {
  const std::uint32_t gen = hdr_->barrier_gen.load(std::memory_order_acquire);
  if (hdr_->barrier_count.fetch_add(1, std::memory_order_acq_rel) + 1 ==
      static_cast<std::uint32_t>(hdr_->world)) {
    hdr_->barrier_count.store(0, std::memory_order_relaxed);
    hdr_->barrier_gen.store(gen + 1, std::memory_order_release);
    return;
  }
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
  int spins = 0;
  while (hdr_->barrier_gen.load(std::memory_order_acquire) == gen) {
    if (honour_abort && hdr_->abort_flag.load(std::memory_order_relaxed))
      throw TimeoutError("engine: job aborted by a peer");
    if (++spins > 1000) {
      std::this_thread::sleep_for(std::chrono::microseconds(50));
      if (std::chrono::steady_clock::now() > deadline) throw TimeoutError("engine: barrier timed out");
    }
  }
}

std::uint64_t SharedBlock::reserve_nic(int node, std::uint64_t ns) const {
  auto& clock = hdr_->node_blocks[node].nic_busy_until_ns;
  const std::uint64_t now = now_ns();
  std::uint64_t cur = clock.load(std::memory_order_relaxed);
  for (;;) {
    const std::uint64_t start = cur > now ? cur : now;
    if (clock.compare_exchange_weak(cur, start + ns, std::memory_order_acq_rel)) return start + ns;
  }
}

}  // namespace fcdp
