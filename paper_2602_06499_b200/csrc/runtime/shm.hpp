// Job-wide shared control block (POSIX shared memory, one per job).
//
// Every rank maps the same segment and registers it with CUDA (pinned,
// host-mapped), so one region carries:
//   * per-rank 32-bit signal flags, written by GPU streams (cuStreamWriteValue32)
//     or by the NIC thread, waited on by peer GPU streams (cuStreamWaitValue32),
//   * per-emulated-node NIC state: the pacing clock that serialises all of a
//     node's GPUs on its single NIC (reference topology.hpp:23-25),
//   * per-rank byte counters (the measured side of comm_volume, costmodel.cpp:21-98),
//   * per-rank inter-node staging slots (the "host-staged" wire of the NIC
//     emulator) and the CUDA IPC handles of every rank's peer-visible arena.
// Nothing here needs a GPU, so the host protocol is testable on CPU.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>

namespace fcdp {

inline constexpr std::uint64_t kShmMagic = 0x46434450'42323030ull;  // "FCDPB200"
inline constexpr int kMaxRanks = 64;
inline constexpr int kProgRing = 8;  // program hashes kept per rank (begin() agreement check)

enum Flag : int {
  kAgTxReady = 0,  // inter AG: my staged piece <= id has crossed the emulated wire
  kRsTxReady,      // inter RS: same, reduce-scatter class
  kSliceReady,     // intra gather: my slice buffer holds gather seq
  kSliceFree,      // intra gather: I finished pulling peers' slices of seq
  kGradReady,      // intra RS: my natural gradient buffer holds rs seq
  kGradFree,       // intra RS: I finished pulling peers' gradients of seq
  kAgStaged,       // inter AG: my staging D2H of piece id landed in host memory (for my NIC thread)
  kRsStaged,       // inter RS: same
  // consumed markers, one per SENDER node: "I no longer need any piece <= v of
  // node n's sender" -> that sender may reuse the ring slots of those pieces
  kAgConsumed0,
  kRsConsumed0 = kAgConsumed0 + 8,
  kNumFlags = kRsConsumed0 + 8
};

enum Counter : int {
  kTxFwdAg = 0, kTxBwdAg, kTxRs, kRxFwdAg, kRxBwdAg, kRxRs, kNvlinkRx, kCacheH2D, kCacheD2H,
  kStagingH2D, kStagingD2H, kAgEventsFwd, kAgEventsBwd, kNicBusyNs, kResidentHits, kTxGradSync, kRxGradSync,
  kNumCounters
};

struct alignas(64) FlagLine {
  volatile std::uint32_t v;
  char pad[60];
};

struct alignas(64) RankBlock {
  FlagLine flags[kNumFlags];
  // Host-side "posted" counters: the value this rank's host has ENQUEUED a
  // write of, per flag.  A rank only enqueues a stream wait on a peer flag once
  // the peer has posted the matching write, so no GPU wait ever depends on
  // work a (possibly blocked) peer host has not issued yet.
  std::atomic<std::uint32_t> posted[kNumFlags];
  std::atomic<std::uint64_t> counters[kNumCounters];
  unsigned char ipc_handle[64];  // cudaIpcMemHandle_t of the peer arena
  std::uint64_t arena_bytes;
  std::int32_t pid, device;
  std::atomic<std::uint32_t> attached;
  // Hash of the k-th program this rank began, in slot k % kProgRing.
  std::atomic<std::uint64_t> prog_hash[kProgRing];
  std::atomic<std::uint32_t> prog_seq[kProgRing];
};

struct alignas(64) NodeBlock {
  std::atomic<std::uint64_t> nic_busy_until_ns;  // pacing clock of the node's NIC (tx)
};

struct alignas(64) ShmHeader {
  std::atomic<std::uint64_t> magic;
  std::int32_t world, nodes, local, inter_slots;
  std::uint64_t slot_bytes;   // bytes of one staging slot
  std::uint64_t total_bytes;
  // Rank 0's pid and a per-creation nonce, written before the magic: a rank
  // that attached to a stale segment of a crashed job (same name) sees a dead
  // creator and re-opens the name.
  std::int32_t creator_pid;
  std::uint64_t creator_nonce;
  alignas(64) std::atomic<std::uint32_t> barrier_count;
  alignas(64) std::atomic<std::uint32_t> barrier_gen;
  alignas(64) std::atomic<std::uint32_t> abort_flag;
  RankBlock ranks[kMaxRanks];
  NodeBlock node_blocks[kMaxRanks];
};

// A named POSIX shared-memory segment (one per rank) used for memory other
// ranks must read directly, e.g. the FCDP-Cache host tier when staged shards
// are served to the wire from it.
class ShmSegment {
 public:
  ShmSegment(const std::string& name, std::size_t bytes, bool create, double timeout_s);
  ~ShmSegment();
  ShmSegment(const ShmSegment&) = delete;
  ShmSegment& operator=(const ShmSegment&) = delete;
  unsigned char* base() const { return base_; }
  std::size_t bytes() const { return bytes_; }

 private:
  std::string name_;
  unsigned char* base_ = nullptr;
  std::size_t bytes_ = 0;
  bool owner_ = false;
};

class SharedBlock {
 public:
  // Rank 0 creates (and later unlinks) the segment; others attach, waiting up
  // to `timeout_s` for it to appear.  slot_bytes / inter_slots size the
  // per-rank staging area: 2 classes (AG, RS) x inter_slots x slot_bytes.
  SharedBlock(const std::string& name, int rank, int world, int nodes, int local, int inter_slots,
              std::uint64_t slot_bytes, double timeout_s);
  ~SharedBlock();
  SharedBlock(const SharedBlock&) = delete;
  SharedBlock& operator=(const SharedBlock&) = delete;

  ShmHeader* header() const { return hdr_; }
  void* base() const { return hdr_; }
  std::size_t bytes() const { return bytes_; }
  RankBlock& rank_block(int r) const { return hdr_->ranks[r]; }
  // Staging ring slot of (rank, class 0 = AG / 1 = RS, slot index).
  unsigned char* slot(int rank, int cls, int idx) const;
  volatile std::uint32_t* flag(int rank, Flag f) const { return &hdr_->ranks[rank].flags[f].v; }
  void add(int rank, Counter c, std::uint64_t v) const {
    hdr_->ranks[rank].counters[c].fetch_add(v, std::memory_order_relaxed);
  }
  std::uint64_t counter(int rank, Counter c) const {
    return hdr_->ranks[rank].counters[c].load(std::memory_order_relaxed);
  }
  void reset_counters(int rank) const;
  void post(int rank, Flag f, std::uint32_t v) const {
    hdr_->ranks[rank].posted[f].store(v, std::memory_order_release);
  }
  // Spin (host) until `rank` has posted >= v for flag f.
  void await_posted(int rank, Flag f, std::uint32_t v, double timeout_s) const;

  // Host barrier over all ranks (sense-reversing on a generation counter).
  // honour_abort = false: the teardown barrier, which must still gather every
  // rank after a peer aborted (no rank may free memory a peer still reads).
  void barrier(double timeout_s, bool honour_abort = true) const;
  // Reserve `ns` of wire time on node n's NIC; returns the finish time (ns,
  // steady clock).  Reservations from the node's ranks serialise.
  std::uint64_t reserve_nic(int node, std::uint64_t ns) const;
  static std::uint64_t now_ns();

  int rank() const { return rank_; }

 private:
  std::string name_;
  int rank_;
  ShmHeader* hdr_ = nullptr;
  std::size_t bytes_ = 0;
  std::size_t slots_offset_ = 0;
};

}  // namespace fcdp
