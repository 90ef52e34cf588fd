// NIC emulator: one thread per rank that turns "my staged payload is in host
// memory" (a flag the staging stream writes after its D2H) into "my payload has crossed the
// emulated network" (a flag peers' streams wait on), after charging the
// payload's wire time to the sending node's single NIC (reference
// topology.hpp:23-25 "one NIC per node"; "Per-node NIC serializes
// all its GPUs' inter-node traffic").  Wire time = bytes / inter-node
// bandwidth of the topology preset (topology.cpp:22-34 in the reference).
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "runtime/shm.hpp"

namespace fcdp {

struct NicJob {
  int cls;               // 0 = all-gather, 1 = reduce-scatter
  std::uint32_t seq;     // per-class sequence number, monotone
  // The thread makes NO CUDA calls: a host thread blocked inside a launch
  // (full pushbuffer) can hold driver locks, and the NIC thread must keep
  // publishing or the stalled streams it feeds would never drain.
  std::uint64_t wire_bytes;  // bytes this rank puts on its node's NIC
  Counter counter;       // which tx counter to charge
};

// One paced payload on the emulated wire (the NIC bandwidth profile, PAPER.md
// Fig. 10 "peak inter-node network bandwidth during forward and backward"):
// [start_ns, end_ns) of steady_clock on the node's NIC clock, its bytes and
// the traffic kind (the tx Counter it is charged to).
struct WireRecord {
  std::uint64_t start_ns, end_ns, bytes;
  std::int32_t kind, node;
};

class NicEmulator {
 public:
  NicEmulator(SharedBlock& shm, int rank, int node, double bytes_per_s, bool pacing);
  ~NicEmulator();
  void submit(const NicJob& job);
  std::uint64_t published(int cls) const;
  // Wire log: off by default; take_log drains what was recorded since the last call.
  void set_log(bool on);
  std::size_t take_log(WireRecord* out, std::size_t capacity);

 private:
  void loop();
  struct Flight {
    NicJob job;
    std::uint64_t finish_ns;
  };
  SharedBlock& shm_;
  int rank_, node_;
  double bytes_per_ns_;
  bool pacing_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<NicJob> queue_[2];
  std::deque<Flight> flight_[2];
  bool stop_ = false;
  bool log_on_ = false;
  std::vector<WireRecord> log_;
  std::thread thread_;
};

}  // namespace fcdp
