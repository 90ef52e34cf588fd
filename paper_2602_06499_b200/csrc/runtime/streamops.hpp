// Stream memory operations (cuStreamWaitValue32 / cuStreamWriteValue32),
// resolved at run time through cudaGetDriverEntryPoint so the library does
// not link libcuda.  They carry every cross-rank ordering edge of the data
// plane: a GPU stream waits on a 32-bit flag in the shared control block
// (pinned, host-mapped) that a peer's stream or NIC thread writes.  No host
// thread blocks on a peer, and no kernel spins.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace fcdp {

struct StreamOps {
  // Block `s` until *flag >= value (wrap-free: values stay < 2^31 per job).
  static void wait_geq(cudaStream_t s, const volatile std::uint32_t* dev_flag, std::uint32_t value);
  // Write `value` to *flag once all prior work on `s` is complete and visible.
  static void write(cudaStream_t s, volatile std::uint32_t* dev_flag, std::uint32_t value);
  static bool available();
};

}  // namespace fcdp
