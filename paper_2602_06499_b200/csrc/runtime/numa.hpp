// NUMA placement for the pinned host tiers.
//
// On a multi-socket host the FCDP-Cache and the NIC staging traffic of a GPU
// should live in the DRAM of the socket its PCIe root hangs off, and the
// threads that drive them (the rank's host thread and its NIC emulator) should
// run there.  libnuma is not available, so this uses sysfs plus the raw mbind
// and sched_setaffinity syscalls.  Single-node hosts: everything is a no-op.
#pragma once

#include <cstddef>
#include <string>
#include <vector>

namespace fcdp {

struct NumaPlacement {
  int gpu_node = -1;     // NUMA node of the GPU's PCIe device (-1: unknown)
  int num_nodes = 1;     // online memory nodes
  bool cpus_bound = false;
  std::size_t bytes_bound = 0;  // host bytes given a preferred-node policy
};

int numa_online_nodes();
int numa_node_of_gpu(int device);
std::vector<int> numa_node_cpus(int node);
// Parse a sysfs cpulist ("0-3,8,10-11").
std::vector<int> parse_cpulist(const std::string& s);
// Preferred-node policy for [p, p + bytes) before first touch.  Returns false
// when the kernel refuses (the memory still works, just not placed).
bool numa_prefer(void* p, std::size_t bytes, int node);
// Pin the calling thread (and threads it creates later) to the node's cores.
bool numa_pin_thread(int node);
// The calling thread's CPU affinity, saved and restored around a temporary pin
// (the engine pins only while it first-touches its host tiers and starts its
// NIC thread; the caller's own thread gets its affinity back).
struct SavedAffinity {
  bool valid = false;
  unsigned char set[128] = {};  // cpu_set_t bytes
};
SavedAffinity numa_save_affinity();
void numa_restore_affinity(const SavedAffinity& a);
// Node of the page holding p (get_mempolicy MPOL_F_NODE|MPOL_F_ADDR), -1 on error.
int numa_node_of_page(const void* p);

}  // namespace fcdp
