#include "numa.hpp"

#include <cuda_runtime.h>
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

namespace fcdp {

namespace {

std::string read_line(const std::string& path) {
  std::ifstream f(path);
  std::string s;
  if (f) std::getline(f, s);
  return s;
}

}  // namespace

std::vector<int> parse_cpulist(const std::string& s) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string part;
  while (std::getline(ss, part, ',')) {
    while (!part.empty() && std::isspace(static_cast<unsigned char>(part.back()))) part.pop_back();
    if (part.empty()) continue;
    const auto dash = part.find('-');
    try {
      if (dash == std::string::npos) {
        out.push_back(std::stoi(part));
      } else {
        const int a = std::stoi(part.substr(0, dash)), b = std::stoi(part.substr(dash + 1));
        for (int c = a; c <= b; ++c) out.push_back(c);
      }
    } catch (...) {
      return {};
    }
  }
  return out;
}

int numa_online_nodes() {
  const std::vector<int> nodes = parse_cpulist(read_line("/sys/devices/system/node/has_memory"));
  return nodes.empty() ? 1 : static_cast<int>(nodes.size());
}

int numa_node_of_gpu(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  std::string id(bus);
  for (char& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  const std::string v = read_line("/sys/bus/pci/devices/" + id + "/numa_node");
  try {
    return v.empty() ? -1 : std::stoi(v);
  } catch (...) {
    return -1;
  }
}

std::vector<int> numa_node_cpus(int node) {
  if (node < 0) return {};
  return parse_cpulist(read_line("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist"));
}

bool numa_prefer(void* p, std::size_t bytes, int node) {
  if (node < 0 || node >= 1024 || !p || bytes == 0) return false;
  const long page = sysconf(_SC_PAGESIZE);
  const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(p);
  const std::uintptr_t lo = a & ~static_cast<std::uintptr_t>(page - 1);
  const std::size_t len = bytes + (a - lo);
  unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
  mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
  constexpr int kMpolPreferred = 1;
  return syscall(SYS_mbind, lo, len, kMpolPreferred, mask, 1024ul, 0u) == 0;
}

bool numa_pin_thread(int node) {
  const std::vector<int> cpus = numa_node_cpus(node);
  if (cpus.empty()) return false;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus)
    if (c >= 0 && c < CPU_SETSIZE) CPU_SET(c, &set);
  return sched_setaffinity(0, sizeof(set), &set) == 0;
}

SavedAffinity numa_save_affinity() {
  SavedAffinity a;
  static_assert(sizeof(cpu_set_t) <= sizeof(a.set), "cpu_set_t size");
  cpu_set_t set;
  CPU_ZERO(&set);
  if (sched_getaffinity(0, sizeof(set), &set) == 0) {
    std::memcpy(a.set, &set, sizeof(set));
    a.valid = true;
  }
  return a;
}

void numa_restore_affinity(const SavedAffinity& a) {
  if (!a.valid) return;
  cpu_set_t set;
  std::memcpy(&set, a.set, sizeof(set));
  sched_setaffinity(0, sizeof(set), &set);
}

int numa_node_of_page(const void* p) {
  int node = -1;
  constexpr unsigned long kMpolFNode = 1, kMpolFAddr = 2;
  if (syscall(SYS_get_mempolicy, &node, nullptr, 0ul, p, kMpolFNode | kMpolFAddr) != 0) return -1;
  return node;
}

}  // namespace fcdp
