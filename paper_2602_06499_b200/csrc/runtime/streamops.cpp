#include "runtime/streamops.hpp"

#include <mutex>
#include <stdexcept>
#include <string>

#include "capi_util.hpp"

namespace fcdp {
namespace {

// CUresult cuStreamWaitValue32(CUstream, CUdeviceptr, cuuint32_t, unsigned int)
using WaitFn = int (*)(cudaStream_t, unsigned long long, std::uint32_t, unsigned int);
using WriteFn = int (*)(cudaStream_t, unsigned long long, std::uint32_t, unsigned int);
constexpr unsigned kWaitGeq = 0x0;      // CU_STREAM_WAIT_VALUE_GEQ
constexpr unsigned kWriteDefault = 0x0; // CU_STREAM_WRITE_VALUE_DEFAULT (with memory barrier)

WaitFn g_wait = nullptr;
WriteFn g_write = nullptr;
std::once_flag g_once;

void resolve() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait = reinterpret_cast<WaitFn>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write = reinterpret_cast<WriteFn>(p);
  });
  if (!g_wait || !g_write) throw CudaError("stream memory operations (cuStreamWaitValue32) unavailable");
}

}  // namespace

bool StreamOps::available() {
  try {
    resolve();
    return true;
  } catch (...) {
    return false;
  }
}

void StreamOps::wait_geq(cudaStream_t s, const volatile std::uint32_t* flag, std::uint32_t value) {
  resolve();
  const int rc = g_wait(s, reinterpret_cast<unsigned long long>(flag), value, kWaitGeq);
  if (rc != 0) throw CudaError("cuStreamWaitValue32 failed (CUresult " + std::to_string(rc) + ")");
}

void StreamOps::write(cudaStream_t s, volatile std::uint32_t* flag, std::uint32_t value) {
  resolve();
  const int rc = g_write(s, reinterpret_cast<unsigned long long>(flag), value, kWriteDefault);
  if (rc != 0) throw CudaError("cuStreamWriteValue32 failed (CUresult " + std::to_string(rc) + ")");
}

}  // namespace fcdp
