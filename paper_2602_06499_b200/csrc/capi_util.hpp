// Exception firewall for the C ABI: every extern "C" entry point runs its body
// through guarded(), which maps C++ exceptions to FCDP_ERR_* codes and stores
// the message for fcdp_last_error().
#pragma once

#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "fcdp.h"
#include "shardsim/error.hpp"
#include "shardsim/schedule.hpp"

namespace fcdp {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OomError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TimeoutError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);
void check_cuda(cudaError_t e, const char* what);

template <typename F>
int guarded(F&& body) {
  try {
    body();
    return FCDP_OK;
  } catch (const shardsim::ConfigError& e) {
    set_last_error(e.what());
    return FCDP_ERR_CONFIG;
  } catch (const shardsim::ProtocolError& e) {
    set_last_error(e.what());
    return FCDP_ERR_PROTOCOL;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return FCDP_ERR_CUDA;
  } catch (const OomError& e) {
    set_last_error(e.what());
    return FCDP_ERR_OOM;
  } catch (const TimeoutError& e) {
    set_last_error(e.what());
    return FCDP_ERR_TIMEOUT;
  } catch (const std::bad_alloc& e) {
    set_last_error("host allocation failed");
    return FCDP_ERR_OOM;
  } catch (const std::out_of_range& e) {
    set_last_error(std::string("index out of range: ") + e.what());
    return FCDP_ERR_CONFIG;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return FCDP_ERR_CONFIG;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FCDP_ERR_INTERNAL;
  } catch (...) {
    set_last_error("unknown exception");
    return FCDP_ERR_INTERNAL;
  }
}

// Accessors into the opaque control-plane handles (capi_control.cpp).
shardsim::ClusterTopology topo_from_c(const fcdp_topology* t);
shardsim::StrategyPlan plan_from_c(const fcdp_plan* p);
const shardsim::ModelSpec& model_from_c(const fcdp_model* m);
const shardsim::EventProgram& program_from_c(const fcdp_program* p);
std::vector<shardsim::ParamState>& states_from_c(fcdp_states* s);

}  // namespace fcdp
