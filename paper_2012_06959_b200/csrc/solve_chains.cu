// Lane-chain lockstep executor — placeholder until the scheduler lands.
#include "plan.hpp"
#include "kernels.cuh"

namespace sptrsv {
int plan_fail(int code, const char* msg);
int DevicePlan::build_chains() {
  chains.ready = false;
  return SPTRSV_OK;
}
bool DevicePlan::chains_preferred() const { return false; }
int DevicePlan::solve_chains(const double*, double*, cudaStream_t) {
  return plan_fail(SPTRSV_E_UNSUPPORTED, "chains executor not built");
}
}  // namespace sptrsv
