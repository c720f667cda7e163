// K2 placeholder: tcgen05 path not built yet.
#include "internal.h"
namespace fw {
bool tc_supported(const CellDims&, int, std::string* why) {
  if (why) *why = "not built";
  return false;
}
int tc_create(Handle&, const fw_cell_desc*) { return FW_ERR_UNSUPPORTED; }
void tc_destroy(Handle&) {}
cudaError_t launch_cell_tc(Handle&, const CellRun&, cudaStream_t, int64_t*) {
  return cudaErrorNotSupported;
}
}  // namespace fw
