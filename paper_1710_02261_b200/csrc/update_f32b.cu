// update_f32b.cu -- instantiations of the fused row-update kernel: TS=float, TF=float, LAST64=true.
#include "update.cuh"

namespace pt {
namespace {
#define PT_ENTRY(N, J) {0, 1, N, J, &launch_update<float, float, N, J, true>, &occupancy_update<float, float, N, J, true>},
const UpdateKernel kTable[] = {PT_NJ_LIST(PT_ENTRY)};
#undef PT_ENTRY
}  // namespace
const UpdateKernel* update_kernels_f32b(int* count) {
    *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
    return kTable;
}
}  // namespace pt
