// update_f32c.cu -- instantiations of the fused row-update kernel: TS=float, TF=float, l64=N - 2.
#include "update.cuh"

namespace pt {
namespace {
#define PT_ENTRY(N, J) {0, N - 2, N, J, &launch_update<float, float, N, J, N - 2>, &occupancy_update<float, float, N, J, N - 2>},
const UpdateKernel kTable[] = {PT_NJ_LIST_N45(PT_ENTRY)};
#undef PT_ENTRY
}  // namespace
const UpdateKernel* update_kernels_f32c(int* count) {
    *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
    return kTable;
}
}  // namespace pt
