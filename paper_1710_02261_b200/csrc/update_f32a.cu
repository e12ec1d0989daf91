// update_f32a.cu -- instantiations of the fused row-update kernel: TS=float, TF=float, l64=0.
#include "update.cuh"

namespace pt {
namespace {
#define PT_ENTRY(N, J) {0, 0, N, J, &launch_update<float, float, N, J, 0>, &occupancy_update<float, float, N, J, 0>},
const UpdateKernel kTable[] = {PT_NJ_LIST(PT_ENTRY)};
#undef PT_ENTRY
}  // namespace
const UpdateKernel* update_kernels_f32a(int* count) {
    *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
    return kTable;
}
}  // namespace pt
