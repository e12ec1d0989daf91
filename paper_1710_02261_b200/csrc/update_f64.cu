// update_f64.cu -- instantiations of the fused row-update kernel: TS=double, TF=double, l64=1.
#include "update.cuh"

namespace pt {
namespace {
#define PT_ENTRY(N, J) {1, 1, N, J, &launch_update<double, double, N, J, 1>, &occupancy_update<double, double, N, J, 1>},
const UpdateKernel kTable[] = {PT_NJ_LIST(PT_ENTRY)};
#undef PT_ENTRY
}  // namespace
const UpdateKernel* update_kernels_f64(int* count) {
    *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
    return kTable;
}
}  // namespace pt
