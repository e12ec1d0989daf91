// update_f32c2.cu -- instantiations of the fused row-update kernel for order 5: TS=float,
// TF=float, l64 = N - 3 ("F32-C2": every outer level in fp64 except the one next to the
// innermost, so J^3 instead of J^4 fp32 -> fp64 conversions per entry; policy 3).
#include "update.cuh"

namespace pt {
namespace {
#define PT_ENTRY(N, J) {0, N - 3, N, J, &launch_update<float, float, N, J, N - 3>, &occupancy_update<float, float, N, J, N - 3>},
const UpdateKernel kTable[] = {PT_ENTRY(5, 2) PT_ENTRY(5, 3) PT_ENTRY(5, 4) PT_ENTRY(5, 5)};
#undef PT_ENTRY
}  // namespace
const UpdateKernel* update_kernels_f32c2(int* count) {
    *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
    return kTable;
}
}  // namespace pt
