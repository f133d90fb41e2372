// tcgen05 tensor-core full search (B in {4, 8}) -- see DESIGN.md.  Placeholder
// dispatcher until the UMMA kernel lands: reports "not handled" so the exact
// CUDA-core path runs.
#include "mns_common.cuh"

namespace mns {
int full_search_tc(const uint8_t *, int, int, int, int, int, int, int, const uint16_t *, const int32_t *,
                   const long long *, long long, unsigned long long *, cudaStream_t, bool *handled) {
    *handled = false;
    return 0;
}
}  // namespace mns
