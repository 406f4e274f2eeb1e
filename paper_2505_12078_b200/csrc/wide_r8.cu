// k_T_wide instantiations with 8 row block(s) per lane (wide_impl.cuh)
#include "wide_impl.cuh"

namespace spock {
SPOCK_WIDE_TU(8)
}  // namespace spock
