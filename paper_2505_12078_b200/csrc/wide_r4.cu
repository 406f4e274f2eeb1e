// k_T_wide instantiations with 4 row block(s) per lane (wide_impl.cuh)
#include "wide_impl.cuh"

namespace spock {
SPOCK_WIDE_TU(4)
}  // namespace spock
