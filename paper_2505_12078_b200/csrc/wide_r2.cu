// k_T_wide instantiations with 2 row block(s) per lane (wide_impl.cuh)
#include "wide_impl.cuh"

namespace spock {
SPOCK_WIDE_TU(2)
}  // namespace spock
