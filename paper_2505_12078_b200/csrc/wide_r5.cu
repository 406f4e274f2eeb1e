// k_T_wide instantiations with 5 row block(s) per lane (wide_impl.cuh)
#include "wide_impl.cuh"

namespace spock {
SPOCK_WIDE_TU(5)
}  // namespace spock
