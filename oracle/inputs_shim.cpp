// TEST / BASELINE INFRASTRUCTURE: the seeded BASELINE input generator
// (paper_2003_04345_b200/csrc/inputs_host.cpp, host C++) compiled by g++ alone into
// oracle/libinputs.so, so that bench.py's reference arm builds the same V / psi
// arrays as the GPU arm without mapping the product library libmb4cu.so.
// Same source file, same arithmetic: the arrays are bit-identical (tests/test_oracle_pins.py).
#include <cstddef>
#include <string>

#include "mb4cu.h"
#include "mb4cu_internal.hpp"

extern "C" {

int orc_make_inputs(const mb4cu_inputs* spec, int x0, int y0, int lnx, int lny, double* V, double* psi,
                    double* psum) {
    std::string why;
    return mb4cu::make_inputs(spec, x0, y0, lnx, lny, V, psi, psum, why);
}

int orc_scale_state(double* psi, size_t nsites, double s, int threads) {
    return mb4cu::scale_state(psi, nsites, s, threads);
}

}  // extern "C"
