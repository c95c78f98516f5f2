// assign_tc.cu -- tcgen05/TMEM 3xTF32 assignment engine (placeholder until the
// tensor-core kernel lands; the runtime only selects it when tc_supported()).
#include <stdio.h>
#include <stdlib.h>

#include "aakm_dev.cuh"

namespace aakm {

float tau_gamma_tc(int d) { return 4.0f * (3.0f * 9.5367432e-7f + (3.0f * d / 8.0f + 8.0f) * 2.3841858e-7f); }

void setup_tc() {}

bool tc_supported(int d, int K) { (void)d; (void)K; return false; }

void launch_assign_tc(const Dev& d, const GEval& g, cudaStream_t s) {
    (void)d; (void)g; (void)s;
    fprintf(stderr, "aakm: tensor-core assignment engine not built\n");
    abort();
}

}  // namespace aakm
