// sample.cu -- posterior sampling: placeholder until the sampling path lands.
#include "love_internal.h"

namespace love {

void build_sampling_cache(Cache& c, cudaStream_t s) {
    (void)c;
    (void)s;
    throw LoveError{LOVE_ERR_ARG, "k_sample > 0 is not implemented yet"};
}

template <typename V>
void launch_sample(const Cache& c, const double* Xs, int64_t t, int64_t ns, uint64_t seed, const double* zeta,
                   V* out, cudaStream_t s) {
    throw LoveError{LOVE_ERR_STATE, "sampling not implemented yet"};
}

template void launch_sample<float>(const Cache&, const double*, int64_t, int64_t, uint64_t, const double*, float*,
                                   cudaStream_t);
template void launch_sample<double>(const Cache&, const double*, int64_t, int64_t, uint64_t, const double*,
                                    double*, cudaStream_t);

}  // namespace love
