// TT (separable trapezoid footprint) projector pair — placeholder until the
// kernels land; the entry points report "not implemented" loudly.
#include "kernels.hpp"

namespace cvpb {

cudaError_t launch_tt(const TTLaunch&, bool, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace cvpb
