// AMG setup on the device: the reference's coarsening
// (amg.cpp:172-227) with the sparse algebra on the GPU and the greedy
// aggregation passes on the host; bit-identical to amg_setup (host).
#pragma once

#include "../host/setup.hpp"

namespace irkb {

Hierarchy amg_setup_device(const Csr& A, const AmgParams& p, int device);

}  // namespace irkb
