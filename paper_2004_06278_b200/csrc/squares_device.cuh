// squares_device.cuh -- the kernels' arithmetic core lives in the public header-only device
// API (include/squares_dev.cuh) so that user kernels and libsquares.so share one definition.
#pragma once
#include "../../include/squares_dev.cuh"
