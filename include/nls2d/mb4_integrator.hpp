// Reference header name (proj/include/nls2d/mb4_integrator.hpp); the GPU path declares
// everything in mb4cu_api.hpp.
#pragma once

#include "nls2d/mb4cu_api.hpp"
