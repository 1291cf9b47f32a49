// Reference header name (proj/include/nls2d/integrators.hpp); the GPU path declares
// everything in mb4cu_api.hpp.
#pragma once

#include "nls2d/mb4cu_api.hpp"
