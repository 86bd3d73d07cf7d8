// Forwarding header: reference clients that include "drot/fused.hpp"
// (proj/core/include/drot/fused.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
