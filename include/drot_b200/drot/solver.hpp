// Forwarding header: reference clients that include "drot/solver.hpp"
// (proj/core/include/drot/solver.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
