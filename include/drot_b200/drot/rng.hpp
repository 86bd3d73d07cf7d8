// Forwarding header: reference clients that include "drot/rng.hpp"
// (proj/core/include/drot/rng.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
