// Forwarding header: reference clients that include "drot/probgen.hpp"
// (proj/core/include/drot/probgen.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
