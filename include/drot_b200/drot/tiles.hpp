// Forwarding header: reference clients that include "drot/tiles.hpp"
// (proj/core/include/drot/tiles.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
