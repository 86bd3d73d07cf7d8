// Forwarding header: reference clients that include "drot/matrix.hpp"
// (proj/core/include/drot/matrix.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
