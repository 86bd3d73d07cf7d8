// Forwarding header: reference clients that include "drot/drot.hpp"
// (proj/core/include/drot/drot.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
