// Forwarding header: reference clients that include "drot/errors.hpp"
// (proj/core/include/drot/errors.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
