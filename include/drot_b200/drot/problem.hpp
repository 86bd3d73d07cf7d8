// Forwarding header: reference clients that include "drot/problem.hpp"
// (proj/core/include/drot/problem.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
