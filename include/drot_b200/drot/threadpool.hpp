// Forwarding header: reference clients that include "drot/threadpool.hpp"
// (proj/core/include/drot/threadpool.hpp) compile unchanged with -I include/drot_b200.
#pragma once
#include "../drot.hpp"
