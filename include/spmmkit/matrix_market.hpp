// Forwarding header: spmmkit/matrix_market.hpp of the reference API.
#pragma once
#include "spmmkit/mm_io.hpp"
