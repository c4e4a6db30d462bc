// Forwarding header: spmmkit/partition.hpp of the reference API (proj/include/spmmkit),
// served by the B200 implementation in b200.hpp.
#pragma once
#include "spmmkit/b200.hpp"
