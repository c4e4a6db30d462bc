// Umbrella header (reference: spmmkit/spmmkit.hpp) for the B200 implementation.
#pragma once
#include "spmmkit/b200.hpp"
#include "spmmkit/mm_io.hpp"
