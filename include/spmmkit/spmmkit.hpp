// Umbrella header (reference: spmmkit/spmmkit.hpp) for the B200 implementation.
#pragma once
#include "spmmkit/b200.hpp"
#include "spmmkit/mm_io.hpp"
// The reference's umbrella also exports its R-MAT test-matrix generator (rmat.hpp). It is
// not on the SpMM path and this tree does not ship one; when a build puts the reference's
// generator on the include path (the reference suites compiled unchanged against these
// headers, tests/cpp/Makefile), the umbrella exports it as the reference's does.
#if __has_include(<spmmkit/rmat.hpp>)
#include <spmmkit/rmat.hpp>
#endif
