// Drop-in forwarding header: reference code that includes "yeeblock/probe.hpp"
// compiles against the B200 shim (include/yeeb200/yeeblock.hpp) with
// -I include/yeeb200/compat. See that header for what is mirrored.
#pragma once
#include "yeeblock.hpp"
