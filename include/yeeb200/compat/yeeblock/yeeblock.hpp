// Drop-in umbrella: with -I include/yeeb200/compat, reference code written
// against namespace yeeblock (/root/reference/proj/include/yeeblock) compiles
// unchanged against the B200 shim and links libyeeb200.so.
#pragma once
#include "../../yeeblock.hpp"

namespace yeeblock = yeeb200;
