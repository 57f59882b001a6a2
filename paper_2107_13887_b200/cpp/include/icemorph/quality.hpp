// icemorph/quality.hpp — forwarding header: the reference's per-module include
// (proj/include/icemorph/quality.hpp) resolves to the B200 library's single public
// header, so a reference caller's #include "icemorph/quality.hpp" compiles unchanged.
#pragma once
#include "icemorph/icemorph.hpp"
