// icemorph/vec.hpp — forwarding header: the reference's per-module include
// (proj/include/icemorph/vec.hpp) resolves to the B200 library's single public
// header, so a reference caller's #include "icemorph/vec.hpp" compiles unchanged.
#pragma once
#include "icemorph/icemorph.hpp"
