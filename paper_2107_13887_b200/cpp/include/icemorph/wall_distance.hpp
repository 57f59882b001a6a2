// icemorph/wall_distance.hpp — forwarding header: the reference's per-module include
// (proj/include/icemorph/wall_distance.hpp) resolves to the B200 library's single public
// header, so a reference caller's #include "icemorph/wall_distance.hpp" compiles unchanged.
#pragma once
#include "icemorph/icemorph.hpp"
