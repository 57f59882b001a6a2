// icemorph/pipeline.hpp — forwarding header: the reference's per-module include
// (proj/include/icemorph/pipeline.hpp) resolves to the B200 library's single public
// header, so a reference caller's #include "icemorph/pipeline.hpp" compiles unchanged.
#pragma once
#include "icemorph/icemorph.hpp"
