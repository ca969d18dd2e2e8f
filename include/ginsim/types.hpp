// ginsim/types.hpp -- the reference's header name for the core value types
// (proj/core/include/ginsim/types.hpp: SignalOp, CompletionAction, Team,
// team_translate, Window).  Here they live in runtime.hpp with the rest of the
// reference-shaped C++ layer; this header lets reference sources that include
// it by name compile unchanged.
#pragma once

#include "ginsim/runtime.hpp"
