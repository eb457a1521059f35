// Drop-in header name of the reference i8t_core (clip.hpp); the declarations
// live in i8t/i8t.hpp.
#pragma once
#include "i8t/i8t.hpp"
