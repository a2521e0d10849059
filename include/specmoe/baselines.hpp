// specmoe/baselines.hpp -- drop-in header name of the reference module; the declarations live in api.hpp.
#pragma once
#include "specmoe/api.hpp"
