// Drop-in for the reference header proj/include/eigmod/types.hpp: the B200
// implementation declares the whole hot-path API in one header.
#pragma once
#include "eigmod_b200/eigmod.hpp"
