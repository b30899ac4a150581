// Drop-in for the reference header proj/include/eigmod/locate.hpp: the B200
// implementation declares the whole hot-path API in one header (the location
// vector entry is eigmod::locate_update).
#pragma once
#include "eigmod_b200/eigmod.hpp"
