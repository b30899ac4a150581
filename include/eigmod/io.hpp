// Drop-in for the reference header proj/include/eigmod/io.hpp: the B200
// implementation declares the whole API in one header.
#pragma once
#include "eigmod_b200/eigmod.hpp"
