// Compatibility include: the whole libdelta API lives in deltasim.hpp.
#pragma once
#include "deltasim/deltasim.hpp"
