#pragma once
// Drop-in path of the reference header glu/baseline.hpp; declared in glu_b200.hpp.
#include "glu/glu_b200.hpp"
