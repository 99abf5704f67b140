#pragma once
// Drop-in path of the reference header glu/jointopt.hpp; everything is declared in
// glu_b200.hpp (same names and signatures).
#include "glu/glu_b200.hpp"
