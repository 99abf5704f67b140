#pragma once
// Drop-in path of the reference header glu/image.hpp; everything is declared in
// glu_b200.hpp (same names and signatures).
#include "glu/glu_b200.hpp"
