#pragma once
// Drop-in path of the reference header glu/io.hpp (GLUP parameter files only;
// PNG/PPM image I/O is out of scope); declared in glu_b200.hpp.
#include "glu/glu_b200.hpp"
