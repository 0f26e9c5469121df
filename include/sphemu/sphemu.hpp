// sphemu/sphemu.hpp — umbrella header of the C++ drop-in API.
#pragma once

#include "sphemu/grid.hpp"
#include "sphemu/mpchol.hpp"
#include "sphemu/sht.hpp"
#include "sphemu/stochastic.hpp"
#include "sphemu/trend.hpp"
#include "sphemu/version.hpp"
#include "sphemu/wigner.hpp"
