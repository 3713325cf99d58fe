// ib_b200/ib/ib.hpp -- overlay of the reference's umbrella header ib/ib.hpp.
#pragma once

#include "grid.hpp"
#include "interpolate.hpp"
#include "kernel.hpp"
#include "reduce.hpp"
#include "sort.hpp"
#include "spread.hpp"
#include "stats.hpp"
