// ib_b200/ib.hpp -- one-include form of the drop-in (include/ib_b200/ib/).
//
// Two ways to switch a reference caller to the B200:
//  * one include:  #include "ib/ib.hpp"  ->  #include "ib_b200/ib.hpp";
//  * no source change at all: put include/ib_b200 AHEAD of the reference's
//    include directory (-I include/ib_b200 -I include -I <reference>/include):
//    every "ib/<name>.hpp" the caller (or the reference's own bench/verify
//    headers) includes then resolves to the overlay of the same name, and
//    the caller links libibcuda.so.
#pragma once

#include "ib/ib.hpp"
