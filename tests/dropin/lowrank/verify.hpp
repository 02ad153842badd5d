// Drop-in: lowrank/verify.hpp is off the B200 path; the reference header is compiled
// in place (its own code over the B200 primitives resolved through this directory).
#pragma once
#include "lowrank_b200/lowrank.hpp"
#include REF_HEADER(verify)
