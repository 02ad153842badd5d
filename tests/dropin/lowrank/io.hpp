// Drop-in: lowrank/io.hpp (MatrixMarket / binary matrices / results CSV) is host file IO
// off the B200 path; the reference header is compiled in place over the drop-in types,
// so a reference user's readers and writers work unchanged.
#pragma once
#include "lowrank_b200/lowrank.hpp"
#include REF_HEADER(io)
