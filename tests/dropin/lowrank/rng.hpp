// Drop-in: the reference header lowrank/rng.hpp resolved to the B200 implementation.
#pragma once
#include "lowrank_b200/lowrank.hpp"
