// Drop-in: the reference header lowrank/sketch.hpp resolved to the B200 implementation.
#pragma once
#include "lowrank_b200/lowrank.hpp"
