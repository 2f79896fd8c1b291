// Drop-in forwarder: the reference header cbct/vec.hpp maps onto the GPU-backed API.
#pragma once
#include "cbct_b200/cbct.hpp"
