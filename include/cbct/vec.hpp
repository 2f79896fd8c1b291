// Drop-in forwarder: the reference header cbct/vec.hpp maps onto cbct_b200/vec.hpp.
#pragma once
#include "cbct_b200/vec.hpp"
