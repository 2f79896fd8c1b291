// Drop-in forwarder: the reference header cbct/polygon.hpp maps onto cbct_b200/polygon.hpp.
#pragma once
#include "cbct_b200/polygon.hpp"
