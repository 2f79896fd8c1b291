// Drop-in forwarder: the reference header cbct/den.hpp maps onto cbct_b200/den.hpp.
#pragma once
#include "cbct_b200/den.hpp"
