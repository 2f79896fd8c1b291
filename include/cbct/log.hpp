// Drop-in forwarder: the reference header cbct/log.hpp maps onto cbct_b200/log.hpp.
#pragma once
#include "cbct_b200/log.hpp"
