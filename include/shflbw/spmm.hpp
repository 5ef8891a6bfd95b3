// spmm.hpp -- forwarding header; the API lives in shflbw/shflbw.hpp
// (same name as the reference header so its includes resolve unchanged).
#pragma once
#include "shflbw/shflbw.hpp"
