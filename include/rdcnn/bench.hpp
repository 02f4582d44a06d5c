// Drop-in header name of the reference API (proj/include/rdcnn/bench.hpp);
// the implementation for the cuda backend lives in cuda_api.hpp.
#pragma once
#include "rdcnn/cuda_api.hpp"
