// Drop-in header name of the reference API (proj/include/rdcnn/sweep.hpp);
// the implementation for the cuda backend lives in cuda_api.hpp.
#pragma once
#include "rdcnn/cuda_api.hpp"
