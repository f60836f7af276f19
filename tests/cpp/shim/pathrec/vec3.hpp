// Include shim: the reference's <pathrec/vec3.hpp> resolves to the B200 engine's C++ mirror
// (include/pathrec_gpu.hpp) in namespace pathrec, so reference callers build unchanged.
#pragma once
#ifndef PATHREC_GPU_NAMESPACE
#define PATHREC_GPU_NAMESPACE pathrec
#endif
#include "pathrec_gpu.hpp"
