// Fixed-width integer types for headers shared by the nvcc build and the
// NVRTC-compiled DSL programs (NVRTC has no host standard library).
#pragma once
#ifdef __CUDACC_RTC__
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#endif
