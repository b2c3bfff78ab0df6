// types.h -- fixed-width integer types for both the offline build (nvcc/g++)
// and the runtime compiler (NVRTC has no C++ standard library headers).
#pragma once
#if defined(__CUDACC_RTC__)
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#ifndef UINT32_MAX
#define UINT32_MAX 0xffffffffu
#endif
#else
#include <cstdint>
#endif
