// jit.h -- run-time compiled structure classes (jit.cpp, jit_lane.cuh).
#pragma once
#include <string>
#include <vector>

#include "types.h"

namespace oob {

// One structure class: the compiled code words of host.cpp compile_query
// (ncon constraint words, ncode node words, 4 membership words per variable).
struct JitClass {
    const uint32_t* words;
    uint32_t nv, ncon, ncode, nlit;
    int bits = 64;  // value type: 64 = int64 regime, 32 = x32 regime (engine.cuh Ext<int>), 128 = int128
};

// Compiles (or finds in the process-wide cache) every class and returns the
// loaded kernels (cudaKernel_t as launchable function pointers) and their
// register counts; *compile_ms = NVRTC time of the classes' compiles.  With
// load = false only the NVRTC step runs (no device needed).
std::string jit_prepare(const std::vector<JitClass>& classes, std::vector<const void*>& kernels,
                        std::vector<int>& regs, double* compile_ms, bool load = true);

// The generated CUDA source of a class (tests / debugging).
std::string jit_source(const JitClass& c);

}  // namespace oob
