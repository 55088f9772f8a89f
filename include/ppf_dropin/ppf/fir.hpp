// Drop-in shim: reference callers that #include "ppf/fir.hpp" get the B200
// implementation in namespace ppf (include/ppf_gpu/ppf.hpp over libppfg.so).
#pragma once
#ifndef PPF_GPU_NS
#define PPF_GPU_NS ppf
#endif
#include "ppf_gpu/ppf.hpp"
