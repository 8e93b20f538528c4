// driver.hpp -- lazily dlopen'ed CUDA driver API.
//
// libktc.so must load (and export every ktc.h symbol) on hosts without a GPU
// driver -- the build container has only the link stub.  The driver entry
// points are therefore resolved at first use from libcuda.so.1; when that
// fails every device call returns KTC_ERR_NO_DRIVER instead of crashing.
#pragma once

#include <cuda.h>

#include <string>

namespace ktc {

#define KTC_STR_(x) #x
#define KTC_XSTR(x) KTC_STR_(x)

// X(symbol): `symbol` is the cuda.h name; macros in cuda.h map it to the
// versioned export (cuMemAlloc -> cuMemAlloc_v2), and KTC_XSTR stringifies
// after that expansion, so dlsym looks up the right versioned symbol.
#define KTC_DRIVER_FUNCS(X)              \
    X(cuInit)                            \
    X(cuDriverGetVersion)                \
    X(cuGetErrorString)                  \
    X(cuGetErrorName)                    \
    X(cuDeviceGetCount)                  \
    X(cuDeviceGet)                       \
    X(cuDeviceGetName)                   \
    X(cuDeviceGetAttribute)              \
    X(cuDeviceTotalMem)                  \
    X(cuDevicePrimaryCtxRetain)          \
    X(cuDevicePrimaryCtxRelease)         \
    X(cuDevicePrimaryCtxReset)           \
    X(cuCtxSetCurrent)                   \
    X(cuCtxSynchronize)                  \
    X(cuStreamCreate)                    \
    X(cuStreamDestroy)                   \
    X(cuStreamSynchronize)               \
    X(cuEventCreate)                     \
    X(cuEventDestroy)                    \
    X(cuEventRecord)                     \
    X(cuEventSynchronize)                \
    X(cuEventQuery)                      \
    X(cuEventElapsedTime)                \
    X(cuMemAlloc)                        \
    X(cuMemFree)                         \
    X(cuMemcpyHtoD)                      \
    X(cuMemcpyDtoH)                      \
    X(cuMemcpyHtoDAsync)                 \
    X(cuMemcpyDtoHAsync)                 \
    X(cuMemcpyDtoDAsync)                 \
    X(cuMemcpy2D)                        \
    X(cuMemsetD32Async)                  \
    X(cuMemHostAlloc)                    \
    X(cuMemFreeHost)                     \
    X(cuModuleLoadData)                  \
    X(cuModuleUnload)                    \
    X(cuModuleGetFunction)               \
    X(cuModuleGetGlobal)                 \
    X(cuFuncSetAttribute)                \
    X(cuFuncGetAttribute)                \
    X(cuLaunchKernel)                    \
    X(cuLaunchKernelEx)                  \
    X(cuTensorMapEncodeTiled)            \
    X(cuOccupancyMaxActiveBlocksPerMultiprocessor)

struct Driver {
#define KTC_DECLARE(fn) decltype(&::fn) fn = nullptr;
    KTC_DRIVER_FUNCS(KTC_DECLARE)
#undef KTC_DECLARE
    bool ok = false;
    std::string error;
};

// Loads libcuda.so.1 and calls cuInit(0) once; thread-safe.
const Driver& driver();

// "cuFoo failed: CUDA_ERROR_X (description)"
std::string cu_error_text(CUresult rc, const char* what);

}  // namespace ktc
