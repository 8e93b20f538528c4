// driver.cpp -- see driver.hpp.
#include "driver.hpp"

#include <dlfcn.h>

#include <mutex>

namespace ktc {

const Driver& driver() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        void* lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
        if (!lib) {
            const char* why = dlerror();
            d.error = std::string("cannot load libcuda.so.1 (no NVIDIA driver on this host): ") +
                      (why ? why : "");
            return;
        }
#define KTC_RESOLVE(fn)                                                         \
    d.fn = reinterpret_cast<decltype(d.fn)>(dlsym(lib, KTC_XSTR(fn)));          \
    if (!d.fn) {                                                                \
        d.error = std::string("libcuda.so.1 lacks ") + KTC_XSTR(fn);            \
        return;                                                                 \
    }
        KTC_DRIVER_FUNCS(KTC_RESOLVE)
#undef KTC_RESOLVE
        CUresult rc = d.cuInit(0);
        if (rc != CUDA_SUCCESS) {
            d.error = cu_error_text(rc, "cuInit");
            return;
        }
        d.ok = true;
    });
    return d;
}

std::string cu_error_text(CUresult rc, const char* what) {
    const Driver& d = driver();
    const char* name = nullptr;
    const char* desc = nullptr;
    if (d.cuGetErrorName) d.cuGetErrorName(rc, &name);
    if (d.cuGetErrorString) d.cuGetErrorString(rc, &desc);
    std::string out = std::string(what) + " failed: ";
    out += name ? name : ("CUresult " + std::to_string(static_cast<int>(rc)));
    if (desc) out += std::string(" (") + desc + ")";
    return out;
}

}  // namespace ktc
