// crash_trace.cpp -- KTC_SEGV_TRACE=1: on SIGSEGV/SIGBUS/SIGABRT print the
// native stack (module + offset per frame, for addr2line against the -g
// build) before dying.  Diagnostic only; off unless the variable is set.
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>

namespace {

void on_fatal(int sig) {
    void* frames[64];
    const int n = backtrace(frames, 64);
    char line[512];
    int len = std::snprintf(line, sizeof line, "ktc: fatal signal %d, native stack:\n", sig);
    (void)!write(2, line, size_t(len));
    for (int i = 0; i < n; ++i) {
        Dl_info info{};
        if (dladdr(frames[i], &info) && info.dli_fname) {
            len = std::snprintf(line, sizeof line, "  #%d %s+0x%lx (%s)\n", i, info.dli_fname,
                                (unsigned long)((char*)frames[i] - (char*)info.dli_fbase),
                                info.dli_sname ? info.dli_sname : "?");
        } else {
            len = std::snprintf(line, sizeof line, "  #%d %p\n", i, frames[i]);
        }
        (void)!write(2, line, size_t(len));
    }
    signal(sig, SIG_DFL);
    raise(sig);
}

struct Installer {
    Installer() {
        const char* e = std::getenv("KTC_SEGV_TRACE");
        if (!e || std::strcmp(e, "0") == 0) return;
        for (int sig : {SIGSEGV, SIGBUS, SIGABRT}) signal(sig, on_fatal);
    }
} installer;

}  // namespace
