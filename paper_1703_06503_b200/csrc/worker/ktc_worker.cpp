// ktc-worker -- one isolated evaluation backend (csrc/isolate.cpp): requests
// on stdin, replies on stdout.  Started by ktc_backend_open when
// ktc_backend_options.isolate is set; exits when its CUDA context is lost.
#include "ktc.h"

int main() { return ktc_worker_serve(0, 1); }
