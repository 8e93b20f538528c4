// isolate.hpp -- process isolation of the evaluation backend.
//
// A CUDA context that took a sticky fault (illegal address, trap, ...) can
// never be used again by its process: the driver refuses even a fresh
// primary context (tools/fault_recovery_probe.cpp, measured on the B200).
// The reference isolates every evaluation in a subprocess with a
// timeout-and-kill (external.hpp:278-286,394-411).  Here an *isolated*
// backend (ktc_backend_options.isolate) forwards every call to one
// persistent worker process per device (ktc-worker, the same libktc behind
// a pipe), so the compile pool, inputs, device reference and modules stay
// warm across evaluations; when a configuration faults or hangs the worker
// reports the runtime_error and exits (or is killed), and the next request
// starts a fresh worker that rebuilds the inputs and re-binds the reference.
#pragma once

#include <cstddef>
#include <string>

#include "ktc.h"

namespace ktc {

struct RemoteBackend;

RemoteBackend* remote_open(int ordinal, const ktc_backend_options& opts, const std::string& cache_dir,
                           std::string* name, std::string* error);
void remote_close(RemoteBackend* rb);
int remote_evaluate(RemoteBackend* rb, const ktc_request* req, ktc_result* out);
int remote_prefetch(RemoteBackend* rb, const ktc_request* req);
size_t remote_prefetch_depth(RemoteBackend* rb);
int remote_begin_search(RemoteBackend* rb);
int remote_set_reference(RemoteBackend* rb, const ktc_request* req, int n_buffers,
                         const void* const* buffers, const size_t* lengths, const int* types);
int remote_read_output(RemoteBackend* rb, int index, void* dst, size_t bytes);
int remote_read_reference(RemoteBackend* rb, const ktc_request* req, int index, void* dst,
                          size_t bytes, char digest_hex[17]);

// Set in the worker process: a sticky fault is reported and the context left
// alone (the worker exits) instead of an in-process reset attempt.
extern bool g_isolated_worker;

}  // namespace ktc
