// isolate.cpp -- isolated evaluation backend: the parent-side proxy and the
// worker's serve loop (see isolate.hpp).
//
// Wire format: frames of [u32 type][u64 length][payload] over two pipes.
// Requests carry the ktc_request fields (strings length-prefixed); replies
// carry the ktc_result struct verbatim (same binary on both ends).
#include "isolate.hpp"

#include <dlfcn.h>
#include <poll.h>
#include <signal.h>
#include <spawn.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "core.hpp"

extern char** environ;

namespace ktc {

bool g_isolated_worker = false;

namespace {

enum Msg : uint32_t {
    kOpen = 1,
    kEval,
    kPrefetch,
    kSetRef,
    kReadOut,
    kReadRef,
    kBegin,
    kClose,
    kReply,
};

// ------------------------------------------------------------ serialization
struct Writer {
    std::string b;
    void raw(const void* p, size_t n) { b.append(static_cast<const char*>(p), n); }
    void u32(uint32_t v) { raw(&v, 4); }
    void u64(uint64_t v) { raw(&v, 8); }
    void i64(int64_t v) { raw(&v, 8); }
    void f64(double v) { raw(&v, 8); }
    void str(const char* s) {
        const size_t n = s ? std::strlen(s) : 0;
        u64(n);
        raw(s, n);
    }
    void blob(const void* p, size_t n) {
        u64(n);
        raw(p, n);
    }
};

struct Reader {
    const char* p;
    const char* end;
    explicit Reader(const std::string& s) : p(s.data()), end(s.data() + s.size()) {}
    void raw(void* dst, size_t n) {
        if (size_t(end - p) < n) throw std::runtime_error("isolated backend: truncated frame");
        std::memcpy(dst, p, n);
        p += n;
    }
    uint32_t u32() { uint32_t v; raw(&v, 4); return v; }
    uint64_t u64() { uint64_t v; raw(&v, 8); return v; }
    int64_t i64() { int64_t v; raw(&v, 8); return v; }
    double f64() { double v; raw(&v, 8); return v; }
    std::string str() {
        const uint64_t n = u64();
        std::string s(n, '\0');
        raw(s.data(), n);
        return s;
    }
};

void put_request(Writer& w, const ktc_request& r) {
    w.str(r.kernel_name);
    w.str(r.source_ref);
    w.u32(uint32_t(r.n_params));
    for (int i = 0; i < r.n_params; ++i) {
        w.str(r.param_names[i]);
        w.i64(r.param_values[i]);
    }
    w.u32(uint32_t(r.ndim));
    for (int d = 0; d < 3; ++d) {
        w.u64(r.global[d]);
        w.u64(r.local[d]);
    }
    w.u32(uint32_t(r.n_args));
    for (int i = 0; i < r.n_args; ++i) {
        w.u32(uint32_t(r.args[i].role));
        w.u32(uint32_t(r.args[i].type));
        w.u64(r.args[i].length);
        w.f64(r.args[i].value);
        w.str(r.args[i].fill);
    }
    w.str(r.device_name);
    w.u32(uint32_t(r.repetitions));
    w.u32(uint32_t(r.want_outputs));
}

// A request decoded into owned storage (the ktc_request points into it).
struct OwnedRequest {
    std::string kernel, source, device;
    std::vector<std::string> names, fills;
    std::vector<const char*> name_ptrs;
    std::vector<long long> values;
    std::vector<ktc_arg> args;
    ktc_request req{};
};

std::unique_ptr<OwnedRequest> get_request(Reader& rd) {
    auto o = std::make_unique<OwnedRequest>();
    o->kernel = rd.str();
    o->source = rd.str();
    const uint32_t np = rd.u32();
    for (uint32_t i = 0; i < np; ++i) {
        o->names.push_back(rd.str());
        o->values.push_back(rd.i64());
    }
    for (const std::string& n : o->names) o->name_ptrs.push_back(n.c_str());
    ktc_request& r = o->req;
    r.ndim = int(rd.u32());
    for (int d = 0; d < 3; ++d) {
        r.global[d] = rd.u64();
        r.local[d] = rd.u64();
    }
    const uint32_t na = rd.u32();
    o->args.resize(na);
    o->fills.resize(na);
    for (uint32_t i = 0; i < na; ++i) {
        o->args[i].role = int(rd.u32());
        o->args[i].type = int(rd.u32());
        o->args[i].length = rd.u64();
        o->args[i].value = rd.f64();
        o->fills[i] = rd.str();
    }
    for (uint32_t i = 0; i < na; ++i) o->args[i].fill = o->fills[i].c_str();
    o->device = rd.str();
    r.repetitions = int(rd.u32());
    r.want_outputs = int(rd.u32());
    r.kernel_name = o->kernel.c_str();
    r.source_ref = o->source.c_str();
    r.n_params = int(np);
    r.param_names = o->name_ptrs.data();
    r.param_values = o->values.data();
    r.n_args = int(na);
    r.args = o->args.data();
    r.device_name = o->device.c_str();
    return o;
}

// ------------------------------------------------------------------ frames
bool write_all(int fd, const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    while (n) {
        const ssize_t k = ::write(fd, c, n);
        if (k < 0 && errno == EINTR) continue;
        if (k <= 0) return false;
        c += k;
        n -= size_t(k);
    }
    return true;
}

bool send_frame(int fd, uint32_t type, const std::string& payload) {
    const uint64_t n = payload.size();
    return write_all(fd, &type, 4) && write_all(fd, &n, 8) && write_all(fd, payload.data(), n);
}

// Reads exactly n bytes; `deadline` < 0 waits forever.  false on EOF,
// error or timeout (*timed_out set).
bool read_all(int fd, void* p, size_t n, double deadline_s, bool* timed_out) {
    char* c = static_cast<char*>(p);
    const auto t0 = std::chrono::steady_clock::now();
    while (n) {
        if (deadline_s >= 0) {
            const double el =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (el >= deadline_s) {
                if (timed_out) *timed_out = true;
                return false;
            }
            pollfd pf{fd, POLLIN, 0};
            const int ms = int(std::min(1000.0, (deadline_s - el) * 1e3)) + 1;
            const int pr = ::poll(&pf, 1, ms);
            if (pr < 0 && errno == EINTR) continue;
            if (pr <= 0) continue;
        }
        const ssize_t k = ::read(fd, c, n);
        if (k < 0 && errno == EINTR) continue;
        if (k <= 0) return false;
        c += k;
        n -= size_t(k);
    }
    return true;
}

bool recv_frame(int fd, uint32_t* type, std::string* payload, double deadline_s = -1,
                bool* timed_out = nullptr) {
    uint64_t n = 0;
    if (!read_all(fd, type, 4, deadline_s, timed_out) || !read_all(fd, &n, 8, deadline_s, timed_out))
        return false;
    payload->assign(n, '\0');
    return read_all(fd, payload->data(), n, deadline_s, timed_out);
}

std::string worker_binary() {
    if (const char* e = std::getenv("KTC_WORKER_BIN")) return e;
    Dl_info info{};
    if (dladdr(reinterpret_cast<void*>(&remote_open), &info) && info.dli_fname) {
        std::string lib = info.dli_fname;
        const size_t slash = lib.rfind('/');
        return (slash == std::string::npos ? std::string(".") : lib.substr(0, slash)) + "/ktc-worker";
    }
    return "ktc-worker";
}

// Generous parent-side limit for one reply: the worker's own watchdog
// (KTC_WATCHDOG_S per launch batch) normally answers long before.
double reply_limit_s() {
    const char* e = std::getenv("KTC_WATCHDOG_S");
    const double wd = e && std::atof(e) > 0 ? std::atof(e) : 30.0;
    return 4.0 * wd + 120.0;
}

}  // namespace

// ================================================================= parent
struct RemoteBackend {
    int ordinal = 0;
    ktc_backend_options opts{};
    std::string cache_dir;
    pid_t pid = -1;
    int to = -1, from = -1;
    size_t prefetch_depth = 0;
    std::string name;
    std::string bound_ref;  // SETREF frame payload to replay after a respawn
    std::string last_status;

    bool alive() const { return pid > 0; }

    void reap(bool kill_it) {
        if (pid <= 0) return;
        if (kill_it) ::kill(pid, SIGKILL);
        int status = 0;
        for (int i = 0; i < 200; ++i) {  // up to ~10 s for an orderly exit
            const pid_t r = ::waitpid(pid, &status, WNOHANG);
            if (r == pid || r < 0) break;
            if (i == 100) ::kill(pid, SIGKILL);
            ::usleep(50000);
        }
        if (WIFSIGNALED(status)) last_status = "signal " + std::to_string(WTERMSIG(status));
        else last_status = "exit " + std::to_string(WEXITSTATUS(status));
        ::close(to);
        ::close(from);
        to = from = -1;
        pid = -1;
    }

    bool spawn(std::string* err) {
        int down[2], up[2];
        if (::pipe(down) || ::pipe(up)) {
            *err = "pipe() failed";
            return false;
        }
        posix_spawn_file_actions_t fa;
        posix_spawn_file_actions_init(&fa);
        posix_spawn_file_actions_adddup2(&fa, down[0], 0);
        posix_spawn_file_actions_adddup2(&fa, up[1], 1);
        posix_spawn_file_actions_addclose(&fa, down[1]);
        posix_spawn_file_actions_addclose(&fa, up[0]);
        const std::string bin = worker_binary();
        char* argv[] = {const_cast<char*>(bin.c_str()), nullptr};
        const int rc = posix_spawn(&pid, bin.c_str(), &fa, nullptr, argv, environ);
        posix_spawn_file_actions_destroy(&fa);
        ::close(down[0]);
        ::close(up[1]);
        to = down[1];
        from = up[0];
        if (rc != 0) {
            ::close(to);
            ::close(from);
            pid = -1;
            *err = "cannot start the evaluation worker " + bin + ": " + std::strerror(rc);
            return false;
        }
        Writer w;
        w.u32(uint32_t(ordinal));
        w.raw(&opts, sizeof opts);
        w.str(cache_dir.c_str());
        uint32_t type = 0;
        std::string reply;
        if (!send_frame(to, kOpen, w.b) || !recv_frame(from, &type, &reply, 600.0)) {
            reap(true);
            *err = "evaluation worker did not start (" + last_status + ")";
            return false;
        }
        Reader rd(reply);
        const int st = int(rd.u32());
        name = rd.str();
        prefetch_depth = size_t(rd.u64());
        if (st != KTC_OK) {
            *err = rd.str();
            reap(false);
            return false;
        }
        if (!bound_ref.empty()) {  // re-bind the reference in the fresh worker
            if (!send_frame(to, kSetRef, bound_ref) || !recv_frame(from, &type, &reply, 600.0)) {
                reap(true);
                *err = "evaluation worker lost while re-binding the reference";
                return false;
            }
        }
        return true;
    }

    bool ensure(std::string* err) { return alive() || spawn(err); }

    // One request/reply round trip; on a dead or hung worker, kills it and
    // reports why in *why.
    bool call(uint32_t type, const std::string& payload, std::string* reply, std::string* why) {
        if (!ensure(why)) return false;
        uint32_t rtype = 0;
        bool timed_out = false;
        if (!send_frame(to, type, payload) ||
            !recv_frame(from, &rtype, reply, reply_limit_s(), &timed_out)) {
            reap(true);
            *why = timed_out ? "evaluation worker timed out and was killed"
                             : "evaluation worker died (" + last_status + ")";
            return false;
        }
        return true;
    }
};

RemoteBackend* remote_open(int ordinal, const ktc_backend_options& opts, const std::string& cache_dir,
                           std::string* name, std::string* error) {
    auto rb = std::make_unique<RemoteBackend>();
    rb->ordinal = ordinal;
    rb->opts = opts;
    rb->opts.cache_dir = nullptr;
    rb->opts.isolate = 0;
    rb->cache_dir = cache_dir;
    if (!rb->spawn(error)) return nullptr;
    *name = rb->name;
    return rb.release();
}

void remote_close(RemoteBackend* rb) {
    if (!rb) return;
    if (rb->alive()) {
        send_frame(rb->to, kClose, "");
        rb->reap(false);
    }
    delete rb;
}

int remote_evaluate(RemoteBackend* rb, const ktc_request* req, ktc_result* out) {
    std::memset(out, 0, sizeof *out);
    Writer w;
    put_request(w, *req);
    std::string reply, why;
    if (!rb->call(kEval, w.b, &reply, &why)) {
        // The configuration took its worker down: a per-configuration
        // failure, never a harness error (backend.hpp:21-31).
        out->status = KTC_STATUS_RUNTIME_ERROR;
        std::snprintf(out->message, sizeof out->message, "%s", why.c_str());
        return KTC_OK;
    }
    Reader rd(reply);
    const int rc = int(rd.u32());
    rd.raw(out, sizeof *out);
    const uint32_t exiting = rd.u32();
    if (exiting) rb->reap(false);  // the worker's context is poisoned; it exits
    if (rc != KTC_OK) set_error(rd.str());
    return rc;
}

int remote_prefetch(RemoteBackend* rb, const ktc_request* req) {
    std::string err;
    if (!rb->ensure(&err)) return KTC_OK;  // a hint only
    Writer w;
    put_request(w, *req);
    if (!send_frame(rb->to, kPrefetch, w.b)) rb->reap(true);
    return KTC_OK;
}

size_t remote_prefetch_depth(RemoteBackend* rb) { return rb->prefetch_depth; }

int remote_begin_search(RemoteBackend* rb) {
    std::string err;
    if (!rb->ensure(&err)) {
        set_error(err);
        return KTC_ERR_CUDA;
    }
    if (!send_frame(rb->to, kBegin, "")) rb->reap(true);
    return KTC_OK;
}

int remote_set_reference(RemoteBackend* rb, const ktc_request* req, int n_buffers,
                         const void* const* buffers, const size_t* lengths, const int* types) {
    Writer w;
    put_request(w, *req);
    w.u32(uint32_t(n_buffers));
    for (int k = 0; k < n_buffers; ++k) {
        w.u64(lengths[k]);
        w.u32(uint32_t(types[k]));
        w.blob(buffers[k], lengths[k] * 4);
    }
    std::string reply, why;
    if (!rb->call(kSetRef, w.b, &reply, &why)) {
        set_error(why);
        return KTC_ERR_CUDA;
    }
    Reader rd(reply);
    const int rc = int(rd.u32());
    if (rc != KTC_OK) {
        set_error(rd.str());
        return rc;
    }
    rb->bound_ref = std::move(w.b);
    return KTC_OK;
}

int remote_read_output(RemoteBackend* rb, int index, void* dst, size_t bytes) {
    Writer w;
    w.u32(uint32_t(index));
    w.u64(bytes);
    std::string reply, why;
    if (!rb->call(kReadOut, w.b, &reply, &why)) {
        set_error(why);
        return KTC_ERR_CUDA;
    }
    Reader rd(reply);
    const int rc = int(rd.u32());
    const std::string data = rd.str();
    if (rc != KTC_OK) {
        set_error(data);
        return rc;
    }
    std::memcpy(dst, data.data(), std::min(bytes, data.size()));
    return KTC_OK;
}

int remote_read_reference(RemoteBackend* rb, const ktc_request* req, int index, void* dst,
                          size_t bytes, char digest_hex[17]) {
    Writer w;
    put_request(w, *req);
    w.u32(uint32_t(index));
    w.u64(bytes);
    std::string reply, why;
    if (!rb->call(kReadRef, w.b, &reply, &why)) {
        set_error(why);
        return KTC_ERR_CUDA;
    }
    Reader rd(reply);
    const int rc = int(rd.u32());
    const std::string data = rd.str();
    if (rc != KTC_OK) {
        set_error(data);
        return rc;
    }
    std::memcpy(dst, data.data(), std::min(bytes, data.size()));
    const std::string dig = rd.str();
    if (digest_hex) std::snprintf(digest_hex, 17, "%s", dig.c_str());
    return KTC_OK;
}

}  // namespace ktc

// ================================================================= worker
extern "C" int ktc_worker_serve(int in_fd, int out_fd) {
    using namespace ktc;
    g_isolated_worker = true;
    ktc_backend* be = nullptr;
    for (;;) {
        uint32_t type = 0;
        std::string payload;
        if (!recv_frame(in_fd, &type, &payload)) break;  // parent went away
        Reader rd(payload);
        Writer w;
        try {
            if (type == kOpen) {
                const int ordinal = int(rd.u32());
                ktc_backend_options o{};
                rd.raw(&o, sizeof o);
                const std::string dir = rd.str();
                o.cache_dir = dir.empty() ? nullptr : dir.c_str();
                o.isolate = 0;
                const int st = ktc_backend_open(ordinal, &o, &be);
                w.u32(uint32_t(st));
                w.str(st == KTC_OK ? ktc_backend_name(be) : "");
                w.u64(st == KTC_OK ? ktc_backend_prefetch_depth(be) : 0);
                w.str(st == KTC_OK ? "" : ktc_last_error(nullptr));
            } else if (type == kEval) {
                auto r = get_request(rd);
                ktc_result res{};
                const int rc = ktc_backend_evaluate(be, &r->req, &res);
                const ktc_ctx* ctx = ktc_backend_ctx(be);
                const bool poisoned = ctx && ctx->sticky;
                w.u32(uint32_t(rc));
                w.raw(&res, sizeof res);
                w.u32(poisoned ? 1u : 0u);
                w.str(rc == KTC_OK ? "" : ktc_last_error(nullptr));
                send_frame(out_fd, kReply, w.b);
                // A poisoned context cannot be recovered in this process:
                // leave without touching the driver again.
                if (poisoned) ::_exit(0);
                continue;
            } else if (type == kPrefetch) {
                auto r = get_request(rd);
                ktc_backend_prefetch(be, &r->req);
                continue;
            } else if (type == kBegin) {
                ktc_backend_begin_search(be);
                continue;
            } else if (type == kSetRef) {
                auto r = get_request(rd);
                const uint32_t n = rd.u32();
                std::vector<std::string> bufs(n);
                std::vector<const void*> ptrs(n);
                std::vector<size_t> lens(n);
                std::vector<int> types(n);
                for (uint32_t k = 0; k < n; ++k) {
                    lens[k] = rd.u64();
                    types[k] = int(rd.u32());
                    bufs[k] = rd.str();
                    ptrs[k] = bufs[k].data();
                }
                const int rc = ktc_backend_set_reference(be, &r->req, int(n), ptrs.data(),
                                                         lens.data(), types.data());
                w.u32(uint32_t(rc));
                w.str(rc == KTC_OK ? "" : ktc_last_error(nullptr));
            } else if (type == kReadOut) {
                const int index = int(rd.u32());
                const uint64_t bytes = rd.u64();
                std::string data(bytes, '\0');
                const int rc = ktc_backend_read_output(be, index, data.data(), bytes);
                w.u32(uint32_t(rc));
                if (rc == KTC_OK) w.blob(data.data(), data.size());
                else w.str(ktc_last_error(nullptr));
            } else if (type == kReadRef) {
                auto r = get_request(rd);
                const int index = int(rd.u32());
                const uint64_t bytes = rd.u64();
                std::string data(bytes, '\0');
                char dig[17] = {0};
                const int rc =
                    ktc_backend_read_reference(be, &r->req, index, data.data(), bytes, dig);
                if (rc == KTC_OK) {
                    w.u32(0);
                    w.blob(data.data(), data.size());
                    w.str(dig);
                } else {
                    w.u32(uint32_t(rc));
                    w.str(ktc_last_error(nullptr));
                }
            } else if (type == kClose) {
                break;
            } else {
                w.u32(uint32_t(KTC_ERR_INVALID));
                w.str("isolated backend: unknown message");
            }
        } catch (const std::exception& e) {
            w.b.clear();
            w.u32(uint32_t(KTC_ERR_INVALID));
            w.str(e.what());
        }
        if (!send_frame(out_fd, kReply, w.b)) break;
    }
    if (be) ktc_backend_close(be);
    return 0;
}
