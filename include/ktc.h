/*
 * ktc.h -- C ABI of the B200-native evaluation backend for the ktune tuner
 * (the tuner of arXiv 1703.06503 / CLTune, as re-implemented by the
 * reference at proj/include/ktune/).
 *
 * The reference prices configurations through ONE virtual call,
 *     ktune::Backend::evaluate(const EvaluationRequest&)      backend.hpp:72-80
 * made from exactly one site, the evaluator inside run_tuning (tuner.hpp:247).
 * That call is the drop-in boundary.  This header is what a ktune-side
 * `CudaBackend : ktune::Backend` binds: plain C types,
 * plain pointers and sizes, integer status codes, never an exception.
 *
 * Three layers:
 *   1. device primitives  (SURVEY 8(b) "C ABI"): device query, NVRTC
 *      compilation for sm_100a, module load, buffers, timed launch, device
 *      verification against a bound reference;
 *   2. the evaluation backend: ktc_backend_evaluate() takes the exact content
 *      of ktune::EvaluationRequest (backend.hpp:45-55) and returns the exact
 *      content of ktune::EvaluationResult (backend.hpp:57-67) plus the device
 *      verification report;
 *   3. the tuner (ktc_tuner_*): the CLTune-named API (Tuner, AddKernel,
 *      AddParameter, AddConstraint, Mul/DivGlobalSize, Mul/DivLocalSize,
 *      SetReference, AddArgumentInput/Output/Scalar, UseFullSearch,
 *      UseRandomSearch, UseAnnealing, UsePSO, Tune, GetBestResult) over the
 *      native ktune-compatible search layer, with search-space execution
 *      sharded over the GPUs given to it.
 *
 * All functions return KTC_OK (0) on success.  Per-configuration failures
 * are NOT errors of the call: they come back as ktc_result.status
 * (compile_error / runtime_error / missing), mirroring ktune::Status
 * (backend.hpp:21).  The message of the last failing call on a handle is
 * available from ktc_last_error(handle) (thread-local for NULL).
 */
#ifndef KTC_H_
#define KTC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KTC_ABI_VERSION 1

/* Call status codes. */
enum {
    KTC_OK = 0,
    KTC_ERR_INVALID = 1,     /* bad argument / malformed request (ktune::Error) */
    KTC_ERR_NO_DRIVER = 2,   /* libcuda.so.1 absent or cuInit failed            */
    KTC_ERR_NO_DEVICE = 3,   /* ordinal out of range                            */
    KTC_ERR_CUDA = 4,        /* driver API failure outside a configuration      */
    KTC_ERR_NVRTC = 5,       /* NVRTC compilation failed (see log)              */
    KTC_ERR_LAUNCH = 6,      /* launch / execution failure                      */
    KTC_ERR_OOM = 7,         /* device allocation failed                        */
    KTC_ERR_UNSUPPORTED = 8, /* unknown kernel family, layout, ...              */
    KTC_ERR_EMPTY_SPACE = 9, /* tuner: no valid configuration (EmptySpace*)     */
    KTC_ERR_IO = 10
};

/* Per-configuration status: same values and order as ktune::Status. */
enum { KTC_STATUS_SUCCESS = 0, KTC_STATUS_COMPILE_ERROR = 1, KTC_STATUS_RUNTIME_ERROR = 2,
       KTC_STATUS_MISSING = 3 };

/* Verification verdict of one evaluation (ktune::Verification, tuner.hpp:112). */
enum { KTC_VERIFY_SKIPPED = 0, KTC_VERIFY_PASS = 1, KTC_VERIFY_FAIL = 2 };

/* Argument roles / element types (ktune::ArgRole, ktune::ElementType). */
enum { KTC_ARG_INPUT = 0, KTC_ARG_OUTPUT = 1, KTC_ARG_SCALAR = 2 };
enum { KTC_F32 = 0, KTC_I32 = 1 };

typedef struct ktc_ctx ktc_ctx;
typedef struct ktc_fn ktc_fn;
typedef struct ktc_backend ktc_backend;
typedef struct ktc_tuner ktc_tuner;
typedef uint64_t ktc_buf; /* device pointer */

int ktc_abi_version(void);
const char* ktc_status_name(int status); /* "ok", "compile_error", ... */
const char* ktc_last_error(const void* handle);

/* ======================================================================= */
/* 1. Device primitives                                                     */
/* ======================================================================= */

typedef struct {
    int ordinal;
    char name[128];
    int cc_major, cc_minor;
    int sm_count;
    int max_threads_per_block;
    int max_block_dim[3];
    int max_grid_dim[3];
    size_t smem_per_block_optin; /* expected 232448 on B200 */
    size_t smem_per_sm;
    size_t l2_bytes;
    size_t global_mem_bytes;
    int sm_clock_khz;
    int mem_clock_khz;
    int mem_bus_width_bits;
    double peak_fp32_gflops; /* sm_count * 128 lanes * 2 * sm clock */
    double peak_hbm_gbs;     /* nominal, from memory clock and bus width */
} ktc_limits;

int ktc_device_count(int* count);
int ktc_open(int ordinal, ktc_ctx** out);
void ktc_close(ktc_ctx* ctx);
int ktc_query_limits(ktc_ctx* ctx, ktc_limits* out);
/* Destroys and recreates the device context after a sticky error (illegal
 * address, trap, ...).  All buffers and modules of `ctx` become invalid. */
int ktc_reset(ktc_ctx* ctx);

/* NVRTC: compiles CUDA C++ `src` for sm_100a into a cubin.  No device needed.
 * `opts` are extra NVRTC options (e.g. "-DXWG=32").  On failure returns
 * KTC_ERR_NVRTC and writes the head of the NVRTC log into `log`. */
int ktc_compile(const char* src, const char* const* opts, int nopts, void** cubin,
                size_t* cubin_size, char* log, size_t log_cap);
void ktc_free_host(void* p);
/* The convolution family's direct code generator (the tuning-time default):
 * emits the PTX of one configuration of kernels/conv.cu -- `defines` are its
 * "NAME=VALUE" compile-time parameters plus "FS=<filter>" -- and compiles it
 * with ptxas for sm_100a, entry "conv2d_k0".  No device needed.  `ptx`
 * (optional) receives the PTX text (free with ktc_free_host). */
int ktc_codegen_conv(const char* const* defines, int ndefines, void** cubin, size_t* cubin_size,
                     char** ptx, char* log, size_t log_cap);
/* The same for the SGEMM family (kernels/gemm.cu semantics, entry "gemm_k0";
 * defines: the 14 parameters plus DBUF / OCC / F2). */
int ktc_codegen_gemm(const char* const* defines, int ndefines, void** cubin, size_t* cubin_size,
                     char** ptx, char* log, size_t log_cap);

int ktc_load(ktc_ctx* ctx, const void* cubin, size_t size, const char* kernel_name, ktc_fn** fn);
void ktc_unload(ktc_fn* fn);
/* Copies `bytes` from host into a __constant__/__device__ symbol of fn's module. */
int ktc_set_symbol(ktc_fn* fn, const char* symbol, const void* src, size_t bytes);

int ktc_alloc(ktc_ctx* ctx, size_t bytes, ktc_buf* out);
int ktc_free(ktc_ctx* ctx, ktc_buf buf);
int ktc_upload(ktc_ctx* ctx, ktc_buf dst, const void* src, size_t bytes);
int ktc_upload_pitched(ktc_ctx* ctx, ktc_buf dst, size_t dst_pitch, const void* src,
                       size_t src_pitch, size_t width_bytes, size_t rows);
int ktc_download(ktc_ctx* ctx, void* dst, ktc_buf src, size_t bytes);
int ktc_memset32(ktc_ctx* ctx, ktc_buf dst, uint32_t value, size_t count);

/* One warm-up launch (if warmup > 0; untimed), then `reps` launches, each
 * bracketed by CUDA events on the context's stream and preceded by an L2
 * flush when flush_l2 == 1.  best_ms = min over reps ("best of N",
 * backend.hpp:41-44); all_ms (optional, reps entries) gets every time.
 * flush_l2 == 2: the reps launches back to back between one event pair;
 * best_ms and every all_ms entry = the mean launch duration. */
int ktc_launch_timed(ktc_ctx* ctx, ktc_fn* fn, const unsigned grid[3], const unsigned block[3],
                     unsigned smem_bytes, void** params, int warmup, int reps, int flush_l2,
                     float* best_ms, float* all_ms);

/* Verification report: field-for-field ktune::VerificationReport (tuner.hpp:30-37). */
typedef struct {
    int pass;
    double max_abs_error;
    double max_rel_error;
    size_t buffer_index;
    size_t element_index;
    size_t elements_compared;
} ktc_verify_report;

/* Binds a device buffer as the trusted output (one buffer).  The buffer is
 * referenced, not copied; it must stay alive while bound. */
int ktc_bind_reference(ktc_ctx* ctx, ktc_buf ref, size_t count, int elem_type, double rel_tol,
                       double abs_tol);
/* Compares `cand` (same count/type) against the bound reference on the
 * device with verify_outputs' exact rule (tuner.hpp:39-106). */
int ktc_verify(ktc_ctx* ctx, ktc_buf cand, ktc_verify_report* out);
/* Same, for an explicit pair of device buffers. */
int ktc_verify_pair(ktc_ctx* ctx, ktc_buf cand, ktc_buf ref, size_t count, int elem_type,
                    double rel_tol, double abs_tol, ktc_verify_report* out);

/* FNV-1a-64 digest over 4-byte little-endian words (arguments.hpp:184-205)
 * and its 16-digit hex form (arguments.hpp:208-216). */
uint64_t ktc_digest_words(const void* data, size_t n_words);
void ktc_digest_hex(uint64_t digest, char out[17]);
/* f32 `uniform:<seed>` recipe (arguments.hpp:126-180): out[i] =
 * float(uniform01) of the i-th std::mt19937_64(seed) draw, bit-identical to
 * the sequential stream, on up to `threads` host threads (jump-ahead). */
int ktc_fill_uniform_f32(uint64_t seed, float* out, size_t n, int threads);

/* ======================================================================= */
/* 2. Evaluation backend: ktune::Backend::evaluate over the C ABI           */
/* ======================================================================= */

/* ktune::ArgumentSpec (arguments.hpp:56-62). */
typedef struct {
    int role;         /* KTC_ARG_* */
    int type;         /* KTC_F32 / KTC_I32 */
    size_t length;    /* buffers */
    double value;     /* scalars */
    const char* fill; /* "none" | "constant:<v>" | "ramp" | "uniform:<seed>" */
} ktc_arg;

/* ktune::EvaluationRequest (backend.hpp:45-55). */
typedef struct {
    const char* kernel_name; /* "conv", "gemm", "gemm_tf32", or a custom kernel */
    const char* source_ref;  /* custom kernels: path of the .cu source */
    int n_params;
    const char* const* param_names;
    const long long* param_values;
    int ndim;
    size_t global[3];
    size_t local[3];
    int n_args;
    const ktc_arg* args;
    const char* device_name;
    int repetitions; /* best of N timed runs */
    /* The caller wants the outputs checked (ktune sets this to job.verify):
     * the backend verifies them on the device against the bound reference
     * (ktc_result.verification) and keeps them on the device for
     * ktc_backend_read_output. */
    int want_outputs;
} ktc_request;

#define KTC_MAX_OUTPUTS 8

/* ktune::EvaluationResult (backend.hpp:57-67) + device verification. */
typedef struct {
    int status;     /* KTC_STATUS_* */
    double time_ms; /* best of `repetitions`, CUDA events; > 0 on success */
    int n_outputs;
    char output_digests[KTC_MAX_OUTPUTS][17];
    int verification; /* KTC_VERIFY_*: device verification against the bound reference */
    ktc_verify_report report;
    char message[512];
    /* Where the wall time went (host clock), for throughput accounting. */
    double compile_ms;    /* NVRTC (0 on a cache hit) */
    double load_ms;       /* cuModuleLoadData + function setup */
    double run_ms;        /* warm-up + timed repetitions + flushes */
    double verify_ms;     /* device verification */
    int compile_cache_hit;
    int kernel_launches;  /* kernels of this library launched for this evaluation */
    double mean_ms;       /* mean over the timed repetitions (time_ms is the min) */
} ktc_result;

typedef struct {
    int warmup;             /* untimed launches before timing (default 1) */
    int flush_l2;           /* flush L2 before every timed launch (default 1); 2 = stream
                             * timing: the repetitions back to back between one event pair,
                             * time = mean launch duration (no flushes) */
    int verify;             /* device verification of every successful run (default 1) */
    double rel_tol;         /* default 1e-4 (tuner.hpp:148) */
    double abs_tol;         /* default 1e-6 (tuner.hpp:149) */
    int compile_threads;    /* NVRTC pool size; 0 = hardware threads */
    const char* cache_dir;  /* on-disk cubin cache; NULL = memory only */
    int digest_outputs;     /* also FNV-digest outputs (D2H + host hash); default 0 */
    /* Early-out for device-bound searches; 0 (default) = off.  When > 0 and
     * this backend has a verified best for the argument list, the warm-up
     * launch of a configuration is flushed and timed (the probe); if it takes
     * more than prune_factor x that best, the probe is the row's time and no
     * further launches are made (the output is still verified).  Otherwise
     * the repetitions follow as usual (the probe was their warm-up).  Such a
     * configuration cannot become the best unless its best-of-N time is below
     * 1/prune_factor of its first flushed launch. */
    double prune_factor;
    /* Process isolation (default 0): every call is forwarded to a persistent
     * worker process per device (ktc-worker).  A configuration that faults
     * (illegal address, trap: the CUDA context is lost for good) or hangs is
     * a runtime_error row and the next evaluation gets a fresh worker, as
     * the reference's external runner is isolated (external.hpp:278-286).
     * The tuner turns it on for custom (user) kernels; KTC_ISOLATE=0/1
     * overrides. */
    int isolate;
} ktc_backend_options;

void ktc_backend_default_options(ktc_backend_options* opts);
int ktc_backend_open(int ordinal, const ktc_backend_options* opts, ktc_backend** out);
void ktc_backend_close(ktc_backend* be);
/* Name as ktune::Backend::name(): "cuda:sm_100a:<device>". */
const char* ktc_backend_name(ktc_backend* be);
ktc_ctx* ktc_backend_ctx(ktc_backend* be);

int ktc_backend_evaluate(ktc_backend* be, const ktc_request* req, ktc_result* out);
/* Starts compiling req's kernel in the background NVRTC pool, so a later
 * evaluate of the same configuration finds the cubin ready. */
int ktc_backend_prefetch(ktc_backend* be, const ktc_request* req);
/* How many requests ahead a caller should keep prefetching so that every
 * NVRTC pool thread has work: 2 x pool threads x configurations per program. */
size_t ktc_backend_prefetch_depth(ktc_backend* be);
/* Starts a new search on this backend: forgets the prune_factor bar (the
 * best verified time seen), so a search is never pruned against another
 * search's (or another stats replica's) best. */
int ktc_backend_begin_search(ktc_backend* be);
/* Process-wide caches (measurement hygiene: a cold end-to-end run).
 * KTC_DROP_COMPILED    the in-memory cubin cache of the compile pool (the
 *                      next evaluation of any configuration compiles again;
 *                      the optional on-disk cache is not touched)
 * KTC_DROP_HOST_INPUTS the pinned host copies of materialized argument
 *                      recipes (the next fresh job materializes its inputs
 *                      on the host again) */
#define KTC_DROP_COMPILED 1
#define KTC_DROP_HOST_INPUTS 2
int ktc_drop_caches(int flags);
/* The isolated backend's worker loop (the ktc-worker executable is just
 * this): serves one backend over framed requests on in_fd / out_fd until the
 * parent closes it.  Not for direct use. */
int ktc_worker_serve(int in_fd, int out_fd);

/* SetReference: binds host reference outputs (one buffer per output
 * argument, in order) for the argument list of `req`.  Built-in families
 * compute their reference on the device (bit-identical to the CPU oracle)
 * and need no call. */
int ktc_backend_set_reference(ktc_backend* be, const ktc_request* req, int n_buffers,
                              const void* const* buffers, const size_t* lengths,
                              const int* types);
/* Output `index` of the last evaluation (host copy; want_outputs). */
int ktc_backend_read_output(ktc_backend* be, int index, void* dst, size_t bytes);
/* The device reference output of the current argument list and its digest. */
int ktc_backend_read_reference(ktc_backend* be, const ktc_request* req, int index, void* dst,
                               size_t bytes, char digest_hex[17]);

/* ======================================================================= */
/* 3. Tuner (CLTune names over the ktune search layer)                      */
/* ======================================================================= */

enum { KTC_SEARCH_FULL = 0, KTC_SEARCH_RANDOM = 1, KTC_SEARCH_ANNEALING = 2, KTC_SEARCH_PSO = 3 };

/* ktune::DeviceModel (device.hpp:14-21). */
typedef struct {
    char name[64];
    size_t max_work_group_total;
    size_t max_work_group_dim[3];
    size_t local_mem_bytes;
    double peak_gflops;
    double peak_gbs;
} ktc_device_model;

/* Presets: "K40m", "GTX480", "HD7970", "Iris5100", "B200" (static), or
 * "cuda:<ordinal>" (queried from the driver). */
int ktc_device_preset(const char* name, ktc_device_model* out);

int ktc_tuner_create(ktc_tuner** out);
void ktc_tuner_destroy(ktc_tuner* t);

/* Built-in case studies (template jobs): kernel + space + device reference. */
int ktc_tuner_template_conv(ktc_tuner* t, size_t x, size_t y, int filter, float weight,
                            uint64_t seed);
int ktc_tuner_template_gemm(ktc_tuner* t, size_t m, size_t n, size_t k, float alpha, float beta,
                            uint64_t seed);
int ktc_tuner_template_gemm_tf32(ktc_tuner* t, size_t m, size_t n, size_t k, float alpha,
                                 float beta, uint64_t seed);

/* CLTune: AddKernel(files, name, global, local). */
int ktc_tuner_add_kernel(ktc_tuner* t, const char* source_ref, const char* name, int ndim,
                         const size_t* global, const size_t* local);
int ktc_tuner_add_parameter(ktc_tuner* t, const char* name, const long long* values, int n);
int ktc_tuner_add_constraint(ktc_tuner* t, const char* expr);
/* target 0 = global, 1 = local; op 0 = multiply, 1 = divide. */
int ktc_tuner_add_modifier(ktc_tuner* t, int target, int op, const char* const* factors, int n);
int ktc_tuner_set_local_memory(ktc_tuner* t, const char* expr);
int ktc_tuner_add_argument(ktc_tuner* t, const ktc_arg* arg);
/* CLTune SetReference(files, name, global, local): a reference kernel (no
 * tuning parameters) run once on the device over the job's arguments at the
 * start of Tune(); its outputs become the reference every configuration is
 * verified against (on the device).  Replaces ktune's TuningJob::reference
 * callback (tuner.hpp:147) for custom kernels. */
int ktc_tuner_set_reference_kernel(ktc_tuner* t, const char* source_ref, const char* name,
                                   int ndim, const size_t* global, const size_t* local);
/* The same with host reference outputs (one buffer per output argument, in
 * order; types KTC_F32 / KTC_I32), copied. */
int ktc_tuner_set_reference_outputs(ktc_tuner* t, int n, const void* const* buffers,
                                    const size_t* lengths, const int* types);
int ktc_tuner_set_device(ktc_tuner* t, const ktc_device_model* dev);
int ktc_tuner_set_strategy(ktc_tuner* t, int kind, double fraction, double temperature,
                           double alpha, double beta, double gamma, size_t swarm);
int ktc_tuner_set_seed(ktc_tuner* t, uint64_t seed);
int ktc_tuner_set_repetitions(ktc_tuner* t, int reps);
int ktc_tuner_set_verification(ktc_tuner* t, int verify, double rel_tol, double abs_tol);
/* Backend: "cuda" (devices below), or "replay:<csv path>". */
int ktc_tuner_set_backend(ktc_tuner* t, const char* spec, const ktc_backend_options* opts);
int ktc_tuner_set_devices(ktc_tuner* t, const int* ordinals, int n);
/* Optional: restrict the search to these enumeration indices of the
 * composed space (used for fixed throughput samples and sharding). */
int ktc_tuner_set_subset(ktc_tuner* t, const uint64_t* indices, size_t n);
/* Checkpoint/resume for full and random searches: successful rows are
 * appended to `path` (replay format `config,time_ms`) as they complete, and
 * configurations already recorded there are served from it instead of being
 * re-evaluated.  NULL or "" disables. */
int ktc_tuner_set_checkpoint(ktc_tuner* t, const char* path);

/* Space funnel: raw, constraint-satisfying, valid after device limits. */
int ktc_tuner_space_counts(ktc_tuner* t, unsigned long long* raw,
                           unsigned long long* constrained, unsigned long long* valid);
/* Canonical string of enumeration index i of the composed space. */
int ktc_tuner_space_config(ktc_tuner* t, uint64_t index, char* out, size_t cap);

int ktc_tuner_tune(ktc_tuner* t);

/* One row of the results table (ktune::TuningRow, tuner.hpp:125-134). */
typedef struct {
    size_t step;
    int status;
    double time_ms;   /* NaN when absent */
    int verification; /* KTC_VERIFY_* */
    double best_so_far; /* NaN when absent */
    size_t global[3];
    size_t local[3];
    int ndim;
    uint64_t space_index; /* enumeration index in the composed space */
    int device;           /* ordinal that evaluated it (-1: not a device backend) */
    ktc_verify_report report;
} ktc_row;

typedef struct {
    size_t rows;
    long long best_index; /* -1 when nothing succeeded */
    double best_time_ms;
    size_t budget;
    size_t unique_evaluations;
    size_t failed_evaluations;
    size_t total_steps;
    unsigned long long space_size;
    double wall_s;           /* Tune() wall time */
    double configs_per_s;    /* rows / wall_s */
    double compile_s;        /* summed NVRTC time (all pool threads) */
    double device_s;         /* summed device-side evaluation wall time */
    size_t compile_cache_hits;
    size_t kernel_launches;
} ktc_summary;

int ktc_tuner_summary(ktc_tuner* t, ktc_summary* out);
int ktc_tuner_row(ktc_tuner* t, size_t i, ktc_row* out, char* config, size_t cap,
                  char* message, size_t msg_cap);
/* GetBestResult: canonical config + time of the best row. */
int ktc_tuner_best(ktc_tuner* t, char* config, size_t cap, double* time_ms);
/* RFC 4180 results CSV, byte-compatible with write_results_csv (report.hpp:62-77). */
int ktc_tuner_write_csv(ktc_tuner* t, const char* path);
/* Replay table `config,time_ms` of the successful rows (backend.hpp:551-562). */
int ktc_tuner_write_replay(ktc_tuner* t, const char* path);

/* Repeated searches (`ktune stats`, tools/ktune.cpp:120-258): `runs` searches
 * with seeds base_seed..base_seed+runs-1, spread as replicas over the tuner's
 * devices (one whole search per device at a time).  Writes `out_csv` (best-of-
 * run statistics + density, report.hpp:98-112), `<stem>_runs<ext>` (one row
 * per run, report.hpp:87-96) and, for spaces of at most 100,000
 * configurations, `<stem>_space<ext>` (the whole-space distribution from one
 * full sweep sharded over every device).  Byte-identical to the reference's
 * reports on the same per-configuration times. */
typedef struct {
    size_t runs;
    double mean, stddev, min, max; /* best-of-run times (ms) */
    int space_written;             /* 1 when <stem>_space was written */
    size_t space_count;            /* successful rows in the full sweep */
    double space_min, space_mean;
    double wall_s;
} ktc_stats_summary;
int ktc_tuner_stats(ktc_tuner* t, size_t runs, uint64_t base_seed, const char* out_csv,
                    ktc_stats_summary* out);

/* Report writers for replicas gathered across processes (one process per
 * GPU): the best-of-run statistics (or a whole-space distribution) of
 * `values` in the given order, and the per-run table -- the files
 * ktc_tuner_stats writes (report.hpp:87-112). */
typedef struct {
    size_t run;
    uint64_t seed;
    double best_time_ms;
    const char* best_config;
} ktc_run_summary;
int ktc_stats_write(const double* values, size_t n, const char* path);
int ktc_runs_write(const ktc_run_summary* runs, size_t n, const char* path);

/* What the CLI prints around a run (tools/ktune.cpp:84-117): the kernel and
 * device names, the backend (its name() after Tune(), else the job's kind),
 * the job's `output` path and the device ordinals the tuner will use. */
typedef struct {
    char kernel[128];
    char device[128];
    char backend[256];
    char output[1024];
    int is_cuda; /* 1 when the backend kind is "cuda" */
    int ndevices;
    int devices[64];
} ktc_job_info;
int ktc_tuner_job_info(ktc_tuner* t, ktc_job_info* out);

/* Job files: the reference's JSON schema (jobfile.hpp) + backend kind
 * "cuda" ({"kind":"cuda","devices":[0],"flush_l2":true,...}). */
int ktc_tuner_load_job(ktc_tuner* t, const char* json_text, const char* base_dir);

#ifdef __cplusplus
}
#endif
#endif /* KTC_H_ */
