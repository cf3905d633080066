/* hiccl — C ABI of the B200-native HiCCL collective execution path.
 *
 * This is the drop-in boundary. The reference (`hiercoll`, a C++20
 * library) has no FFI of its own; its public interface is the C++ API
 * listed beside each entry point below, and the paper's user API is
 * Comm<T>::add_multicast/add_reduction/add_fence, init(hierarchy,
 * library, ring, stripe, pipeline), start(), wait() (PAPER.md:231-233,
 * 304-327). Every entry point takes plain pointers and sizes, returns an
 * hc_status, never throws, and records a thread-local message readable
 * with hc_last_error(). Status values are 1 + the reference ErrorCode
 * (proj/include/hiercoll/types.hpp:50-64) in its order, plus
 * HC_CUDA_ERROR / HC_TIMEOUT for the device path.
 *
 * Strings returned through char** are heap-allocated: release with hc_free.
 */
#ifndef HICCL_H_
#define HICCL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int hc_status;
enum {
  HC_OK = 0,
  HC_EMPTY_LEAF_SET = 1,
  HC_RANK_OUT_OF_RANGE = 2,
  HC_EMPTY_STEP = 3,
  HC_WRITE_WRITE_RACE = 4,
  HC_READ_WRITE_RACE = 5,
  HC_BAD_BUFFER_REF = 6,
  HC_UNSUPPORTED_FORMULATION = 7,
  HC_INVALID_MACHINE = 8,
  HC_INVALID_CONFIG = 9,
  HC_UNINITIALIZED_READ = 10,
  HC_DEPENDENCY_VIOLATION = 11,
  HC_NO_INTER_NODE_BOUND = 12,
  HC_PARSE_ERROR = 13,
  HC_CUDA_ERROR = 14,
  HC_TIMEOUT = 15,
  HC_INTERNAL = 99
};

/* Reduce operators (types.hpp:28) and element types the executor folds. */
enum { HC_OP_SUM = 0, HC_OP_MAX = 1 };
enum {
  HC_F32 = 0,  /* IEEE add per fold, no contraction */
  HC_BF16 = 1, /* widen to f32, add, round-to-nearest-even after every fold */
  HC_F16 = 2,  /* same rule as bf16 */
  HC_I32 = 3,  /* wrapping add */
  HC_I64 = 4,
  HC_F64 = 5,
  HC_U8 = 6    /* byte copies / wrapping add */
};

const char* hc_last_error(void);
void hc_free(void* p);
const char* hc_version(void);

/* ---------------------------------------------------------------------
 * Composition — replaces hiercoll::CollectiveProgram
 * (composition.hpp:66-122; composition.cpp:66-194, 239-441).
 * ------------------------------------------------------------------- */
typedef struct hc_program hc_program;

hc_status hc_program_create(int world_size, hc_program** out);
void hc_program_destroy(hc_program* prog);
/* CollectiveProgram::declare_buffer (composition.hpp:75-76) */
hc_status hc_program_declare_buffer(hc_program* prog, const char* id, int64_t length,
                                    int input, int internal);
/* CollectiveProgram::add_multicast(send, recv, root, leaves) (composition.hpp:81-82) */
hc_status hc_program_add_multicast(hc_program* prog, const char* send_buf, int64_t send_off,
                                   const char* recv_buf, int64_t recv_off, int64_t count,
                                   int root, const int* leaves, int n_leaves);
/* CollectiveProgram::add_reduction(send, recv, leaves, root, op) (composition.hpp:85-87) */
hc_status hc_program_add_reduction(hc_program* prog, const char* send_buf, int64_t send_off,
                                   const char* recv_buf, int64_t recv_off, int64_t count,
                                   const int* leaves, int n_leaves, int root, int op);
/* CollectiveProgram::add_fence (composition.hpp:91) */
hc_status hc_program_add_fence(hc_program* prog);
/* CollectiveProgram::validate (composition.hpp:103): one line per
 * violation, "Code|step|primitive|rank|buffer|lo|hi|message\n". */
hc_status hc_program_validate(const hc_program* prog, char** report);
/* serialize / deserialize / id (composition.hpp:105-109), hiercoll-program-v1 */
hc_status hc_program_serialize(const hc_program* prog, char** json);
hc_status hc_program_deserialize(const char* json, hc_program** out);
hc_status hc_program_id(const hc_program* prog, char** id);
/* presets::build(CollectiveSpec, p) (presets.hpp:62). kind: 0 scatter,
 * 1 broadcast, 2 gather, 3 reduce, 4 all_to_all, 5 all_gather,
 * 6 reduce_scatter, 7 all_reduce; formulation 0 single, 1 multi, 2 multi_alt. */
hc_status hc_program_preset(int kind, int formulation, int p, int64_t count, int root,
                            int op, hc_program** out);

/* ---------------------------------------------------------------------
 * Lowering — replaces hiercoll::lower + hiercoll::pipeline
 * (factorize.hpp:107-109, pipeline.hpp:40) and the machine description
 * (machine.hpp:48-89). `transport` labels are the paper's per-level
 * library; NULL means "IPC" at every level.
 * ------------------------------------------------------------------- */
typedef struct {
  const int* hierarchy;
  int num_levels;
  int gpus_per_node;
  const char* const* transport;
} hc_machine_desc;

typedef struct hc_plan hc_plan; /* a PipelinedPlan */

/* Argument order follows the paper's init(hierarchy, library, ring,
 * stripe, pipeline). */
hc_status hc_plan_lower(const hc_program* prog, const hc_machine_desc* machine, int ring,
                        int stripe, int pipeline, hc_plan** out);
/* lower() alone, hiercoll-plan-v1 text (factorize.hpp:65-67) */
hc_status hc_plan_lower_staged_json(const hc_program* prog, const hc_machine_desc* machine,
                                    int ring, int stripe, char** json);
hc_status hc_plan_serialize(const hc_plan* plan, char** json); /* hiercoll-pipelined-v1 */
hc_status hc_plan_deserialize(const char* json, hc_plan** out);
void hc_plan_destroy(hc_plan* plan);

typedef struct {
  int world_size;
  int num_transfers;
  int num_buffers;
  int num_stages;
  int slots;
  int depth;
  int stripe;
  int ring;
} hc_plan_info;

typedef struct {
  int32_t id, src, dst, src_buf, dst_buf; /* buffer ids index hc_plan_buffer */
  int32_t reduce, op, stage, slot, channel, stripe, level, step, n_deps;
  int64_t src_off, dst_off, count;
} hc_transfer;

hc_status hc_plan_get_info(const hc_plan* plan, hc_plan_info* out);
/* Buffer table in name order (the plan's std::map order). */
hc_status hc_plan_get_buffer(const hc_plan* plan, int index, const char** name,
                             int64_t* length, int* input, int* internal);
/* Fills num_transfers records in id order. */
hc_status hc_plan_get_transfers(const hc_plan* plan, hc_transfer* out);
/* Bytes src->dst at `slot` (pipeline.hpp:44), row-major p*p. */
hc_status hc_plan_comm_matrix(const hc_plan* plan, int slot, int64_t* out);

/* Executor schedule diagnostics (host only, no GPU needed): builds the
 * write groups / phases / wait edges the executor would run for this
 * mapping, replays them against a sequential (slot, id) execution with an
 * order-sensitive fold, and returns a JSON summary. verify = 0 skips the
 * O(items^2) replay checks (large plans). */
hc_status hc_plan_schedule_summary(const hc_plan* plan, int num_execs, const int* rank_to_exec,
                                   int copy_mode, int element_size, int verify, char** json);

/* Device layout diagnostics (host only): the items, tiles and tile-granular
 * waits every executor would run when the buffers named in
 * `multicast_buffers` (comma-separated, may be empty) sit in an NVLS window
 * — multimem lowering and the reduce+multicast fusion included — checked
 * pair by pair (verify_sync). dtype is an hc_dtype code. JSON per executor:
 * per step the item kinds ("p2p", "mc_reduce", "mc_store",
 * "mc_reduce_store") and the number of fused pairs. */
hc_status hc_plan_layout_summary(const hc_plan* plan, int num_execs, const int* rank_to_exec,
                                 int copy_mode, int dtype, int ctas, const char* multicast_buffers,
                                 char** json);

/* ---------------------------------------------------------------------
 * Cost model and tuner (include/hiccl/model.hpp) — the reference's
 * slot-synchronous simulate() (perf.cpp:48-106) re-targeted at the B200
 * executor, plus its closed forms Eq. (1)/(2), Table-4 bounds and d*p/t
 * (perf.cpp:108-140).
 * ------------------------------------------------------------------- */
typedef struct {
  double launch;   /* s: launch + entry/exit barriers */
  double step;     /* s: one dependent step */
  double push_bw;  /* B/s: peer stores per GPU per direction */
  double pull_bw;  /* B/s: peer loads per GPU per direction */
  double hbm_bw;   /* B/s: local copy, read + write bytes */
  double ll_launch; /* s: launch in tagged-line mode (no barriers) */
  double ll_step;   /* s: one dependent step in tagged-line mode */
  double ll_bw;     /* B/s: tagged-line bytes (2x payload) a GPU stores to peers */
  double ll_in_bw;  /* B/s: tagged-line bytes a GPU receives */
  double ll_bidir_bw; /* B/s: tagged-line bytes stored + received */
  double nvls_read_bw;  /* B/s: bytes a GPU serves to NVSwitch reads (multimem.ld_reduce) */
  double nvls_store_bw; /* B/s: bytes multicast stores (multimem.st) land on a GPU */
  double nvls_bidir_bw; /* B/s: both of the above together, both directions busy */
  double nvls_reduce_bw; /* B/s: multimem.ld_reduce results one GPU draws */
  double pull_uni_bw;    /* B/s: peer loads when the opposite direction is idle */
  double push_uni_bw;    /* B/s: peer stores when the opposite direction is idle */
  double nvls_launch;    /* s: extra fixed cost of a launch with multimem items */
} hc_model;

typedef struct {
  int formulation;
  int ring;
  int pipeline;
  double seconds;
  int copy_mode;   /* 1 push or 3 ll */
  int nvls;        /* 1: user buffers in an NVLS window (hc_tune_nvls only) */
} hc_tune_result;

hc_status hc_model_default(hc_model* out);
hc_status hc_plan_predict(const hc_plan* plan, int element_size, const hc_model* model,
                          int ranks_per_gpu, int copy_mode, double* seconds);
hc_status hc_tune(int kind, int p, int64_t count, int element_size, const hc_model* model,
                  hc_tune_result* out);
/* With user buffers in an NVLS window (one rank per GPU, dtype = hc_dtype):
 * the executors' device layout, multimem lowering and fusion included. */
hc_status hc_plan_predict_nvls(const hc_plan* plan, int dtype, const hc_model* model,
                               double* seconds);
/* hc_tune, also weighing the NVLS library (out->nvls). */
hc_status hc_tune_nvls(int kind, int p, int64_t count, int dtype, const hc_model* model,
                       hc_tune_result* out);
hc_status hc_t_ring(double alpha, double d, int k, double f, int m, int n, double intra,
                    double* seconds);
hc_status hc_t_tree(double alpha, double d, int k, double f, int m, int n, double intra,
                    double* seconds);
hc_status hc_bound(int kind, int p, int g, int k, double f, double* bytes_per_second);
hc_status hc_throughput(double d_bytes, int p, double t, double* bytes_per_second);

/* ---------------------------------------------------------------------
 * Executor — replaces hiercoll::execute_plan / run_transfers
 * (engine.hpp:127, engine.cpp:285-347). One hc_exec per (process, GPU);
 * an executor serves every logical rank mapped to it (several ranks per
 * GPU emulate larger worlds). Not thread-safe per handle.
 * ------------------------------------------------------------------- */
typedef struct hc_exec hc_exec;

typedef struct {
  int device;              /* CUDA ordinal this executor drives */
  int exec_index;          /* 0..num_execs-1 */
  int num_execs;           /* executors in the world */
  const int* rank_to_exec; /* world_size entries */
  int dtype;               /* HC_F32 ... */
  int ctas;                /* persistent CTAs; 0 = one per SM */
  int threads;             /* threads per CTA; 0 = default */
  int copy_mode;           /* 0 pull (dst runs copies), 1 push (src runs copies),
                              2 staged (push, and remote reduction sources are
                              pushed into staging on the dst, folded locally),
                              3 ll (low latency: every remote source is pushed
                              into staging as tagged lines; no barriers, no
                              system-scope fences; small messages),
                              4 auto (push or ll, whichever the B200 cost
                              model predicts faster for this plan; ll only
                              while every user buffer is <= 64 MiB) */
  double timeout_s;        /* watchdog for flag waits; <= 0 disables */
  int execs_per_device;    /* executors of this world sharing `device` (0 or 1:
                              one). With n > 1 every grid is capped at 1/n of
                              the device's co-resident CTAs so all n persistent
                              grids run at once, and a NULL stream in
                              hc_exec_start selects the executor's own
                              non-blocking stream. Same cross-executor protocol
                              (system-scope flags, entry/exit barriers) as
                              executors on different GPUs. */
} hc_exec_config;

hc_status hc_exec_create(const hc_plan* plan, const hc_exec_config* cfg, hc_exec** out);
void hc_exec_destroy(hc_exec* ex);

/* Bind a user buffer (plan buffer `name`, logical `rank`) to a device
 * address usable from this executor's device: local memory for ranks
 * this executor serves, a peer-mapped or IPC-opened address otherwise. */
hc_status hc_exec_bind_buffer(hc_exec* ex, int rank, const char* name, void* ptr,
                              size_t bytes);
/* Internal staging (__acc.*, __stage.*, __tmp) for this executor's ranks
 * lives in one arena allocated by hc_exec_create; its layout is a pure
 * function of (plan, rank_to_exec), so peers only exchange the base. */
hc_status hc_exec_local_arena(hc_exec* ex, void** ptr, size_t* bytes);
hc_status hc_exec_bind_peer_arena(hc_exec* ex, int peer_exec, void* ptr);
/* Per-executor flag words (epoch-tagged completion counters). */
hc_status hc_exec_local_flags(hc_exec* ex, void** ptr, size_t* bytes);
hc_status hc_exec_bind_peer_flags(hc_exec* ex, int peer_exec, void* ptr);
/* Resolve every address and upload the device program. */
hc_status hc_exec_commit(hc_exec* ex);
/* Launch the persistent kernel for one execution on `stream`
 * (cudaStream_t, NULL = legacy default). Non-blocking. */
hc_status hc_exec_start(hc_exec* ex, void* stream);
/* Block until this executor's buffers are reusable. */
hc_status hc_exec_wait(hc_exec* ex);
/* Non-blocking completion poll: *done = 1 when finished. */
hc_status hc_exec_query(hc_exec* ex, int* done);

typedef struct {
  int num_steps;        /* global (slot, phase) steps */
  int num_items;        /* work items this executor runs */
  int num_waits;        /* cross-executor wait edges */
  int ctas;
  int threads;
  int64_t bytes_in;     /* bytes this executor's items read */
  int64_t bytes_out;    /* bytes this executor's items write */
  int64_t remote_bytes; /* bytes read from or written to other executors */
  int64_t arena_bytes;
  int nvls_items;       /* items lowered to multimem (NVLS) */
  int paired_waits;     /* waits on one producer CTA (tile-granular) */
  int whole_waits;      /* waits on every CTA of a producer executor */
  int copy_mode;        /* the mode in effect (copy_mode 4 = auto resolves to 1 or 3) */
  int tma_steps;        /* steps of local copies streamed by TMA bulk copies */
  int staged_steps;     /* steps of folds staged through shared memory (HICCL_STAGED) */
} hc_exec_stats;
hc_status hc_exec_get_stats(const hc_exec* ex, hc_exec_stats* out);
/* Device timeline of the most recent launch (%globaltimer, ns): [0] grid
 * entry, [1] entry barrier passed, [2+s] CTA 0 published global step s
 * (stale when nobody waits on it), [S+2] last CTA done, [S+3] exit barrier.
 * n must be >= num_steps + 4. Blocks until the launch completes. */
hc_status hc_exec_get_trace(hc_exec* ex, int64_t* out, int n);

/* ---------------------------------------------------------------------
 * NVLS windows — symmetric memory bound to an NVSwitch multicast object
 * (the paper's per-level "library" NVLS). Buffers placed in a window and
 * declared with hc_exec_bind_multicast let the executor lower reduction
 * groups over every rank to one multimem.ld_reduce (reduced inside the
 * switch; fp sums then differ from the plan's fold order within a stated
 * tolerance) and multicasts to every rank to one multimem.st.
 * ------------------------------------------------------------------- */
typedef struct hc_window hc_window;

hc_status hc_nvls_supported(int device, int* supported);
/* One process driving all members: `bytes` per device on devices[0..n). */
hc_status hc_window_create(const int* devices, int n, size_t bytes, hc_window** out);
/* One process per member: the creator passes handle = NULL and publishes
 * hc_window_export(); the others open with that handle. After EVERY member
 * has opened (caller's barrier), every member calls hc_window_bind. */
hc_status hc_window_open(int device, int n_members, size_t bytes, const unsigned char* handle,
                         hc_window** out);
hc_status hc_window_export(hc_window* w, unsigned char handle[64]);
hc_status hc_window_bind(hc_window* w);
/* One process per member: unicast access to another member's memory.
 * The owner exports (after bind), the peer imports and gets its address. */
hc_status hc_window_export_memory(hc_window* w, unsigned char handle[64]);
hc_status hc_window_import_memory(hc_window* w, const unsigned char handle[64], void** uc);
/* Unicast and multicast base of a member driven by this process. */
hc_status hc_window_pointers(hc_window* w, int member, void** uc, void** mc, size_t* bytes);
void hc_window_destroy(hc_window* w);
/* Every rank's buffer `name` lies in one window; `mc_ptr` is the
 * multicast address, on this executor's device, of the buffer's offset 0. */
hc_status hc_exec_bind_multicast(hc_exec* ex, const char* name, void* mc_ptr);

/* Single-process convenience: enable peer access between every pair of
 * `devices` (cudaDeviceEnablePeerAccess). */
hc_status hc_enable_peer_access(const int* devices, int n);

/* Multi-process bootstrap: CUDA IPC export/import of a device address.
 * The handle is 64 opaque bytes; `offset` is ptr minus its allocation base. */
hc_status hc_ipc_export(void* ptr, unsigned char handle[64], size_t* offset);
hc_status hc_ipc_import(const unsigned char handle[64], size_t offset, int device, void** ptr);
hc_status hc_ipc_close(void* base_ptr);
/* The device allocation containing ptr: its base address and size. */
hc_status hc_device_range(const void* ptr, void** base, size_t* bytes);

/* Device memory helpers (so callers need no CUDA runtime of their own). */
hc_status hc_device_alloc(int device, size_t bytes, void** ptr);
hc_status hc_device_free(int device, void* ptr);
hc_status hc_device_count(int* n);
hc_status hc_device_sync(int device);
/* Fill with the counter-hash generator shared with the oracle:
 * h = splitmix64(seed ^ (rank << 40) ^ index), f32 = ((h>>40)*2^-24)*2-1,
 * bf16/f16 = RNE(f32), i32 = (h>>33) & 0xFFFF, i64 likewise, u8 = h>>56. */
hc_status hc_device_fill(int device, void* ptr, int64_t count, int dtype, uint64_t seed,
                         int rank, int64_t index_base, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HICCL_H_ */
