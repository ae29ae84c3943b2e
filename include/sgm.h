/*
 * sgm.h — C ABI of the B200 sGraph-candidate backend (libsgm.so).
 *
 * The backend executes *instantiated sGraph candidates* (a block graph with a
 * concrete mapping and concrete grid / for-loop sizes) on one B200 (sm_100a),
 * times them, and runs finite-field equivalence checks on device.  It is the
 * drop-in replacement for the reference's CPU interpreter:
 *
 *   reference interface                          replaced by
 *   ------------------------------------------   ------------------------------------
 *   symfuse.interp.run_concrete                  sgm_plan_create + sgm_plan_run
 *     (pkg/src/symfuse/interp.py:128-212)          (+ sgm_plan_run_host for host buffers)
 *   symfuse.interp.run_program                   sgm_plan_create(program-as-plan) + run
 *     (interp.py:69-83)
 *   symfuse.tuner.score_interp                   sgm_plan_time / sgm_timer_* (batched)
 *     (pkg/src/symfuse/tuner.py:160-174)
 *   symfuse.interp.random_equiv_test             sgm_ff_fill + sgm_plan_run (SGM_FF) +
 *     (interp.py:238-286)                          sgm_compare_u32 / sgm_rel_err
 *   errors.py exception classes                  sgm_status codes + sgm_last_error()
 *     (pkg/src/symfuse/errors.py:1-38)
 *
 * Everything is plain C: POD descriptors, raw device pointers, sizes and an
 * opaque stream handle (a CUstream / cudaStream_t, or NULL for the legacy
 * stream).  No torch types cross this boundary.
 *
 * Conventions
 *  - Every entry point returns an sgm_status; on failure a thread-local message
 *    is available from sgm_last_error().
 *  - Tensors are dense row-major.  Input slot k of a plan reads program input k
 *    (program order, symfuse `Program.inputs`); output slot k writes program
 *    output k (`Program.outputs`).  Element type follows the plan's number
 *    system: SGM_F64 double, SGM_F32 float, SGM_BF16 bfloat16 (uint16 bits),
 *    SGM_FF uint32 residues modulo 2^31-1.
 *  - Threading: one host thread drives one device; plan handles are not
 *    thread-safe, sgm_plan_create may be called concurrently (compilation is
 *    independent per plan).
 */
#ifndef SGM_H_
#define SGM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGM_ABI_VERSION 2

#define SGM_MAX_RANK 4
#define SGM_MAX_GRID 3
#define SGM_MAX_NODES 64
#define SGM_MAX_SLOTS 16

/* Status codes.  1..6 map onto the reference's errors.py classes. */
typedef enum {
  SGM_OK = 0,
  SGM_ERR_SHAPE = 1,          /* ShapeError           (errors.py:5)  */
  SGM_ERR_DIVISIBILITY = 2,   /* DivisibilityError    (errors.py:9)  */
  SGM_ERR_WRITE_CONFLICT = 3, /* WriteConflictError   (errors.py:33) */
  SGM_ERR_UNSUPPORTED = 4,    /* UnsupportedOpError   (errors.py:25) */
  SGM_ERR_CONSTRAINT = 5,     /* ConstraintError      (errors.py:17) */
  SGM_ERR_INVALID = 6,        /* malformed descriptor / numpy-style ValueError */
  SGM_ERR_CUDA = 100,         /* CUDA driver failure */
  SGM_ERR_NVRTC = 101,        /* kernel compilation failure */
  SGM_ERR_RESOURCE = 102,     /* smem / cluster / memory limits */
  SGM_ERR_NOT_INIT = 103
} sgm_status;

/* Number systems a plan computes in. */
typedef enum {
  SGM_F64 = 0,  /* fp64 storage + compute (the reference's dtype)            */
  SGM_F32 = 1,  /* fp32 storage + compute                                    */
  SGM_BF16 = 2, /* bf16 storage, fp32 compute                                */
  SGM_FF = 3    /* uint32 residues mod p = 2^31-1; exp/silu/sqrt keyed hashes */
} sgm_numsys;

/* Block-graph node kinds (symfuse graph.py:49-65). */
typedef enum {
  SGM_INPUT = 0, SGM_OUTPUT = 1, SGM_MATMUL = 2, SGM_EXP = 3, SGM_SILU = 4,
  SGM_SQUARE = 5, SGM_SQRT = 6, SGM_DIV = 7, SGM_MUL = 8, SGM_ADD = 9,
  SGM_SUM = 10, SGM_ACCUM = 11, SGM_SCALE = 12
} sgm_kind;

/* One program tensor seen through a loader (input slot) or saver (output slot). */
typedef struct {
  int32_t rank;
  int32_t _pad;
  int64_t dims[SGM_MAX_RANK];
} sgm_slot_desc;

/* One block-graph node.  Mirrors symfuse BlockNode (graph.py:190-208) plus the
 * concrete tile shape of ConcreteGraph.shapes (graph.py:406-441) and, for
 * loaders / savers, the partition of each data dim:
 *   grid_mask[d] bit g set  <=> mapping[MapVar(tensor, d, grid[g])] == 1
 *   loop_split[d] != 0      <=> mapping[MapVar(tensor, d, loop)] == 1 (loaders only)
 * Splits nest in grid order, then the loop (interp.py:90-113). */
typedef struct {
  int32_t kind;            /* sgm_kind */
  int32_t n_inputs;
  int32_t inputs[2];
  int32_t slot;            /* loader: input slot; saver: output slot; else -1 */
  int32_t axis;            /* sum axis (left-indexed data dim), else -1 */
  int64_t const_num;       /* scale factor numerator / denominator */
  int64_t const_den;
  int32_t rank;
  int32_t _pad;
  int64_t shape[SGM_MAX_RANK];       /* concrete per-block tile shape */
  uint32_t grid_mask[SGM_MAX_RANK];
  int32_t loop_split[SGM_MAX_RANK];
} sgm_node_desc;

/* Planner hints (0 = automatic). */
typedef struct {
  int32_t max_cluster;     /* cap on CTAs per logical block sharing a cluster (1..16) */
  int32_t target_ctas;     /* desired total CTAs (default 2 x SMs) */
  int32_t threads;         /* threads per CTA (default 256) */
  int32_t smem_budget;     /* bytes of dynamic smem per CTA the planner may use */
  int32_t no_loop_split;   /* 1: run the for-loop sequentially inside every CTA */
  int32_t no_hoist;        /* 1: do not hoist loop-invariant body nodes */
  int32_t use_tcgen05;     /* -1 off, 0 auto, 1 force where legal */
  int32_t no_tma;          /* 1: stream matmul operands with plain loads, no TMA producer warp */
  int32_t trace;           /* 1: record %globaltimer at schedule events (sgm_plan_trace) */
  int32_t variant;         /* v > 0: the v-th best split the planner scored (physical-plan tuning) */
  int32_t one_cta;         /* 1: size the TMA ring for one CTA per SM (32 KB slots) */
  int32_t max_gsplit;      /* cap on gsplit parts per reduction group (0 = none) */
  int32_t slot_kb;         /* TMA ring slot size in KB at one CTA per SM: 0 = planner (32), 16 = twice the slots */
  int32_t wd_test;         /* test only: 1 = the TMA producer issues nothing, so the watchdog must fire */
  int32_t small_plain;     /* 1: small streamed operands (<= 64 KB per item, <= 1/8 of the largest stream)
                              are read with plain loads by the compute warps instead of the TMA ring */
  int32_t big_first;       /* 1: schedule the largest streamed matmul first (its ring fill starts at once;
                              small chains run after it, their operands already in flight) */
  int32_t item_cost_ns;    /* planner's fixed cost per work item (0 = calibrated 4 us): lower values favour
                              many small items (finer gsplit), i.e. less wave quantisation on 148 SMs */
  int32_t min_gsplit;      /* only plans with at least this many gsplit parts per reduction group (more,
                              smaller work items: finer load balance over 148 SMs) */
  int32_t no_wd;           /* 1: unbounded (canonical) mbarrier waits, no kernel watchdog; 2-7% faster ring
                              loops.  The sweep runs watchdog kernels; the best-kernel phase reports no_wd ones */
  int32_t interleave;      /* 1: issue the first ring-full of the largest tcgen05 stream before a small
                              independent stream chain scheduled ahead of it (LoRA's X@A -> T@B), the
                              rest after it: the chain runs while the ring refills */
  int32_t ff_tma;          /* 1: finite-field plans stream their residues through the TMA ring too */
  int32_t no_xcache;       /* 1: no x-cache (nodes independent of the grid coordinate recomputed per item) */
  int32_t no_prefetch;     /* 1: loop-body tiles are not prefetched into registers one iteration ahead */
  int32_t _reserved[3];
} sgm_plan_hints;

typedef struct {
  int32_t abi_version;     /* must be SGM_ABI_VERSION */
  int32_t numsys;          /* sgm_numsys */
  int32_t n_inputs;
  int32_t n_outputs;
  sgm_slot_desc inputs[SGM_MAX_SLOTS];
  sgm_slot_desc outputs[SGM_MAX_SLOTS];
  int32_t n_nodes;
  int32_t n_grid;          /* number of grid dims (1..3) */
  int64_t grid[SGM_MAX_GRID]; /* concrete grid sizes (params[x], params[y], params[z]) */
  int64_t n_loop;          /* params[i] */
  sgm_node_desc nodes[SGM_MAX_NODES];
  sgm_plan_hints hints;
} sgm_plan_desc;

/* What the planner decided (for reports, tests and the profiler). */
typedef struct {
  int64_t logical_blocks;  /* prod(grid) */
  int64_t ctas;            /* launched CTAs */
  int32_t cluster;         /* CTAs per cluster */
  int32_t threads;
  int32_t smem_bytes;      /* dynamic smem per CTA */
  int32_t loop_parts;      /* loop iterations spread over this many CTAs */
  int64_t free_parts;      /* independent CTAs per logical block */
  int64_t scratch_bytes;   /* global scratch for tiles that do not fit smem */
  double compile_ms;       /* 0 on a cache hit */
  int32_t cache_hit;
  int32_t n_tcgen05;       /* matmul nodes realised with tcgen05 */
  uint64_t source_hash;
  char kernel_name[64];
  char plan_summary[448];
} sgm_plan_info;

typedef struct sgm_plan sgm_plan;

int sgm_abi_version(void);
const char* sgm_last_error(void);
/* Kernel launches issued by this library so far (generated + utility kernels;
 * graph launches count every node executed). */
long long sgm_launch_count(void);

/* Bind the calling thread to `device` (primary context) and load the driver. */
int sgm_init(int device);
/* Directory for the persistent cubin cache (NULL = default next to libsgm.so). */
int sgm_set_cache_dir(const char* path);

/* Validate + plan + generate + compile (or cache-hit) a candidate kernel. */
int sgm_plan_create(const sgm_plan_desc* desc, sgm_plan** out);
int sgm_plan_info_get(const sgm_plan* plan, sgm_plan_info* info);
/* The B200 resource model without compiling: validate + plan + generate only.
 * SGM_OK iff the candidate has a feasible physical plan on this device (shared
 * memory <= 227 KB per CTA incl. the TMA ring, TMEM columns, cluster size <= 16,
 * TMA box limits, scratch); `info` (may be NULL) receives the plan (no
 * compile_ms / cache_hit).  Replaces the reference's 2-byte / 164 KiB budget
 * filter (tuner.py:36-37,67-71) for backend "b200". */
int sgm_plan_feasible(const sgm_plan_desc* desc, sgm_plan_info* info);
/* Copy the generated CUDA source (NUL-terminated, truncated to cap). Returns length via *len. */
int sgm_plan_source(const sgm_plan* plan, char* buf, size_t cap, size_t* len);
/* The sm_100a cubin of a compile-only plan (created before sgm_init bound a
 * device), for cuobjdump / SASS inspection; *len receives its size. */
int sgm_plan_cubin(const sgm_plan* plan, void* buf, size_t cap, size_t* len);
int sgm_plan_destroy(sgm_plan* plan);

/* Outputs are first filled with NaN (fp) / 0xFFFFFFFF (FF) when init_outputs != 0,
 * reproducing the reference's NaN-initialised outputs (interp.py:147-152).
 * Every input and output pointer must be 16-byte aligned (SGM_ERR_INVALID otherwise). */
int sgm_plan_run(sgm_plan* plan, const void* const* inputs, void* const* outputs,
                 int init_outputs, void* stream);
/* Timeline of the last run of a plan created with hints.trace = 1: for every
 * launched CTA, SGM_TRACE_N (time_ns, event) pairs; entries [0, N/2) come from
 * compute thread 0, [N/2, N) from the TMA producer lane; unused entries are 0.
 * Events: 0 entry, 1 start (setup + item-invariant prologue done), 2 item start,
 * 1000+n node n, 2000+p flush at schedule position p, 5 item end, 7 exit;
 * producer 3 item start, 4000+n stream of node n, 6 done. */
#define SGM_TRACE_N 512
int sgm_plan_trace(const sgm_plan* plan, uint64_t* host, int64_t cap_pairs, int64_t* n_pairs);
/* Host-buffer variant: H2D of inputs, run, D2H of outputs, all on `stream`
 * (pinned staging owned by the plan).  This is the e2e path. */
int sgm_plan_run_host(sgm_plan* plan, const void* const* host_inputs,
                      void* const* host_outputs, void* stream);
/* Time `iters` back-to-back launches (after `warmup`) with CUDA events on
 * `stream`.  If `rot` > 1, `inputs` holds rot*n_inputs pointers (rotating input
 * sets, so successive launches miss L2).  Writes mean microseconds per launch. */
int sgm_plan_time(sgm_plan* plan, const void* const* inputs, void* const* outputs,
                  int rot, int warmup, int iters, void* stream, double* mean_us);

/* Batched, sync-free profiling of many plans (the candidate sweep).  Slot k
 * times `reps` launches of a CUDA graph holding `rot` back-to-back launches (one
 * per rotating input set; `inputs` = rot*n_inputs pointers), after `warmup`
 * untimed launches of that graph, between two events recorded on `stream`.
 * Nothing synchronises until sgm_timer_read, which waits for the last event and
 * returns the mean microseconds per kernel launch of slots 0..n-1. */
typedef struct sgm_timer sgm_timer;
int sgm_timer_create(int capacity, sgm_timer** out);
int sgm_timer_enqueue(sgm_timer* t, int slot, sgm_plan* plan, const void* const* inputs, void* const* outputs,
                      int rot, int warmup, int reps, void* stream);
int sgm_timer_read(sgm_timer* t, int n, double* us_per_launch);
int sgm_timer_destroy(sgm_timer* t);

/* Counter-based uniform residues in [0, p): value(i) = mix64(key + i*G) mod p with
 * key = mix64(seed ^ mix64(salt)).  Same function as oracle/ff_np.py:ff_uniform. */
int sgm_ff_fill(uint32_t* dst, int64_t n, uint64_t seed, uint64_t salt, void* stream);
/* Number of positions where a != b (uint32). */
int sgm_compare_u32(const uint32_t* a, const uint32_t* b, int64_t n, void* stream,
                    int64_t* mismatches);
/* Asynchronous variant: adds the number of mismatching positions to
 * *dev_counter (a device int64), no synchronisation. */
int sgm_compare_u32_acc(const uint32_t* a, const uint32_t* b, int64_t n, void* stream, int64_t* dev_counter);
/* rel_err(a, b) = max|a-b| / (1 + max|b|), +inf if a is non-finite (interp.py:228-231).
 * numsys selects the element type of both buffers (F64/F32/BF16). */
int sgm_rel_err(const void* a, const void* b, int64_t n, int numsys, void* stream,
                double* out);
/* Asynchronous, mixed-type rel_err accumulation (the sweep's deployment-dtype
 * parity gate): `a` holds n elements of number system `numsys` (F64/F32/BF16),
 * `b` n fp64 values.  Folds into dev_slot[0..2] (device uint64, zeroed by the
 * caller): [0] max|a-b| and [1] max|b| as non-negative double bit patterns
 * (atomicMax), [2] += count of non-finite elements of a.  The host computes
 * rel_err = slot[2] ? inf : slot[0] / (1 + slot[1]), as interp.py:228-231. */
int sgm_rel_err_acc(const void* a, int numsys, const double* b, int64_t n, void* stream, uint64_t* dev_slot);
/* Watchdog of a plan's kernel: generated kernels bound every wait on an
 * asynchronous completion (TMA bytes, MMA commits, remote cluster arrivals) to
 * 2 s; a wait that times out sets a flag in the plan's module and gives up,
 * so a broken kernel terminates (with wrong results) instead of hanging the
 * device.  Synchronises `stream`, sets *tripped = 1 if any launch since the
 * last reset timed out, and clears the flag when `reset` != 0.  The Python
 * layer reports it as the reference's "run: ..." verdict (interp.py:278-281). */
int sgm_plan_watchdog(sgm_plan* plan, void* stream, int reset, int* tripped);
/* Programmatic dependent launch for every later launch (and graph capture):
 * 1 on (default unless the SGM_NO_PDL environment variable is set), 0 off.
 * With PDL a launch may begin while the previous kernel in the stream drains;
 * generated kernels gate every global access on griddepcontrol.wait. */
int sgm_set_pdl(int on);
/* Fill with a standard-normal-like deterministic pattern (for timing inputs). */
int sgm_fill_normal(void* dst, int64_t n, int numsys, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SGM_H_ */
