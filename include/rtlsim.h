/*
 * rtlsim.h -- C ABI of the B200-native RTeAAL Sim hot path.
 *
 * The library evaluates a synchronous circuit cycle by cycle, batched over
 * many independent stimulus lanes, as the cascade of extended Einsums of
 * PAPER.md Cascade 1 (box:einsum):
 *
 *   per cycle c:
 *     1. input injection   LI[in_k]  = stimulus & M(w)      (§2.1; §6.2)
 *     2. for each level i (iterative rank I, stop condition "i == I"):
 *          a. gather  OI_{i,n,o,r,s} = LI_{i,r} . OIM_{i,n,o,r,s}  :: AND <-(->)   (eq:split_einsum1 P:809-812)
 *          b. op      LO = OI :: AND op_u[n](<-) OR op_r[n](->),   LO_sel :: populate op_s[n]
 *                     (eq:step4c P:826-830, eq:step5b P:839-843, alg:opn P:753-775, App. A)
 *          c. write   LI_{i+1,s} = LO | LO_sel  :: OR ANY(->)    (Cascade 1 P:956-966; alg:RU P:1012)
 *          d. level barrier
 *     3. per-cycle signal hash (reading R12), fused
 *     4. register commit (Fig. 1 caption P:187), simultaneous
 *
 * Op semantics are FIRRTL unsigned semantics masked to the op's declared
 * width <= 64 (readings R1-R5).  All arithmetic is exact integer.
 *
 * Process model: one process per GPU.  A graph is loaded onto ONE device;
 * multi-GPU lane sharding uses one rs_lanes per process with a global lane
 * offset (rs_lane_opts.lane0), so results never depend on the GPU count.
 *
 * Conventions (all functions):
 *   - Never abort or throw across the ABI.  On a non-RS_OK status outputs are
 *     unspecified and rs_last_error() (thread-local) explains.
 *   - The caller owns every input array; the library copies what it keeps.
 *   - Handles are not thread-safe; free lanes before their graph.
 *   - rs_step_cycles is asynchronous on the lanes' stream unless it writes a
 *     HOST hash buffer; rs_read_signals / rs_write_registers synchronise.
 */
#ifndef RTLSIM_H
#define RTLSIM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RS_OK = 0,
  RS_E_INVALID_ARG = -1,  /* NULL pointer, zero/oversized count, bad option value */
  RS_E_GRAPH = -2,        /* comb. loop, bad arity/width/id/param, multiple or missing driver, bad level */
  RS_E_CAPACITY = -3,     /* > 2^30 rows in a width class, arity > 63, lane count overflow */
  RS_E_OOM = -4,          /* device or host allocation failed */
  RS_E_CUDA = -5,         /* CUDA runtime error (message has the CUDA error string) */
  RS_E_STATE = -6,        /* call order: e.g. staged mode with cycles not staged */
  RS_E_RANGE = -7,        /* lane / signal / cycle index out of range */
  RS_E_UNSUPPORTED = -8   /* valid request this build does not implement */
} rs_status;

/* Opcodes: the interchange format's numbering (same values in synth/circuit.py). */
enum {
  RS_OP_AND = 0, RS_OP_OR = 1, RS_OP_XOR = 2, RS_OP_NOT = 3, RS_OP_ADD = 4, RS_OP_SUB = 5,
  RS_OP_MUL = 6, RS_OP_EQ = 7, RS_OP_LT = 8, RS_OP_SHL = 9, RS_OP_SHR = 10, RS_OP_BITS = 11,
  RS_OP_CAT = 12, RS_OP_MUX = 13, RS_NUM_OPS = 14
};

/* Execution modes for rs_load_graph. */
enum {
  RS_MODE_LANES = 0,   /* many lanes: a CTA owns a lane tile; CTA barrier between levels */
  RS_MODE_SINGLE = 1   /* one lane: ops of a level spread over the grid; grid barrier between levels */
};
/* Flag OR-ed into rs_load_graph's mode: run the compiler's data-level graph passes
 * (§6.1, App. B.1) --
 * constant propagation (ops of constant operands, and a few absorbing cases, become
 * constant signals) and copy propagation (an op whose result always equals an
 * operand's value becomes an alias of it: no row, no evaluation; reads of it read
 * the operand, and its hash weight is folded into the operand's, so every result
 * -- hashes, rs_read_signals, waveforms -- is unchanged).  rs_graph_info reports
 * what was removed. */
#define RS_LOAD_PASSES 0x100u

/* Where a pointer lives. */
enum { RS_MEM_NONE = 0, RS_MEM_HOST = 1, RS_MEM_DEVICE = 2 };

/*
 * Circuit in canonical-id form; signal id = index into width[].
 * Every signal has exactly one driver: an input, a register, a constant or
 * one op.  All arrays are host-side and caller-owned; rs_load_graph copies.
 *   width[n_signals]          1..64 (reading R2)
 *   input_id[n_inputs]        input k = position k (the stimulus index)
 *   reg_id/reg_next_id[n_regs]; reg_init[n_regs] or NULL (-> 0); init is masked
 *   const_id/const_val[n_consts]; values are masked to the width
 *   opcode/out_id[n_ops]; operands of op j are arg_id[arg_off[j] .. arg_off[j+1])
 *     in O-rank order (PAPER.md eq:custom_reduce P:778-796).  Arity: and/or/xor/
 *     add/sub/mul 2..63 (left fold), eq/lt/cat 2, not/shl/shr/bits 1, mux 3
 *     (selector, then O=1 value chosen when selector != 0, then O=2 value).
 *   param[n_ops][2]           shl/shr: [0] = n (n >= 64 gives 0); bits: [0] = hi,
 *                             [1] = lo (lo <= hi <= 63); other ops: ignored.
 *                             cat's w_b is the declared width of operand 1.
 *   level[n_ops] or NULL      optional level per op; must satisfy level(op) >
 *                             level(producer of each operand).  NULL -> ASAP
 *                             levels (§6.1).  Results do not
 *                             depend on levels (§4.2).
 */
typedef struct {
  uint32_t n_signals;  const uint8_t* width;
  uint32_t n_inputs;   const uint32_t* input_id;
  uint32_t n_regs;     const uint32_t* reg_id;   const uint32_t* reg_next_id; const uint64_t* reg_init;
  uint32_t n_consts;   const uint32_t* const_id; const uint64_t* const_val;
  uint32_t n_ops;      const uint8_t* opcode;    const uint32_t* out_id;
                       const uint32_t* arg_off;  const uint32_t* arg_id;
                       const uint32_t* param;    const uint32_t* level;
} rs_graph_desc;

/* Compiled-graph statistics (filled by rs_graph_info). */
typedef struct {
  uint32_t mode;
  uint32_t n_levels;
  uint32_t n_ops;                 /* canonical ops */
  uint32_t n_copy_ops;            /* identity ops the compiler inserted (register -> source next edges) */
  uint32_t n_runs;                /* (level, opcode, arity, out class) runs */
  uint32_t n_coords;
  uint32_t rows[4];               /* rows per width class (1, 2, 4, 8-byte containers) */
  uint64_t state_bytes_per_lane;  /* sum_c rows[c] * 2^c */
  uint64_t graph_device_bytes;    /* bytes of the device graph format */
  uint64_t graph_alg_bytes;       /* G: int32 operand coords + one u32 param word per op */
  uint64_t alg_bytes_per_lane_cycle;  /* SURVEY §8(d) B_alg per lane per cycle, excluding G */
  uint64_t identity_ops_naive;    /* copies a naive §4.2 construction would need */
  uint32_t rows_bit;              /* class-0 rows [0, rows_bit) are the 1-bit signals (bit planes in lane kernel 6) */
  uint32_t n_alias;               /* RS_LOAD_PASSES: ops removed by copy propagation (signals aliased) */
  uint32_t n_folded;              /* RS_LOAD_PASSES: ops removed by constant propagation */
  uint32_t n_mux_chain;           /* RS_LOAD_PASSES: muxes whose else-branch is another mux (counted, not fused) */
} rs_graph_info;

/* Options for rs_alloc_lanes (NULL -> all defaults). */
typedef struct {
  uint64_t lane0;          /* global index of this allocation's first lane (stimulus, hashes) */
  uint32_t lane_tile;      /* RS_MODE_LANES: lanes per CTA tile, 0 = auto, else 8, 16 or 32 (kernel 2)
                              or 32, 64 or 128 (kernel 1) */
  uint32_t threads;        /* threads per CTA, 0 = auto; a multiple of 32, at most the CTA size the kernel's
                              register budget is compiled for: 768 for lane kernels 1 and 6, 640 for lane
                              kernel 2, 896 for lane kernel 7 (768 when it pairs ops: >= 2,048 ops per CTA
                              and level), 1024 single-lane */
  uint32_t stage_cycles;   /* capacity (cycles) of the staged-input ring, 0 = none */
  uint32_t cluster;        /* RS_MODE_LANES: CTAs (a thread-block cluster on as many SMs) sharing one
                              lane tile, 0 = auto, else 1, 2, 4 or 8, or 16 (a non-portable cluster size)
                              for kernel 7 */
  void* stream;            /* cudaStream_t to run on; NULL = a stream the library creates */
  uint32_t parts;          /* RS_MODE_SINGLE level cut: 0/1 = off, else 2..8 partitions,
                              each owning a contiguous level range (balanced by op weight) and a full
                              state replica; partitions hand each cycle on through release/acquire
                              flags and push the signals a later partition reads (cut signals, register
                              values) into its replica.  On one device the partitions are CTA groups of
                              one cooperative launch.  RS_E_CAPACITY if the slices do not fit
                              co-resident, RS_E_INVALID_ARG if parts > n_levels or > 8. */
  uint32_t kernel;         /* RS_MODE_LANES step kernel (results identical): 0 = auto (7 at >= 2048
                              lanes, and for designs with <= 1,024 ops per level at >= 1,024 or
                              <= 256 lanes with 32-lane tiles; else 2); 1 = tile-interleaved: tile = 32 * P lanes (P = 1, 2, 4),
                              thread t owns lanes t + 32k, one op per warp, operand container widths
                              dispatched once per op through a jump table on the class signature;
                              2 = two adjacent lanes per thread, 8/16/32-lane tiles, aligned 64-bit
                              word gathers + extraction; 6 = kernel 1's tiles with the 1-bit signals as
                              bit planes (32 lanes per word); 7 = kernel 1's
                              tiles driven by 32-byte per-op records (one jump into the gather, one
                              into an (opcode, arity, out class) tail).  lane_tile must match (32/64/128
                              for 1 and 7, 8/16/32 for 2, 64/128 for 6).  RS_E_INVALID_ARG otherwise.
                              RS_MODE_SINGLE: 0 = auto (RepCut with one partition when the whole design
                              fits one SM's shared memory, else the level-synchronous grid); 3 = RepCut,
                              shared-memory slices; 4 = RepCut, global replicas; 5 = level-synchronous
                              grid (k_single2; the level cut uses it).
                              Both modes: 8 = the design's own specialised kernel (rs_specialize: every op
                              a straight-line expression with its operands, widths and hash weight baked
                              in, one thread per lane, the SU analog of PAPER.md
                              P:1215-1216); lane_tile 0/32/64/128 sets the state layout only; excludes
                              parts / repcut / part_world and waveform capture.  Errors of rs_specialize. */
  uint32_t repcut;         /* RS_MODE_SINGLE replicated cut (App. C, Cascade 2; SURVEY.md §8(f)
                              NEXT-2): 0 = off, else P >= 1 partitions = CTAs of one cooperative launch; the
                              registers are cut into P contiguous blocks, partition p evaluates the cone of
                              its registers' next values (shared logic replicated) on its own state replica
                              with CTA barriers only, and after each cycle delivers its registers' new
                              values to the partitions that read them (the Register Update Map).  Pays off on
                              designs whose cones barely overlap (e.g. multi-core SoCs).  RS_E_INVALID_ARG
                              if P > n_regs, > 255, > the SMs of the device, or combined with parts.
                              Each partition keeps its working set (op descriptors + a compact copy of the
                              signals it touches) in shared memory when it fits (k_repcut_smem), else works
                              on its state replica in global memory (k_repcut).  P = 1 runs a design that
                              fits one SM's shared memory on a single CTA with CTA barriers only. */
  uint32_t repcut_global;  /* RepCut kernel choice: 0 = auto (shared-memory slices with 8-byte signal
                              slots if they fit, else width-packed slots, else global replicas);
                              1 = global replicas; 2 = width-packed shared-memory slices */
  uint32_t part_world;     /* RS_MODE_SINGLE level cut ACROSS PROCESSES / GPUs: 0 = off,
                              else 2..8 partitions, one per process; this allocation runs partition
                              part_rank only, on its own state replica, and reaches the other partitions'
                              replicas and cycle flags through peer-mapped device memory (CUDA IPC over
                              NVLink: rs_ipc_handle / rs_ipc_connect).  Excludes parts and repcut. */
  uint32_t part_rank;      /* this process's partition, < part_world */
  uint32_t l2_policy;      /* RS_MODE_LANES L2-residency policy (north star: "an L2-residency policy for
                              state"), applied per launch as a CUDA access-policy window: 0 = none;
                              1 = the stage schedule (graph tensor, re-read by every CTA every cycle)
                              persisting; 2 = the signal state persisting (hit ratio = the device's
                              persisting-L2 limit / state bytes, the rest streaming).  Results are
                              identical; only speed differs (measured in DESIGN.md §8). */
  uint32_t defer_state;    /* 1: do not allocate the signal state; the caller binds its own device buffer
                              (e.g. a torch tensor) with rs_lanes_bind_state before stepping, sized by
                              rs_lanes_state_bytes.  Not with part_world. */
  uint32_t op_pairs;       /* RS_MODE_LANES kernel 7: 0 = auto (ops with <= 2 operands evaluated in pairs,
                              both pairs' loads in flight before either is computed, when a CTA has
                              >= 2,048 ops per level), 1 = one op at a time, 2 = pairs (CTAs of at most
                              768 threads).  Results identical.  RS_E_INVALID_ARG if > 2. */
} rs_lane_opts;

typedef struct rs_graph rs_graph;
typedef struct rs_lanes rs_lanes;

const char* rs_version(void);
/* Thread-local message for the last non-RS_OK status (never NULL). */
const char* rs_last_error(void);

/* device value for rs_load_graph: compile and validate only (no device
 * memory; the handle supports rs_graph_info_get / rs_graph_export and
 * rs_free_graph only -- rs_alloc_lanes returns RS_E_STATE). */
#define RS_DEVICE_NONE (-1)

/* Validate + compile the circuit into the GPU graph format (levelize, insert
 * identity copies for register->source next edges, group each level by
 * (opcode, arity, width class) as in PAPER.md Format c P:1123-1129, renumber
 * signals so op outputs are implicit, pack operand coords as int32) and copy
 * it to `device`.  mode: RS_MODE_LANES or RS_MODE_SINGLE. */
rs_status rs_load_graph(const rs_graph_desc* desc, int device, uint32_t mode, rs_graph** out);
rs_status rs_graph_info_get(const rs_graph* g, rs_graph_info* out);

/* Copy one array of the compiled graph format to host memory `out` (or,
 * with out == NULL, only report its element count in *count).  Element
 * types: RUNS = 5 x u32 per run {op_begin, count, coord_begin, out_row0,
 * meta = opcode | arity<<8 | out_class<<16}; OPK = u64; all others u32.
 * For inspection and tests of the format; never needed to simulate. */
enum {
  RS_EXPORT_RUNS = 0, RS_EXPORT_LEVEL_RUN_BEGIN = 1, RS_EXPORT_LEVEL_OP_BEGIN = 2, RS_EXPORT_OPW = 3,
  RS_EXPORT_OPK = 4, RS_EXPORT_COORD_OFF = 5, RS_EXPORT_COORD = 6, RS_EXPORT_SIG_COORD = 7,
  RS_EXPORT_REG_COORD = 8, RS_EXPORT_REG_NEXT_COORD = 9, RS_EXPORT_IN_COORD = 10
};
rs_status rs_graph_export(const rs_graph* g, uint32_t what, void* out, uint64_t* count);
void rs_free_graph(rs_graph* g);

/* RepCut plan statistics for P partitions (host-only; works on a RS_DEVICE_NONE
 * graph): *ops_total = sum of the partitions' op counts (replication factor =
 * ops_total / ops), *max_ops = the largest partition, *push = (register,
 * reader) pairs of the Register Update Map.  Any output may be NULL. */
rs_status rs_repcut_stats(const rs_graph* g, uint32_t P, uint64_t* ops_total, uint32_t* max_ops, uint64_t* push);

/* Level ranges of a `parts`-way level cut (rs_lane_opts.parts):
 * partition k owns levels [cut[k], cut[k+1]); cut[0] = 0, cut[parts] = n_levels,
 * every range non-empty, boundaries balanced by op weight (1 + arity).  `cut`
 * is caller-owned host memory of parts + 1 entries.  Host-only (works on a
 * RS_DEVICE_NONE graph).  RS_E_INVALID_ARG if parts is 0, > 8 or > n_levels. */
rs_status rs_level_cut(const rs_graph* g, uint32_t parts, uint32_t* cut);

/* Per-design specialisation (rs_lane_opts.kernel = 8; §5.2
 * P:1215-1216 "S fully unrolled; OIM embedded in the binary", Tables 4-6): generate the
 * design's step kernel as PTX for sm_100a -- each op of the compiled graph (after
 * RS_LOAD_PASSES, if given) a few register instructions with its operands, widths,
 * parameters and hash weight as immediates, the design's registers held in registers
 * across cycles, one thread per lane -- and load it (the driver JIT-compiles it).  Cached
 * in the graph; rs_alloc_lanes(kernel = 8) calls it.  With RS_DEVICE_NONE it only
 * generates the PTX (see rs_specialized_ptx).
 * Errors: RS_E_CAPACITY above 4,096 ops (ptxas time grows superlinearly with the
 * straight-line cycle: 0.4 s for C1's 256 ops, 25 min for C2's 20k); RS_E_CUDA if the JIT
 * or the module load fails. */
rs_status rs_specialize(rs_graph* g);

/* The PTX rs_specialize generated (host memory, caller-owned): copies at most cap - 1
 * bytes + a NUL into buf (buf may be NULL), *len = the full length.  RS_E_STATE before
 * rs_specialize. */
rs_status rs_specialized_ptx(const rs_graph* g, char* buf, uint64_t cap, uint64_t* len);

/* Allocate the signal state for n_lanes lanes (RS_MODE_SINGLE: n_lanes must
 * be 1), initialised to: registers = init & M(w), constants = value, all
 * other signals 0; the absolute cycle counter = 0; input source = seed 0. */
rs_status rs_alloc_lanes(rs_graph* g, uint32_t n_lanes, const rs_lane_opts* opts, rs_lanes** out);
void rs_free_lanes(rs_lanes* s);
/* Device bytes held by this allocation. */
uint64_t rs_lanes_bytes(const rs_lanes* s);
/* Caller-owned state (rs_lane_opts.defer_state = 1; SURVEY.md §8(b) "torch-owned memory"):
 * rs_lanes_state_bytes = the bytes the signal state needs; rs_lanes_bind_state binds `state`
 * (device memory of the graph's device, 256-byte aligned, >= those bytes, owned by the caller,
 * kept alive until rs_free_lanes) and initialises it (registers = init, constants, all else 0;
 * synchronises the lanes' stream).  Stepping or reading before binding returns RS_E_STATE;
 * RS_E_CAPACITY if the buffer is too small, RS_E_INVALID_ARG if not such device memory. */
uint64_t rs_lanes_state_bytes(const rs_lanes* s);
rs_status rs_lanes_bind_state(rs_lanes* s, void* state, uint64_t bytes);

/* Input source = counter-based stimulus of (seed, input k, absolute cycle,
 * global lane) (reading R13). */
rs_status rs_set_input_seed(rs_lanes* s, uint64_t seed);
/* Input source = staged values for absolute cycles [first_cycle,
 * first_cycle + n_cycles): values[n_cycles][n_inputs][n_lanes] (u64, masked to
 * each input's width when injected), host (on_device = 0) or device memory
 * of the lanes' device (on_device = 1).  n_cycles <= stage_cycles.  The
 * ring keeps the last stage_cycles staged cycles.  Asynchronous, on a copy
 * stream of the allocation: the copy waits for the last launch that read the
 * ring slots it overwrites, and a later rs_step_cycles waits for the copies
 * of its cycles only -- so with a ring of two chunks the next chunk's
 * transfer overlaps the current chunk's simulation.  Pinned host memory must
 * stay valid until the step that reads it has run (rs_sync covers both);
 * device values are copied after all work already queued on the lanes'
 * stream (so a producer kernel on that stream is complete). */
rs_status rs_set_inputs(rs_lanes* s, uint64_t first_cycle, uint32_t n_cycles,
                        const uint64_t* values, int on_device);

/* Advance n_cycles cycles.  hashes: RS_MEM_NONE (no hash computed, pointer
 * ignored), RS_MEM_DEVICE ([n_cycles][n_lanes] u64 on the lanes' device) or
 * RS_MEM_HOST ([n_cycles][n_lanes] u64 host; the call synchronises).
 * H[c][l] = sum over all canonical signals of value * K_s mod 2^64, taken
 * after the combinational evaluation of cycle c and before the commit. */
rs_status rs_step_cycles(rs_lanes* s, uint32_t n_cycles, uint64_t* hashes, int hashes_mem);

/* Read canonical signals ids[n_ids] for lanes [lane_begin, lane_begin+n_lanes)
 * (allocation-relative) into out[n_ids][n_lanes] (host).  Registers hold the
 * committed values; other signals hold the values of the last cycle. Syncs. */
rs_status rs_read_signals(rs_lanes* s, const uint32_t* ids, uint32_t n_ids,
                          uint32_t lane_begin, uint32_t n_lanes, uint64_t* out);
/* Checkpoint restore: overwrite registers reg_ids[n] (canonical ids of
 * registers) for lanes [lane_begin, lane_begin+n_lanes) from values[n][n_lanes]
 * (host, masked).  RS_E_RANGE if an id is not a register. Syncs. */
rs_status rs_write_registers(rs_lanes* s, const uint32_t* reg_ids, uint32_t n,
                             uint32_t lane_begin, uint32_t n_lanes, const uint64_t* values);
rs_status rs_get_cycle(const rs_lanes* s, uint64_t* cycle);
rs_status rs_set_cycle(rs_lanes* s, uint64_t cycle);
/* Kernel launches issued by this allocation so far (evidence counter). */
uint64_t rs_launch_count(const rs_lanes* s);
/* Chosen launch shape: lane tile, threads per CTA, CTAs, CTAs per cluster
 * (any output pointer may be NULL). */
rs_status rs_launch_shape(const rs_lanes* s, uint32_t* lane_tile, uint32_t* threads, uint32_t* ctas,
                          uint32_t* cluster);
/* Step kernel in use: lane mode 1 or 2 (rs_lane_opts.kernel); single-lane mode 3 = RepCut with
 * shared-memory slices (k_repcut_smem), 4 = RepCut on global replicas (k_repcut), 5 = the
 * level-synchronous single-lane grid (k_single2, also the level cut); 0 for NULL. */
uint32_t rs_lanes_kernel(const rs_lanes* s);
rs_status rs_sync(rs_lanes* s);
/* ---- Waveform capture (§6.2: the
 * DMI dumps waveforms of selected signals).  rs_watch selects up to 8192
 * canonical signal ids of an allocation; every later rs_step_cycles then
 * records, fused into the step kernel (lane mode: one extra stage per cycle;
 * single lane: a pass over the watched signals, plus one grid barrier on the
 * level-synchronous grid, after the last level and before the commit), a CHANGE
 * record for each (watched signal, lane) whose value after the combinational
 * evaluation of cycle c -- the snapshot the per-cycle hash covers -- differs
 * from its value at cycle c - 1, and for every (signal, lane) at the first
 * stepped cycle after rs_watch.  Records are appended to a device buffer of
 * `capacity` records in no particular order; records beyond capacity are
 * counted as dropped.  n_ids = 0 stops watching (and frees the buffers).
 * RS_E_RANGE for an unknown id; RS_E_UNSUPPORTED for a level cut (parts > 1)
 * or the global-replica RepCut kernel. */
typedef struct {
  uint64_t cycle;   /* absolute cycle */
  uint64_t lane;    /* global lane id (rs_lane_opts.lane0 + allocation lane) */
  uint32_t watch;   /* index into the rs_watch id list */
  uint32_t pad_;
  uint64_t value;   /* the signal's value at that cycle (masked to its width) */
} rs_change;
rs_status rs_watch(rs_lanes* s, const uint32_t* ids, uint32_t n_ids, uint64_t capacity);
/* Copy the records collected so far to host memory `out` (up to cap; caller-
 * owned) and clear the buffer; *n_out = records copied, *dropped = records
 * lost to capacity since the last read (either pointer may be NULL).
 * Synchronises the lanes' stream. */
rs_status rs_wave_read(rs_lanes* s, rs_change* out, uint64_t cap, uint64_t* n_out, uint64_t* dropped);

/* ---- Level cut across processes / GPUs (rs_lane_opts.part_world > 1; SURVEY.md §8(e) row 2;
 * PAPER.md App. B P:1961-1963 partition synchronisation, App. C Cascade 2's per-cycle exchange
 * P:2053-2059).  Every process loads the same graph, allocates its partition with
 * part_world / part_rank, exports the handle of its replica + cycle flag with rs_ipc_handle
 * (RS_IPC_HANDLE_BYTES bytes, host memory, caller-owned), gathers all ranks' handles (e.g. a
 * torch.distributed all_gather; rank order) and passes them to rs_ipc_connect, which maps the
 * peers' memory (cudaIpcOpenMemHandle; NVLink peer access when the devices differ).  Then
 * rs_step_cycles on every rank advances the single lane: partition k evaluates its level range,
 * stores the cut signals and register values other partitions read straight into their
 * replicas (peer stores) and releases its cycle flag (system scope); partition k + 1 acquires it.
 * hashes (RS_MEM_HOST / DEVICE, [n_cycles] u64) receive THIS partition's share of each cycle's
 * hash (its levels' ops, its registers, and for partition 0 the inputs and constants): the
 * cycle's hash is the sum over ranks mod 2^64.  rs_read_signals reads this rank's replica, which
 * holds the partition's own signals, the registers and inputs.  Partitions wait on one another
 * inside the kernel, so they must run on distinct devices to step freely; ranks that share a
 * device must step one cycle per call, in rank order, with a host barrier between calls (the
 * flags then never wait).  A hash-off step followed by a hash-on step returns RS_E_UNSUPPORTED
 * (the per-partition register carry is only kept by hashed steps).  rs_ipc_connect:
 * RS_E_STATE if not a part_world allocation, RS_E_CUDA if a handle cannot be opened. */
#define RS_IPC_HANDLE_BYTES 64
rs_status rs_ipc_handle(rs_lanes* s, void* handle);
rs_status rs_ipc_connect(rs_lanes* s, const void* handles);

/* Diagnostics (builds with -DRS_TRACE only, else RS_E_UNSUPPORTED): the first
 * call arms a per-stage clock64 trace of CTA 0; later calls copy up to n u64
 * stamps to host `out` (layout: per stage [top, after stage wait, after
 * barrier, work end of each warp]). */
rs_status rs_debug_trace(rs_lanes* s, uint64_t* out, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
