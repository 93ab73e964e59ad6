// compiler.hpp -- host graph-tensor compiler.
//
// Turns an rs_graph_desc (canonical ids) into the GPU graph format:
//   * levelization (§4.2; §6.1 P:1266 "slicing the graph
//     into layers via topological sort");
//   * identity elision by coordinate assignment (§4.3 P:1030-1039,
//     P:1272-1273): every signal keeps ONE row for the whole cycle, so no
//     identity copies are stored; the only copies inserted are for register
//     next edges that point at a source (an input or a register), which the
//     single-pass commit of the kernel needs (DESIGN.md §"Register commit");
//   * Format-c swizzle (§5.1, alg:NU P:1171-1174): each level's
//     ops grouped into runs by (opcode, arity, width class) so a warp never
//     diverges on the op, and each run writes consecutive rows of its class
//     (the S coordinate array vanishes: out rows are implicit);
//   * operand coordinates (the R coordinates of OIM) packed as int32:
//     bits 31..30 = width class, bits 29..0 = row in that class array.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rtlsim.h"

namespace rtlsim {

constexpr uint32_t OP_COPY = 14;         // internal identity op (never in a desc)
constexpr uint32_t ROW_MASK = 0x3FFFFFFFu;
constexpr uint32_t MAX_ROWS = 1u << 30;
constexpr uint32_t MAX_ARITY = 63;

inline uint32_t width_class(uint32_t w) { return w <= 8 ? 0 : w <= 16 ? 1 : w <= 32 ? 2 : 3; }
inline uint32_t make_coord(uint32_t cls, uint32_t row) { return (cls << 30) | row; }

// Param word of one op (u32):
//   [6:0] w_out  [13:7] p0  [19:14] p1  [21:20] out class  [25:22] opcode  [31:26] arity
//   p0 = shl/shr amount clamped to 64 | bits hi | cat w_b;  p1 = bits lo.
inline uint32_t pack_pw(uint32_t w_out, uint32_t p0, uint32_t p1, uint32_t cls, uint32_t op,
                        uint32_t arity) {
  return (w_out & 127u) | ((p0 & 127u) << 7) | ((p1 & 63u) << 14) | ((cls & 3u) << 20) |
         ((op & 15u) << 22) | ((arity & 63u) << 26);
}

struct DevRun {            // one (level, opcode, arity, kind, out class) run
  uint32_t op_begin;       // index of the run's first op in the per-op arrays
  uint32_t count;
  uint32_t coord_begin;    // index of the first operand coord
  uint32_t out_row0;       // first output row in the out class array
  uint32_t meta;           // opcode | arity << 8 | out_cls << 16 | kind << 18 (kind: 0 all-1-bit, 1 1-bit out, 2 wider)
};

struct CompiledGraph {
  uint32_t mode = 0;
  uint32_t n_signals = 0, n_inputs = 0, n_regs = 0, n_consts = 0;
  uint32_t n_ops = 0, n_copy = 0, n_levels = 0;
  uint32_t rows[4] = {0, 0, 0, 0};
  uint32_t rows_bit = 0;            // class-0 rows [0, rows_bit) are exactly the 1-bit signals
  // graph passes (RS_LOAD_PASSES): canonical id -> representative (itself, or the
  // signal an alias reads), ops removed as aliases / folded to constants, mux chains
  std::vector<uint32_t> sig_rep;
  uint32_t n_alias = 0, n_folded = 0, n_mux_chain = 0, n_ops_input = 0;
  // per-op arrays in device order (level-major, run-major)
  std::vector<uint32_t> opw;        // param word
  std::vector<uint64_t> opk;        // hash weight of the op's output (0 for copies)
  std::vector<uint32_t> coord_off;  // [n_ops_total + 1]
  std::vector<uint32_t> coord;      // packed operand coords
  std::vector<DevRun> runs;
  std::vector<uint32_t> level_run_begin;  // [n_levels + 1]
  std::vector<uint32_t> level_op_begin;   // [n_levels + 1]
  // inputs (stimulus index k = position)
  std::vector<uint32_t> in_coord;
  std::vector<uint32_t> in_w;
  std::vector<uint64_t> in_k;
  // registers (latch)
  std::vector<uint32_t> reg_coord, reg_next_coord, reg_w;
  std::vector<uint64_t> reg_k, reg_init;
  // constants
  std::vector<uint32_t> const_coord;
  std::vector<uint64_t> const_val;
  // canonical id -> coord; kind 0 input 1 reg 2 const 3 op
  std::vector<uint32_t> sig_coord;
  std::vector<uint8_t> sig_kind;
  std::vector<int32_t> sig_reg_index;
  uint64_t const_hash = 0;
  uint64_t init_reg_hash = 0;
  // statistics
  uint64_t alg_bytes_per_lane_cycle = 0;
  uint64_t graph_alg_bytes = 0;
  uint64_t identity_ops_naive = 0;

  uint32_t n_ops_total() const { return (uint32_t)opw.size(); }
  uint64_t state_bytes_per_lane() const {
    return (uint64_t)rows[0] + 2ull * rows[1] + 4ull * rows[2] + 8ull * rows[3];
  }
  uint64_t device_bytes() const;
};

// splitmix64 (public algorithm; independent implementation of DESIGN.md R12/R13)
inline uint64_t splitmix_next(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t hash_weight(uint64_t s) { return splitmix_next(0x5EED000000000000ull + s) | 1ull; }
inline uint64_t width_mask(uint32_t w) { return w >= 64 ? ~0ull : ((1ull << w) - 1ull); }

// Returns RS_OK or an error status with *err set.  mode: RS_MODE_LANES or
// RS_MODE_SINGLE, optionally | RS_LOAD_PASSES (constant / copy propagation,
// passes.cpp).
rs_status compile_graph(const rs_graph_desc* d, uint32_t mode, CompiledGraph* out, std::string* err);

// ---------------------------------------------------------------- graph passes (NEXT-1)
// Result of run_passes: the rewritten circuit (surviving ops, operands renamed to
// their representatives, folded signals turned into constants) plus, per
// canonical signal, its representative (itself unless it became an alias).
struct PassResult {
  std::vector<uint32_t> rep;       // [n_signals]
  std::vector<uint32_t> folded;    // signals turned into constants
  uint32_t n_alias = 0, n_mux_chain = 0;
  std::vector<uint8_t> width, opcode;
  std::vector<uint32_t> input_id, reg_id, reg_next_id, const_id, out_id, arg_off, arg_id, param, level, cat_wb;
  std::vector<uint64_t> reg_init, const_val;
  rs_graph_desc desc;              // points into the vectors above
};
// topo: the ops in a topological order.
void run_passes(const rs_graph_desc* d, const std::vector<int64_t>& drv, const std::vector<uint32_t>& topo,
                PassResult* out);

// ---------------------------------------------------------------- stages
// The lane kernel walks a fixed per-cycle schedule of *stages*; each stage's
// descriptors live in one contiguous, 16-byte aligned block of the stage blob
// so a single TMA bulk copy (cp.async.bulk) brings it into shared memory,
// prefetched one stage ahead.  Schedule per cycle:
//   INJECT chunks (inputs) | OPS chunks, level by level | LATCH chunks (registers)
// with a CTA barrier after every stage.  A level larger than one stage is
// split into several OPS stages (barrier after each; only the last one ends
// the level, but an extra barrier is harmless).
enum StageType : uint32_t { ST_INJECT = 1, ST_OPS = 2, ST_LATCH = 3, ST_NOP = 4, ST_WATCH = 6 };

struct StageHdr {          // first 64 bytes of a stage block
  uint32_t type;
  uint32_t n;              // ops / inputs / registers in the stage
  uint32_t n_runs;
  uint32_t n_coords;
  uint32_t first;          // index of the first input / register / op (global numbering)
  uint32_t level;
  uint32_t off_w;          // u32[n]: op param words / input widths / register widths
  uint32_t off_k;          // u64[n]: hash weights
  uint32_t off_c;          // u32[..]: op operand coords | input coords | (next, reg) coord pairs
  uint32_t off_runs;       // StageRun[n_runs]
  uint32_t bytes;
  uint32_t n_items;        // OPS: work items (run-aligned batches of <= `batch` ops)
  uint32_t off_items;      // u32[n_items]: run << 16 | (count - 1) << 13 | first op (stage-relative)
  uint32_t pad[3];
};

// Ops per work item of an OPS stage: kernel 2's gather batch (its items never
// hold more), and kernel 1's default; kernel 1 takes items of kBatchWide ops
// when a CTA has many ops per level (build_stages' `batch`; runtime.cu).
#ifndef RS_BATCH
#define RS_BATCH 2
#endif
constexpr uint32_t kBatch = RS_BATCH;   // <= 8 (3-bit count field of a work item)
#ifndef RS_BATCH_WIDE
#define RS_BATCH_WIDE 4
#endif
constexpr uint32_t kBatchWide = RS_BATCH_WIDE;  // <= 8

struct StageRun {          // a run clipped to the stage; indices relative to the stage
  uint32_t op_begin;
  uint32_t count;
  uint32_t coord_begin;
  uint32_t out_row0;
  uint32_t meta;           // opcode | arity << 8 | out_cls << 16
  uint32_t pad[3];
};

struct StageRef {
  uint64_t off;            // byte offset of the block in the blob
  uint32_t bytes;
  uint32_t type;
};

// Build the per-cycle stage schedule with blocks of at most stage_bytes.
void build_stages(const CompiledGraph& g, uint32_t stage_bytes, uint32_t batch, std::vector<uint8_t>* blob,
                  std::vector<StageRef>* table);

// ---------------------------------------------------------------- single-lane slices
// Single-lane mode: CTA g of a G-CTA persistent grid owns a fixed contiguous
// chunk of every level's ops (and of the registers / inputs); its descriptors
// stay resident in shared memory for the whole launch.  Layout of one slice
// (16-byte aligned sections, offsets in SliceHdr):
//   head: SliceLvl[n_levels] | SliceSeg[...] | pw u32[ops] | coords u32[...]
//   tail: push {coord, dmask} u32x2[n_push]
//         | latch {next coord, reg coord, w | own << 7 | dmask << 8, reg index} u32x4[n_latch]
//         | inject {coord, width} u32x2[n_inj]
// The head (read every level) must fit shared memory; the tail (read once
// per cycle, coalesced) is copied there too when every slice fits whole,
// else it is streamed from global memory (L2).
//
// Level cut: with P > 1 partitions, partition k owns the
// contiguous level range [level_cut[k], level_cut[k+1]) (balanced by op
// weight) and keeps a full replica of the signal state.  Its slices hold
// only its levels; its latch list holds every register whose next value is
// produced by a partition <= k (the register's owner), own == 1 for its own
// registers, whose new value it also pushes to the replicas in dmask (the
// partitions < k, which have finished the cycle); its push list holds the
// op outputs it produces that a later partition reads (operands, or the next
// value of a register that partition latches), dmask = the consumers.
struct SliceHdr {
  uint32_t bytes;
  uint32_t n_levels;
  uint32_t off_lvl, off_seg, off_pw, off_push, off_coord, off_latch, off_inj;
  uint32_t n_push, n_latch;
  uint32_t inj_first, n_inj;       // inputs [inj_first, inj_first + n_inj)
  uint32_t part;                   // level-cut partition of the slice
  uint32_t head_bytes;             // bytes of the head (= off_push)
  uint32_t pad;
};
constexpr uint32_t kMaxParts = 8;
struct SliceLvl {
  uint32_t op_begin;   // global op index of the chunk's first op (hash weights)
  uint32_t n;          // ops in the chunk
  uint32_t pw_base;    // index of its first op in the slice's pw / cofs arrays
  uint32_t coord_base; // index of its first coord in the slice's coords array
  uint32_t seg_begin, n_seg;
  uint32_t pad[2];
};
struct SliceSeg {      // a run piece inside a chunk: one arity, outputs consecutive rows of one class
  uint32_t first;      // chunk-relative index of the piece's first op
  uint32_t count;
  uint32_t out_coord0; // (class << 30) | row of the first op's output
  uint32_t coord0;     // first coord of the piece, relative to the level's coord_base (arity-strided)
};
// Level ranges of P partitions balanced by op weight (1 + arity): [cut[k], cut[k+1]).
std::vector<uint32_t> level_cut(const CompiledGraph& g, uint32_t P);
// Partition (of `cut`) that produces each signal row, per class (sources: 0).
void row_owner(const CompiledGraph& g, const std::vector<uint32_t>& cut, std::vector<uint8_t> owner[4]);
// Slices of P partitions x Gp CTAs (partition-major).  Returns false (and
// builds nothing) if a slice head would exceed max_bytes.
bool build_single_slices(const CompiledGraph& g, uint32_t P, uint32_t Gp, uint32_t max_bytes,
                         std::vector<uint8_t>* blob, std::vector<uint64_t>* slice_off);

// ---------------------------------------------------------------- RepCut
// Replicated-cut partitioning for single-lane simulation (SURVEY.md §8(f)
// NEXT-2; App. C, Cascade 2 P:2021-2078): registers are split into P
// contiguous blocks; partition p evaluates the combinational cone of its
// registers' next values (ops shared between cones are replicated), keeps its
// own state replica, and after every cycle pushes each of its registers'
// new values into the replicas of the partitions that read it -- the Register
// Update Map (RUM) of Cascade 2's last Einsum.  Every op is hashed by exactly
// one partition (its lowest-numbered holder); ops outside every cone are
// given to partition (op index mod P) with their own cones.
struct RepCutPlan {
  uint32_t P = 0;
  std::vector<uint32_t> lvl_begin;   // [P][n_levels + 1]: offsets into ops (partition-major)
  std::vector<uint32_t> ops;         // device op index | owned << 31, per partition in level order
  std::vector<uint32_t> reg_begin;   // [P + 1]
  std::vector<uint32_t> regs;        // register indices, partition-major
  std::vector<uint32_t> push_begin;  // [P + 1]
  std::vector<uint32_t> push;        // (register index, reader partition) pairs, by owner partition
  std::vector<uint8_t> sig_owner;    // [n_signals]: the partition whose replica holds the signal's value
  uint64_t ops_total = 0;            // sum of partition op counts (replication = ops_total / n_ops_total)
  uint32_t max_ops = 0;              // largest partition
};
// Returns false (with *err) if P is 0, > 255 or > the number of registers.
bool build_repcut(const CompiledGraph& g, uint32_t P, RepCutPlan* out, std::string* err);

// Partition-local RepCut slices (repcut.cuh k_repcut_smem): partition p keeps
// the values of the signals it touches (its ops' outputs and operands, its
// registers, the inputs it reads or owns) in shared memory, renumbered into a
// compact local state of byte offsets < 64 KiB -- u64 region first, then u32,
// u16, u8, so an offset's width class follows from three comparisons -- and
// its op descriptors next to them.  Registers cross partitions through a
// global mailbox (value by register index): owners post after the commit,
// readers pull after the one grid barrier per cycle.  Layout of one slice
// (16-byte aligned sections, offsets relative to the slice; the smem part is
// [0, smem_bytes), the map is read from global memory at launch start / end):
//   lvl u32[n_levels + 1] | pw u32[ops] | cw u16x4[ops] {out, c0, c1, c2 | ovf index}
//   | ovf u16[...] (operands 2.. of ops with arity > 3) | commit u32x4[n_commit]
//   {reg | next << 16, register index | width << 24, hash weight lo, hi}
//   | pull u32x2[n_pull] {local, register index}
//   | inject u32x4[n_inj] {local | width << 16, input index, hash weight lo, hi (0: not owned)}
//   | [kop u64[ops]: the op hash weights, when they fit]
//   | (state: state_bytes at state_off, not in the blob) | map u32x2[n_map] {local, coord}
struct RepSliceHdr {
  uint32_t smem_bytes;    // bytes copied to shared memory (16-aligned)
  uint32_t state_off;     // shared-memory offset of the local state (16-aligned; = smem_bytes)
  uint32_t state_bytes;   // 16-aligned
  uint32_t b1, b2, b3;    // local offsets where the u32 / u16 / u8 regions start
  uint32_t n_levels, n_ops;
  uint32_t off_lvl, off_pw, off_cw, off_ovf;
  uint32_t off_commit, n_commit, off_pull, n_pull;
  uint32_t off_inj, n_inj, off_map, n_map;
  uint32_t k_base;        // first entry of the partition in the op hash-weight array
  uint32_t max_level;     // largest level of the partition (ops)
  uint32_t off_kop;       // u64[ops]: op hash weights in shared memory (kop_smem), else in global memory
  uint32_t kop_smem;
  uint32_t wide;          // every local signal in an 8-byte slot (no width-class logic in the gathers)
  uint32_t pad_[3];
};
// Builds the P slices of `plan` (blob, slice offsets) and the per-partition op
// hash weights (owned ops: opk, else 0) in slice op order.  in_owner[k] = the
// partition that hashes input k (and whose replica holds it for read-back).
// Returns false (with *err) if a slice's smem part + local state exceeds
// max_smem or its local state exceeds 64 KiB.
// wide: 8-byte slots for every local signal (faster gathers; fails sooner).
bool build_repcut_slices(const CompiledGraph& g, const RepCutPlan& plan, uint32_t max_smem, bool wide,
                         std::vector<uint8_t>* blob, std::vector<uint64_t>* slice_off,
                         std::vector<uint64_t>* op_k, std::vector<uint8_t>* in_owner, std::string* err);

}  // namespace rtlsim
