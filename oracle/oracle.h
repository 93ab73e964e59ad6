/*
 * oracle.h -- plain CPU reference interpreter for the RTeAAL Sim hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2601_18140_b200/) never links, imports or calls it.
 *
 * What it computes (DESIGN.md §"Oracle"):
 *   The cascade of PAPER.md Cascade 1 (box:einsum) plus register
 *   commit (Fig. 1 caption P:187) and input injection (§6.2)
 *   computes exactly the synchronous-circuit semantics: every cycle each
 *   combinational op is evaluated on its operands in dependency order, then
 *   every register simultaneously takes its next value.  Levelization and
 *   identity elision change traversal, never results (§4.2 P:900-904,
 *   §4.3).  This file is that plain definition written out:
 *   a topological interpreter with no OIM, no levels and no code shared
 *   with the CUDA path.
 *
 * Opcode numbers are the interchange format's (same values as
 * include/rtlsim.h and synth/circuit.py; written independently here).
 */
#ifndef RTL_ORACLE_H
#define RTL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_AND = 0, ORC_OR = 1, ORC_XOR = 2, ORC_NOT = 3, ORC_ADD = 4, ORC_SUB = 5,
  ORC_MUL = 6, ORC_EQ = 7, ORC_LT = 8, ORC_SHL = 9, ORC_SHR = 10, ORC_BITS = 11,
  ORC_CAT = 12, ORC_MUX = 13, ORC_NUM_OPS = 14
};

typedef struct {
  uint32_t n_signals; const uint8_t* width;            /* [n_signals], 1..64 */
  uint32_t n_inputs;  const uint32_t* input_id;         /* [n_inputs] */
  uint32_t n_regs;    const uint32_t* reg_id;           /* [n_regs] */
                      const uint32_t* reg_next_id;      /* [n_regs] */
                      const uint64_t* reg_init;         /* [n_regs] or NULL */
  uint32_t n_consts;  const uint32_t* const_id;         /* [n_consts] */
                      const uint64_t* const_val;        /* [n_consts] */
  uint32_t n_ops;     const uint8_t* opcode;            /* [n_ops] */
                      const uint32_t* out_id;           /* [n_ops] */
                      const uint32_t* arg_off;          /* [n_ops+1] */
                      const uint32_t* arg_id;           /* [arg_off[n_ops]] */
                      const uint32_t* param;            /* [n_ops][2] */
} orc_circuit;

/* M(w) = 2^w - 1 for w in 1..64 (2^64-1 at w = 64). */
uint64_t orc_mask(uint32_t w);

/* splitmix64 generator step as a pure function of the state x:
 * returns the output for state x + 0x9E3779B97F4A7C15 (Steele, Lea, Flood,
 * "Fast splittable pseudorandom number generators", OOPSLA 2014). */
uint64_t orc_splitmix_next(uint64_t x);

/* Stimulus of input k (index into input_id) at absolute cycle c for global
 * lane l, before masking: DESIGN.md reading R13. */
uint64_t orc_stimulus(uint64_t seed, uint64_t k, uint64_t c, uint64_t lane);

/* Hash weight K_s of canonical signal s (odd): DESIGN.md reading R12. */
uint64_t orc_hash_weight(uint64_t s);

/* One op: x[0..n-1] are the operand values in O order (PAPER.md
 * eq:custom_reduce P:778-796), wb = declared width of operand 1 (cat only).
 * Result is masked to w_out.  Returns 0 and sets *ok=0 for an unknown
 * opcode or bad arity. */
uint64_t orc_apply_op(uint32_t opcode, uint32_t n, const uint64_t* x,
                      uint32_t p0, uint32_t p1, uint32_t wb, uint32_t w_out, int* ok);

/* Topological order of the ops (Kahn).  Returns 0 on success, -1 if some
 * signal has != 1 driver, -2 on a combinational loop, -3 on a bad op. */
int orc_topo_order(const orc_circuit* g, uint32_t* order /* [n_ops] */);

/*
 * Simulate lanes [lane0, lane0+n_lanes) for cycles [cycle0, cycle0+n_cycles).
 *   staged      : NULL -> stimulus from (seed, k, c, lane); else values
 *                 [n_cycles][n_inputs][n_lanes] (masked to the input width)
 *   reg_state0  : NULL -> registers start at reg_init & M(w); else
 *                 [n_regs][n_lanes] start values (masked)
 *   hashes      : NULL or [n_cycles][n_lanes]: H[c,l] = sum_s v_s*K_s mod 2^64
 *                 over all signals after the combinational evaluation of
 *                 cycle c, before the register commit (reading R12)
 *   watch/trace : NULL or trace[n_cycles][n_watch][n_lanes] = pre-commit
 *                 value of signal watch[i] at each cycle
 *   final_state : NULL or [n_signals][n_lanes]: values after the last
 *                 commit; non-register signals hold their last-cycle values
 * Returns 0 or the negative orc_topo_order error.
 */
int orc_simulate(const orc_circuit* g, uint64_t seed, const uint64_t* staged,
                 const uint64_t* reg_state0, uint64_t cycle0, uint32_t n_cycles,
                 uint64_t lane0, uint32_t n_lanes,
                 uint64_t* hashes, const uint32_t* watch, uint32_t n_watch,
                 uint64_t* trace, uint64_t* final_state);

#ifdef __cplusplus
}
#endif
#endif
