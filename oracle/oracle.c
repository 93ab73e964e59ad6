/*
 * oracle.c -- plain, slow, obviously correct CPU interpreter.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Written from PAPER.md; each
 * function cites the passage it follows.  No blocking, fusion or reordering
 * beyond the plain definition: per lane, per cycle, inject -> evaluate every
 * op in a topological order -> hash -> simultaneous register commit.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* M(w): DESIGN.md reading R2 ("width masking to 64 bits", BASELINE.json
 * north_star).  w == 64 must not shift by 64 (undefined in C). */
uint64_t orc_mask(uint32_t w) {
  if (w >= 64) return ~(uint64_t)0;
  return (((uint64_t)1) << w) - 1;
}

/* splitmix64 (public algorithm): state += golden gamma; output = mix(state). */
uint64_t orc_splitmix_next(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* Reading R13: "uniform-random values per cycle" (BASELINE.json configs)
 * as a counter-based function of (seed, input index, cycle, global lane). */
uint64_t orc_stimulus(uint64_t seed, uint64_t k, uint64_t c, uint64_t lane) {
  uint64_t x = orc_splitmix_next(seed);
  x = orc_splitmix_next(x + k);
  x = orc_splitmix_next(x + c);
  x = orc_splitmix_next(x + lane);
  return x;
}

/* Reading R12: K_s odd, so a single differing signal always changes H. */
uint64_t orc_hash_weight(uint64_t s) {
  return orc_splitmix_next(0x5EED000000000000ULL + s) | 1ULL;
}

/*
 * op_u / op_r / op_s of Cascade 1 (box:einsum P:950-952) for one op.
 *   reducible ops: fold op_r over the O rank in ascending o (Alg. opn
 *     P:753-775; O-rank order P:778-788): cur = op_r(prev, map_tmp).
 *   unary ops: the map compute operator op_u (eq:step4c P:826-830).
 *   select op: op_s on the whole O fiber; O=0 is the selector choosing O=1
 *     or O=2 (App. A); nonzero selects O=1 (reading R4).
 * Operator meanings beyond "multiply" and mux are not defined in the paper;
 * they follow FIRRTL unsigned semantics (reading R1).
 */
uint64_t orc_apply_op(uint32_t opcode, uint32_t n, const uint64_t* x,
                      uint32_t p0, uint32_t p1, uint32_t wb, uint32_t w_out, int* ok) {
  uint64_t r = 0;
  uint32_t o;
  *ok = 1;
  switch (opcode) {
    case ORC_AND: case ORC_OR: case ORC_XOR: case ORC_ADD: case ORC_SUB: case ORC_MUL:
      if (n < 2) { *ok = 0; return 0; }
      r = x[0];                       /* o = 0: reduce temporary := map temporary */
      for (o = 1; o < n; ++o) {       /* o ascending: cur = op_r(prev, map_tmp) */
        switch (opcode) {
          case ORC_AND: r = r & x[o]; break;
          case ORC_OR:  r = r | x[o]; break;
          case ORC_XOR: r = r ^ x[o]; break;
          case ORC_ADD: r = r + x[o]; break;     /* mod 2^64 */
          case ORC_SUB: r = r - x[o]; break;     /* left fold: ((x0-x1)-x2)... */
          default:      r = r * x[o]; break;     /* low 64 bits */
        }
      }
      break;
    case ORC_EQ:
      if (n != 2) { *ok = 0; return 0; }
      r = (x[0] == x[1]) ? 1 : 0;
      break;
    case ORC_LT:
      if (n != 2) { *ok = 0; return 0; }
      r = (x[0] < x[1]) ? 1 : 0;      /* unsigned */
      break;
    case ORC_NOT:
      if (n != 1) { *ok = 0; return 0; }
      r = ~x[0];                      /* reading R3: then masked to w_out */
      break;
    case ORC_SHL:
      if (n != 1) { *ok = 0; return 0; }
      r = (p0 >= 64) ? 0 : (x[0] << p0);   /* reading R5 */
      break;
    case ORC_SHR:
      if (n != 1) { *ok = 0; return 0; }
      r = (p0 >= 64) ? 0 : (x[0] >> p0);
      break;
    case ORC_BITS:                    /* p0 = hi, p1 = lo, lo <= hi <= 63 */
      if (n != 1 || p1 > p0 || p0 > 63) { *ok = 0; return 0; }
      r = (x[0] >> p1) & orc_mask(p0 - p1 + 1);
      break;
    case ORC_CAT:                     /* x0 is the high part; wb = width(x1) */
      if (n != 2) { *ok = 0; return 0; }
      r = (wb >= 64) ? x[1] : ((x[0] << wb) | x[1]);
      break;
    case ORC_MUX:
      if (n != 3) { *ok = 0; return 0; }
      r = (x[0] != 0) ? x[1] : x[2];
      break;
    default:
      *ok = 0;
      return 0;
  }
  return r & orc_mask(w_out);
}

/* Levelization "via topological sort" (§6.1) -- here only an
 * evaluation order: Kahn's algorithm over op -> op dependencies. */
int orc_topo_order(const orc_circuit* g, uint32_t* order) {
  const uint32_t NS = g->n_signals, NO = g->n_ops;
  int64_t* drv = (int64_t*)malloc(sizeof(int64_t) * (NS ? NS : 1)); /* -2 none, -1 source, >=0 op */
  uint32_t* indeg = (uint32_t*)calloc(NO ? NO : 1, sizeof(uint32_t));
  uint32_t* cnt = (uint32_t*)calloc((size_t)NS + 1, sizeof(uint32_t));
  uint32_t* users = NULL;
  uint32_t* queue = order;
  uint32_t i, j, head = 0, tail = 0;
  int rc = 0;
  for (i = 0; i < NS; ++i) drv[i] = -2;
#define CLAIM(s, v) do { if ((s) >= NS || drv[(s)] != -2) { rc = -1; goto done; } drv[(s)] = (v); } while (0)
  for (i = 0; i < g->n_inputs; ++i) CLAIM(g->input_id[i], -1);
  for (i = 0; i < g->n_regs; ++i) CLAIM(g->reg_id[i], -1);
  for (i = 0; i < g->n_consts; ++i) CLAIM(g->const_id[i], -1);
  for (j = 0; j < NO; ++j) CLAIM(g->out_id[j], (int64_t)j);
#undef CLAIM
  for (i = 0; i < NS; ++i) if (drv[i] == -2) { rc = -1; goto done; }
  for (i = 0; i < g->n_regs; ++i) if (g->reg_next_id[i] >= NS) { rc = -1; goto done; }
  for (j = 0; j < NO; ++j) {
    if (g->opcode[j] >= ORC_NUM_OPS || g->arg_off[j + 1] < g->arg_off[j]) { rc = -3; goto done; }
    for (i = g->arg_off[j]; i < g->arg_off[j + 1]; ++i) {
      uint32_t s = g->arg_id[i];
      if (s >= NS) { rc = -3; goto done; }
      if (drv[s] >= 0) { indeg[j]++; cnt[s]++; }
    }
  }
  /* CSR of signal -> consuming ops */
  {
    uint32_t* off = (uint32_t*)calloc((size_t)NS + 1, sizeof(uint32_t));
    uint32_t* fill;
    for (i = 0; i < NS; ++i) off[i + 1] = off[i] + cnt[i];
    users = (uint32_t*)malloc(sizeof(uint32_t) * (off[NS] ? off[NS] : 1));
    fill = (uint32_t*)calloc((size_t)NS + 1, sizeof(uint32_t));
    for (j = 0; j < NO; ++j)
      for (i = g->arg_off[j]; i < g->arg_off[j + 1]; ++i) {
        uint32_t s = g->arg_id[i];
        if (drv[s] >= 0) users[off[s] + fill[s]++] = j;
      }
    for (j = 0; j < NO; ++j) if (indeg[j] == 0) queue[tail++] = j;
    while (head < tail) {
      uint32_t op = queue[head++], s = g->out_id[op];
      for (i = off[s]; i < off[s + 1]; ++i)
        if (--indeg[users[i]] == 0) queue[tail++] = users[i];
    }
    free(off);
    free(fill);
    if (tail != NO) rc = -2;
  }
done:
  free(drv);
  free(indeg);
  free(cnt);
  free(users);
  return rc;
}

int orc_simulate(const orc_circuit* g, uint64_t seed, const uint64_t* staged,
                 const uint64_t* reg_state0, uint64_t cycle0, uint32_t n_cycles,
                 uint64_t lane0, uint32_t n_lanes,
                 uint64_t* hashes, const uint32_t* watch, uint32_t n_watch,
                 uint64_t* trace, uint64_t* final_state) {
  const uint32_t NS = g->n_signals, NO = g->n_ops;
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (NO ? NO : 1));
  uint64_t* v = (uint64_t*)malloc(sizeof(uint64_t) * (NS ? NS : 1));
  uint64_t* K = (uint64_t*)malloc(sizeof(uint64_t) * (NS ? NS : 1));
  uint64_t* t = (uint64_t*)malloc(sizeof(uint64_t) * (g->n_regs ? g->n_regs : 1));
  uint64_t x[64];
  uint32_t l, c, i, j;
  int rc = orc_topo_order(g, order);
  if (rc != 0) goto out;
  for (i = 0; i < NS; ++i) K[i] = orc_hash_weight(i);
  for (l = 0; l < n_lanes; ++l) {
    /* init: everything 0, registers at init, constants at their value */
    memset(v, 0, sizeof(uint64_t) * NS);
    for (i = 0; i < g->n_regs; ++i) {
      uint64_t init = reg_state0 ? reg_state0[(size_t)i * n_lanes + l]
                                 : (g->reg_init ? g->reg_init[i] : 0);
      v[g->reg_id[i]] = init & orc_mask(g->width[g->reg_id[i]]);
    }
    for (i = 0; i < g->n_consts; ++i)
      v[g->const_id[i]] = g->const_val[i] & orc_mask(g->width[g->const_id[i]]);
    for (c = 0; c < n_cycles; ++c) {
      /* (1) input injection: testbench values into LI (§2.1, §6.2) */
      for (i = 0; i < g->n_inputs; ++i) {
        uint32_t s = g->input_id[i];
        uint64_t val = staged ? staged[((size_t)c * g->n_inputs + i) * n_lanes + l]
                              : orc_stimulus(seed, i, cycle0 + c, lane0 + l);
        v[s] = val & orc_mask(g->width[s]);
      }
      /* (2) every op in dependency order: gather (eq:split_einsum1 P:809-812),
       *     op_u / op_r / op_s (eq:step4c, eq:step5b), write LI[s] (Alg. RU) */
      for (j = 0; j < NO; ++j) {
        uint32_t op = order[j], a0 = g->arg_off[op], n = g->arg_off[op + 1] - a0, wb = 0;
        int ok;
        if (n > 64) { rc = -3; goto out; }
        for (i = 0; i < n; ++i) x[i] = v[g->arg_id[a0 + i]];
        if (n >= 2) wb = g->width[g->arg_id[a0 + 1]];
        v[g->out_id[op]] = orc_apply_op(g->opcode[op], n, x, g->param[2 * op],
                                        g->param[2 * op + 1], wb, g->width[g->out_id[op]], &ok);
        if (!ok) { rc = -3; goto out; }
      }
      /* (3) per-cycle hash over all signals, pre-commit (reading R12) */
      if (hashes) {
        uint64_t h = 0;
        for (i = 0; i < NS; ++i) h += v[i] * K[i];
        hashes[(size_t)c * n_lanes + l] = h;
      }
      if (trace)
        for (i = 0; i < n_watch; ++i)
          trace[((size_t)c * n_watch + i) * n_lanes + l] = v[watch[i]];
      /* (4) simultaneous register commit (Fig. 1 caption P:187; reading R8) */
      for (i = 0; i < g->n_regs; ++i)
        t[i] = v[g->reg_next_id[i]] & orc_mask(g->width[g->reg_id[i]]);
      for (i = 0; i < g->n_regs; ++i) v[g->reg_id[i]] = t[i];
    }
    if (final_state)
      for (i = 0; i < NS; ++i) final_state[(size_t)i * n_lanes + l] = v[i];
  }
out:
  free(order);
  free(v);
  free(K);
  free(t);
  return rc;
}
