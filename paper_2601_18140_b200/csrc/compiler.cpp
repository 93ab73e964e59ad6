// compiler.cpp -- see compiler.hpp.
#include "compiler.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <functional>
#include <unordered_map>

namespace rtlsim {

uint64_t CompiledGraph::device_bytes() const {
  return opw.size() * 4ull + opk.size() * 8ull + coord_off.size() * 4ull + coord.size() * 4ull +
         runs.size() * sizeof(DevRun) + (level_run_begin.size() + level_op_begin.size()) * 4ull +
         in_coord.size() * 16ull + reg_coord.size() * 28ull;
}

namespace {

bool fixed_arity_ok(uint32_t op, uint32_t n) {
  switch (op) {
    case RS_OP_AND: case RS_OP_OR: case RS_OP_XOR: case RS_OP_ADD: case RS_OP_SUB: case RS_OP_MUL:
      return n >= 2 && n <= MAX_ARITY;
    case RS_OP_EQ: case RS_OP_LT: case RS_OP_CAT: return n == 2;
    case RS_OP_NOT: case RS_OP_SHL: case RS_OP_SHR: case RS_OP_BITS: return n == 1;
    case RS_OP_MUX: return n == 3;
    default: return false;
  }
}

rs_status fail(std::string* err, rs_status st, const char* fmt, unsigned long long a = 0,
               unsigned long long b = 0) {
  char buf[256];
  snprintf(buf, sizeof buf, fmt, a, b);
  *err = buf;
  return st;
}

}  // namespace

// alias (optional, graph passes): alias[s] != s marks signal s as an alias of
// alias[s] -- no driver, no row, its hash weight added to its representative's.
static rs_status compile_core(const rs_graph_desc* d, uint32_t mode, CompiledGraph* out, std::string* err,
                              const std::vector<uint32_t>* alias, const std::vector<uint32_t>* cat_wb = nullptr) {
  if (!d || !out) return fail(err, RS_E_INVALID_ARG, "NULL desc or out");
  if (mode != RS_MODE_LANES && mode != RS_MODE_SINGLE)
    return fail(err, RS_E_INVALID_ARG, "unknown mode %llu", mode);
  const uint32_t NS = d->n_signals, NO = d->n_ops;
  if (NS > 0 && !d->width) return fail(err, RS_E_INVALID_ARG, "width is NULL");
  if ((d->n_inputs && !d->input_id) || (d->n_regs && (!d->reg_id || !d->reg_next_id)) ||
      (d->n_consts && (!d->const_id || !d->const_val)) ||
      (NO && (!d->opcode || !d->out_id || !d->arg_off || !d->arg_id)))
    return fail(err, RS_E_INVALID_ARG, "NULL array with nonzero count");
  if (NO && d->arg_off[0] != 0) return fail(err, RS_E_GRAPH, "arg_off[0] must be 0");

  CompiledGraph& g = *out;
  g = CompiledGraph();
  g.mode = mode;
  g.n_signals = NS;
  g.n_inputs = d->n_inputs;
  g.n_regs = d->n_regs;
  g.n_consts = d->n_consts;
  g.n_ops = NO;

  for (uint32_t s = 0; s < NS; ++s)
    if (d->width[s] < 1 || d->width[s] > 64)
      return fail(err, RS_E_GRAPH, "signal %llu has width %llu (must be 1..64)", s, d->width[s]);

  // ---- drivers: exactly one per signal
  // driver: -1 none, -2 input, -3 reg, -4 const, >=0 op index
  std::vector<int64_t> drv(NS, -1);
  auto claim = [&](uint32_t s, int64_t v) -> bool {
    if (s >= NS || drv[s] != -1) return false;
    drv[s] = v;
    return true;
  };
  for (uint32_t i = 0; i < d->n_inputs; ++i)
    if (!claim(d->input_id[i], -2)) return fail(err, RS_E_GRAPH, "input %llu: bad id or multiple drivers", i);
  for (uint32_t i = 0; i < d->n_regs; ++i)
    if (!claim(d->reg_id[i], -3)) return fail(err, RS_E_GRAPH, "register %llu: bad id or multiple drivers", i);
  for (uint32_t i = 0; i < d->n_consts; ++i)
    if (!claim(d->const_id[i], -4)) return fail(err, RS_E_GRAPH, "const %llu: bad id or multiple drivers", i);
  for (uint32_t j = 0; j < NO; ++j)
    if (!claim(d->out_id[j], j)) return fail(err, RS_E_GRAPH, "op %llu: bad out id or multiple drivers", j);
  auto is_alias = [&](uint32_t s) -> bool { return alias && (*alias)[s] != s; };
  for (uint32_t s = 0; s < NS; ++s)
    if (drv[s] == -1 && !is_alias(s)) return fail(err, RS_E_GRAPH, "signal %llu has no driver", s);
  // hash weights (reading R12): an alias's weight moves to its representative
  std::vector<uint64_t> W(NS);
  for (uint32_t s = 0; s < NS; ++s) W[s] = is_alias(s) ? 0ull : hash_weight(s);
  for (uint32_t s = 0; s < NS; ++s)
    if (is_alias(s)) W[(*alias)[s]] += hash_weight(s);
  for (uint32_t i = 0; i < d->n_regs; ++i)
    if (d->reg_next_id[i] >= NS) return fail(err, RS_E_GRAPH, "register %llu: next id out of range", i);

  // ---- ops: opcode, arity, params, operand ids
  for (uint32_t j = 0; j < NO; ++j) {
    const uint32_t op = d->opcode[j];
    if (d->arg_off[j + 1] < d->arg_off[j]) return fail(err, RS_E_GRAPH, "op %llu: arg_off decreasing", j);
    const uint32_t n = d->arg_off[j + 1] - d->arg_off[j];
    if (op >= RS_NUM_OPS) return fail(err, RS_E_GRAPH, "op %llu: unknown opcode %llu", j, op);
    if (n > MAX_ARITY && (op == RS_OP_AND || op == RS_OP_OR || op == RS_OP_XOR || op == RS_OP_ADD ||
                          op == RS_OP_SUB || op == RS_OP_MUL))
      return fail(err, RS_E_CAPACITY, "op %llu: arity %llu > 63", j, n);
    if (!fixed_arity_ok(op, n)) return fail(err, RS_E_GRAPH, "op %llu: bad arity %llu", j, n);
    for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a)
      if (d->arg_id[a] >= NS) return fail(err, RS_E_GRAPH, "op %llu: operand id out of range", j);
    if (op == RS_OP_BITS) {
      if (!d->param) return fail(err, RS_E_GRAPH, "op %llu: bits needs param", j);
      const uint32_t hi = d->param[2 * j], lo = d->param[2 * j + 1];
      if (lo > hi || hi > 63) return fail(err, RS_E_GRAPH, "op %llu: bits hi=%llu lo out of range", j, hi);
    }
    if ((op == RS_OP_SHL || op == RS_OP_SHR) && !d->param)
      return fail(err, RS_E_GRAPH, "op %llu: shift needs param", j);
  }

  // ---- levels (ASAP via Kahn, or validated given levels)
  std::vector<uint32_t> lev(NO, 0);
  {
    std::vector<uint32_t> indeg(NO, 0), cnt(NS + 1, 0);
    for (uint32_t j = 0; j < NO; ++j)
      for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a)
        if (drv[d->arg_id[a]] >= 0) { indeg[j]++; cnt[d->arg_id[a]]++; }
    std::vector<uint32_t> off(NS + 1, 0);
    for (uint32_t s = 0; s < NS; ++s) off[s + 1] = off[s] + cnt[s];
    std::vector<uint32_t> users(off[NS]), fill(NS, 0);
    for (uint32_t j = 0; j < NO; ++j)
      for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a) {
        uint32_t s = d->arg_id[a];
        if (drv[s] >= 0) users[off[s] + fill[s]++] = j;
      }
    std::vector<uint32_t> q;
    q.reserve(NO);
    for (uint32_t j = 0; j < NO; ++j) if (indeg[j] == 0) q.push_back(j);
    for (size_t h = 0; h < q.size(); ++h) {
      const uint32_t j = q[h], s = d->out_id[j];
      for (uint32_t u = off[s]; u < off[s + 1]; ++u) {
        const uint32_t k = users[u];
        lev[k] = std::max(lev[k], lev[j] + 1);
        if (--indeg[k] == 0) q.push_back(k);
      }
    }
    if (q.size() != NO) return fail(err, RS_E_GRAPH, "combinational loop (%llu ops unreachable)", NO - q.size());
  }
  if (d->level) {
    for (uint32_t j = 0; j < NO; ++j) {
      for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a) {
        const int64_t p = drv[d->arg_id[a]];
        if (p >= 0 && d->level[p] >= d->level[j])
          return fail(err, RS_E_GRAPH, "op %llu: level not above operand producer op %llu", j, p);
      }
      if (d->level[j] > (1u << 24)) return fail(err, RS_E_CAPACITY, "op %llu: level too large", j);
    }
    for (uint32_t j = 0; j < NO; ++j) lev[j] = d->level[j];
  }
  uint32_t n_levels = 0;
  for (uint32_t j = 0; j < NO; ++j) n_levels = std::max(n_levels, lev[j] + 1);

  // ---- identity copies for register next edges that point at an input or a
  // register: the kernel commits registers in one pass and injects the next
  // cycle's inputs in the same phase, so the latch must only read op rows.
  struct Copy { uint32_t src; };
  std::vector<Copy> copies;
  std::unordered_map<uint32_t, uint32_t> copy_of;  // source signal -> copy index
  std::vector<uint32_t> reg_src(d->n_regs);          // effective next: signal id or NS + copy index
  for (uint32_t i = 0; i < d->n_regs; ++i) {
    const uint32_t nx = d->reg_next_id[i];
    if (drv[nx] == -2 || drv[nx] == -3) {
      auto it = copy_of.find(nx);
      uint32_t ci;
      if (it == copy_of.end()) {
        ci = (uint32_t)copies.size();
        copies.push_back({nx});
        copy_of[nx] = ci;
      } else {
        ci = it->second;
      }
      reg_src[i] = NS + ci;
    } else {
      reg_src[i] = nx;
    }
  }
  if (!copies.empty() && n_levels == 0) n_levels = 1;
  g.n_copy = (uint32_t)copies.size();
  g.n_levels = n_levels;
  const uint32_t NT = NO + g.n_copy;  // total ops (canonical + copies); copies are op NO + ci

  auto op_code = [&](uint32_t t) -> uint32_t { return t < NO ? d->opcode[t] : OP_COPY; };
  auto op_arity = [&](uint32_t t) -> uint32_t { return t < NO ? d->arg_off[t + 1] - d->arg_off[t] : 1; };
  auto op_width = [&](uint32_t t) -> uint32_t {
    return t < NO ? d->width[d->out_id[t]] : d->width[copies[t - NO].src];
  };
  auto op_level = [&](uint32_t t) -> uint32_t { return t < NO ? lev[t] : 0; };

  // ---- group each level by (opcode, arity, kind, out class): Format-c swizzle.
  // kind (bit-sliced lane kernel, lanes_b.cuh): 0 = a 1-bit result whose
  // operands are all 1-bit (evaluated on 32-lane bit-plane words), 1 = another
  // 1-bit result, 2 = a wider result; the other kernels ignore it.
  auto op_kind = [&](uint32_t t) -> uint32_t {
    if (op_width(t) != 1) return 2;
    if (t >= NO) return d->width[copies[t - NO].src] == 1 ? 0 : 1;
    for (uint32_t a = d->arg_off[t]; a < d->arg_off[t + 1]; ++a)
      if (d->width[d->arg_id[a]] != 1) return 1;
    return 0;
  };
  std::vector<uint32_t> order(NT);
  std::iota(order.begin(), order.end(), 0u);
  std::vector<uint8_t> kind(NT);
  for (uint32_t t = 0; t < NT; ++t) kind[t] = (uint8_t)op_kind(t);
  auto key = [&](uint32_t t) -> uint64_t {
    // arity first: consecutive work items then share the gather code path, so
    // sub-warps of one warp stay converged even across short runs
    return ((uint64_t)op_level(t) << 32) | ((uint64_t)op_arity(t) << 16) | ((uint64_t)op_code(t) << 8) |
           ((uint64_t)kind[t] << 4) | width_class(op_width(t));
  };
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key(a) < key(b); });

  // ---- rows: per class, [consts][inputs][registers][ops in device order];
  // class 0 holds every 1-bit signal first (rows [0, rows_bit)), so a lane
  // allocation may keep them as bit planes (lanes_b.cuh)
  std::vector<uint32_t> sig_coord(NS + g.n_copy, 0);
  uint32_t n_bit = 0;
  for (uint32_t s = 0; s < NS; ++s) n_bit += d->width[s] == 1 && !is_alias(s);
  for (const Copy& c : copies) n_bit += d->width[c.src] == 1;
  uint32_t rows[4] = {0, 0, 0, 0}, bit_row = 0;
  rows[0] = n_bit;
  auto assign = [&](uint32_t sig, uint32_t w) -> bool {
    const uint32_t c = width_class(w);
    if (rows[c] >= MAX_ROWS) return false;
    sig_coord[sig] = make_coord(c, w == 1 ? bit_row++ : rows[c]++);
    return true;
  };
  for (uint32_t i = 0; i < d->n_consts; ++i)
    if (!assign(d->const_id[i], d->width[d->const_id[i]])) return fail(err, RS_E_CAPACITY, "> 2^30 rows in a class");
  for (uint32_t i = 0; i < d->n_inputs; ++i)
    if (!assign(d->input_id[i], d->width[d->input_id[i]])) return fail(err, RS_E_CAPACITY, "> 2^30 rows in a class");
  for (uint32_t i = 0; i < d->n_regs; ++i)
    if (!assign(d->reg_id[i], d->width[d->reg_id[i]])) return fail(err, RS_E_CAPACITY, "> 2^30 rows in a class");

  g.level_run_begin.assign(n_levels + 1, 0);
  g.level_op_begin.assign(n_levels + 1, 0);
  g.opw.reserve(NT);
  g.opk.reserve(NT);
  g.coord_off.reserve(NT + 1);
  g.coord_off.push_back(0);
  {
    // out rows first (implicit S coordinates), run by run
    size_t i = 0;
    uint32_t cur_level = 0;
    while (i < NT) {
      const uint32_t t0 = order[i];
      const uint64_t k0 = key(t0);
      size_t e = i;
      while (e < NT && key(order[e]) == k0) ++e;
      const uint32_t L = op_level(t0);
      while (cur_level < L) { ++cur_level; g.level_run_begin[cur_level] = (uint32_t)g.runs.size(); g.level_op_begin[cur_level] = (uint32_t)i; }
      DevRun r;
      r.op_begin = (uint32_t)i;
      r.count = (uint32_t)(e - i);
      r.coord_begin = 0;  // filled below
      const uint32_t cls = width_class(op_width(t0));
      r.out_row0 = op_width(t0) == 1 ? bit_row : rows[cls];
      r.meta = op_code(t0) | (op_arity(t0) << 8) | (cls << 16) | ((uint32_t)kind[t0] << 18);
      for (size_t k = i; k < e; ++k) {
        const uint32_t t = order[k];
        const uint32_t sig = t < NO ? d->out_id[t] : NS + (t - NO);
        if (!assign(sig, op_width(t))) return fail(err, RS_E_CAPACITY, "> 2^30 rows in a class");
      }
      g.runs.push_back(r);
      i = e;
    }
    while (cur_level < n_levels) { ++cur_level; g.level_run_begin[cur_level] = (uint32_t)g.runs.size(); g.level_op_begin[cur_level] = (uint32_t)NT; }
    g.level_run_begin[n_levels] = (uint32_t)g.runs.size();
    g.level_op_begin[n_levels] = NT;
  }
  for (int c = 0; c < 4; ++c) g.rows[c] = rows[c];
  g.rows_bit = n_bit;
  for (uint32_t s = 0; s < NS; ++s)
    if (is_alias(s)) sig_coord[s] = sig_coord[(*alias)[s]];
  if (bit_row != n_bit) return fail(err, RS_E_GRAPH, "internal: 1-bit rows %llu != %llu", bit_row, n_bit);

  // ---- per-op arrays in device order
  size_t run_i = 0;
  for (uint32_t k = 0; k < NT; ++k) {
    while (run_i + 1 < g.runs.size() && g.runs[run_i + 1].op_begin <= k) ++run_i;
    if (!g.runs.empty() && g.runs[run_i].op_begin == k) g.runs[run_i].coord_begin = (uint32_t)g.coord.size();
    const uint32_t t = order[k];
    const uint32_t op = op_code(t), n = op_arity(t), w = op_width(t);
    uint32_t p0 = 0, p1 = 0;
    if (t < NO) {
      const uint32_t a0 = d->arg_off[t];
      if (op == RS_OP_SHL || op == RS_OP_SHR) p0 = std::min<uint32_t>(d->param[2 * t], 64u);
      if (op == RS_OP_BITS) { p0 = d->param[2 * t]; p1 = d->param[2 * t + 1]; }
      if (op == RS_OP_CAT) p0 = cat_wb ? (*cat_wb)[t] : d->width[d->arg_id[a0 + 1]];
      for (uint32_t a = a0; a < a0 + n; ++a) g.coord.push_back(sig_coord[d->arg_id[a]]);
      g.opk.push_back(W[d->out_id[t]]);
    } else {
      g.coord.push_back(sig_coord[copies[t - NO].src]);
      g.opk.push_back(0);
    }
    g.opw.push_back(pack_pw(w, p0, p1, width_class(w), op, n));
    g.coord_off.push_back((uint32_t)g.coord.size());
  }

  // ---- inputs, registers, constants
  uint64_t B = 0;
  for (uint32_t i = 0; i < d->n_inputs; ++i) {
    const uint32_t s = d->input_id[i];
    g.in_coord.push_back(sig_coord[s]);
    g.in_w.push_back(d->width[s]);
    g.in_k.push_back(W[s]);
    B += 1ull << width_class(d->width[s]);
  }
  for (uint32_t i = 0; i < d->n_regs; ++i) {
    const uint32_t s = d->reg_id[i];
    const uint32_t w = d->width[s];
    g.reg_coord.push_back(sig_coord[s]);
    g.reg_next_coord.push_back(sig_coord[reg_src[i]]);
    g.reg_w.push_back(w);
    g.reg_k.push_back(W[s]);
    const uint64_t init = (d->reg_init ? d->reg_init[i] : 0) & width_mask(w);
    g.reg_init.push_back(init);
    g.init_reg_hash += init * W[s];
    B += (1ull << width_class(w)) + (1ull << width_class(d->width[d->reg_next_id[i]]));
  }
  for (uint32_t i = 0; i < d->n_consts; ++i) {
    const uint32_t s = d->const_id[i];
    const uint64_t v = d->const_val[i] & width_mask(d->width[s]);
    g.const_coord.push_back(sig_coord[s]);
    g.const_val.push_back(v);
    g.const_hash += v * W[s];
  }
  // canonical maps
  g.sig_coord.assign(sig_coord.begin(), sig_coord.begin() + NS);
  g.sig_kind.assign(NS, 3);
  g.sig_reg_index.assign(NS, -1);
  for (uint32_t i = 0; i < d->n_inputs; ++i) g.sig_kind[d->input_id[i]] = 0;
  for (uint32_t i = 0; i < d->n_regs; ++i) { g.sig_kind[d->reg_id[i]] = 1; g.sig_reg_index[d->reg_id[i]] = (int32_t)i; }
  for (uint32_t i = 0; i < d->n_consts; ++i) g.sig_kind[d->const_id[i]] = 2;
  g.sig_rep.resize(NS);
  for (uint32_t s = 0; s < NS; ++s) {
    g.sig_rep[s] = alias ? (*alias)[s] : s;
    if (is_alias(s)) {  // read back like its representative
      g.sig_kind[s] = g.sig_kind[(*alias)[s]];
      g.sig_reg_index[s] = g.sig_reg_index[(*alias)[s]];
    }
  }

  // ---- statistics: B_alg per lane-cycle, G, naive identity count
  uint64_t G = 0;
  for (uint32_t j = 0; j < NO; ++j) {
    const uint32_t a0 = d->arg_off[j], a1 = d->arg_off[j + 1];
    for (uint32_t a = a0; a < a1; ++a) B += 1ull << width_class(d->width[d->arg_id[a]]);
    B += 1ull << width_class(d->width[d->out_id[j]]);
    G += 4ull * (a1 - a0) + 4ull;
  }
  g.alg_bytes_per_lane_cycle = B;
  g.graph_alg_bytes = G;
  {
    // naive §4.2 construction: a value produced at level l (sources: -1) and
    // last needed at level u needs u - l - 1 identity copies; register next
    // values are needed after the last level (level n_levels).
    std::vector<int64_t> plev(NS, -1), last(NS, -1);
    for (uint32_t j = 0; j < NO; ++j) plev[d->out_id[j]] = lev[j];
    for (uint32_t j = 0; j < NO; ++j)
      for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a)
        last[d->arg_id[a]] = std::max<int64_t>(last[d->arg_id[a]], lev[j]);
    for (uint32_t i = 0; i < d->n_regs; ++i) last[d->reg_next_id[i]] = std::max<int64_t>(last[d->reg_next_id[i]], n_levels);
    uint64_t ids = 0;
    for (uint32_t s = 0; s < NS; ++s)
      if (last[s] - plev[s] - 1 > 0) ids += (uint64_t)(last[s] - plev[s] - 1);
    g.identity_ops_naive = ids;
  }
  return RS_OK;
}

rs_status compile_graph(const rs_graph_desc* d, uint32_t mode, CompiledGraph* out, std::string* err) {
  if (!(mode & RS_LOAD_PASSES)) return compile_core(d, mode, out, err, nullptr);
  mode &= ~RS_LOAD_PASSES;
  // validate the circuit as given (drivers, arities, params, loops) first
  rs_status st = compile_core(d, mode, out, err, nullptr);
  if (st != RS_OK) return st;
  // a topological order: the ops by their (valid) levels
  const uint32_t NO = d->n_ops, NS = d->n_signals;
  std::vector<int64_t> drv(NS, -1);
  for (uint32_t j = 0; j < NO; ++j) drv[d->out_id[j]] = j;
  std::vector<uint32_t> lev(NO, 0), topo(NO);
  {
    // ASAP levels by a Kahn sweep over the producers (the core run proved acyclicity)
    std::vector<uint32_t> indeg(NO, 0), off(NS + 1, 0);
    for (uint32_t j = 0; j < NO; ++j)
      for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a)
        if (drv[d->arg_id[a]] >= 0) { indeg[j]++; off[d->arg_id[a] + 1]++; }
    for (uint32_t s2 = 0; s2 < NS; ++s2) off[s2 + 1] += off[s2];
    std::vector<uint32_t> users(off[NS]), fill(off.begin(), off.end() - 1);
    for (uint32_t j = 0; j < NO; ++j)
      for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a)
        if (drv[d->arg_id[a]] >= 0) users[fill[d->arg_id[a]]++] = j;
    size_t h = 0, t = 0;
    for (uint32_t j = 0; j < NO; ++j) if (indeg[j] == 0) topo[t++] = j;
    while (h < t) {
      const uint32_t j = topo[h++], o = d->out_id[j];
      for (uint32_t u = off[o]; u < off[o + 1]; ++u)
        if (--indeg[users[u]] == 0) topo[t++] = users[u];
    }
  }
  PassResult pr;
  run_passes(d, drv, topo, &pr);
  st = compile_core(&pr.desc, mode, out, err, &pr.rep, &pr.cat_wb);
  if (st != RS_OK) return st;
  out->n_alias = pr.n_alias;
  out->n_folded = (uint32_t)pr.folded.size();
  out->n_mux_chain = pr.n_mux_chain;
  out->n_ops_input = NO;
  return RS_OK;
}

namespace {
inline uint32_t al16(uint32_t x) { return (x + 15u) & ~15u; }

struct StageWriter {
  std::vector<uint8_t>* blob;
  std::vector<StageRef>* table;
  void emit(StageHdr h, const uint32_t* w, const uint64_t* k, const uint32_t* c, const StageRun* runs,
            const uint32_t* items = nullptr) {
    h.off_w = al16((uint32_t)sizeof(StageHdr));
    h.off_k = al16(h.off_w + 4 * h.n);
    h.off_c = al16(h.off_k + 8 * h.n);
    h.off_runs = al16(h.off_c + 4 * h.n_coords);
    h.off_items = al16(h.off_runs + (uint32_t)sizeof(StageRun) * h.n_runs);
    h.bytes = al16(h.off_items + 4 * h.n_items);
    const size_t base = (blob->size() + 15) & ~(size_t)15;
    blob->resize(base + h.bytes, 0);
    uint8_t* p = blob->data() + base;
    std::memcpy(p, &h, sizeof h);
    if (h.n && w) std::memcpy(p + h.off_w, w, 4ull * h.n);
    if (h.n && k) std::memcpy(p + h.off_k, k, 8ull * h.n);
    if (h.n_coords && c) std::memcpy(p + h.off_c, c, 4ull * h.n_coords);
    if (h.n_runs && runs) std::memcpy(p + h.off_runs, runs, sizeof(StageRun) * h.n_runs);
    if (h.n_items && items) std::memcpy(p + h.off_items, items, 4ull * h.n_items);
    table->push_back({base, h.bytes, h.type});
  }
};

// Upper bound of a stage's bytes (OPS items bounded by n / batch + n_runs).
uint32_t stage_size(uint32_t n, uint32_t n_coords, uint32_t n_runs, uint32_t batch) {
  uint32_t off_w = al16((uint32_t)sizeof(StageHdr));
  uint32_t off_k = al16(off_w + 4 * n);
  uint32_t off_c = al16(off_k + 8 * n);
  uint32_t off_r = al16(off_c + 4 * n_coords);
  uint32_t off_i = al16(off_r + (uint32_t)sizeof(StageRun) * n_runs);
  const uint32_t items = n_runs ? n / batch + n_runs : 0;
  return al16(off_i + 4 * items);
}

constexpr uint32_t kMaxStageOps = 8191;   // 13-bit op field of a work item
}  // namespace

void build_stages(const CompiledGraph& g, uint32_t stage_bytes, uint32_t batch, std::vector<uint8_t>* blob,
                  std::vector<StageRef>* table) {
  stage_bytes = std::max<uint32_t>(stage_bytes, 4096);  // room for >= 1 entry per stage (always progresses)
  blob->clear();
  table->clear();
  StageWriter W{blob, table};
  // inputs: w, K, coord
  {
    uint32_t i = 0;
    while (i < g.n_inputs) {
      uint32_t n = 0;
      while (i + n < g.n_inputs && stage_size(n + 1, n + 1, 0, batch) <= stage_bytes) ++n;
      StageHdr h{};
      h.type = ST_INJECT;
      h.n = n;
      h.n_coords = n;
      h.first = i;
      W.emit(h, &g.in_w[i], &g.in_k[i], &g.in_coord[i], nullptr);
      i += n;
    }
  }
  // ops, level by level
  for (uint32_t l = 0; l < g.n_levels; ++l) {
    const uint32_t ob = g.level_op_begin[l], oe = g.level_op_begin[l + 1];
    uint32_t r = g.level_run_begin[l];
    uint32_t j = ob;
    while (j < oe) {
      // grow the stage op by op
      uint32_t e = j, nruns = 0, ncoords = 0, rr = r;
      while (e < oe) {
        while (rr + 1 < g.level_run_begin[l + 1] && g.runs[rr + 1].op_begin <= e) ++rr;
        const bool new_run = (e == j) || (g.runs[rr].op_begin == e);
        const uint32_t ar = g.coord_off[e + 1] - g.coord_off[e];
        if ((stage_size(e - j + 1, ncoords + ar, nruns + (new_run ? 1 : 0), batch) > stage_bytes || e - j >= kMaxStageOps) &&
            e > j)
          break;
        nruns += new_run ? 1 : 0;
        ncoords += ar;
        ++e;
      }
      std::vector<StageRun> runs;
      uint32_t k = j;
      while (k < e) {
        while (r + 1 < g.level_run_begin[l + 1] && g.runs[r + 1].op_begin <= k) ++r;
        const DevRun& R = g.runs[r];
        const uint32_t se = std::min(e, R.op_begin + R.count);
        StageRun sr{};
        sr.op_begin = k - j;
        sr.count = se - k;
        sr.coord_begin = g.coord_off[k] - g.coord_off[j];
        sr.out_row0 = R.out_row0 + (k - R.op_begin);
        sr.meta = R.meta;
        runs.push_back(sr);
        k = se;
      }
      // work items: run-aligned batches of <= batch ops
      std::vector<uint32_t> items;
      for (uint32_t q = 0; q < runs.size(); ++q)
        for (uint32_t o = 0; o < runs[q].count; o += batch) {
          const uint32_t cnt = std::min(batch, runs[q].count - o);
          items.push_back((q << 16) | ((cnt - 1) << 13) | (runs[q].op_begin + o));
        }
      StageHdr h{};
      h.type = ST_OPS;
      h.n = e - j;
      h.n_runs = (uint32_t)runs.size();
      h.n_coords = g.coord_off[e] - g.coord_off[j];
      h.first = j;
      h.level = l;
      h.n_items = (uint32_t)items.size();
      W.emit(h, &g.opw[j], &g.opk[j], &g.coord[g.coord_off[j]], runs.data(), items.data());
      j = e;
    }
  }
  // registers: w, K, (next, reg) coord pairs
  {
    uint32_t i = 0;
    while (i < g.n_regs) {
      uint32_t n = 0;
      while (i + n < g.n_regs && stage_size(n + 1, 2 * (n + 1), 0, batch) <= stage_bytes) ++n;
      std::vector<uint32_t> pairs(2 * n);
      for (uint32_t q = 0; q < n; ++q) {
        pairs[2 * q] = g.reg_next_coord[i + q];
        pairs[2 * q + 1] = g.reg_coord[i + q];
      }
      StageHdr h{};
      h.type = ST_LATCH;
      h.n = n;
      h.n_coords = 2 * n;
      h.first = i;
      W.emit(h, &g.reg_w[i], &g.reg_k[i], pairs.data(), nullptr);
      i += n;
    }
  }
  if (table->empty()) {
    StageHdr h{};
    h.type = ST_NOP;
    W.emit(h, nullptr, nullptr, nullptr, nullptr);
  }
}

std::vector<uint32_t> level_cut(const CompiledGraph& g, uint32_t P) {
  // cumulative op weight (1 + arity) at each level boundary
  const uint32_t nl = g.n_levels;
  auto wl = [&](uint32_t l) -> uint64_t {
    const uint32_t o = g.level_op_begin[l];
    return (uint64_t)o + g.coord_off[o];
  };
  const uint64_t W = wl(nl);
  std::vector<uint32_t> cut(P + 1, nl);
  cut[0] = 0;
  for (uint32_t k = 1; k < P; ++k) {
    const uint64_t target = (W * k + P / 2) / P;
    uint32_t l = cut[k - 1] + 1;                      // every partition gets >= 1 level
    while (l < nl - (P - 1 - k) && wl(l) < target) ++l;
    cut[k] = std::min(l, nl - (P - k));
  }
  return cut;
}

void row_owner(const CompiledGraph& g, const std::vector<uint32_t>& cut, std::vector<uint8_t> owner[4]) {
  for (int c = 0; c < 4; ++c) owner[c].assign(g.rows[c], 0);
  uint32_t k = 0;
  for (uint32_t l = 0; l < g.n_levels; ++l) {
    while (l >= cut[k + 1]) ++k;
    for (uint32_t r = g.level_run_begin[l]; r < g.level_run_begin[l + 1]; ++r) {
      const DevRun& R = g.runs[r];
      const uint32_t cls = (R.meta >> 16) & 3u;
      for (uint32_t i = 0; i < R.count; ++i) owner[cls][R.out_row0 + i] = (uint8_t)k;
    }
  }
}

bool build_single_slices(const CompiledGraph& g, uint32_t P, uint32_t Gp, uint32_t max_bytes,
                         std::vector<uint8_t>* blob, std::vector<uint64_t>* slice_off) {
  blob->clear();
  slice_off->assign((size_t)P * Gp, 0);
  if (P == 0 || P > kMaxParts || P > std::max<uint32_t>(1, g.n_levels)) return false;
  auto chunk = [](uint32_t n, uint32_t part, uint32_t parts, uint32_t& b, uint32_t& e) {
    const uint32_t c = (n + parts - 1) / parts;
    b = std::min(n, part * c);
    e = std::min(n, b + c);
  };
  const std::vector<uint32_t> cut = level_cut(g, P);
  std::vector<uint8_t> owner[4];
  row_owner(g, cut, owner);
  auto own_of = [&](uint32_t c) -> uint32_t { return owner[c >> 30][c & ROW_MASK]; };
  // register owner = partition producing its next value (an op row: the
  // compiler routes source next values through identity copies at level 0)
  std::vector<uint32_t> reg_owner(g.n_regs);
  for (uint32_t i = 0; i < g.n_regs; ++i) reg_owner[i] = own_of(g.reg_next_coord[i]);
  // cut signals: producer partition -> (coord -> consumer mask)
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> push(P);
  if (P > 1) {
    std::vector<uint32_t> mask[4];
    for (int c = 0; c < 4; ++c) mask[c].assign(g.rows[c], 0);
    uint32_t k = 0;
    for (uint32_t l = 0; l < g.n_levels; ++l) {
      while (l >= cut[k + 1]) ++k;
      for (uint32_t j = g.level_op_begin[l]; j < g.level_op_begin[l + 1]; ++j)
        for (uint32_t q = g.coord_off[j]; q < g.coord_off[j + 1]; ++q) {
          const uint32_t c = g.coord[q];
          mask[c >> 30][c & ROW_MASK] |= 1u << k;
        }
    }
    for (uint32_t i = 0; i < g.n_regs; ++i) {  // partitions after the owner latch it locally
      const uint32_t c = g.reg_next_coord[i];
      for (uint32_t m = reg_owner[i] + 1; m < P; ++m) mask[c >> 30][c & ROW_MASK] |= 1u << m;
    }
    // only op rows produced by an earlier partition travel; sources are in every replica
    std::vector<uint8_t> is_op[4];
    for (int c = 0; c < 4; ++c) is_op[c].assign(g.rows[c], 0);
    for (const DevRun& R : g.runs)
      for (uint32_t i = 0; i < R.count; ++i) is_op[(R.meta >> 16) & 3u][R.out_row0 + i] = 1;
    for (uint32_t c = 0; c < 4; ++c)
      for (uint32_t r = 0; r < g.rows[c]; ++r) {
        if (!is_op[c][r]) continue;
        const uint32_t k0 = owner[c][r];
        const uint32_t m = mask[c][r] & ~((2u << k0) - 1u);  // consumers after the producer
        if (m) push[k0].push_back({make_coord(c, r), m});
      }
  }
  for (uint32_t k = 0; k < P; ++k) {
    // latch list of partition k: registers owned by partitions <= k
    std::vector<uint32_t> regs;
    for (uint32_t i = 0; i < g.n_regs; ++i)
      if (reg_owner[i] <= k) regs.push_back(i);
    for (uint32_t cta = 0; cta < Gp; ++cta) {
      std::vector<SliceLvl> lv(cut[k + 1] - cut[k]);
      std::vector<SliceSeg> seg;
      std::vector<uint32_t> pw, coords, latch, inj, pu;
      for (uint32_t l = cut[k]; l < cut[k + 1]; ++l) {
        const uint32_t ob = g.level_op_begin[l], oe = g.level_op_begin[l + 1];
        // chunk boundaries balanced by weight 1 + arity (ops are sorted by arity
        // inside a level, so equal op counts would give the last CTAs all the
        // 3-operand ops: unequal work and shared memory)
        auto wpos = [&](uint32_t j) -> uint64_t { return (uint64_t)(j - ob) + (g.coord_off[j] - g.coord_off[ob]); };
        const uint64_t W = wpos(oe);
        auto cutw = [&](uint32_t part) -> uint32_t {
          const uint64_t target = (W * part + Gp - 1) / Gp;
          uint32_t lo = ob, hi = oe;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) / 2;
            if (wpos(mid) < target) lo = mid + 1; else hi = mid;
          }
          return lo;
        };
        const uint32_t b = cutw(cta), e = cutw(cta + 1);
        SliceLvl& L = lv[l - cut[k]];
        L = SliceLvl{};
        L.op_begin = b;
        L.n = e - b;
        L.pw_base = (uint32_t)pw.size();
        L.coord_base = (uint32_t)coords.size();
        L.seg_begin = (uint32_t)seg.size();
        for (uint32_t r = g.level_run_begin[l]; r < g.level_run_begin[l + 1]; ++r) {
          const DevRun& R = g.runs[r];
          const uint32_t s0 = std::max(b, R.op_begin), s1 = std::min(e, R.op_begin + R.count);
          if (s0 >= s1) continue;
          SliceSeg sg{};
          sg.first = s0 - b;
          sg.count = s1 - s0;
          sg.out_coord0 = make_coord((R.meta >> 16) & 3u, R.out_row0 + (s0 - R.op_begin));
          sg.coord0 = g.coord_off[s0] - g.coord_off[b];
          seg.push_back(sg);
        }
        L.n_seg = (uint32_t)seg.size() - L.seg_begin;
        for (uint32_t j = b; j < e; ++j) {
          pw.push_back(g.opw[j]);
          for (uint32_t q = g.coord_off[j]; q < g.coord_off[j + 1]; ++q) coords.push_back(g.coord[q]);
        }
      }
      uint32_t rb, re, ib, ie, pb, pe;
      chunk((uint32_t)regs.size(), cta, Gp, rb, re);
      chunk(g.n_inputs, cta, Gp, ib, ie);
      chunk((uint32_t)push[k].size(), cta, Gp, pb, pe);
      for (uint32_t q = rb; q < re; ++q) {
        const uint32_t i = regs[q];
        const uint32_t own = reg_owner[i] == k ? 1u : 0u;
        const uint32_t dmask = own ? ((1u << k) - 1u) : 0u;  // earlier replicas are done with the cycle
        latch.push_back(g.reg_next_coord[i]);
        latch.push_back(g.reg_coord[i]);
        latch.push_back(g.reg_w[i] | (own << 7) | (dmask << 8));
        latch.push_back(i);
      }
      for (uint32_t i = ib; i < ie; ++i) {
        inj.push_back(g.in_coord[i]);
        inj.push_back(g.in_w[i]);
      }
      for (uint32_t i = pb; i < pe; ++i) {
        pu.push_back(push[k][i].first);
        pu.push_back(push[k][i].second);
      }
      SliceHdr h{};
      h.n_levels = (uint32_t)lv.size();
      h.off_lvl = al16((uint32_t)sizeof(SliceHdr));
      h.off_seg = al16(h.off_lvl + (uint32_t)(lv.size() * sizeof(SliceLvl)));
      h.off_pw = al16(h.off_seg + (uint32_t)(seg.size() * sizeof(SliceSeg)));
      h.off_coord = al16(h.off_pw + 4u * (uint32_t)pw.size());
      h.head_bytes = al16(h.off_coord + 4u * (uint32_t)coords.size());
      h.off_push = h.head_bytes;
      h.off_latch = al16(h.off_push + 4u * (uint32_t)pu.size());
      h.off_inj = al16(h.off_latch + 4u * (uint32_t)latch.size());
      h.bytes = al16(h.off_inj + 4u * (uint32_t)inj.size());
      h.n_push = pe - pb;
      h.n_latch = re - rb;
      h.inj_first = ib;
      h.n_inj = ie - ib;
      h.part = k;
      if (h.head_bytes > max_bytes) {
        blob->clear();
        return false;
      }
      const size_t base = (blob->size() + 127) & ~(size_t)127;
      blob->resize(base + h.bytes, 0);
      uint8_t* p = blob->data() + base;
      std::memcpy(p, &h, sizeof h);
      auto put = [&](uint32_t off, const void* src, size_t n) {
        if (n) std::memcpy(p + off, src, n);
      };
      put(h.off_lvl, lv.data(), lv.size() * sizeof(SliceLvl));
      put(h.off_seg, seg.data(), seg.size() * sizeof(SliceSeg));
      put(h.off_pw, pw.data(), pw.size() * 4);
      put(h.off_push, pu.data(), pu.size() * 4);
      put(h.off_coord, coords.data(), coords.size() * 4);
      put(h.off_latch, latch.data(), latch.size() * 4);
      put(h.off_inj, inj.data(), inj.size() * 4);
      (*slice_off)[(size_t)k * Gp + cta] = base;
    }
  }
  return true;
}

namespace {

// Register partition by cone clustering (the partitioning step of RepCut, PAPER.md
// P:1981-1982, which uses a hypergraph partitioner; reading R20): a register's
// replication cost is the overlap of its next-value cone with other partitions' cones,
// and cones only meet inside connected combinational logic -- registers and inputs end
// a cone.  So the ops are joined with their operands' producers (union-find), each
// register goes with the component of its next value's producer, and the components
// (the cores of a multi-core design, coupled only through registers) are cut to size
// and bin-packed, largest first, into P partitions.  Returns an empty vector when the
// logic is one component (a random single core: nothing to find).
std::vector<uint32_t> cone_cluster_partition(const CompiledGraph& g, uint32_t P,
                                             const std::function<int32_t(uint32_t)>& producer,
                                             std::vector<int32_t>* op_home) {
  const uint32_t NT = g.n_ops_total(), R = g.n_regs;
  std::vector<uint32_t> uf(NT);
  for (uint32_t j = 0; j < NT; ++j) uf[j] = j;
  auto find = [&](uint32_t x) {
    while (uf[x] != x) x = uf[x] = uf[uf[x]];
    return x;
  };
  for (uint32_t j = 0; j < NT; ++j)
    for (uint32_t a = g.coord_off[j]; a < g.coord_off[j + 1]; ++a) {
      const int32_t q = producer(g.coord[a]);
      if (q >= 0) uf[find(j)] = find((uint32_t)q);
    }
  std::unordered_map<uint32_t, std::vector<uint32_t>> comp;
  for (uint32_t i = 0; i < R; ++i) {
    const int32_t q = producer(g.reg_next_coord[i]);
    comp[q >= 0 ? find((uint32_t)q) : NT + i].push_back(i);
  }
  if (comp.size() <= 1) return {};
  // pieces of at most ~R / P registers (index order within a component), bin-packed
  const uint32_t target = std::max<uint32_t>(1, (R + P - 1) / P);
  std::vector<std::vector<uint32_t>> pieces;
  for (auto& kv : comp) {
    std::vector<uint32_t>& v = kv.second;
    if (v.size() <= target + target / 2) {
      pieces.push_back(std::move(v));
      continue;
    }
    for (size_t b = 0; b < v.size(); b += target)
      pieces.emplace_back(v.begin() + b, v.begin() + std::min(v.size(), b + target));
  }
  std::sort(pieces.begin(), pieces.end(), [](const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
    return a.size() != b.size() ? a.size() > b.size() : a[0] < b[0];
  });
  std::vector<uint32_t> part(R, 0), load(P, 0);
  for (const auto& pc : pieces) {
    const uint32_t p = (uint32_t)(std::min_element(load.begin(), load.end()) - load.begin());
    for (uint32_t i : pc) part[i] = p;
    load[p] += (uint32_t)pc.size();
  }
  for (uint32_t p = 0; p < P; ++p)
    if (!load[p]) return {};  // a partition without registers: keep the blocks
  // home of every op: the partition of its component's (first) registers -- where dead
  // logic of that component goes, so it drags no cone into another partition
  std::unordered_map<uint32_t, int32_t> home;
  for (uint32_t i = 0; i < R; ++i) {
    const int32_t q = producer(g.reg_next_coord[i]);
    if (q >= 0) home.emplace(find((uint32_t)q), (int32_t)part[i]);
  }
  op_home->assign(NT, -1);
  for (uint32_t j = 0; j < NT; ++j) {
    auto it = home.find(find(j));
    if (it != home.end()) (*op_home)[j] = it->second;
  }
  return part;
}

bool build_repcut_with(const CompiledGraph& g, uint32_t P, const std::vector<uint32_t>& reg_part,
                       const std::function<int32_t(uint32_t)>& producer, const std::vector<int32_t>* op_home,
                       RepCutPlan* out);

}  // namespace

bool build_repcut(const CompiledGraph& g, uint32_t P, RepCutPlan* out, std::string* err) {
  const uint32_t R = g.n_regs;
  if (P == 0 || P > 255 || (R && P > R) || (!R && P > 1)) {
    *err = "repcut: partitions must be in [1, min(255, n_regs)]";
    return false;
  }
  // producing op of every (class, row); -1 = a source
  std::vector<int32_t> prod[4];
  for (int c = 0; c < 4; ++c) prod[c].assign(g.rows[c], -1);
  for (const DevRun& r : g.runs) {
    const uint32_t cls = (r.meta >> 16) & 3u;
    for (uint32_t k = 0; k < r.count; ++k) prod[cls][r.out_row0 + k] = (int32_t)(r.op_begin + k);
  }
  const std::function<int32_t(uint32_t)> producer = [&](uint32_t c) -> int32_t { return prod[c >> 30][c & ROW_MASK]; };
  // register partition: contiguous index blocks (a netlist lists each module's registers
  // together), or the cone clustering when it replicates less (the largest partition
  // first, then the total)
  std::vector<uint32_t> blocks(R);
  for (uint32_t i = 0; i < R; ++i) blocks[i] = (uint32_t)((uint64_t)i * P / R);
  build_repcut_with(g, P, blocks, producer, nullptr, out);
  if (P > 1) {
    std::vector<int32_t> home;
    const std::vector<uint32_t> cc = cone_cluster_partition(g, P, producer, &home);
    if (!cc.empty() && cc != blocks) {
      RepCutPlan alt;
      build_repcut_with(g, P, cc, producer, &home, &alt);
      if (alt.max_ops < out->max_ops || (alt.max_ops == out->max_ops && alt.ops_total < out->ops_total))
        *out = std::move(alt);
    }
  }
  return true;
}

namespace {

bool build_repcut_with(const CompiledGraph& g, uint32_t P, const std::vector<uint32_t>& reg_part,
                       const std::function<int32_t(uint32_t)>& producer, const std::vector<int32_t>* op_home,
                       RepCutPlan* out) {
  const uint32_t NT = g.n_ops_total(), NL = g.n_levels, R = g.n_regs;
  // cones: member[p] bitmaps over ops
  std::vector<std::vector<uint8_t>> member(P, std::vector<uint8_t>(NT, 0));
  std::vector<uint32_t> stack;
  auto close = [&](uint32_t p, int32_t j0) {
    if (j0 < 0 || member[p][j0]) return;
    stack.assign(1, (uint32_t)j0);
    member[p][j0] = 1;
    while (!stack.empty()) {
      const uint32_t j = stack.back();
      stack.pop_back();
      for (uint32_t a = g.coord_off[j]; a < g.coord_off[j + 1]; ++a) {
        const int32_t q = producer(g.coord[a]);
        if (q >= 0 && !member[p][q]) {
          member[p][q] = 1;
          stack.push_back((uint32_t)q);
        }
      }
    }
  };
  for (uint32_t i = 0; i < R; ++i) close(reg_part[i], producer(g.reg_next_coord[i]));
  std::vector<int32_t> owner(NT, -1);
  for (uint32_t j = 0; j < NT; ++j)
    for (uint32_t p = 0; p < P && owner[j] < 0; ++p)
      if (member[p][j]) owner[j] = (int32_t)p;
  // ops outside every register cone (dead logic: its values are still hashed
  // and readable) join the partition of their first operand's producer (the
  // producers have lower device indices -- level order -- so they already have
  // an owner), else of their first register operand, else j mod P; with their
  // cone, so they replicate and push no more than they must
  std::unordered_map<uint32_t, uint32_t> reg_of_coord;
  for (uint32_t i = 0; i < R; ++i) reg_of_coord[g.reg_coord[i]] = i;
  std::unordered_map<uint32_t, uint32_t> in_of_coord;
  for (uint32_t i = 0; i < g.n_inputs; ++i) in_of_coord[g.in_coord[i]] = i;
  // canonical id of each op's output (identity copies: none)
  std::vector<uint32_t> out_sig(NT, UINT32_MAX);
  for (uint32_t s2 = 0; s2 < g.n_signals; ++s2)
    if (g.sig_kind[s2] == 3 && (g.sig_rep.empty() || g.sig_rep[s2] == s2)) {
      const int32_t q = producer(g.sig_coord[s2]);
      if (q >= 0) out_sig[q] = s2;
    }
  for (uint32_t j = 0; j < NT; ++j)
    if (owner[j] < 0) {
      int32_t p = op_home ? (*op_home)[j] : -1;  // the clustering's home of its logic component
      for (uint32_t a = g.coord_off[j]; a < g.coord_off[j + 1] && p < 0; ++a) {
        const int32_t q = producer(g.coord[a]);
        if (q >= 0) p = owner[q];
      }
      // then inputs, then registers, both in contiguous index blocks (a multi-core
      // design's inputs and registers follow its module order); inputs first: an
      // operand that is another block's register is how cores couple, and a dead op
      // placed by it would drag its dependents' cones into that block (the graph
      // passes turn copies of inputs into direct input operands, exposing this)
      for (uint32_t a = g.coord_off[j]; a < g.coord_off[j + 1] && p < 0; ++a) {
        auto it = in_of_coord.find(g.coord[a]);
        if (it != in_of_coord.end()) p = (int32_t)((uint64_t)it->second * P / g.n_inputs);
      }
      // else the block its own canonical id falls in (signals in contiguous id blocks, like
      // registers: a netlist lists each module's signals together); not a register
      // operand's block -- registers are how cores couple, so an op reading only a
      // foreign register (and constants) would drag its dependents' cones there
      if (p < 0 && out_sig[j] != UINT32_MAX) p = (int32_t)((uint64_t)out_sig[j] * P / g.n_signals);
      if (p < 0) p = (int32_t)(j % P);
      close((uint32_t)p, (int32_t)j);
      owner[j] = p;
    }
  RepCutPlan& o = *out;
  o = RepCutPlan{};
  o.P = P;
  o.lvl_begin.assign((size_t)P * (NL + 1), 0);
  for (uint32_t p = 0; p < P; ++p) {
    uint32_t cnt = 0;
    for (uint32_t l = 0; l < NL; ++l) {
      o.lvl_begin[(size_t)p * (NL + 1) + l] = (uint32_t)o.ops.size();
      for (uint32_t j = g.level_op_begin[l]; j < g.level_op_begin[l + 1]; ++j)
        if (member[p][j]) {
          o.ops.push_back(j | ((uint32_t)(owner[j] == (int32_t)p) << 31));
          ++cnt;
        }
    }
    o.lvl_begin[(size_t)p * (NL + 1) + NL] = (uint32_t)o.ops.size();
    o.ops_total += cnt;
    o.max_ops = std::max(o.max_ops, cnt);
  }
  // own registers and the Register Update Map (push to the partitions that read a register)
  o.reg_begin.assign(P + 1, 0);
  for (uint32_t i = 0; i < R; ++i) o.reg_begin[reg_part[i] + 1]++;
  for (uint32_t p = 0; p < P; ++p) o.reg_begin[p + 1] += o.reg_begin[p];
  o.regs.resize(R);
  {
    std::vector<uint32_t> fill(o.reg_begin.begin(), o.reg_begin.end() - 1);
    for (uint32_t i = 0; i < R; ++i) o.regs[fill[reg_part[i]]++] = i;
  }
  std::vector<std::vector<uint8_t>> reads(P, std::vector<uint8_t>(R, 0));
  for (uint32_t p = 0; p < P; ++p)
    for (uint32_t j = 0; j < NT; ++j)
      if (member[p][j])
        for (uint32_t a = g.coord_off[j]; a < g.coord_off[j + 1]; ++a) {
          auto it = reg_of_coord.find(g.coord[a]);
          if (it != reg_of_coord.end()) reads[p][it->second] = 1;
        }
  o.push_begin.assign(P + 1, 0);
  for (uint32_t p = 0; p < P; ++p) {
    o.push_begin[p] = (uint32_t)(o.push.size() / 2);
    for (uint32_t k = o.reg_begin[p]; k < o.reg_begin[p + 1]; ++k) {
      const uint32_t i = o.regs[k];
      for (uint32_t q = 0; q < P; ++q)
        if (q != p && reads[q][i]) {
          o.push.push_back(i);
          o.push.push_back(q);
        }
    }
  }
  o.push_begin[P] = (uint32_t)(o.push.size() / 2);
  // read-back: the replica holding each signal's value
  o.sig_owner.assign(g.n_signals, 0);
  for (uint32_t s = 0; s < g.n_signals; ++s) {
    if (g.sig_kind[s] == 1) {
      o.sig_owner[s] = (uint8_t)reg_part[g.sig_reg_index[s]];
    } else if (g.sig_kind[s] == 3) {
      const int32_t j = producer(g.sig_coord[s]);
      o.sig_owner[s] = (uint8_t)(j >= 0 ? owner[j] : 0);
    }
  }
  return true;
}

}  // namespace


bool build_repcut_slices(const CompiledGraph& g, const RepCutPlan& plan, uint32_t max_smem, bool wide,
                         std::vector<uint8_t>* blob, std::vector<uint64_t>* slice_off,
                         std::vector<uint64_t>* op_k, std::vector<uint8_t>* in_owner, std::string* err) {
  const uint32_t P = plan.P, NL = g.n_levels, NT = g.n_ops_total(), R = g.n_regs, NI = g.n_inputs;
  blob->clear();
  slice_off->assign(P, 0);
  op_k->clear();
  if (R >= (1u << 24)) {
    *err = "repcut slices: more than 2^24 registers";
    return false;
  }
  in_owner->assign(NI, 0);
  // output coord of every op
  std::vector<uint32_t> out_coord(NT, 0);
  for (const DevRun& r : g.runs) {
    const uint32_t cls = (r.meta >> 16) & 3u;
    for (uint32_t k = 0; k < r.count; ++k) out_coord[r.op_begin + k] = (cls << 30) | (r.out_row0 + k);
  }
  std::unordered_map<uint32_t, uint32_t> reg_of_coord, in_of_coord;
  for (uint32_t i = 0; i < R; ++i) reg_of_coord[g.reg_coord[i]] = i;
  for (uint32_t k = 0; k < NI; ++k) in_of_coord[g.in_coord[k]] = k;
  // who reads each input; its owner is the lowest reader (none: partition 0)
  std::vector<std::vector<uint8_t>> reads_in(P, std::vector<uint8_t>(NI, 0));
  for (uint32_t p = 0; p < P; ++p)
    for (uint32_t x = plan.lvl_begin[(size_t)p * (NL + 1)]; x < plan.lvl_begin[(size_t)p * (NL + 1) + NL]; ++x) {
      const uint32_t j = plan.ops[x] & 0x7FFFFFFFu;
      for (uint32_t a = g.coord_off[j]; a < g.coord_off[j + 1]; ++a) {
        auto it = in_of_coord.find(g.coord[a]);
        if (it != in_of_coord.end()) reads_in[p][it->second] = 1;
      }
    }
  for (uint32_t k = 0; k < NI; ++k) {
    uint32_t o = 0;
    while (o < P && !reads_in[o][k]) ++o;
    (*in_owner)[k] = (uint8_t)(o < P ? o : 0);
  }
  std::vector<uint32_t> reg_owner(R, 0);
  for (uint32_t p = 0; p < P; ++p)
    for (uint32_t k = plan.reg_begin[p]; k < plan.reg_begin[p + 1]; ++k) reg_owner[plan.regs[k]] = p;
  auto align16 = [](size_t n) { return (n + 15) & ~(size_t)15; };
  for (uint32_t p = 0; p < P; ++p) {
    const uint32_t* lb = plan.lvl_begin.data() + (size_t)p * (NL + 1);
    // ---- local signal set, by class
    std::vector<uint32_t> sigs;
    for (uint32_t x = lb[0]; x < lb[NL]; ++x) {
      const uint32_t j = plan.ops[x] & 0x7FFFFFFFu;
      sigs.push_back(out_coord[j]);
      for (uint32_t a = g.coord_off[j]; a < g.coord_off[j + 1]; ++a) sigs.push_back(g.coord[a]);
    }
    for (uint32_t k = plan.reg_begin[p]; k < plan.reg_begin[p + 1]; ++k) {
      sigs.push_back(g.reg_coord[plan.regs[k]]);
      sigs.push_back(g.reg_next_coord[plan.regs[k]]);
    }
    for (uint32_t k = 0; k < NI; ++k)
      if (reads_in[p][k] || (*in_owner)[k] == p) sigs.push_back(g.in_coord[k]);
    std::sort(sigs.begin(), sigs.end());
    sigs.erase(std::unique(sigs.begin(), sigs.end()), sigs.end());
    std::unordered_map<uint32_t, uint32_t> local;
    local.reserve(sigs.size() * 2);
    uint32_t off = 0, bnd[4] = {0, 0, 0, 0};
    for (int cls = 3; cls >= 0; --cls) {
      bnd[cls] = off;
      for (uint32_t c : sigs)
        if ((c >> 30) == (uint32_t)cls || (wide && cls == 3)) {
          local[c] = off;
          off += wide ? 8u : 1u << cls;
        }
      if (wide) {  // one region of 8-byte slots: every offset reads as class 3
        bnd[2] = bnd[1] = bnd[0] = off;
        break;
      }
    }
    const uint32_t state_bytes = (uint32_t)align16(off + 8);  // + 8: the aligned-word gather may read past the end
    if (off > 65535u) {
      *err = "repcut slice " + std::to_string(p) + ": local state of " + std::to_string(off) + " bytes > 64 KiB";
      return false;
    }
    auto L = [&](uint32_t c) -> uint16_t { return (uint16_t)local.at(c); };
    // ---- sections
    const uint32_t n_ops = lb[NL] - lb[0];
    std::vector<uint32_t> lvl(NL + 1), pw(n_ops);
    std::vector<uint16_t> cw((size_t)n_ops * 4), ovf;
    uint32_t max_level = 0;
    for (uint32_t l = 0; l <= NL; ++l) lvl[l] = lb[l] - lb[0];
    for (uint32_t l = 0; l < NL; ++l) max_level = std::max(max_level, lb[l + 1] - lb[l]);
    // within a level, ops by (output class, opcode, arity): the warps of a
    // level then mostly store one width and take one path
    std::vector<uint32_t> order(lb[NL] - lb[0]);
    for (uint32_t l = 0; l < NL; ++l) {
      auto first = order.begin() + (lb[l] - lb[0]), last = order.begin() + (lb[l + 1] - lb[0]);
      std::iota(first, last, lb[l]);
      auto key = [&](uint32_t x) {
        const uint32_t j = plan.ops[x] & 0x7FFFFFFFu;
        return ((out_coord[j] >> 30) << 16) | (((g.opw[j] >> 22) & 15u) << 8) | (g.opw[j] >> 26);
      };
      std::stable_sort(first, last, [&](uint32_t u, uint32_t v) { return key(u) < key(v); });
    }
    for (uint32_t x0 = lb[0]; x0 < lb[NL]; ++x0) {
      const uint32_t x = order[x0 - lb[0]];
      const uint32_t i = x0 - lb[0], j = plan.ops[x] & 0x7FFFFFFFu;
      const uint32_t n = g.coord_off[j + 1] - g.coord_off[j];
      pw[i] = g.opw[j];
      cw[4 * i] = L(out_coord[j]);
      const uint32_t* cp = g.coord.data() + g.coord_off[j];
      cw[4 * i + 1] = L(cp[0]);
      cw[4 * i + 2] = n >= 2 ? L(cp[1]) : cw[4 * i + 1];
      if (n <= 3) {
        cw[4 * i + 3] = n >= 3 ? L(cp[2]) : cw[4 * i + 1];
      } else {
        if (ovf.size() + n > 65535u) {
          *err = "repcut slice: too many long-fold operands";
          return false;
        }
        cw[4 * i + 3] = (uint16_t)ovf.size();
        for (uint32_t o = 2; o < n; ++o) ovf.push_back(L(cp[o]));
      }
      op_k->push_back((plan.ops[x] >> 31) ? g.opk[j] : 0ull);
    }
    std::vector<uint32_t> commit, pull, inj, map;
    for (uint32_t k = plan.reg_begin[p]; k < plan.reg_begin[p + 1]; ++k) {
      const uint32_t r = plan.regs[k];
      commit.push_back(L(g.reg_coord[r]) | ((uint32_t)L(g.reg_next_coord[r]) << 16));
      commit.push_back(r | (g.reg_w[r] << 24));
      commit.push_back((uint32_t)g.reg_k[r]);
      commit.push_back((uint32_t)(g.reg_k[r] >> 32));
    }
    for (uint32_t c : sigs) {
      auto it = reg_of_coord.find(c);
      if (it != reg_of_coord.end()) {
        const uint32_t r = it->second;
        if (reg_owner[r] != p) {
          pull.push_back(L(c));
          pull.push_back(r);
        }
      }
      map.push_back(L(c));
      map.push_back(c);
    }
    for (uint32_t k = 0; k < NI; ++k)
      if (reads_in[p][k] || (*in_owner)[k] == p) {
        const bool own = (*in_owner)[k] == p;
        inj.push_back(L(g.in_coord[k]) | (g.in_w[k] << 16));
        inj.push_back(k);
        inj.push_back(own ? (uint32_t)g.in_k[k] : 0u);
        inj.push_back(own ? (uint32_t)(g.in_k[k] >> 32) : 0u);
      }
    RepSliceHdr h{};
    size_t o = align16(sizeof(RepSliceHdr));
    h.off_lvl = (uint32_t)o; o = align16(o + lvl.size() * 4);
    h.off_pw = (uint32_t)o; o = align16(o + pw.size() * 4);
    h.off_cw = (uint32_t)o; o = align16(o + cw.size() * 2);
    h.off_ovf = (uint32_t)o; o = align16(o + ovf.size() * 2);
    h.off_commit = (uint32_t)o; o = align16(o + commit.size() * 4);
    h.off_pull = (uint32_t)o; o = align16(o + pull.size() * 4);
    h.off_inj = (uint32_t)o; o = align16(o + inj.size() * 4);
    // the op hash weights join the slice when they fit (else read from global memory)
    h.off_kop = (uint32_t)o;
    if (o + (size_t)n_ops * 8 + state_bytes <= max_smem) {
      h.kop_smem = 1;
      o = align16(o + (size_t)n_ops * 8);
    }
    h.smem_bytes = (uint32_t)o;
    h.state_off = (uint32_t)o;
    h.state_bytes = state_bytes;
    h.off_map = (uint32_t)o; o = align16(o + map.size() * 4);
    h.b1 = bnd[2]; h.b2 = bnd[1]; h.b3 = bnd[0];
    h.n_levels = NL; h.n_ops = n_ops; h.max_level = max_level; h.wide = wide ? 1u : 0u;
    h.n_commit = (uint32_t)commit.size() / 4; h.n_pull = (uint32_t)pull.size() / 2;
    h.n_inj = (uint32_t)inj.size() / 4; h.n_map = (uint32_t)map.size() / 2;
    h.k_base = (uint32_t)(op_k->size() - n_ops);
    if ((size_t)h.smem_bytes + state_bytes > max_smem) {
      *err = "repcut slice " + std::to_string(p) + ": " + std::to_string(h.smem_bytes + state_bytes) +
             " bytes of shared memory > " + std::to_string(max_smem);
      return false;
    }
    const size_t base = align16(blob->size());
    (*slice_off)[p] = base;
    blob->resize(base + o, 0);
    uint8_t* b = blob->data() + base;
    std::memcpy(b, &h, sizeof h);
    auto cp = [&](uint32_t at, const void* src, size_t n) { if (n) std::memcpy(b + at, src, n); };
    cp(h.off_lvl, lvl.data(), lvl.size() * 4);
    cp(h.off_pw, pw.data(), pw.size() * 4);
    cp(h.off_cw, cw.data(), cw.size() * 2);
    cp(h.off_ovf, ovf.data(), ovf.size() * 2);
    cp(h.off_commit, commit.data(), commit.size() * 4);
    cp(h.off_pull, pull.data(), pull.size() * 4);
    cp(h.off_inj, inj.data(), inj.size() * 4);
    if (h.kop_smem) cp(h.off_kop, op_k->data() + h.k_base, (size_t)n_ops * 8);
    cp(h.off_map, map.data(), map.size() * 4);
  }
  return true;
}

}  // namespace rtlsim
