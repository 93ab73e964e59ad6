// passes.cpp -- data-level graph passes of the graph-tensor compiler (SURVEY.md
// §8(f) NEXT-1; §6.1 P:1259-1264 "copy propagation, constant
// propagation", App. B.1), run by compile_graph when rs_load_graph
// is called with RS_LOAD_PASSES.
//
// Constant propagation: an op whose operands are all constants becomes a
// constant signal (its value computed here once); some ops with one constant
// operand are constants too (and with 0, mul by 0, x ^ x, ...).
// Copy propagation: an op whose result provably equals one operand's value for
// every input (shift by 0, bits(x, hi >= w(x) - 1, 0), and with all ones, or /
// xor / add with 0, sub of 0, mul by 1, mux with a constant selector or equal
// branches, cat(0, x) -- each only when the declared width keeps every bit of
// the operand) is removed, and its signal becomes an ALIAS of that operand:
// it has no row, reads of it read the operand's row, and its hash weight is
// added to the operand's (sum_s v_s K_s is unchanged because v_alias = v_rep
// every cycle; reading R12).  Chains collapse (rep of a rep).
//
// Mux chains (mux whose O=2 branch is another mux): counted, not fused -- the
// per-cycle hash covers every inner mux's value, so a fused chain would still
// have to materialise each inner value.
#include <cstring>

#include "compiler.hpp"

namespace rtlsim {

namespace {

uint64_t fold_value(uint32_t op, const uint64_t* x, uint32_t n, uint32_t w_out, uint32_t p0, uint32_t p1,
                    uint32_t wb) {
  uint64_t r = 0;
  switch (op) {
    case RS_OP_AND: r = x[0]; for (uint32_t i = 1; i < n; ++i) r &= x[i]; break;
    case RS_OP_OR: r = x[0]; for (uint32_t i = 1; i < n; ++i) r |= x[i]; break;
    case RS_OP_XOR: r = x[0]; for (uint32_t i = 1; i < n; ++i) r ^= x[i]; break;
    case RS_OP_ADD: r = x[0]; for (uint32_t i = 1; i < n; ++i) r += x[i]; break;
    case RS_OP_SUB: r = x[0]; for (uint32_t i = 1; i < n; ++i) r -= x[i]; break;
    case RS_OP_MUL: r = x[0]; for (uint32_t i = 1; i < n; ++i) r *= x[i]; break;
    case RS_OP_EQ: r = x[0] == x[1]; break;
    case RS_OP_LT: r = x[0] < x[1]; break;
    case RS_OP_NOT: r = ~x[0]; break;
    case RS_OP_SHL: r = p0 >= 64 ? 0 : x[0] << p0; break;
    case RS_OP_SHR: r = p0 >= 64 ? 0 : x[0] >> p0; break;
    case RS_OP_BITS: r = (x[0] >> p1) & width_mask(p0 - p1 + 1); break;
    case RS_OP_CAT: r = wb >= 64 ? x[1] : ((x[0] << wb) | x[1]); break;
    case RS_OP_MUX: r = x[0] != 0 ? x[1] : x[2]; break;
    default: break;
  }
  return r & width_mask(w_out);
}

}  // namespace

void run_passes(const rs_graph_desc* d, const std::vector<int64_t>& drv, const std::vector<uint32_t>& topo,
                PassResult* out) {
  const uint32_t NS = d->n_signals, NO = d->n_ops;
  PassResult& r = *out;
  r = PassResult();
  r.rep.resize(NS);
  for (uint32_t s = 0; s < NS; ++s) r.rep[s] = s;
  std::vector<uint8_t> is_const(NS, 0), is_reg(NS, 0);
  std::vector<uint64_t> cval(NS, 0);
  for (uint32_t i = 0; i < d->n_regs; ++i) is_reg[d->reg_id[i]] = 1;
  for (uint32_t i = 0; i < d->n_consts; ++i) {
    is_const[d->const_id[i]] = 1;
    cval[d->const_id[i]] = d->const_val[i] & width_mask(d->width[d->const_id[i]]);
  }
  std::vector<uint8_t> removed(NO, 0);
  std::vector<uint32_t> args;
  std::vector<uint64_t> vals;
  for (uint32_t j : topo) {
    const uint32_t op = d->opcode[j], out_s = d->out_id[j], w = d->width[out_s];
    const uint32_t a0 = d->arg_off[j], n = d->arg_off[j + 1] - a0;
    args.assign(n, 0);
    vals.assign(n, 0);
    bool all_const = true;
    for (uint32_t i = 0; i < n; ++i) {
      args[i] = r.rep[d->arg_id[a0 + i]];
      all_const = all_const && is_const[args[i]];
      vals[i] = cval[args[i]];
    }
    const uint32_t p0 = (op == RS_OP_SHL || op == RS_OP_SHR || op == RS_OP_BITS) ? d->param[2 * j] : 0;
    const uint32_t p1 = op == RS_OP_BITS ? d->param[2 * j + 1] : 0;
    const uint32_t wb = op == RS_OP_CAT ? d->width[d->arg_id[a0 + 1]] : 0;
    auto wid = [&](uint32_t s) -> uint32_t { return d->width[s]; };
    auto make_const = [&](uint64_t v) {
      is_const[out_s] = 1;
      cval[out_s] = v & width_mask(w);
      removed[j] = 1;
      r.folded.push_back(out_s);
    };
    auto make_alias = [&](uint32_t x) {  // result == value of x for every input
      // never a register: after the commit a register holds its NEXT value, while
      // an op's signal keeps the cycle's value (rs_read_signals would differ)
      if (is_reg[x]) return false;
      r.rep[out_s] = x;
      removed[j] = 1;
      r.n_alias++;
      return true;
    };
    auto kc = [&](uint32_t i, uint64_t v) { return is_const[args[i]] && (cval[args[i]] & width_mask(w)) == v; };
    auto ones = [&](uint32_t i, uint32_t other) {  // constant i covers every bit of the other operand
      const uint64_t m = width_mask(wid(args[other]));
      return is_const[args[i]] && (cval[args[i]] & m) == m;
    };
    if (all_const) {
      make_const(fold_value(op, vals.data(), n, w, p0, p1, wb));
      continue;
    }
    if (n == 2) {
      const uint32_t x0 = args[0], x1 = args[1];
      const bool same = x0 == x1;
      switch (op) {
        case RS_OP_AND:
          if (kc(0, 0) || kc(1, 0)) { make_const(0); continue; }
          if (ones(1, 0) && w >= wid(x0)) { if (make_alias(x0)) continue; }
          if (ones(0, 1) && w >= wid(x1)) { if (make_alias(x1)) continue; }
          if (same && w >= wid(x0)) { if (make_alias(x0)) continue; }
          break;
        case RS_OP_OR:
        case RS_OP_XOR:
        case RS_OP_ADD:
          if (op == RS_OP_XOR && same) { make_const(0); continue; }
          if (op == RS_OP_OR && same && w >= wid(x0)) { if (make_alias(x0)) continue; }
          if (is_const[x1] && cval[x1] == 0 && w >= wid(x0)) { if (make_alias(x0)) continue; }
          if (is_const[x0] && cval[x0] == 0 && w >= wid(x1)) { if (make_alias(x1)) continue; }
          break;
        case RS_OP_SUB:
          if (same) { make_const(0); continue; }
          if (is_const[x1] && cval[x1] == 0 && w >= wid(x0)) { if (make_alias(x0)) continue; }
          break;
        case RS_OP_MUL:
          if (kc(0, 0) || kc(1, 0)) { make_const(0); continue; }
          if (is_const[x1] && cval[x1] == 1 && w >= wid(x0)) { if (make_alias(x0)) continue; }
          if (is_const[x0] && cval[x0] == 1 && w >= wid(x1)) { if (make_alias(x1)) continue; }
          break;
        case RS_OP_EQ:
          if (same) { make_const(1); continue; }
          break;
        case RS_OP_LT:
          if (same) { make_const(0); continue; }
          break;
        case RS_OP_CAT:
          if (is_const[x0] && cval[x0] == 0 && w >= wid(x1)) { if (make_alias(x1)) continue; }
          break;
        default:
          break;
      }
    } else if (n == 1) {
      const uint32_t x0 = args[0];
      if ((op == RS_OP_SHL || op == RS_OP_SHR) && p0 == 0 && w >= wid(x0)) { if (make_alias(x0)) continue; }
      if (op == RS_OP_BITS && p1 == 0 && p0 + 1 >= wid(x0) && w >= wid(x0)) { if (make_alias(x0)) continue; }
      if ((op == RS_OP_SHL && p0 >= w) || (op == RS_OP_SHR && p0 >= wid(x0)) || (op == RS_OP_BITS && p1 >= wid(x0))) {
        make_const(0);
        continue;
      }
    } else if (op == RS_OP_MUX) {
      const uint32_t s = args[0], xa = args[1], xb = args[2];
      if (is_const[s]) {
        const uint32_t x = cval[s] != 0 ? xa : xb;
        if (w >= wid(x)) { if (make_alias(x)) continue; }
      }
      if (xa == xb && w >= wid(xa)) { if (make_alias(xa)) continue; }
    }
  }
  // mux chains: a mux whose O=2 (else) branch is produced by another mux
  {
    std::vector<uint8_t> is_mux(NS, 0);
    for (uint32_t j = 0; j < NO; ++j)
      if (!removed[j] && d->opcode[j] == RS_OP_MUX) is_mux[d->out_id[j]] = 1;
    for (uint32_t j = 0; j < NO; ++j)
      if (!removed[j] && d->opcode[j] == RS_OP_MUX && is_mux[r.rep[d->arg_id[d->arg_off[j] + 2]]]) r.n_mux_chain++;
  }
  // the rewritten graph: surviving ops with operands renamed to their reps;
  // folded signals become constants
  r.width.assign(d->width, d->width + NS);
  r.input_id.assign(d->input_id, d->input_id + d->n_inputs);
  r.reg_id.assign(d->reg_id, d->reg_id + d->n_regs);
  r.reg_next_id.resize(d->n_regs);
  for (uint32_t i = 0; i < d->n_regs; ++i) r.reg_next_id[i] = r.rep[d->reg_next_id[i]];
  if (d->reg_init) r.reg_init.assign(d->reg_init, d->reg_init + d->n_regs);
  else r.reg_init.assign(d->n_regs, 0);
  r.const_id.assign(d->const_id, d->const_id + d->n_consts);
  r.const_val.assign(d->const_val, d->const_val + d->n_consts);
  for (uint32_t s : r.folded) {
    r.const_id.push_back(s);
    r.const_val.push_back(cval[s]);
  }
  r.arg_off.push_back(0);
  for (uint32_t j = 0; j < NO; ++j) {
    if (removed[j]) continue;
    r.opcode.push_back(d->opcode[j]);
    r.out_id.push_back(d->out_id[j]);
    for (uint32_t a = d->arg_off[j]; a < d->arg_off[j + 1]; ++a) r.arg_id.push_back(r.rep[d->arg_id[a]]);
    r.arg_off.push_back((uint32_t)r.arg_id.size());
    r.param.push_back(d->param ? d->param[2 * j] : 0);
    r.param.push_back(d->param ? d->param[2 * j + 1] : 0);
    // cat's w_b is its ORIGINAL operand 1's declared width (a renamed operand may
    // be narrower: same value, different w_b)
    r.cat_wb.push_back(d->opcode[j] == RS_OP_CAT ? d->width[d->arg_id[d->arg_off[j] + 1]] : 0u);
    if (d->level) r.level.push_back(d->level[j]);
  }
  std::memset(&r.desc, 0, sizeof r.desc);
  r.desc.n_signals = NS;
  r.desc.width = r.width.data();
  r.desc.n_inputs = (uint32_t)r.input_id.size();
  r.desc.input_id = r.input_id.data();
  r.desc.n_regs = (uint32_t)r.reg_id.size();
  r.desc.reg_id = r.reg_id.data();
  r.desc.reg_next_id = r.reg_next_id.data();
  r.desc.reg_init = r.reg_init.data();
  r.desc.n_consts = (uint32_t)r.const_id.size();
  r.desc.const_id = r.const_id.data();
  r.desc.const_val = r.const_val.data();
  r.desc.n_ops = (uint32_t)r.opcode.size();
  r.desc.opcode = r.opcode.data();
  r.desc.out_id = r.out_id.data();
  r.desc.arg_off = r.arg_off.data();
  r.desc.arg_id = r.arg_id.data();
  r.desc.param = r.param.data();
  r.desc.level = d->level ? r.level.data() : nullptr;
  (void)drv;
}

}  // namespace rtlsim
