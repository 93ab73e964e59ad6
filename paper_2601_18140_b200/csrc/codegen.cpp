// codegen.cpp -- per-design specialised step kernel (kernel 8) as PTX; see codegen.hpp.
//
// Op semantics are those of kernels.cuh apply_op (Cascade 1 op_u / op_r / op_s, PAPER.md
// eq:step4c P:826-830, alg:opn P:753-775 with the O-rank fold order P:778-796, op_s
// P:839-843, mux App. A); the cycle order is that of every other step kernel:
// inject inputs, evaluate the levels in order, hash, latch the registers simultaneously
// (alg:RU P:1012; R12 / R13 for the hash and the stimulus).
//
// Register types: a signal of width class 0..2 (<= 32 bits) lives in a .b32 register,
// class 3 in a .b64.  An op whose result bits depend only on its operands' low bits
// (and / or / xor / add / sub / mul / not / shl / cat / mux data / copy) is computed at
// the width of its result (operands truncated); shr / bits / eq / lt / the mux selector
// at the width of their operands.  The hash Σ v·K mod 2^64 is kept as a 64-bit low
// accumulator plus a 32-bit high one: v·K = lo·Klo + 2^32 (lo·Khi + hi·Klo) mod 2^64.
#include "codegen.hpp"

#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <unordered_map>
#include <unordered_set>

namespace rtlsim {
namespace {

std::string hex(uint64_t v) {
  char b[32];
  std::snprintf(b, sizeof b, "0x%016" PRIx64, v);
  return b;
}
std::string num(uint64_t v) { return std::to_string(v); }

struct Val {
  bool w64 = false;
  std::string reg;  // register name
};

struct Emit {
  std::string s;
  uint32_t n32 = 0, n64 = 0, np = 0;
  std::string r32() { return "%r" + num(n32++); }
  std::string r64() { return "%d" + num(n64++); }
  std::string reg(bool w64) { return w64 ? r64() : r32(); }
  std::string pr() { return "%p" + num(np++); }
  void ins(const std::string& x) { s += "\t" + x + ";\n"; }
  void label(const std::string& l) { s += l + ":\n"; }
};

// SuArgs field offsets (codegen.hpp)
enum : uint32_t {
  F_STATE = 0, F_TILE_BYTES = 8, F_REGION = 16, F_LT = 48, F_N_LANES = 56, F_LANE0 = 64, F_CYCLE0 = 72,
  F_N_CYCLES = 80, F_STAGED = 88, F_SEED = 96, F_STAGE = 104, F_STAGE_CAP = 112, F_HASHES = 120, F_HCARRY = 128
};

class Gen {
 public:
  // single-lane graphs: one warp runs the lane, all 32 threads on the same values (no
  // divergence), thread t computing the stimulus of inputs t, t + 32, ... in parallel
  // (broadcast with shfl); thread 0 alone stores
  explicit Gen(const CompiledGraph& cg) : cg_(cg), warp_((cg.mode & 0xFFu) == RS_MODE_SINGLE) {}
  std::string run();

 private:
  const CompiledGraph& cg_;
  const bool warp_;
  Emit e_;
  std::unordered_map<uint32_t, Val> sig_;  // coordinate -> register holding the signal's value
  std::vector<uint32_t> out_coord_;
  // kernel-wide registers
  std::string lane_, gl_, tb_, lin_, base_[4], stride_[4], sk0_;
  std::vector<std::string> sk_;                  // (seed, k) stimulus prefixes
  std::string c_, ci_, nlast_, hp_, hstride_, pstaged_, phash_, stage_, stage_cap_, nl8_;
  // hash accumulators: kAcc independent (lo, hi) pairs, dealt round-robin, so the Σ v·K
  // chain does not serialise the cycle on the multiply-add latency
  static constexpr int kAcc = 8;
  std::string hl_[kAcc], hh_[kAcc], wl_, wid_, pw0_, pst_;
  int acc_ = 0;
  void acc_zero(uint64_t init);
  std::string acc_sum();  // H = Σ hl + (Σ hh << 32)
  std::string pred_st() const { return warp_ ? "@" + pw0_ + " " : std::string(); }

  static bool cls64(uint32_t coord) { return (coord >> 30) == 3u; }
  const Val& sig(uint32_t coord) { return sig_.at(coord); }
  std::string as(const Val& v, bool w64);
  void sm64(const std::string& d, const std::string& x);
  void hash_add(const Val& v, uint64_t K);
  void store(uint32_t coord, const Val& v);
  std::string op_expr(uint32_t j);
  void body(bool wb);
  void inputs(const std::string& sfx, bool do_hash, bool do_store);
  // multi-warp single lane (W_ > 1): ops of every level dealt to W_ warps, values another
  // warp reads exchanged through shared memory, one named barrier per level
  uint32_t W_ = 1;
  std::vector<uint32_t> owner_;          // op -> warp
  std::vector<int32_t> xslot_;           // op -> shared slot of its value (another warp reads it), or -1
  uint32_t n_x_ = 0, off_reg_ = 0, off_hs_ = 0, smem_bytes_ = 0;
  std::string smb_, ci_par_;             // shared base address (u32), cycle parity
  void plan_warps();
  void body_mw(uint32_t w, bool wb);
 public:
  uint32_t threads() const { return warp_ ? 32u * W_ : 128u; }
};

std::string Gen::as(const Val& v, bool w64) {
  if (v.w64 == w64) return v.reg;
  const std::string t = e_.reg(w64);
  e_.ins(std::string(w64 ? "cvt.u64.u32 " : "cvt.u32.u64 ") + t + ", " + v.reg);
  return t;
}

// splitmix64 finaliser (R13; kernels.cuh d_splitmix_next): d = sm64(x)
void Gen::sm64(const std::string& d, const std::string& x) {
  const std::string z = e_.r64(), t = e_.r64();
  e_.ins("add.u64 " + z + ", " + x + ", 0x9E3779B97F4A7C15");
  e_.ins("shr.u64 " + t + ", " + z + ", 30");
  e_.ins("xor.b64 " + z + ", " + z + ", " + t);
  e_.ins("mul.lo.u64 " + z + ", " + z + ", 0xBF58476D1CE4E5B9");
  e_.ins("shr.u64 " + t + ", " + z + ", 27");
  e_.ins("xor.b64 " + z + ", " + z + ", " + t);
  e_.ins("mul.lo.u64 " + z + ", " + z + ", 0x94D049BB133111EB");
  e_.ins("shr.u64 " + t + ", " + z + ", 31");
  e_.ins("xor.b64 " + d + ", " + z + ", " + t);
}

void Gen::hash_add(const Val& v, uint64_t K) {
  if (!K) return;
  const uint32_t klo = (uint32_t)K, khi = (uint32_t)(K >> 32);
  const std::string& hl = hl_[acc_], & hh = hh_[acc_];
  acc_ = (acc_ + 1) % kAcc;
  if (!v.w64) {
    e_.ins("mad.wide.u32 " + hl + ", " + v.reg + ", " + num(klo) + ", " + hl);
    e_.ins("mad.lo.u32 " + hh + ", " + v.reg + ", " + num(khi) + ", " + hh);
  } else {
    const std::string lo = e_.r32(), hi = e_.r32();
    e_.ins("mov.b64 {" + lo + ", " + hi + "}, " + v.reg);
    e_.ins("mad.wide.u32 " + hl + ", " + lo + ", " + num(klo) + ", " + hl);
    e_.ins("mad.lo.u32 " + hh + ", " + lo + ", " + num(khi) + ", " + hh);
    e_.ins("mad.lo.u32 " + hh + ", " + hi + ", " + num(klo) + ", " + hh);
  }
}

void Gen::acc_zero(uint64_t init) {
  for (int a = 0; a < kAcc; ++a) {
    e_.ins("mov.u64 " + hl_[a] + ", " + (a == 0 ? hex(init) : std::string("0")));
    e_.ins("mov.u32 " + hh_[a] + ", 0");
  }
  acc_ = 0;
}

std::string Gen::acc_sum() {
  std::string l = hl_[0], h = hh_[0];
  for (int a = 1; a < kAcc; ++a) {
    const std::string l2 = e_.r64(), h2 = e_.r32();
    e_.ins("add.u64 " + l2 + ", " + l + ", " + hl_[a]);
    e_.ins("add.u32 " + h2 + ", " + h + ", " + hh_[a]);
    l = l2;
    h = h2;
  }
  const std::string t = e_.r64(), H = e_.r64();
  e_.ins("cvt.u64.u32 " + t + ", " + h);
  e_.ins("shl.b64 " + t + ", " + t + ", 32");
  e_.ins("add.u64 " + H + ", " + l + ", " + t);
  return H;
}

void Gen::store(uint32_t coord, const Val& v) {
  const uint32_t c = coord >> 30, row = coord & ROW_MASK;
  const std::string a = e_.r64();
  e_.ins("mad.lo.u64 " + a + ", " + stride_[c] + ", " + num(row) + ", " + base_[c]);
  static const char* ty[4] = {"u8", "u16", "u32", "u64"};
  e_.ins(pred_st() + "st.global." + ty[c] + " [" + a + "], " + v.reg);
}

// Emit op j; returns the register holding its (masked) result, of its out class's type.
std::string Gen::op_expr(uint32_t j) {
  const uint32_t pw = cg_.opw[j];
  const uint32_t w = pw & 127u, p0 = (pw >> 7) & 127u, p1 = (pw >> 14) & 63u, op = (pw >> 22) & 15u;
  const uint32_t c0 = cg_.coord_off[j], n = cg_.coord_off[j + 1] - c0;
  const bool o64 = cls64(out_coord_[j]);
  std::vector<const Val*> X(n);
  for (uint32_t o = 0; o < n; ++o) X[o] = &sig(cg_.coord[c0 + o]);
  bool c64 = o64;  // compute width
  std::string d;
  auto T = [&](bool w64) { return std::string(w64 ? "64" : "32"); };
  auto fold = [&](const char* inst) {
    d = as(*X[0], c64);
    for (uint32_t o = 1; o < n; ++o) {
      const std::string t = e_.reg(c64);
      e_.ins(std::string(inst) + T(c64) + " " + t + ", " + d + ", " + as(*X[o], c64));
      d = t;
    }
  };
  switch (op) {
    case RS_OP_AND: fold("and.b"); break;
    case RS_OP_OR: fold("or.b"); break;
    case RS_OP_XOR: fold("xor.b"); break;
    case RS_OP_ADD: fold("add.u"); break;
    case RS_OP_SUB: fold("sub.u"); break;
    case RS_OP_MUL: fold("mul.lo.u"); break;
    case RS_OP_EQ:
    case RS_OP_LT: {
      const bool k64 = X[0]->w64 || X[1]->w64;
      const std::string p = e_.pr();
      e_.ins(std::string(op == RS_OP_EQ ? "setp.eq.u" : "setp.lt.u") + T(k64) + " " + p + ", " + as(*X[0], k64) +
             ", " + as(*X[1], k64));
      d = e_.reg(c64);
      e_.ins("selp.b" + T(c64) + " " + d + ", 1, 0, " + p);
      break;
    }
    case RS_OP_NOT:
      d = e_.reg(c64);
      e_.ins("not.b" + T(c64) + " " + d + ", " + as(*X[0], c64));
      break;
    case RS_OP_SHL:
      d = e_.reg(c64);
      if (p0 >= (c64 ? 64u : 32u)) e_.ins("mov.b" + T(c64) + " " + d + ", 0");
      else e_.ins("shl.b" + T(c64) + " " + d + ", " + as(*X[0], c64) + ", " + num(p0));
      break;
    case RS_OP_SHR:
    case RS_OP_BITS: {
      c64 = o64 || X[0]->w64;
      const uint32_t sh = op == RS_OP_SHR ? p0 : p1;
      d = e_.reg(c64);
      if (sh >= (c64 ? 64u : 32u)) e_.ins("mov.b" + T(c64) + " " + d + ", 0");
      else e_.ins("shr.u" + T(c64) + " " + d + ", " + as(*X[0], c64) + ", " + num(sh));
      if (op == RS_OP_BITS) {
        const uint32_t bw = p0 - p1 + 1u;
        if (bw < (c64 ? 64u : 32u)) {
          const std::string t = e_.reg(c64);
          e_.ins("and.b" + T(c64) + " " + t + ", " + d + ", " + hex(width_mask(bw)));
          d = t;
        }
      }
      break;
    }
    case RS_OP_CAT:
      if (p0 >= (c64 ? 64u : 32u)) {
        d = as(*X[1], c64);
      } else {
        const std::string t = e_.reg(c64);
        e_.ins("shl.b" + T(c64) + " " + t + ", " + as(*X[0], c64) + ", " + num(p0));
        d = e_.reg(c64);
        e_.ins("or.b" + T(c64) + " " + d + ", " + t + ", " + as(*X[1], c64));
      }
      break;
    case RS_OP_MUX: {
      const std::string p = e_.pr();
      e_.ins("setp.ne.u" + T(X[0]->w64) + " " + p + ", " + X[0]->reg + ", 0");
      d = e_.reg(c64);
      e_.ins("selp.b" + T(c64) + " " + d + ", " + as(*X[1], c64) + ", " + as(*X[2], c64) + ", " + p);
      break;
    }
    default: d = as(*X[0], c64); break;  // OP_COPY
  }
  if (w < (c64 ? 64u : 32u)) {
    const std::string t = e_.reg(c64);
    e_.ins("and.b" + T(c64) + " " + t + ", " + d + ", " + hex(width_mask(w)));
    d = t;
  }
  if (c64 && !o64) {
    const std::string t = e_.r32();
    e_.ins("cvt.u32.u64 " + t + ", " + d);
    d = t;
  }
  return d;
}

void Gen::inputs(const std::string& sfx, bool do_hash, bool do_store) {
  // step 1: inputs (staged ring or counter-based stimulus)
  const uint32_t NI = cg_.n_inputs;
  if (NI) {
    e_.ins("@" + pstaged_ + " bra STG" + sfx);
    std::vector<std::string> ys(sk_.size());
    for (size_t m = 0; m < sk_.size(); ++m) {  // one stimulus per input, or per 32 inputs and thread (warp_)
      const std::string x = e_.r64(), z = e_.r64();
      ys[m] = e_.r64();
      e_.ins("add.u64 " + x + ", " + sk_[m] + ", " + c_);
      sm64(z, x);
      e_.ins("add.u64 " + z + ", " + z + ", " + gl_);
      sm64(ys[m], z);
    }
    for (uint32_t k = 0; k < NI; ++k) {
      const Val& v = sig(cg_.in_coord[k]);
      std::string y = ys[warp_ ? k / 32 : k];
      if (warp_) {  // input k's value from thread k % 32
        const std::string lo = e_.r32(), hi = e_.r32(), lo2 = e_.r32(), hi2 = e_.r32();
        e_.ins("mov.b64 {" + lo + ", " + hi + "}, " + y);
        e_.ins("shfl.sync.idx.b32 " + lo2 + ", " + lo + ", " + num(k % 32) + ", 31, -1");
        if (v.w64) {
          e_.ins("shfl.sync.idx.b32 " + hi2 + ", " + hi + ", " + num(k % 32) + ", 31, -1");
          y = e_.r64();
          e_.ins("mov.b64 " + y + ", {" + lo2 + ", " + hi2 + "}");
        } else {
          e_.ins("and.b32 " + v.reg + ", " + lo2 + ", " + hex(width_mask(cg_.in_w[k])));
          continue;
        }
      }
      if (v.w64) e_.ins("and.b64 " + v.reg + ", " + y + ", " + hex(width_mask(cg_.in_w[k])));
      else {
        const std::string t = e_.r32();
        e_.ins("cvt.u32.u64 " + t + ", " + y);
        e_.ins("and.b32 " + v.reg + ", " + t + ", " + hex(width_mask(cg_.in_w[k])));
      }
    }
    e_.ins("bra.uni INJ" + sfx);
    e_.label("STG" + sfx);
    {
      const std::string slot = e_.r64(), a = e_.r64();
      e_.ins("rem.u64 " + slot + ", " + c_ + ", " + stage_cap_);
      e_.ins("mul.lo.u64 " + slot + ", " + slot + ", " + num(NI));
      e_.ins("mul.lo.u64 " + slot + ", " + slot + ", " + nl8_);
      e_.ins("mad.lo.u64 " + a + ", " + lane_ + ", 8, " + stage_);
      e_.ins("add.u64 " + a + ", " + a + ", " + slot);
      for (uint32_t k = 0; k < NI; ++k) {
        const Val& v = sig(cg_.in_coord[k]);
        const std::string y = e_.r64();
        e_.ins("ld.global.u64 " + y + ", [" + a + "]");
        if (k + 1 < NI) e_.ins("add.u64 " + a + ", " + a + ", " + nl8_);
        if (v.w64) e_.ins("and.b64 " + v.reg + ", " + y + ", " + hex(width_mask(cg_.in_w[k])));
        else {
          const std::string t = e_.r32();
          e_.ins("cvt.u32.u64 " + t + ", " + y);
          e_.ins("and.b32 " + v.reg + ", " + t + ", " + hex(width_mask(cg_.in_w[k])));
        }
      }
    }
    e_.label("INJ" + sfx);
    for (uint32_t k = 0; k < NI; ++k) {
      if (do_hash) hash_add(sig(cg_.in_coord[k]), cg_.in_k[k]);
      if (do_store) store(cg_.in_coord[k], sig(cg_.in_coord[k]));
    }
  }
}

void Gen::body(bool wb) {
  const std::string sfx = wb ? "_w" : "_l";
  acc_zero(cg_.const_hash);
  inputs(sfx, true, wb);
  // register term of the hash (values at the start of the cycle)
  for (uint32_t j = 0; j < cg_.n_regs; ++j) hash_add(sig(cg_.reg_coord[j]), cg_.reg_k[j]);
  // steps 2a-2c, level by level (device order is level-major)
  for (uint32_t j = 0; j < cg_.n_ops_total(); ++j) {
    const Val& out = sig_.at(out_coord_[j]);
    const std::string d = op_expr(j);
    e_.ins(std::string(out.w64 ? "mov.b64 " : "mov.b32 ") + out.reg + ", " + d);
    hash_add(out, cg_.opk[j]);
    if (wb) store(out_coord_[j], out);
  }
  // step 3: the cycle's hash H = hl + (hh << 32)
  {
    const std::string H = acc_sum();
    e_.ins("@" + pst_ + " st.global.u64 [" + hp_ + "], " + H);
    e_.ins("add.u64 " + hp_ + ", " + hp_ + ", " + hstride_);
  }
  // step 4: simultaneous register latch
  std::vector<std::string> nx(cg_.n_regs);
  for (uint32_t j = 0; j < cg_.n_regs; ++j) {
    const Val& R = sig(cg_.reg_coord[j]);
    const Val& src = sig(cg_.reg_next_coord[j]);
    std::string v = as(src, R.w64);
    const uint32_t w = cg_.reg_w[j];
    if (w < (R.w64 ? 64u : 32u)) {
      const std::string t = e_.reg(R.w64);
      e_.ins(std::string(R.w64 ? "and.b64 " : "and.b32 ") + t + ", " + v + ", " + hex(width_mask(w)));
      v = t;
    } else {
      const std::string t = e_.reg(R.w64);
      e_.ins(std::string(R.w64 ? "mov.b64 " : "mov.b32 ") + t + ", " + v);
      v = t;
    }
    nx[j] = v;
  }
  for (uint32_t j = 0; j < cg_.n_regs; ++j) {
    const Val& R = sig(cg_.reg_coord[j]);
    e_.ins(std::string(R.w64 ? "mov.b64 " : "mov.b32 ") + R.reg + ", " + nx[j]);
  }
  if (wb) {  // state write-back of the registers and the register term of the next cycle's hash
    acc_zero(0);
    for (uint32_t j = 0; j < cg_.n_regs; ++j) {
      store(cg_.reg_coord[j], sig(cg_.reg_coord[j]));
      hash_add(sig(cg_.reg_coord[j]), cg_.reg_k[j]);
    }
    const std::string H = acc_sum(), a = e_.r64(), hc = e_.r64();
    e_.ins("ld.param.u64 " + hc + ", [rs_su_a+" + num(F_HCARRY) + "]");
    e_.ins("cvta.to.global.u64 " + hc + ", " + hc);
    e_.ins("mad.lo.u64 " + a + ", " + lane_ + ", 8, " + hc);
    e_.ins(pred_st() + "st.global.u64 [" + a + "], " + H);
  }
}

void Gen::plan_warps() {
  const uint32_t NO = cg_.n_ops_total(), NL = cg_.n_levels;
  W_ = 1;
  if (!warp_ || NO == 0) return;
  const uint32_t avg = NO / std::max<uint32_t>(1, NL);
  // measured on C1 (18.6 ops per level; profiles/r02/kernel8): 1 / 2 / 3 / 4 / 6 / 8 warps = 1.53 / 1.33 /
  // 1.18 / 1.05 / 1.02 / 1.09 us per cycle
  W_ = std::min<uint32_t>(8, std::max<uint32_t>(1, avg / 3));
  if (const char* e = std::getenv("RTLSIM_K8_WARPS")) W_ = std::min<uint32_t>(8, std::max(1, std::atoi(e)));
  if (W_ == 1) return;
  std::unordered_map<uint32_t, uint32_t> prod;  // op output coordinate -> op
  for (uint32_t j = 0; j < NO; ++j) prod[out_coord_[j]] = j;
  owner_.assign(NO, 0);
  for (uint32_t l = 0; l < NL; ++l) {
    const uint32_t lb = cg_.level_op_begin[l], le = cg_.level_op_begin[l + 1], cap = (le - lb + W_ - 1) / W_;
    std::vector<uint32_t> load(W_, 0);
    for (uint32_t j = lb; j < le; ++j) {  // the warp that produced most operands, among those with room
      std::vector<uint32_t> score(W_, 0);
      for (uint32_t o = cg_.coord_off[j]; o < cg_.coord_off[j + 1]; ++o) {
        auto it = prod.find(cg_.coord[o]);
        if (it != prod.end()) score[owner_[it->second]]++;
      }
      uint32_t best = W_;
      for (uint32_t w = 0; w < W_; ++w) {
        if (load[w] >= cap) continue;
        if (best == W_ || score[w] > score[best] || (score[w] == score[best] && load[w] < load[best])) best = w;
      }
      owner_[j] = best;
      load[best]++;
    }
  }
  xslot_.assign(NO, -1);
  for (uint32_t j = 0; j < NO; ++j)
    for (uint32_t o = cg_.coord_off[j]; o < cg_.coord_off[j + 1]; ++o) {
      auto it = prod.find(cg_.coord[o]);
      if (it != prod.end() && owner_[it->second] != owner_[j] && xslot_[it->second] < 0)
        xslot_[it->second] = (int32_t)n_x_++;
    }
  off_reg_ = 8 * n_x_;
  off_hs_ = off_reg_ + 16 * cg_.n_regs;
  smem_bytes_ = off_hs_ + 16 * W_;
}

void Gen::body_mw(uint32_t w, bool wb) {
  const std::string sfx = "_" + num(w) + (wb ? "w" : "l");
  const uint32_t NR = cg_.n_regs, NO = cg_.n_ops_total();
  static const char* sty[2] = {"u32", "u64"};
  // this cycle's buffers: registers [2][NR], hash partials [2][W] by cycle parity
  std::string regcur = e_.r32(), regnxt = e_.r32(), hsb = e_.r32();
  {
    const std::string p = e_.r32(), q = e_.r32();
    e_.ins("cvt.u32.u64 " + p + ", " + ci_);
    e_.ins("and.b32 " + p + ", " + p + ", 1");
    e_.ins("xor.b32 " + q + ", " + p + ", 1");
    e_.ins("mad.lo.u32 " + regcur + ", " + p + ", " + num(8 * NR) + ", " + smb_);
    e_.ins("mad.lo.u32 " + regnxt + ", " + q + ", " + num(8 * NR) + ", " + smb_);
    e_.ins("mad.lo.u32 " + hsb + ", " + p + ", " + num(8 * W_) + ", " + smb_);
  }
  acc_zero(w == 0 ? cg_.const_hash : 0);
  inputs(sfx, w == 0, wb && w == 0);
  // registers this warp reads or hashes
  std::unordered_set<uint32_t> regs_read;
  std::unordered_map<uint32_t, uint32_t> reg_of;  // register coordinate -> register index
  for (uint32_t j = 0; j < NR; ++j) reg_of[cg_.reg_coord[j]] = j;
  for (uint32_t j = 0; j < NO; ++j)
    if (owner_[j] == w)
      for (uint32_t o = cg_.coord_off[j]; o < cg_.coord_off[j + 1]; ++o)
        if (reg_of.count(cg_.coord[o])) regs_read.insert(reg_of[cg_.coord[o]]);
  for (uint32_t j = 0; j < NR; ++j) {
    if (!regs_read.count(j) && j % W_ != w) continue;
    const Val& R = sig(cg_.reg_coord[j]);
    e_.ins(std::string("ld.shared.") + sty[R.w64] + " " + R.reg + ", [" + regcur + "+" + num(off_reg_ + 8 * j) + "]");
    if (j % W_ == w) hash_add(R, cg_.reg_k[j]);
  }
  // registers whose next value is not an op's (a constant): warp 0 posts it now
  std::unordered_map<uint32_t, std::vector<uint32_t>> next_of;  // next-source coordinate -> registers
  for (uint32_t j = 0; j < NR; ++j) next_of[cg_.reg_next_coord[j]].push_back(j);
  std::unordered_set<uint32_t> op_out(out_coord_.begin(), out_coord_.end());
  auto post_next = [&](uint32_t r, const Val& src) {
    const Val& R = sig(cg_.reg_coord[r]);
    std::string v = as(src, R.w64);
    if (cg_.reg_w[r] < (R.w64 ? 64u : 32u)) {
      const std::string t = e_.reg(R.w64);
      e_.ins(std::string(R.w64 ? "and.b64 " : "and.b32 ") + t + ", " + v + ", " + hex(width_mask(cg_.reg_w[r])));
      v = t;
    }
    e_.ins("@" + pw0_ + " st.shared." + sty[R.w64] + " [" + regnxt + "+" + num(off_reg_ + 8 * r) + "], " + v);
  };
  if (w == 0)
    for (uint32_t r = 0; r < NR; ++r)
      if (!op_out.count(cg_.reg_next_coord[r])) post_next(r, sig(cg_.reg_next_coord[r]));
  std::unordered_map<uint32_t, uint32_t> prod;
  for (uint32_t j = 0; j < NO; ++j) prod[out_coord_[j]] = j;
  std::unordered_set<uint32_t> loaded;
  const uint32_t NL = std::max<uint32_t>(1, cg_.n_levels);
  for (uint32_t l = 0; l < NL; ++l) {
    const uint32_t lb = cg_.n_levels ? cg_.level_op_begin[l] : 0, le = cg_.n_levels ? cg_.level_op_begin[l + 1] : 0;
    for (uint32_t j = lb; j < le; ++j) {
      if (owner_[j] != w) continue;
      for (uint32_t o = cg_.coord_off[j]; o < cg_.coord_off[j + 1]; ++o) {  // other warps' values
        auto it = prod.find(cg_.coord[o]);
        if (it == prod.end() || owner_[it->second] == w || loaded.count(cg_.coord[o])) continue;
        const Val& v = sig(cg_.coord[o]);
        e_.ins(std::string("ld.shared.") + sty[v.w64] + " " + v.reg + ", [" + smb_ + "+" + num(8 * xslot_[it->second]) + "]");
        loaded.insert(cg_.coord[o]);
      }
      const Val& out = sig_.at(out_coord_[j]);
      const std::string d = op_expr(j);
      e_.ins(std::string(out.w64 ? "mov.b64 " : "mov.b32 ") + out.reg + ", " + d);
      hash_add(out, cg_.opk[j]);
      if (xslot_[j] >= 0)
        e_.ins("@" + pw0_ + " st.shared." + sty[out.w64] + " [" + smb_ + "+" + num(8 * xslot_[j]) + "], " + out.reg);
      auto nx = next_of.find(out_coord_[j]);
      if (nx != next_of.end())
        for (uint32_t r : nx->second) post_next(r, out);
      if (wb) store(out_coord_[j], out);
    }
    if (l + 1 == NL) {  // this warp's share of the cycle's hash
      const std::string H = acc_sum();
      e_.ins("@" + pw0_ + " st.shared.u64 [" + hsb + "+" + num(off_hs_ + 8 * w) + "], " + H);
    }
    e_.ins("bar.sync 1, " + num(32 * W_));
  }
  if (w == 0) {
    std::string H = e_.r64();
    e_.ins("ld.shared.u64 " + H + ", [" + hsb + "+" + num(off_hs_) + "]");
    for (uint32_t k = 1; k < W_; ++k) {
      const std::string t = e_.r64(), H2 = e_.r64();
      e_.ins("ld.shared.u64 " + t + ", [" + hsb + "+" + num(off_hs_ + 8 * k) + "]");
      e_.ins("add.u64 " + H2 + ", " + H + ", " + t);
      H = H2;
    }
    e_.ins("@" + pst_ + " st.global.u64 [" + hp_ + "], " + H);
  }
  e_.ins("add.u64 " + hp_ + ", " + hp_ + ", " + hstride_);
  if (wb && w == 0) {  // the registers after the last latch: state write-back and the hash carry
    acc_zero(0);
    for (uint32_t j = 0; j < NR; ++j) {
      const Val& R = sig(cg_.reg_coord[j]);
      e_.ins(std::string("ld.shared.") + sty[R.w64] + " " + R.reg + ", [" + regnxt + "+" + num(off_reg_ + 8 * j) + "]");
      store(cg_.reg_coord[j], R);
      hash_add(R, cg_.reg_k[j]);
    }
    const std::string H = acc_sum(), a = e_.r64(), hc = e_.r64();
    e_.ins("ld.param.u64 " + hc + ", [rs_su_a+" + num(F_HCARRY) + "]");
    e_.ins("cvta.to.global.u64 " + hc + ", " + hc);
    e_.ins("mad.lo.u64 " + a + ", " + lane_ + ", 8, " + hc);
    e_.ins("@" + pw0_ + " st.global.u64 [" + a + "], " + H);
  }
}

std::string Gen::run() {
  // registers of the design's signals
  out_coord_.resize(cg_.n_ops_total());
  for (const DevRun& r : cg_.runs) {
    const uint32_t cls = (r.meta >> 16) & 3u;
    for (uint32_t i = 0; i < r.count; ++i) out_coord_[r.op_begin + i] = make_coord(cls, r.out_row0 + i);
  }
  auto declare = [&](uint32_t coord) {
    Val v;
    v.w64 = cls64(coord);
    v.reg = e_.reg(v.w64);
    sig_[coord] = v;
  };
  for (uint32_t k = 0; k < cg_.n_inputs; ++k) declare(cg_.in_coord[k]);
  for (uint32_t j = 0; j < cg_.n_regs; ++j) declare(cg_.reg_coord[j]);
  for (size_t k = 0; k < cg_.const_coord.size(); ++k) declare(cg_.const_coord[k]);
  for (uint32_t j = 0; j < cg_.n_ops_total(); ++j) declare(out_coord_[j]);
  plan_warps();

  // prologue: lane, tile, state bases, stimulus prefixes, registers
  auto param = [&](uint32_t off) {
    const std::string r = e_.r64();
    e_.ins("ld.param.u64 " + r + ", [rs_su_a+" + num(off) + "]");
    return r;
  };
  {
    const std::string t = e_.r32(), b = e_.r32(), nt = e_.r32();
    e_.ins("mov.u32 " + t + ", %tid.x");
    e_.ins("mov.u32 " + b + ", %ctaid.x");
    e_.ins("mov.u32 " + nt + ", %ntid.x");
    lane_ = e_.r64();
    if (warp_) {
      wl_ = e_.r32();
      pw0_ = e_.pr();
      e_.ins("and.b32 " + wl_ + ", " + t + ", 31");
      e_.ins("setp.eq.u32 " + pw0_ + ", " + wl_ + ", 0");
      wid_ = e_.r32();
      e_.ins("shr.u32 " + wid_ + ", " + t + ", 5");
      e_.ins("mov.u64 " + lane_ + ", 0");
    } else {
      const std::string t64 = e_.r64();
      e_.ins("mul.wide.u32 " + lane_ + ", " + b + ", " + nt);
      e_.ins("cvt.u64.u32 " + t64 + ", " + t);
      e_.ins("add.u64 " + lane_ + ", " + lane_ + ", " + t64);
    }
  }
  const std::string nlanes = param(F_N_LANES), ncyc = param(F_N_CYCLES);
  {
    const std::string p = e_.pr();
    e_.ins("setp.ge.u64 " + p + ", " + lane_ + ", " + nlanes);
    e_.ins("@" + p + " bra DONE");
    const std::string q = e_.pr();
    e_.ins("setp.eq.u64 " + q + ", " + ncyc + ", 0");
    e_.ins("@" + q + " bra DONE");
  }
  const std::string state = param(F_STATE), tbytes = param(F_TILE_BYTES), LT = param(F_LT);
  e_.ins("cvta.to.global.u64 " + state + ", " + state);
  const std::string tile = e_.r64();
  lin_ = e_.r64();
  tb_ = e_.r64();
  e_.ins("div.u64 " + tile + ", " + lane_ + ", " + LT);
  e_.ins("rem.u64 " + lin_ + ", " + lane_ + ", " + LT);
  e_.ins("mad.lo.u64 " + tb_ + ", " + tile + ", " + tbytes + ", " + state);
  for (int c = 0; c < 4; ++c) {
    const std::string reg = param(F_REGION + 8 * c), t = e_.r64();
    base_[c] = e_.r64();
    stride_[c] = e_.r64();
    e_.ins("shl.b64 " + t + ", " + lin_ + ", " + num(c));
    e_.ins("add.u64 " + base_[c] + ", " + tb_ + ", " + reg);
    e_.ins("add.u64 " + base_[c] + ", " + base_[c] + ", " + t);
    e_.ins("shl.b64 " + stride_[c] + ", " + LT + ", " + num(c));
  }
  const std::string lane0 = param(F_LANE0);
  gl_ = e_.r64();
  e_.ins("add.u64 " + gl_ + ", " + lane0 + ", " + lane_);
  const std::string seed = param(F_SEED);
  sk0_ = e_.r64();
  sm64(sk0_, seed);
  sk_.resize(warp_ ? (cg_.n_inputs + 31) / 32 : cg_.n_inputs);
  for (uint32_t m = 0; m < sk_.size(); ++m) {
    const std::string x = e_.r64();
    sk_[m] = e_.r64();
    if (warp_) {  // this thread's input 32 m + t
      const std::string t64 = e_.r64();
      e_.ins("cvt.u64.u32 " + t64 + ", " + wl_);
      e_.ins("add.u64 " + x + ", " + sk0_ + ", " + t64);
      e_.ins("add.u64 " + x + ", " + x + ", " + num(32ull * m));
    } else {
      e_.ins("add.u64 " + x + ", " + sk0_ + ", " + num(m));
    }
    sm64(sk_[m], x);
  }
  const std::string staged = param(F_STAGED);
  pstaged_ = e_.pr();
  e_.ins("setp.ne.u64 " + pstaged_ + ", " + staged + ", 0");
  stage_ = param(F_STAGE);
  e_.ins("cvta.to.global.u64 " + stage_ + ", " + stage_);
  stage_cap_ = param(F_STAGE_CAP);
  nl8_ = e_.r64();
  e_.ins("shl.b64 " + nl8_ + ", " + nlanes + ", 3");
  // hash output: hashes + (ci * n_lanes + lane) * 8, advancing n_lanes * 8 per cycle
  const std::string hashes = param(F_HASHES);
  phash_ = e_.pr();
  e_.ins("setp.ne.u64 " + phash_ + ", " + hashes + ", 0");
  pst_ = phash_;
  if (warp_) {
    pst_ = e_.pr();
    e_.ins("and.pred " + pst_ + ", " + phash_ + ", " + pw0_);
  }
  e_.ins("cvta.to.global.u64 " + hashes + ", " + hashes);
  hp_ = e_.r64();
  hstride_ = nl8_;
  e_.ins("mad.lo.u64 " + hp_ + ", " + lane_ + ", 8, " + hashes);
  for (int a = 0; a < kAcc; ++a) {
    hl_[a] = e_.r64();
    hh_[a] = e_.r32();
  }
  // constants and registers
  for (size_t k = 0; k < cg_.const_coord.size(); ++k) {
    const Val& v = sig(cg_.const_coord[k]);
    e_.ins(std::string(v.w64 ? "mov.b64 " : "mov.b32 ") + v.reg + ", " +
           (v.w64 ? hex(cg_.const_val[k]) : num((uint32_t)cg_.const_val[k])));
  }
  for (uint32_t j = 0; j < cg_.n_regs; ++j) {
    const uint32_t coord = cg_.reg_coord[j], c = coord >> 30;
    const Val& v = sig(coord);
    const std::string a = e_.r64();
    e_.ins("mad.lo.u64 " + a + ", " + stride_[c] + ", " + num(coord & ROW_MASK) + ", " + base_[c]);
    static const char* ty[4] = {"u8", "u16", "u32", "u64"};
    e_.ins(std::string("ld.global.") + ty[c] + " " + v.reg + ", [" + a + "]");
  }
  // cycle loop: all but the last cycle without stores, the last one with the write-back
  c_ = param(F_CYCLE0);
  ci_ = e_.r64();
  nlast_ = e_.r64();
  e_.ins("mov.u64 " + ci_ + ", 0");
  e_.ins("sub.u64 " + nlast_ + ", " + ncyc + ", 1");
  if (W_ == 1) {
    e_.label("LOOP");
    {
      const std::string p = e_.pr();
      e_.ins("setp.ge.u64 " + p + ", " + ci_ + ", " + nlast_);
      e_.ins("@" + p + " bra FINAL");
    }
    body(false);
    e_.ins("add.u64 " + ci_ + ", " + ci_ + ", 1");
    e_.ins("add.u64 " + c_ + ", " + c_ + ", 1");
    e_.ins("bra.uni LOOP");
    e_.label("FINAL");
    body(true);
  } else {
    // the registers' values for cycle 0 into shared buffer 0, then one stream per warp
    smb_ = e_.r32();
    e_.ins("mov.u32 " + smb_ + ", su_sm");
    {
      const std::string p0 = e_.pr();
      e_.ins("setp.eq.u32 " + p0 + ", " + wid_ + ", 0");
      const std::string pt0 = e_.pr();
      e_.ins("and.pred " + pt0 + ", " + p0 + ", " + pw0_);
      for (uint32_t j = 0; j < cg_.n_regs; ++j) {
        const Val& R = sig(cg_.reg_coord[j]);
        e_.ins("@" + pt0 + " st.shared." + (R.w64 ? std::string("u64") : std::string("u32")) + " [" + smb_ + "+" +
               num(off_reg_ + 8 * j) + "], " + R.reg);
      }
    }
    e_.ins("bar.sync 1, " + num(32 * W_));
    for (uint32_t w = 1; w < W_; ++w) {
      const std::string p = e_.pr();
      e_.ins("setp.eq.u32 " + p + ", " + wid_ + ", " + num(w));
      e_.ins("@" + p + " bra WS_" + num(w));
    }
    for (uint32_t w = 0; w < W_; ++w) {
      e_.label("WS_" + num(w));
      e_.label("LOOP_" + num(w));
      {
        const std::string p = e_.pr();
        e_.ins("setp.ge.u64 " + p + ", " + ci_ + ", " + nlast_);
        e_.ins("@" + p + " bra FINAL_" + num(w));
      }
      body_mw(w, false);
      e_.ins("add.u64 " + ci_ + ", " + ci_ + ", 1");
      e_.ins("add.u64 " + c_ + ", " + c_ + ", 1");
      e_.ins("bra.uni LOOP_" + num(w));
      e_.label("FINAL_" + num(w));
      body_mw(w, true);
      e_.ins("bra.uni DONE");
    }
  }
  e_.label("DONE");
  e_.ins("ret");

  std::string head = ".version 8.7\n.target sm_100a\n.address_size 64\n\n";
  if (W_ > 1) head += ".shared .align 8 .b8 su_sm[" + num(std::max<uint32_t>(8, smem_bytes_)) + "];\n\n";
  head += ".visible .entry rs_su(.param .align 8 .b8 rs_su_a[" + num(sizeof(SuArgs)) + "])\n.maxntid " +
          num(threads()) + ", 1, 1\n{\n";
  head += "\t.reg .pred %p<" + num(e_.np + 1) + ">;\n";
  head += "\t.reg .b32 %r<" + num(e_.n32 + 1) + ">;\n";
  head += "\t.reg .b64 %d<" + num(e_.n64 + 1) + ">;\n";
  return head + e_.s + "}\n";
}

}  // namespace

std::string su_ptx(const CompiledGraph& cg, uint32_t* threads) {
  Gen g(cg);
  std::string p = g.run();
  if (threads) *threads = g.threads();
  return p;
}

}  // namespace rtlsim
