// slice_check.cpp -- host-only diagnostic: compile a circuit dumped by
// tools/dump_circuit.py and report single-lane slice sizes for G CTAs.
//   g++ -O2 -std=c++17 -I include tools/slice_check.cpp paper_2601_18140_b200/csrc/compiler.cpp -o /tmp/slice_check
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2601_18140_b200/csrc/compiler.hpp"

template <class T>
std::vector<T> rd(FILE* f) {
  uint64_t n = 0;
  if (fread(&n, 8, 1, f) != 1) exit(2);
  std::vector<T> v(n);
  if (n && fread(v.data(), sizeof(T), n, f) != n) exit(2);
  return v;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  const unsigned G = argc > 2 ? atoi(argv[2]) : 148;
  auto width = rd<uint8_t>(f);
  auto input_id = rd<uint32_t>(f), reg_id = rd<uint32_t>(f), reg_next = rd<uint32_t>(f);
  auto reg_init = rd<uint64_t>(f);
  auto const_id = rd<uint32_t>(f);
  auto const_val = rd<uint64_t>(f);
  auto opcode = rd<uint8_t>(f);
  auto out_id = rd<uint32_t>(f), arg_off = rd<uint32_t>(f), arg_id = rd<uint32_t>(f), param = rd<uint32_t>(f);
  rs_graph_desc d{};
  d.n_signals = width.size(); d.width = width.data();
  d.n_inputs = input_id.size(); d.input_id = input_id.data();
  d.n_regs = reg_id.size(); d.reg_id = reg_id.data(); d.reg_next_id = reg_next.data(); d.reg_init = reg_init.data();
  d.n_consts = const_id.size(); d.const_id = const_id.data(); d.const_val = const_val.data();
  d.n_ops = opcode.size(); d.opcode = opcode.data(); d.out_id = out_id.data(); d.arg_off = arg_off.data();
  d.arg_id = arg_id.data(); d.param = param.data();
  rtlsim::CompiledGraph g;
  std::string err;
  if (rtlsim::compile_graph(&d, RS_MODE_SINGLE, &g, &err) != RS_OK) { printf("compile: %s\n", err.c_str()); return 1; }
  std::vector<uint8_t> blob;
  std::vector<uint64_t> off;
  bool ok = rtlsim::build_single_slices(g, 1, G, 1u << 30, &blob, &off);  // one partition (no level cut)
  uint32_t mx = 0, mn = ~0u;
  for (unsigned i = 0; i < G; ++i) {
    const auto* h = reinterpret_cast<const rtlsim::SliceHdr*>(blob.data() + off[i]);
    mx = std::max(mx, h->bytes); mn = std::min(mn, h->bytes);
  }
  printf("G=%u ok=%d slice bytes min %u max %u (levels %u)\n", G, ok, mn, mx, g.n_levels);
  for (unsigned i = 0; i < G; i += (G > 8 ? G / 8 : 1)) {
    const auto* h = reinterpret_cast<const rtlsim::SliceHdr*>(blob.data() + off[i]);
    printf("  cta %u: bytes %u (head %u) lvl@%u seg@%u pw@%u coord@%u push@%u latch@%u inj@%u\n", i, h->bytes,
           h->head_bytes, h->off_lvl, h->off_seg, h->off_pw, h->off_coord, h->off_push, h->off_latch, h->off_inj);
  }
  return 0;
}
