// kernels.cuh -- sm_100a step kernels for the RTeAAL Sim cascade.
//
// State layout (SURVEY.md §8(a) "signal-major x lane-minor"): the lanes of an
// allocation are cut into tiles of LT lanes; a tile owns one contiguous block
// [class 0 region | class 1 | class 2 | class 3] where class c holds rows of
// LT containers of 2^c bytes (lane-minor).  The gather of one operand for the
// tile's lanes is one coalesced LT * 2^c byte access (PAPER.md P:1441-1443
// names this gather as the CPU kernels' main D-cache-miss source).
//
// Lane mode (k_lanes): CTA = one lane tile.  Every cycle walks a fixed stage
// schedule (compiler.hpp build_stages); each stage's descriptors are brought
// into shared memory by a TMA bulk copy issued one stage ahead.  Sub-warps
// (LT threads) split a stage's ops into contiguous chunks and walk them run by
// run -- one (opcode, arity) specialisation per run, the NU "switch hoisted out
// of the op loop" (alg:NU P:1175-1202) -- gathering U ops' operands with
// branch-free loads before computing any (the PSU partial S unrolling,
// P:1204-1209, used for memory-level parallelism).  __syncthreads is the level
// barrier (iterative rank I).
//
// Single-lane mode (k_single): one op per thread over a cooperative grid; a
// grid barrier separates levels.
#pragma once
#include <cstdint>

#include "compiler.hpp"

// Build-time tuning knobs (ops gathered per batch for arity <= 2 / 3, and the
// CTA size the lane kernel's register budget is compiled for).
#ifndef RS_U2
#define RS_U2 4
#endif
#ifndef RS_U3
#define RS_U3 2
#endif
#ifndef RS_LANES_MAX_THREADS
#define RS_LANES_MAX_THREADS 1024
#endif

namespace rtlsim {

struct GraphDev {
  const DevRun* runs;
  const uint32_t* level_run_begin;
  const uint32_t* level_op_begin;
  const uint32_t* opw;
  const uint64_t* opk;
  const uint32_t* coord_off;
  const uint32_t* coord;
  const uint32_t* out_coord;
  const uint32_t* in_coord;
  const uint32_t* in_w;
  const uint64_t* in_k;
  const uint32_t* reg_coord;
  const uint32_t* reg_next_coord;
  const uint32_t* reg_w;
  const uint64_t* reg_k;
  uint32_t n_levels, n_inputs, n_regs, n_ops_total;
  uint64_t const_hash;
};

struct StepArgs {
  GraphDev g;
  uint8_t* state;          // [n_tiles][tile_bytes]
  uint64_t tile_bytes;
  uint64_t region[4];      // byte offset of class c's region inside a tile
  uint32_t rows[4];
  uint32_t LT;
  uint32_t n_lanes;        // lanes in this allocation
  uint64_t lane0;          // global id of lane 0
  uint64_t cycle0;         // absolute cycle of the first stepped cycle
  uint32_t n_cycles;
  int staged;              // 0: stimulus from seed; 1: staged ring
  uint64_t seed;
  const uint64_t* stage;   // [stage_cap][n_inputs][n_lanes]
  uint32_t stage_cap;
  uint64_t* hashes;        // [n_cycles][n_lanes] or nullptr
  uint64_t* hcarry_in;     // per-lane register term of the hash for cycle0
  uint64_t* hcarry_out;    // same for cycle0 + n_cycles (may alias hcarry_in in lane mode)
  unsigned long long* bar; // grid barrier counter (single mode)
  const uint8_t* stage_blob;   // lane mode: this allocation's bound stage schedule
  const StageRef* stage_tab;
  uint32_t n_stages;
  uint32_t stage_bytes;        // shared-memory bytes per stage buffer
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint64_t wmask(uint32_t w) { return ~0ull >> (64u - w); }  // w in 1..64

__device__ __forceinline__ uint64_t d_splitmix_next(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// DESIGN.md reading R13 (independent of oracle/; same public algorithm).
__device__ __forceinline__ uint64_t d_stimulus(uint64_t seed, uint64_t k, uint64_t c, uint64_t lane) {
  uint64_t x = d_splitmix_next(seed);
  x = d_splitmix_next(x + k);
  x = d_splitmix_next(x + c);
  return d_splitmix_next(x + lane);
}

// Row-coordinate access ((class << 30) | row): single-lane and aux kernels.
template <int LT>
struct TileP {
  uint8_t* p0;
  uint16_t* p1;
  uint32_t* p2;
  uint64_t* p3;
  // L2-coherent load (single-lane mode: other SMs write the state)
  __device__ __forceinline__ uint64_t ld_cg(uint32_t c) const {
    const size_t r = (size_t)(c & ROW_MASK) * LT;
    switch (c >> 30) {
      case 0: return __ldcg(p0 + r);
      case 1: return __ldcg(p1 + r);
      case 2: return __ldcg(p2 + r);
      default: return __ldcg(p3 + r);
    }
  }
  __device__ __forceinline__ void st(uint32_t cls, uint32_t row, uint64_t v) const {
    const size_t r = (size_t)row * LT;
    switch (cls) {
      case 0: p0[r] = (uint8_t)v; break;
      case 1: p1[r] = (uint16_t)v; break;
      case 2: p2[r] = (uint32_t)v; break;
      default: p3[r] = v; break;
    }
  }
  __device__ __forceinline__ void stc(uint32_t c, uint64_t v) const { st(c >> 30, c & ROW_MASK, v); }
};

template <int LT>
__device__ __forceinline__ TileP<LT> tile_ptrs(const StepArgs& a, uint32_t tile, uint32_t lin) {
  uint8_t* tb = a.state + (size_t)tile * a.tile_bytes;
  TileP<LT> t;
  t.p0 = tb + a.region[0] + lin;
  t.p1 = reinterpret_cast<uint16_t*>(tb + a.region[1]) + lin;
  t.p2 = reinterpret_cast<uint32_t*>(tb + a.region[2]) + lin;
  t.p3 = reinterpret_cast<uint64_t*>(tb + a.region[3]) + lin;
  return t;
}

// op_u / op_r / op_s of Cascade 1 for one op with A operands.
// pw: [6:0] w_out [13:7] p0 [19:14] p1 (compiler.hpp pack_pw).
template <int OP, int A>
__device__ __forceinline__ uint64_t apply_op(const uint64_t* x, uint32_t pw) {
  uint64_t r;
  const uint32_t p0 = (pw >> 7) & 127u;
  if constexpr (OP == RS_OP_AND) { r = x[0]; _Pragma("unroll") for (int o = 1; o < A; ++o) r &= x[o]; }
  else if constexpr (OP == RS_OP_OR) { r = x[0]; _Pragma("unroll") for (int o = 1; o < A; ++o) r |= x[o]; }
  else if constexpr (OP == RS_OP_XOR) { r = x[0]; _Pragma("unroll") for (int o = 1; o < A; ++o) r ^= x[o]; }
  else if constexpr (OP == RS_OP_ADD) { r = x[0]; _Pragma("unroll") for (int o = 1; o < A; ++o) r += x[o]; }
  else if constexpr (OP == RS_OP_SUB) { r = x[0]; _Pragma("unroll") for (int o = 1; o < A; ++o) r -= x[o]; }
  else if constexpr (OP == RS_OP_MUL) { r = x[0]; _Pragma("unroll") for (int o = 1; o < A; ++o) r *= x[o]; }
  else if constexpr (OP == RS_OP_EQ) { r = (x[0] == x[1]) ? 1ull : 0ull; }
  else if constexpr (OP == RS_OP_LT) { r = (x[0] < x[1]) ? 1ull : 0ull; }
  else if constexpr (OP == RS_OP_NOT) { r = ~x[0]; }
  else if constexpr (OP == RS_OP_SHL) { r = p0 >= 64 ? 0ull : (x[0] << p0); }
  else if constexpr (OP == RS_OP_SHR) { r = p0 >= 64 ? 0ull : (x[0] >> p0); }
  else if constexpr (OP == RS_OP_BITS) {
    const uint32_t lo = (pw >> 14) & 63u;
    r = (x[0] >> lo) & wmask(p0 - lo + 1u);
  }
  else if constexpr (OP == RS_OP_CAT) { r = p0 >= 64 ? x[1] : ((x[0] << p0) | x[1]); }
  else if constexpr (OP == RS_OP_MUX) { r = x[0] != 0 ? x[1] : x[2]; }
  else { r = x[0]; }  // OP_COPY
  return r & wmask(pw & 127u);
}

// Runtime-arity fold (arity > 3; rare).
__device__ __forceinline__ uint64_t fold_step(uint32_t op, uint64_t r, uint64_t x) {
  switch (op) {
    case RS_OP_AND: return r & x;
    case RS_OP_OR: return r | x;
    case RS_OP_XOR: return r ^ x;
    case RS_OP_ADD: return r + x;
    case RS_OP_SUB: return r - x;
    default: return r * x;
  }
}

// ------------------------------------------------------------------ lane mode
// Shared-memory helpers (explicit .shared accesses from non-inlined code).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

// mbarrier + TMA 1-D bulk copy (cp.async.bulk) -- the stage prefetch.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Per-thread lane constants for bound coordinates ((class << 30) | byte offset
// of the row's lane 0 inside the tile; rows are 8-byte aligned).
struct Lane {
  uint8_t* tb;     // tile base
  uint32_t off8;   // byte c = (lin << c) & ~7: the lane's container's 8-byte word inside a class-c row
  uint32_t sh8;    // byte c = ((lin << c) & 7) * 8: bit offset of the container inside that word
  uint32_t lin;
};

__device__ __forceinline__ Lane make_lane(uint8_t* tb, uint32_t lin) {
  Lane L;
  L.tb = tb;
  L.lin = lin;
  L.off8 = (lin & ~7u) | (((lin << 1) & ~7u) << 8) | (((lin << 2) & ~7u) << 16) | (((lin << 3) & ~7u) << 24);
  L.sh8 = ((lin & 7u) << 3) | ((((lin << 1) & 7u) << 3) << 8) | ((((lin << 2) & 7u) << 3) << 16);
  return L;
}

// Gather, part 1: one aligned 64-bit load per operand -- the word that holds
// this lane's container, whatever the class -- so a batch issues exactly one
// load per operand, with no branches and no register reused between loads.
__device__ __forceinline__ uint64_t gather_raw(const Lane& L, uint32_t c) {
  const uint32_t cls = c >> 30;
  const uint8_t* p = L.tb + ((c & ROW_MASK) + __byte_perm(L.off8, 0u, cls | 0x4440u));
  return *reinterpret_cast<const uint64_t*>(p);
}

// Gather, part 2 (after every load of the batch is in flight): shift the
// lane's container down and mask it to its class width.
__device__ __forceinline__ uint64_t gather_fix(const Lane& L, uint32_t c, uint64_t w) {
  const uint32_t cls = c >> 30;
  const uint32_t sh = __byte_perm(L.sh8, 0u, cls | 0x4440u);
  const uint64_t v = w >> sh;
  const uint32_t m32 = 0xFFFFFFFFu >> (32u - (8u << min(cls, 2u)));
  return cls == 3u ? w : (uint64_t)((uint32_t)v & m32);
}

__device__ __forceinline__ uint64_t gather(const Lane& L, uint32_t c) { return gather_fix(L, c, gather_raw(L, c)); }

// Store to a bound coordinate (class varies per value: latch / inject).
__device__ __forceinline__ void scatter(const Lane& L, uint32_t c, uint64_t v) {
  const uint32_t cls = c >> 30;
  uint8_t* p = L.tb + (c & ROW_MASK) + (L.lin << cls);
  switch (cls) {
    case 0: *p = (uint8_t)v; break;
    case 1: *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; break;
    case 2: *reinterpret_cast<uint32_t*>(p) = (uint32_t)v; break;
    default: *reinterpret_cast<uint64_t*>(p) = v; break;
  }
}

// op_u / op_r / op_s of Cascade 1 for a batch of U ops of one run (same
// opcode and arity): one uniform switch per batch, the batch's U ops
// unrolled inside each case; only the opcodes of arity A are instantiated.
// Per-op parameters come from the param words (compiler.hpp pack_pw).
template <int U, int A>
__device__ __forceinline__ void batch_compute(uint32_t op, const uint64_t (&x)[U][A], const uint32_t (&pw)[U],
                                              uint64_t (&y)[U]) {
#define RS_EACH(EXPR) _Pragma("unroll") for (int u = 0; u < U; ++u) { y[u] = (EXPR); } break;
  if constexpr (A == 1) {
    switch (op) {
      case RS_OP_NOT: RS_EACH(~x[u][0])
      case RS_OP_SHL: RS_EACH(((pw[u] >> 7) & 127u) >= 64 ? 0ull : (x[u][0] << ((pw[u] >> 7) & 127u)))
      case RS_OP_SHR: RS_EACH(((pw[u] >> 7) & 127u) >= 64 ? 0ull : (x[u][0] >> ((pw[u] >> 7) & 127u)))
      case RS_OP_BITS: RS_EACH((x[u][0] >> ((pw[u] >> 14) & 63u)) &
                               wmask(((pw[u] >> 7) & 127u) - ((pw[u] >> 14) & 63u) + 1u))
      default: RS_EACH(x[u][0])  // OP_COPY
    }
  } else if constexpr (A == 2) {
    switch (op) {
      case RS_OP_AND: RS_EACH(x[u][0] & x[u][1])
      case RS_OP_OR: RS_EACH(x[u][0] | x[u][1])
      case RS_OP_XOR: RS_EACH(x[u][0] ^ x[u][1])
      case RS_OP_ADD: RS_EACH(x[u][0] + x[u][1])
      case RS_OP_SUB: RS_EACH(x[u][0] - x[u][1])
      case RS_OP_MUL: RS_EACH(x[u][0] * x[u][1])
      case RS_OP_EQ: RS_EACH(x[u][0] == x[u][1] ? 1ull : 0ull)
      case RS_OP_LT: RS_EACH(x[u][0] < x[u][1] ? 1ull : 0ull)
      default: RS_EACH(((pw[u] >> 7) & 127u) >= 64 ? x[u][1] : ((x[u][0] << ((pw[u] >> 7) & 127u)) | x[u][1]))  // CAT
    }
  } else {
    switch (op) {
      case RS_OP_AND: RS_EACH(x[u][0] & x[u][1] & x[u][2])
      case RS_OP_OR: RS_EACH(x[u][0] | x[u][1] | x[u][2])
      case RS_OP_XOR: RS_EACH(x[u][0] ^ x[u][1] ^ x[u][2])
      case RS_OP_ADD: RS_EACH(x[u][0] + x[u][1] + x[u][2])
      case RS_OP_SUB: RS_EACH(x[u][0] - x[u][1] - x[u][2])
      case RS_OP_MUL: RS_EACH(x[u][0] * x[u][1] * x[u][2])
      default: RS_EACH(x[u][0] != 0 ? x[u][1] : x[u][2])  // MUX
    }
  }
#undef RS_EACH
#pragma unroll
  for (int u = 0; u < U; ++u) y[u] &= wmask(pw[u] & 127u);
}

// One work item: cnt <= U ops of one run (opcode op, arity A in 1..3, out
// class out_cls), descriptors in shared memory (s_c: first coord, s_w: first
// param word, s_k: first hash weight), outputs at consecutive rows from
// out_byte0.  All operands of the batch are gathered (branch-free; tail slots
// re-read op 0) before any op is computed: memory-level parallelism.
template <int LT, bool HASH, int A>
__device__ __forceinline__ uint64_t batch_ops(const Lane& L, uint32_t op, uint32_t s_c, uint32_t s_w, uint32_t s_k,
                                              uint32_t out_cls, uint32_t out_byte0, uint32_t cnt) {
  constexpr int U = (int)kBatch;
  uint64_t x[U][A];
  uint32_t cc[U][A];
  uint32_t pw[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t uu = (uint32_t)u < cnt ? (uint32_t)u : 0u;
#pragma unroll
    for (int o = 0; o < A; ++o) {
      cc[u][o] = lds32(s_c + 4 * (uu * A + o));
      x[u][o] = gather_raw(L, cc[u][o]);
    }
    pw[u] = lds32(s_w + 4 * uu);
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int o = 0; o < A; ++o) x[u][o] = gather_fix(L, cc[u][o], x[u][o]);
  uint64_t y[U];
  batch_compute<U, A>(op, x, pw, y);
  uint64_t hacc = 0;
  if constexpr (HASH) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((uint32_t)u < cnt) hacc += y[u] * lds64(s_k + 8 * u);
  }
  uint8_t* ob = L.tb + out_byte0 + (L.lin << out_cls);
  const uint32_t ostride = (uint32_t)LT << out_cls;
  switch (out_cls) {
    case 0:
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) ob[u * ostride] = (uint8_t)y[u];
      break;
    case 1:
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) *reinterpret_cast<uint16_t*>(ob + u * ostride) = (uint16_t)y[u];
      break;
    case 2:
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) *reinterpret_cast<uint32_t*>(ob + u * ostride) = (uint32_t)y[u];
      break;
    default:
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) *reinterpret_cast<uint64_t*>(ob + u * ostride) = y[u];
      break;
  }
  return hacc;
}

// Folds with more than 3 operands (left fold over the O rank; rare).
template <int LT, bool HASH>
__device__ __forceinline__ uint64_t seg_generic(const Lane& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t meta,
                                                uint32_t out_byte0, uint32_t n) {
  const uint32_t op = meta & 0xffu, ar = (meta >> 8) & 0xffu, out_cls = (meta >> 16) & 3u;
  uint64_t hacc = 0;
#pragma unroll 1
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t c = s_c + 4 * j * ar;
    uint64_t r = gather(L, lds32(c));
#pragma unroll 1
    for (uint32_t o = 1; o < ar; ++o) r = fold_step(op, r, gather(L, lds32(c + 4 * o)));
    const uint64_t y = r & wmask(lds32(s_w + 4 * j) & 127u);
    scatter(L, (out_cls << 30) | (out_byte0 + j * ((uint32_t)LT << out_cls)), y);
    if constexpr (HASH) hacc += y * lds64(s_k + 8 * j);
  }
  return hacc;
}

__device__ __forceinline__ void chunk_of(uint32_t n, uint32_t part, uint32_t nparts, uint32_t& b, uint32_t& e) {
  const uint32_t c = (n + nparts - 1) / nparts;
  b = min(n, part * c);
  e = min(n, b + c);
}

// OPS stage: the stage's work items (run-aligned batches of <= kBatch ops)
// dealt round-robin to the sub-warps, so every sub-warp gets an even mix of
// arities and classes (static balance; no atomics).
template <int LT, bool HASH>
__device__ __forceinline__ uint64_t stage_ops(const Lane& L, const uint8_t* buf, uint32_t sub, uint32_t nsub) {
  const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
  const StageRun* runs = reinterpret_cast<const StageRun*>(buf + h->off_runs);
  const uint32_t* items = reinterpret_cast<const uint32_t*>(buf + h->off_items);
  const uint32_t base = smem_addr(buf), n_items = h->n_items;
  const uint32_t s_c0 = base + h->off_c, s_w0 = base + h->off_w, s_k0 = base + h->off_k;
  uint64_t hacc = 0;
#pragma unroll 1
  for (uint32_t it = sub; it < n_items; it += nsub) {
    const uint32_t w = items[it];
    const StageRun R = runs[w >> 16];
    const uint32_t b = w & 0x1FFFu, cnt = ((w >> 13) & 7u) + 1u;
    const uint32_t ar = (R.meta >> 8) & 0xffu, k = b - R.op_begin, cls = (R.meta >> 16) & 3u, op = R.meta & 0xffu;
    const uint32_t s_c = s_c0 + 4 * (R.coord_begin + k * ar);
    const uint32_t ob = R.out_row0 + k * ((uint32_t)LT << cls);
    uint64_t hh;
    if (ar == 2) hh = batch_ops<LT, HASH, 2>(L, op, s_c, s_w0 + 4 * b, s_k0 + 8 * b, cls, ob, cnt);
    else if (ar == 1) hh = batch_ops<LT, HASH, 1>(L, op, s_c, s_w0 + 4 * b, s_k0 + 8 * b, cls, ob, cnt);
    else if (ar == 3) hh = batch_ops<LT, HASH, 3>(L, op, s_c, s_w0 + 4 * b, s_k0 + 8 * b, cls, ob, cnt);
    else hh = seg_generic<LT, HASH>(L, s_c, s_w0 + 4 * b, s_k0 + 8 * b, R.meta, ob, cnt);
    if constexpr (HASH) hacc += hh;
  }
  return hacc;
}

// LATCH stage: tmp = LI[next] & M(w_r); LI[r] = tmp.  One pass is hazard-free
// because every next row is an op row (compiler identity copies; reading R8).
template <int LT, bool HASH>
__device__ __forceinline__ uint64_t stage_latch(const Lane& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t b,
                                                uint32_t e) {
  constexpr int U = 8;
  uint64_t h = 0;
#pragma unroll 1
  for (uint32_t j = b; j < e; j += U) {
    uint64_t v[U];
    uint32_t cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cc[u] = lds32(s_c + 8 * min(j + u, e - 1));
      v[u] = gather_raw(L, cc[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < e) {
        const uint64_t x = gather_fix(L, cc[u], v[u]) & wmask(lds32(s_w + 4 * (j + u)));
        scatter(L, lds32(s_c + 8 * (j + u) + 4), x);
        if constexpr (HASH) h += x * lds64(s_k + 8 * (j + u));
      }
  }
  return h;
}

// INJECT stage: LI[in_k] = stimulus & M(w_k) (or the staged value).
template <int LT, bool HASH>
__device__ __forceinline__ uint64_t stage_inject(const Lane& L, uint32_t s_c, uint32_t s_w, uint32_t s_k,
                                                 uint32_t first, uint32_t b, uint32_t e,
                                                 const uint64_t* __restrict__ stage, uint32_t n_inputs,
                                                 uint32_t n_lanes, uint64_t seed, uint64_t glane,
                                                 uint64_t cycle_or_slot, int staged, uint32_t lane, bool valid) {
  uint64_t h = 0;
#pragma unroll 1
  for (uint32_t j = b; j < e; ++j) {
    const uint32_t k = first + j;
    uint64_t v;
    if (staged)
      v = valid ? __ldg(stage + (cycle_or_slot * n_inputs + k) * n_lanes + lane) : 0ull;
    else
      v = d_stimulus(seed, k, cycle_or_slot, glane);
    v &= wmask(lds32(s_w + 4 * j));
    scatter(L, lds32(s_c + 4 * j), v);
    if constexpr (HASH) h += v * lds64(s_k + 8 * j);
  }
  return h;
}

template <int LT, bool HASH>
__global__ void __launch_bounds__(RS_LANES_MAX_THREADS, 1) k_lanes(const StepArgs a) {
  constexpr int LTL = (LT == 32) ? 5 : (LT == 16) ? 4 : (LT == 8) ? 3 : (LT == 4) ? 2 : (LT == 2) ? 1 : 0;
  extern __shared__ __align__(128) uint8_t smem[];
  // shared memory: [mbarriers | stage buffer 0 | stage buffer 1 | red[2][T] | hr[T] | hp[T]]
  // red: per-thread hash partials of a cycle (double buffered, reduced per lane);
  // hr / hp: per-thread register terms of the next / current cycle.  Kept in
  // shared memory, not registers: the hot loop needs every register it has.
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  uint64_t* red = reinterpret_cast<uint64_t*>(smem + 128 + 2 * (size_t)a.stage_bytes);
  uint64_t* hr_s = red + 2 * T;
  uint64_t* hp_s = red + 3 * T;

  const uint32_t lin = tid & (LT - 1);
  const uint32_t sub = tid >> LTL;
  const uint32_t nsub = T >> LTL;
  const Lane L = make_lane(a.state + (size_t)blockIdx.x * a.tile_bytes, lin);

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  if constexpr (HASH) {
    const uint32_t lane = blockIdx.x * LT + lin;
    hr_s[tid] = 0;
    hp_s[tid] = (sub == 0 && lane < a.n_lanes) ? a.hcarry_in[lane] : 0ull;
  }
  __syncthreads();
  const uint32_t S = a.n_stages;
  const uint32_t total = a.n_cycles * S;  // host keeps n_cycles * S < 2^31
  if (tid == 0 && total) {
    const StageRef r = a.stage_tab[0];
    tma_load_1d(smem + 128, a.stage_blob + r.off, r.bytes, &mbar[0]);
  }

  uint64_t hacc = 0;
  uint32_t s = 0, cyc = 0;
#pragma unroll 1
  for (uint32_t gi = 0; gi < total; ++gi) {
    const uint32_t bsel = gi & 1u;
    if (tid == 0 && gi + 1 < total) {
      const StageRef r = a.stage_tab[s + 1 == S ? 0 : s + 1];
      tma_load_1d(smem + 128 + (bsel ^ 1u) * a.stage_bytes, a.stage_blob + r.off, r.bytes, &mbar[bsel ^ 1u]);
    }
    mbar_wait(&mbar[bsel], (gi >> 1) & 1u);
    const uint8_t* buf = smem + 128 + bsel * a.stage_bytes;
    const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
    const uint32_t type = h->type;
    if (type == ST_OPS) {
      const uint64_t hh = stage_ops<LT, HASH>(L, buf, sub, nsub);
      if constexpr (HASH) hacc += hh;
    } else if (type == ST_LATCH) {
      uint32_t b, e;
      chunk_of(h->n, sub, nsub, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        const uint64_t hh = stage_latch<LT, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, b, e);
        if constexpr (HASH) hr_s[tid] += hh;
      }
    } else if (type == ST_INJECT) {
      uint32_t b, e;
      chunk_of(h->n, sub, nsub, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf), lane = blockIdx.x * LT + lin;
        const uint64_t c = a.cycle0 + cyc;
        const uint64_t hh = stage_inject<LT, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, h->first,
                                                   b, e, a.stage, a.g.n_inputs, a.n_lanes, a.seed, a.lane0 + lane,
                                                   a.staged ? c % a.stage_cap : c, a.staged, lane, lane < a.n_lanes);
        if constexpr (HASH) hacc += hh;
      }
    }
    const bool eoc = (s + 1 == S);
    if constexpr (HASH) {
      if (eoc) {
        red[(cyc & 1u) * T + tid] = hacc + hp_s[tid];
        hp_s[tid] = hr_s[tid];
        hr_s[tid] = 0;
        hacc = 0;
      }
    }
    __syncthreads();
    if constexpr (HASH) {
      const uint32_t lane = blockIdx.x * LT + lin;
      if (eoc && sub == 0 && a.hashes != nullptr && lane < a.n_lanes) {
        const uint64_t* rr = red + (cyc & 1u) * T + lin;
        uint64_t sum = a.g.const_hash;
#pragma unroll 4
        for (uint32_t i = 0; i < nsub; ++i) sum += rr[i * LT];
        a.hashes[(size_t)cyc * a.n_lanes + lane] = sum;
      }
    }
    if (eoc) {
      s = 0;
      ++cyc;
    } else {
      ++s;
    }
  }
  if constexpr (HASH) {
    // register term of the hash of the next cycle (hp_s holds the last commit's partials)
    __syncthreads();
    const uint32_t lane = blockIdx.x * LT + lin;
    if (sub == 0 && lane < a.n_lanes) {
      uint64_t sum = 0;
      for (uint32_t i = 0; i < nsub; ++i) sum += hp_s[i * LT + lin];
      a.hcarry_out[lane] = sum;
    }
  }
}

// ------------------------------------------------------------------ single-lane mode
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long& target) {
  __syncthreads();
  if (gridDim.x == 1) return;
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1ull);
    while (ld_acquire(bar) < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ uint64_t block_sum(uint64_t v, uint64_t* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const uint32_t w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) sm[w] = v;
  __syncthreads();
  uint64_t s = 0;
  if (threadIdx.x == 0)
    for (uint32_t i = 0; i < nw; ++i) s += sm[i];
  __syncthreads();
  return s;
}

__device__ __forceinline__ uint64_t single_op(const StepArgs& a, const TileP<1>& t, uint32_t j) {
  const uint32_t pw = __ldg(a.g.opw + j);
  const uint32_t op = (pw >> 22) & 15u, n = pw >> 26;
  const uint32_t* cp = a.g.coord + __ldg(a.g.coord_off + j);
  uint64_t x[3];
  switch (op) {
    case RS_OP_AND: case RS_OP_OR: case RS_OP_XOR: case RS_OP_ADD: case RS_OP_SUB: case RS_OP_MUL: {
      uint64_t r = t.ld_cg(__ldg(cp));
      for (uint32_t o = 1; o < n; ++o) r = fold_step(op, r, t.ld_cg(__ldg(cp + o)));
      return r & wmask(pw & 127u);
    }
    case RS_OP_EQ: x[0] = t.ld_cg(__ldg(cp)); x[1] = t.ld_cg(__ldg(cp + 1)); return apply_op<RS_OP_EQ, 2>(x, pw);
    case RS_OP_LT: x[0] = t.ld_cg(__ldg(cp)); x[1] = t.ld_cg(__ldg(cp + 1)); return apply_op<RS_OP_LT, 2>(x, pw);
    case RS_OP_CAT: x[0] = t.ld_cg(__ldg(cp)); x[1] = t.ld_cg(__ldg(cp + 1)); return apply_op<RS_OP_CAT, 2>(x, pw);
    case RS_OP_NOT: x[0] = t.ld_cg(__ldg(cp)); return apply_op<RS_OP_NOT, 1>(x, pw);
    case RS_OP_SHL: x[0] = t.ld_cg(__ldg(cp)); return apply_op<RS_OP_SHL, 1>(x, pw);
    case RS_OP_SHR: x[0] = t.ld_cg(__ldg(cp)); return apply_op<RS_OP_SHR, 1>(x, pw);
    case RS_OP_BITS: x[0] = t.ld_cg(__ldg(cp)); return apply_op<RS_OP_BITS, 1>(x, pw);
    case RS_OP_MUX:
      x[0] = t.ld_cg(__ldg(cp)); x[1] = t.ld_cg(__ldg(cp + 1)); x[2] = t.ld_cg(__ldg(cp + 2));
      return apply_op<RS_OP_MUX, 3>(x, pw);
    default: x[0] = t.ld_cg(__ldg(cp)); return apply_op<OP_COPY, 1>(x, pw);
  }
}

template <bool HASH>
__global__ void __launch_bounds__(1024, 1) k_single(const StepArgs a) {
  __shared__ uint64_t sm[32];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  const TileP<1> t = tile_ptrs<1>(a, 0, 0);
  unsigned long long target = 0;
  uint64_t hacc = 0;
  if (HASH && tid == 0) hacc = a.hcarry_in[0];
  if (a.n_cycles == 0) return;
  for (uint32_t k = tid; k < a.g.n_inputs; k += T) {
    uint64_t v = a.staged ? __ldg(a.stage + (size_t)(a.cycle0 % a.stage_cap) * a.g.n_inputs + k)
                          : d_stimulus(a.seed, k, a.cycle0, a.lane0);
    v &= wmask(__ldg(a.g.in_w + k));
    t.stc(__ldg(a.g.in_coord + k), v);
    if (HASH) hacc += v * __ldg(a.g.in_k + k);
  }
  grid_barrier(a.bar, target);
  uint64_t hr = 0;
  for (uint32_t cyc = 0; cyc < a.n_cycles; ++cyc) {
    for (uint32_t lev = 0; lev < a.g.n_levels; ++lev) {
      const uint32_t ob = __ldg(a.g.level_op_begin + lev), oe = __ldg(a.g.level_op_begin + lev + 1);
      for (uint32_t j = ob + tid; j < oe; j += T) {
        const uint64_t y = single_op(a, t, j);
        t.stc(__ldg(a.g.out_coord + j), y);
        if (HASH) hacc += y * __ldg(a.g.opk + j);
      }
      grid_barrier(a.bar, target);
    }
    hr = 0;
    for (uint32_t j = tid; j < a.g.n_regs; j += T) {
      const uint64_t x = t.ld_cg(__ldg(a.g.reg_next_coord + j)) & wmask(__ldg(a.g.reg_w + j));
      t.stc(__ldg(a.g.reg_coord + j), x);
      if (HASH) hr += x * __ldg(a.g.reg_k + j);
    }
    uint64_t hin = 0;
    if (cyc + 1 < a.n_cycles) {
      const uint64_t c = a.cycle0 + cyc + 1;
      for (uint32_t k = tid; k < a.g.n_inputs; k += T) {
        uint64_t v = a.staged ? __ldg(a.stage + (size_t)(c % a.stage_cap) * a.g.n_inputs + k)
                              : d_stimulus(a.seed, k, c, a.lane0);
        v &= wmask(__ldg(a.g.in_w + k));
        t.stc(__ldg(a.g.in_coord + k), v);
        if (HASH) hin += v * __ldg(a.g.in_k + k);
      }
    }
    if (HASH) {
      const uint64_t s = block_sum(hacc, sm) + (blockIdx.x == 0 ? a.g.const_hash : 0ull);
      if (threadIdx.x == 0 && a.hashes) atomicAdd((unsigned long long*)(a.hashes + cyc), (unsigned long long)s);
      hacc = hr + hin;
    }
    grid_barrier(a.bar, target);
  }
  if (HASH) {
    const uint64_t s = block_sum(hr, sm);
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)a.hcarry_out, (unsigned long long)s);
  }
}

// ------------------------------------------------------------------ aux kernels
// Row-coordinate addressing for a given lane of the allocation.
__device__ __forceinline__ uint8_t* row_addr(const StepArgs& a, uint32_t c, uint32_t lane) {
  const uint32_t cls = c >> 30, row = c & ROW_MASK;
  const uint32_t tile = lane / a.LT, lin = lane % a.LT;
  return a.state + (size_t)tile * a.tile_bytes + a.region[cls] + (((size_t)row * a.LT + lin) << cls);
}

__device__ __forceinline__ uint64_t ld_any(const uint8_t* p, uint32_t cls) {
  switch (cls) {
    case 0: return *p;
    case 1: return *reinterpret_cast<const uint16_t*>(p);
    case 2: return *reinterpret_cast<const uint32_t*>(p);
    default: return *reinterpret_cast<const uint64_t*>(p);
  }
}

__device__ __forceinline__ void st_any(uint8_t* p, uint32_t cls, uint64_t v) {
  switch (cls) {
    case 0: *p = (uint8_t)v; break;
    case 1: *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; break;
    case 2: *reinterpret_cast<uint32_t*>(p) = (uint32_t)v; break;
    default: *reinterpret_cast<uint64_t*>(p) = v; break;
  }
}

// Fill every lane (padded lanes included) of the given rows with a value
// (constants, register init).
__global__ void k_broadcast(StepArgs a, uint32_t n_lanes_pad, const uint32_t* coords, const uint64_t* vals, uint32_t n) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < (uint64_t)n * n_lanes_pad;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(idx / n_lanes_pad), l = (uint32_t)(idx % n_lanes_pad);
    const uint32_t c = coords[i];
    st_any(row_addr(a, c, l), c >> 30, vals[i]);
  }
}

// out[i][l] = value of coords[i] at lane lane_begin + l (rs_read_signals, step 5)
__global__ void k_read(StepArgs a, const uint32_t* coords, uint32_t n_ids, uint32_t lane_begin, uint32_t n,
                       uint64_t* out) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < (uint64_t)n_ids * n;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(idx / n), l = (uint32_t)(idx % n);
    const uint32_t c = coords[i];
    out[idx] = ld_any(row_addr(a, c, lane_begin + l), c >> 30);
  }
}

__global__ void k_write(StepArgs a, const uint32_t* coords, const uint32_t* widths, uint32_t n_ids, uint32_t lane_begin,
                        uint32_t n, const uint64_t* vals) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < (uint64_t)n_ids * n;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(idx / n), l = (uint32_t)(idx % n);
    const uint32_t c = coords[i];
    st_any(row_addr(a, c, lane_begin + l), c >> 30, vals[idx] & wmask(widths[i]));
  }
}

// hcarry[l] = sum_r v_r * K_r (register term of the next cycle's hash)
__global__ void k_reg_hash(StepArgs a, uint32_t n_lanes, uint64_t* hcarry) {
  for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n_lanes; l += gridDim.x * blockDim.x) {
    uint64_t h = 0;
    for (uint32_t j = 0; j < a.g.n_regs; ++j) {
      const uint32_t c = a.g.reg_coord[j];
      h += ld_any(row_addr(a, c, l), c >> 30) * a.g.reg_k[j];
    }
    hcarry[l] = h;
  }
}

}  // namespace rtlsim
