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
#ifndef RS_LANES_MAX_THREADS
#define RS_LANES_MAX_THREADS 640    // kernel 2 (k_lanes): 96 registers
#endif
#ifndef RS_LANES_T_MAX_THREADS
#define RS_LANES_T_MAX_THREADS 768  // kernel 1 (k_lanes_t): 80 registers, 3-operand batches of 1 op at P = 4
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
  uint32_t cluster;            // lane mode: CTAs (one cluster) sharing one lane tile
  unsigned long long* trace;   // RS_TRACE builds: per-stage clock64 stamps of CTA 0 (tools/, not the product)
  // waveform capture (rs_watch): previous values [n_watch][lanes_pad], change records, record counter
  uint64_t* wave_prev;
  uint64_t* wave_rec;          // [capacity][4] u64: cycle, lane, watch, value
  unsigned long long* wave_count;
  uint64_t wave_cap;
  uint64_t wave_first;         // records are unconditional at this absolute cycle
  // single-lane waveform capture: watch entries (k_single2: signal coords;
  // k_repcut_smem: per-partition {local offset, watch index} pairs from
  // watch_begin[p]), 0 entries = off
  const uint32_t* watch_ent;
  const uint32_t* watch_begin;
  uint32_t n_watch;
  // bit-sliced lane kernel (lanes_b.cuh) allocations: class-0 rows [0, rows_bit)
  // (the 1-bit signals) are bit planes at region_b + row * 16 inside a tile (word k
  // = lanes 32k..32k+31); region[0] is then biased by -rows_bit * LT so that
  // region[0] + row * LT addresses the u8 rows [rows_bit, rows[0])
  uint32_t bitplane;
  uint32_t rows_bit;
  uint64_t region_b;
  uint32_t pairs;    // kernel 7: evaluate <= 2-operand ops in pairs (many ops per CTA and level)
};

// One watched value of the single lane (watch index j) at `cycle`: a change
// record when it differs from the previous cycle's (always at wave_first).
__device__ __forceinline__ void watch_single(const StepArgs& a, uint32_t j, uint64_t v, uint64_t cycle) {
  uint64_t* prev = a.wave_prev + j;
  const bool rec = cycle == a.wave_first || *prev != v;
  *prev = v;
  if (!rec) return;
  const unsigned long long i = atomicAdd(a.wave_count, 1ull);
  if (i < a.wave_cap) {
    uint64_t* r = a.wave_rec + 4 * i;
    r[0] = cycle;
    r[1] = a.lane0;
    r[2] = j;
    r[3] = v;
  }
}

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
  // plain (L1-cached) load: state written by this CTA, or published to it
  // through an acquire (RepCut replicas)
  __device__ __forceinline__ uint64_t ld(uint32_t c) const {
    const size_t r = (size_t)(c & ROW_MASK) * LT;
    switch (c >> 30) {
      case 0: return p0[r];
      case 1: return p1[r];
      case 2: return p2[r];
      default: return p3[r];
    }
  }
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

// WATCH stage (waveform capture, rs_watch): for watches [b, e) of the stage and
// the thread's lanes (tile-relative ids lanes[0..n)), compare each value with
// the previous cycle's and append a change record; the records of a warp are
// reserved with one atomic.  coords: the watched signals' bound coordinates.
template <int N>
__device__ __forceinline__ void stage_watch(const StepArgs& a, const uint8_t* tb, const uint32_t* coords, uint32_t b,
                                            uint32_t e, const uint32_t (&lanes)[N], uint32_t tile, uint64_t cycle) {
  const size_t lanes_pad = (size_t)gridDim.x / a.cluster * a.LT;
#pragma unroll 1
  for (uint32_t j = b; j < e; ++j) {
    const uint32_t c = coords[j], cls = c >> 30;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const uint32_t l = tile * a.LT + lanes[k];  // allocation lane
      const uint8_t* p = tb + (c & ROW_MASK) + ((size_t)lanes[k] << cls);
      uint64_t v;
      switch (cls) {
        case 0: v = *p; break;
        case 1: v = *reinterpret_cast<const uint16_t*>(p); break;
        case 2: v = *reinterpret_cast<const uint32_t*>(p); break;
        default: v = *reinterpret_cast<const uint64_t*>(p); break;
      }
      uint64_t* prev = a.wave_prev + (size_t)j * lanes_pad + l;
      const bool rec = l < a.n_lanes && (cycle == a.wave_first || *prev != v);
      *prev = v;
      // one atomic per warp and step: the leader reserves the warp's records
      const uint32_t am = __activemask();
      const uint32_t m = __ballot_sync(am, rec);
      if (m == 0u) continue;
      const uint32_t me = threadIdx.x & 31u, leader = __ffs(m) - 1;
      unsigned long long base = 0;
      if (me == leader) base = atomicAdd(a.wave_count, (unsigned long long)__popc(m));
      base = __shfl_sync(am, base, leader);
      if (rec) {
        const unsigned long long i = base + __popc(m & ((1u << me) - 1u));
        if (i < a.wave_cap) {
          uint64_t* r = a.wave_rec + 4 * i;
          r[0] = cycle;
          r[1] = a.lane0 + l;
          r[2] = j;
          r[3] = v;
        }
      }
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

// op_u / op_r / op_s for an op of arity <= 3 (n = pw >> 26), branch-free: the
// ops of a warp may have different opcodes (single-lane mode deals a level's
// ops to threads), and a switch compiles to an indirect branch that splits the
// warp into serialized paths; every candidate result is computed and the op's
// one is picked by a selection tree on the opcode bits (depth 4).  Unmasked;
// folds with n > 3 are the caller's.
__device__ __forceinline__ uint64_t select_op(uint32_t pw, uint64_t x0, uint64_t x1, uint64_t x2) {
  const uint32_t op = (pw >> 22) & 15u, n = pw >> 26, p0 = (pw >> 7) & 127u;
  const bool three = n == 3;
  const uint64_t z = three ? x2 : 0ull;
  const uint32_t sh = p0 >= 64 ? 63u : p0;
  const uint64_t shl = p0 >= 64 ? 0ull : (x0 << sh), shr = p0 >= 64 ? 0ull : (x0 >> sh);
  const uint32_t lo = (pw >> 14) & 63u;
  {  // selection tree on the opcode bits (depth 4 instead of a 14-deep chain)
    const uint64_t a0 = x0 & x1 & (three ? x2 : ~0ull), a1 = x0 | x1 | z, a2 = x0 ^ x1 ^ z, a3 = ~x0;
    const uint64_t a4 = x0 + x1 + z, a5 = x0 - x1 - z, a6 = x0 * x1 * (three ? x2 : 1ull);
    const uint64_t a7 = (uint64_t)(x0 == x1), a8 = (uint64_t)(x0 < x1), a9 = shl, a10 = shr;
    const uint64_t a11 = (x0 >> lo) & wmask(p0 - lo + 1u), a12 = p0 >= 64 ? x1 : (shl | x1);
    const uint64_t a13 = x0 != 0 ? x1 : x2, a14 = x0;
    const bool b0 = op & 1u, b1 = op & 2u, b2 = op & 4u, b3 = op & 8u;
    const uint64_t s01 = b0 ? a1 : a0, s23 = b0 ? a3 : a2, s45 = b0 ? a5 : a4, s67 = b0 ? a7 : a6;
    const uint64_t s89 = b0 ? a9 : a8, sab = b0 ? a11 : a10, scd = b0 ? a13 : a12, sef = a14;
    const uint64_t t0 = b1 ? s23 : s01, t1 = b1 ? s67 : s45, t2 = b1 ? sab : s89, t3 = b1 ? sef : scd;
    const uint64_t u0 = b2 ? t1 : t0, u1 = b2 ? t3 : t2;
    return b3 ? u1 : u0;
  }
}

template <bool CG = true>
__device__ __forceinline__ uint64_t single_op(const StepArgs& a, const TileP<1>& t, uint32_t j) {
  auto L = [&](uint32_t c) -> uint64_t { return CG ? t.ld_cg(c) : t.ld(c); };
  const uint32_t pw = __ldg(a.g.opw + j);
  const uint32_t op = (pw >> 22) & 15u, n = pw >> 26;
  const uint32_t* cp = a.g.coord + __ldg(a.g.coord_off + j);
  uint64_t x[3];
  switch (op) {
    case RS_OP_AND: case RS_OP_OR: case RS_OP_XOR: case RS_OP_ADD: case RS_OP_SUB: case RS_OP_MUL: {
      uint64_t r = L(__ldg(cp));
      for (uint32_t o = 1; o < n; ++o) r = fold_step(op, r, L(__ldg(cp + o)));
      return r & wmask(pw & 127u);
    }
    case RS_OP_EQ: x[0] = L(__ldg(cp)); x[1] = L(__ldg(cp + 1)); return apply_op<RS_OP_EQ, 2>(x, pw);
    case RS_OP_LT: x[0] = L(__ldg(cp)); x[1] = L(__ldg(cp + 1)); return apply_op<RS_OP_LT, 2>(x, pw);
    case RS_OP_CAT: x[0] = L(__ldg(cp)); x[1] = L(__ldg(cp + 1)); return apply_op<RS_OP_CAT, 2>(x, pw);
    case RS_OP_NOT: x[0] = L(__ldg(cp)); return apply_op<RS_OP_NOT, 1>(x, pw);
    case RS_OP_SHL: x[0] = L(__ldg(cp)); return apply_op<RS_OP_SHL, 1>(x, pw);
    case RS_OP_SHR: x[0] = L(__ldg(cp)); return apply_op<RS_OP_SHR, 1>(x, pw);
    case RS_OP_BITS: x[0] = L(__ldg(cp)); return apply_op<RS_OP_BITS, 1>(x, pw);
    case RS_OP_MUX:
      x[0] = L(__ldg(cp)); x[1] = L(__ldg(cp + 1)); x[2] = L(__ldg(cp + 2));
      return apply_op<RS_OP_MUX, 3>(x, pw);
    default: x[0] = L(__ldg(cp)); return apply_op<OP_COPY, 1>(x, pw);
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

// Bit-plane word and bit of (coordinate, lane) in a bit-sliced allocation, or
// nullptr when the row is a container row.
__device__ __forceinline__ uint32_t* bit_word(const StepArgs& a, uint32_t c, uint32_t lane, uint32_t& bit) {
  if (!a.bitplane || (c >> 30) != 0u || (c & ROW_MASK) >= a.rows_bit) return nullptr;
  const uint32_t tile = lane / a.LT, lin = lane % a.LT;
  bit = lin & 31u;
  return reinterpret_cast<uint32_t*>(a.state + (size_t)tile * a.tile_bytes + a.region_b + (size_t)(c & ROW_MASK) * 16 +
                                     (lin >> 5) * 4);
}
__device__ __forceinline__ uint64_t ld_sig(const StepArgs& a, uint32_t c, uint32_t lane) {
  uint32_t bit;
  if (const uint32_t* w = bit_word(a, c, lane, bit)) return (*w >> bit) & 1u;
  return ld_any(row_addr(a, c, lane), c >> 30);
}
// one lane of a bit plane is one bit of a word other lanes share: atomic
__device__ __forceinline__ void st_sig(const StepArgs& a, uint32_t c, uint32_t lane, uint64_t v) {
  uint32_t bit;
  if (uint32_t* w = bit_word(a, c, lane, bit)) {
    if (v & 1u) atomicOr(w, 1u << bit);
    else atomicAnd(w, ~(1u << bit));
    return;
  }
  st_any(row_addr(a, c, lane), c >> 30, v);
}

// Fill every lane (padded lanes included) of the given rows with a value
// (constants, register init).
__global__ void k_broadcast(StepArgs a, uint32_t n_lanes_pad, const uint32_t* coords, const uint64_t* vals, uint32_t n) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < (uint64_t)n * n_lanes_pad;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(idx / n_lanes_pad), l = (uint32_t)(idx % n_lanes_pad);
    st_sig(a, coords[i], l, vals[i]);
  }
}

// out[i][l] = value of coords[i] at lane lane_begin + l (rs_read_signals, step 5)
__global__ void k_read(StepArgs a, const uint32_t* coords, uint32_t n_ids, uint32_t lane_begin, uint32_t n,
                       uint64_t* out) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < (uint64_t)n_ids * n;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(idx / n), l = (uint32_t)(idx % n);
    out[idx] = ld_sig(a, coords[i], lane_begin + l);
  }
}

__global__ void k_write(StepArgs a, const uint32_t* coords, const uint32_t* widths, uint32_t n_ids, uint32_t lane_begin,
                        uint32_t n, const uint64_t* vals) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < (uint64_t)n_ids * n;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(idx / n), l = (uint32_t)(idx % n);
    st_sig(a, coords[i], lane_begin + l, vals[idx] & wmask(widths[i]));
  }
}

// hcarry[l] = sum_r v_r * K_r (register term of the next cycle's hash)
__global__ void k_reg_hash(StepArgs a, uint32_t n_lanes, uint64_t* hcarry) {
  for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n_lanes; l += gridDim.x * blockDim.x) {
    uint64_t h = 0;
    for (uint32_t j = 0; j < a.g.n_regs; ++j) h += ld_sig(a, a.g.reg_coord[j], l) * a.g.reg_k[j];
    hcarry[l] = h;
  }
}

}  // namespace rtlsim
