// lanes.cuh -- the lane-mode step kernel (k_lanes): many independent
// stimulus lanes, one CTA per lane tile of LT lanes, every thread owning P
// adjacent lanes of its tile.
//
// Per cycle the CTA walks a fixed stage schedule (compiler.hpp build_stages):
//   INJECT chunks | OPS chunks level by level | LATCH chunks,
// each stage's descriptors brought into shared memory by one TMA bulk copy
// issued a stage ahead; __syncthreads after every stage is the level barrier
// (the iterative rank I of Cascade 1).
//
// Inside an OPS stage the work items -- run-aligned batches of kBatch ops of
// one (opcode, arity, out class) run, PAPER.md Format c -- are
// dealt round-robin to sub-warps of LT/P threads.  A sub-warp gathers every
// operand of its batch (eq:split_einsum1) with one aligned 64-bit
// load per operand (plus one per extra lane for 64-bit operands) before
// computing any op (op_u / op_r / op_s, eq:step4c / eq:step5b): the PSU
// partial S unrolling of P:1204-1209, used here for memory-level parallelism.
// The per-op decode (descriptors, addresses, run bookkeeping) is paid once
// per thread for P lanes.
#pragma once
#include "kernels.cuh"

#ifndef RS_P
#define RS_P 2
#endif

namespace rtlsim {

__device__ __forceinline__ void chunk_of(uint32_t n, uint32_t part, uint32_t nparts, uint32_t& b, uint32_t& e) {
  const uint32_t c = (n + nparts - 1) / nparts;
  b = min(n, part * c);
  e = min(n, b + c);
}

// Per-thread constants.  Bound coordinates are (class << 30) | byte offset of
// the row's lane 0 inside the tile (rows are 8-byte aligned).
template <int P>
struct LaneP {
  uint8_t* tb;       // tile base
  uint32_t lin;      // thread index inside its sub-warp; owns tile lanes lin*P .. lin*P+P-1
  uint32_t off8;     // byte c: ((lin*P) << c) & ~7 -- the 8-byte word holding the thread's first lane
  uint32_t sh8[P];   // byte c (c <= 2): bit offset of lane p's container inside that word
};

template <int P>
__device__ __forceinline__ LaneP<P> make_lanep(uint8_t* tb, uint32_t lin) {
  LaneP<P> L;
  L.tb = tb;
  L.lin = lin;
  const uint32_t l0 = lin * P;
  L.off8 = 0;
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) L.off8 |= (((l0 << c) & ~7u) & 0xFFu) << (8 * c);
#pragma unroll
  for (int p = 0; p < P; ++p) {
    L.sh8[p] = 0;
#pragma unroll
    for (uint32_t c = 0; c < 3; ++c) L.sh8[p] |= ((((l0 + p) << c) & 7u) * 8u) << (8 * c);
  }
  return L;
}

__device__ __forceinline__ uint32_t cls_sel(uint32_t c) { return (c >> 30) | 0x4440u; }

// Gather, part 1: the aligned 64-bit word holding the thread's first lane of
// operand coordinate c (all P lanes for classes <= 32 bit), plus, for 64-bit
// operands only, the next P-1 words -- each in its own register, so no load
// waits for another.
template <int P>
__device__ __forceinline__ void gather_raw(const LaneP<P>& L, uint32_t c, uint64_t (&w)[P]) {
  const uint8_t* q = L.tb + ((c & ROW_MASK) + __byte_perm(L.off8, 0u, cls_sel(c)));
  w[0] = *reinterpret_cast<const uint64_t*>(q);
#pragma unroll
  for (int p = 1; p < P; ++p) {
    w[p] = 0;
    if ((c >> 30) == 3u) w[p] = *reinterpret_cast<const uint64_t*>(q + 8 * p);
  }
}

// Gather, part 2 (after the batch's loads are all in flight): lane p's value.
template <int P>
__device__ __forceinline__ void gather_fix(const LaneP<P>& L, uint32_t c, const uint64_t (&w)[P], uint64_t (&x)[P]) {
  const uint32_t cls = c >> 30, s = cls_sel(c);
  const uint32_t m32 = 0xFFFFFFFFu >> __byte_perm(0x00001018u, 0u, s);  // 0xFF / 0xFFFF / ~0
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint32_t v = (uint32_t)(w[0] >> __byte_perm(L.sh8[p], 0u, s)) & m32;
    x[p] = cls == 3u ? w[p] : (uint64_t)v;
  }
}

// Store the thread's P lanes of one value row (class cls, row byte offset rb).
template <int P>
__device__ __forceinline__ void store_lanes(const LaneP<P>& L, uint32_t cls, uint32_t rb, const uint64_t (&y)[P]) {
  uint8_t* q = L.tb + rb + ((L.lin * P) << cls);
  if constexpr (P == 2) {
    switch (cls) {
      case 0: *reinterpret_cast<uint16_t*>(q) = (uint16_t)(((uint32_t)y[1] << 8) | ((uint32_t)y[0] & 0xFFu)); break;
      case 1: *reinterpret_cast<uint32_t*>(q) = ((uint32_t)y[1] << 16) | ((uint32_t)y[0] & 0xFFFFu); break;
      case 2: *reinterpret_cast<uint64_t*>(q) = (y[1] << 32) | (y[0] & 0xFFFFFFFFull); break;
      default: *reinterpret_cast<ulonglong2*>(q) = make_ulonglong2(y[0], y[1]); break;
    }
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      uint8_t* r = q + (p << cls);
      switch (cls) {
        case 0: *r = (uint8_t)y[p]; break;
        case 1: *reinterpret_cast<uint16_t*>(r) = (uint16_t)y[p]; break;
        case 2: *reinterpret_cast<uint32_t*>(r) = (uint32_t)y[p]; break;
        default: *reinterpret_cast<uint64_t*>(r) = y[p]; break;
      }
    }
  }
}

// op_u / op_r / op_s of Cascade 1 for the U ops x P lanes of a batch of one
// run: one uniform switch per batch, the batch unrolled inside each case; only
// the opcodes of arity A are instantiated.  Parameters come from the param
// words (compiler.hpp pack_pw).
template <int U, int A, int P>
__device__ __forceinline__ void batch_compute(uint32_t op, const uint64_t (&x)[U][A][P], const uint32_t (&pw)[U],
                                              uint64_t (&y)[U][P]) {
#define RS_EACH(EXPR)                                   \
  _Pragma("unroll") for (int u = 0; u < U; ++u) {       \
    _Pragma("unroll") for (int p = 0; p < P; ++p) {     \
      y[u][p] = (EXPR);                                 \
    }                                                   \
  }                                                     \
  break;
#define X0 x[u][0][p]
#define X1 x[u][A > 1 ? 1 : 0][p]
#define X2 x[u][A > 2 ? 2 : 0][p]
#define P0 ((pw[u] >> 7) & 127u)
#define P1 ((pw[u] >> 14) & 63u)
  if constexpr (A == 1) {
    switch (op) {
      case RS_OP_NOT: RS_EACH(~X0)
      case RS_OP_SHL: RS_EACH(P0 >= 64 ? 0ull : (X0 << P0))
      case RS_OP_SHR: RS_EACH(P0 >= 64 ? 0ull : (X0 >> P0))
      case RS_OP_BITS: RS_EACH((X0 >> P1) & wmask(P0 - P1 + 1u))
      default: RS_EACH(X0)  // OP_COPY
    }
  } else if constexpr (A == 2) {
    switch (op) {
      case RS_OP_AND: RS_EACH(X0 & X1)
      case RS_OP_OR: RS_EACH(X0 | X1)
      case RS_OP_XOR: RS_EACH(X0 ^ X1)
      case RS_OP_ADD: RS_EACH(X0 + X1)
      case RS_OP_SUB: RS_EACH(X0 - X1)
      case RS_OP_MUL: RS_EACH(X0 * X1)
      case RS_OP_EQ: RS_EACH(X0 == X1 ? 1ull : 0ull)
      case RS_OP_LT: RS_EACH(X0 < X1 ? 1ull : 0ull)
      default: RS_EACH(P0 >= 64 ? X1 : ((X0 << P0) | X1))  // CAT
    }
  } else {
    switch (op) {
      case RS_OP_AND: RS_EACH(X0 & X1 & X2)
      case RS_OP_OR: RS_EACH(X0 | X1 | X2)
      case RS_OP_XOR: RS_EACH(X0 ^ X1 ^ X2)
      case RS_OP_ADD: RS_EACH(X0 + X1 + X2)
      case RS_OP_SUB: RS_EACH(X0 - X1 - X2)
      case RS_OP_MUL: RS_EACH(X0 * X1 * X2)
      default: RS_EACH(X0 != 0 ? X1 : X2)  // MUX
    }
  }
#undef RS_EACH
#undef X0
#undef X1
#undef X2
#undef P0
#undef P1
}

// Mask to the out width, hash, store: once per batch per out class (uniform
// over the run).  Out classes <= 32 bit take a 32-bit path: 32-bit mask, a
// 32 x 64-bit hash multiply, and the P lanes packed into one store.
template <int LT, int P, bool HASH, int U>
__device__ __forceinline__ void batch_store(const LaneP<P>& L, uint32_t out_cls, uint32_t out_byte0, uint32_t cnt,
                                            uint32_t s_k, const uint32_t (&pw)[U], const uint64_t (&y)[U][P],
                                            uint64_t (&hacc)[P]) {
  uint8_t* ob = L.tb + out_byte0 + ((L.lin * P) << out_cls);
  const uint32_t ostride = (uint32_t)LT << out_cls;
  if (out_cls < 3u) {
    uint32_t v[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t m32 = 0xFFFFFFFFu >> (32u - (pw[u] & 127u));  // w_out <= 32
#pragma unroll
      for (int p = 0; p < P; ++p) v[u][p] = (uint32_t)y[u][p] & m32;
    }
    if constexpr (HASH) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) {
          const uint64_t k = lds64(s_k + 8 * u);
#pragma unroll
          for (int p = 0; p < P; ++p) hacc[p] += (uint64_t)v[u][p] * k;
        }
    }
    if (out_cls == 0u) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) {
          if constexpr (P == 2) *reinterpret_cast<uint16_t*>(ob + u * ostride) = (uint16_t)(v[u][0] | (v[u][1] << 8));
          else _Pragma("unroll") for (int p = 0; p < P; ++p) ob[u * ostride + p] = (uint8_t)v[u][p];
        }
    } else if (out_cls == 1u) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) {
          if constexpr (P == 2) *reinterpret_cast<uint32_t*>(ob + u * ostride) = v[u][0] | (v[u][1] << 16);
          else _Pragma("unroll") for (int p = 0; p < P; ++p)
              reinterpret_cast<uint16_t*>(ob + u * ostride)[p] = (uint16_t)v[u][p];
        }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) {
          if constexpr (P == 2)
            *reinterpret_cast<uint2*>(ob + u * ostride) = make_uint2(v[u][0], v[u][1]);
          else _Pragma("unroll") for (int p = 0; p < P; ++p)
              reinterpret_cast<uint32_t*>(ob + u * ostride)[p] = v[u][p];
        }
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((uint32_t)u < cnt) {
        const uint64_t m = wmask(pw[u] & 127u);
        uint64_t z[P];
#pragma unroll
        for (int p = 0; p < P; ++p) z[p] = y[u][p] & m;
        if constexpr (HASH) {
          const uint64_t k = lds64(s_k + 8 * u);
#pragma unroll
          for (int p = 0; p < P; ++p) hacc[p] += z[p] * k;
        }
        if constexpr (P == 2)
          *reinterpret_cast<ulonglong2*>(ob + u * ostride) = make_ulonglong2(z[0], z[1]);
        else _Pragma("unroll") for (int p = 0; p < P; ++p)
            reinterpret_cast<uint64_t*>(ob + u * ostride)[p] = z[p];
      }
  }
}

// One work item: cnt <= kBatch ops of one run (opcode op, arity A in 1..3,
// out class out_cls); descriptors in shared memory (s_c: first coord, s_w:
// first param word, s_k: first hash weight); outputs at consecutive rows
// from out_byte0.  Tail slots re-read op 0 (no branches in the gather).
template <int LT, int P, bool HASH, int A>
__device__ __forceinline__ void batch_ops(const LaneP<P>& L, uint32_t op, uint32_t s_c, uint32_t s_w, uint32_t s_k,
                                          uint32_t out_cls, uint32_t out_byte0, uint32_t cnt, uint64_t (&hacc)[P]) {
  constexpr int U = (int)kBatch;
  uint64_t x[U][A][P];
  uint32_t cc[U][A];
  uint32_t pw[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t uu = (uint32_t)u < cnt ? (uint32_t)u : 0u;
#pragma unroll
    for (int o = 0; o < A; ++o) {
      cc[u][o] = lds32(s_c + 4 * (uu * A + o));
      gather_raw<P>(L, cc[u][o], x[u][o]);
    }
    pw[u] = lds32(s_w + 4 * uu);
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int o = 0; o < A; ++o) {
      uint64_t w[P];
#pragma unroll
      for (int p = 0; p < P; ++p) w[p] = x[u][o][p];
      gather_fix<P>(L, cc[u][o], w, x[u][o]);
    }
  uint64_t y[U][P];
  batch_compute<U, A, P>(op, x, pw, y);
  batch_store<LT, P, HASH, U>(L, out_cls, out_byte0, cnt, s_k, pw, y, hacc);
}

// Folds with more than 3 operands (left fold over the O rank; rare).
template <int LT, int P, bool HASH>
__device__ __forceinline__ void seg_generic(const LaneP<P>& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t meta,
                                            uint32_t out_byte0, uint32_t n, uint64_t (&hacc)[P]) {
  const uint32_t op = meta & 0xffu, ar = (meta >> 8) & 0xffu, out_cls = (meta >> 16) & 3u;
#pragma unroll 1
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t c0 = s_c + 4 * j * ar;
    uint64_t w[P], r[P], x[P];
    uint32_t c = lds32(c0);
    gather_raw<P>(L, c, w);
    gather_fix<P>(L, c, w, r);
#pragma unroll 1
    for (uint32_t o = 1; o < ar; ++o) {
      c = lds32(c0 + 4 * o);
      gather_raw<P>(L, c, w);
      gather_fix<P>(L, c, w, x);
#pragma unroll
      for (int p = 0; p < P; ++p) r[p] = fold_step(op, r[p], x[p]);
    }
    const uint64_t m = wmask(lds32(s_w + 4 * j) & 127u);
#pragma unroll
    for (int p = 0; p < P; ++p) r[p] &= m;
    if constexpr (HASH) {
      const uint64_t k = lds64(s_k + 8 * j);
#pragma unroll
      for (int p = 0; p < P; ++p) hacc[p] += r[p] * k;
    }
    store_lanes<P>(L, out_cls, out_byte0 + j * ((uint32_t)LT << out_cls), r);
  }
}

// OPS stage: the stage's work items dealt round-robin to the sub-warps (an
// even mix of arities and classes per sub-warp; no atomics).
template <int LT, int P, bool HASH>
__device__ __forceinline__ void stage_ops(const LaneP<P>& L, const uint8_t* buf, uint32_t sub, uint32_t nsub,
                                          uint64_t (&hacc)[P]) {
  const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
  const StageRun* runs = reinterpret_cast<const StageRun*>(buf + h->off_runs);
  const uint32_t* items = reinterpret_cast<const uint32_t*>(buf + h->off_items);
  const uint32_t base = smem_addr(buf), n_items = h->n_items;
  const uint32_t s_c0 = base + h->off_c, s_w0 = base + h->off_w, s_k0 = base + h->off_k;
#pragma unroll 1
  for (uint32_t it = sub; it < n_items; it += nsub) {
    const uint32_t w = items[it];
    const StageRun R = runs[w >> 16];
    const uint32_t b = w & 0x1FFFu, cnt = ((w >> 13) & 7u) + 1u;
    const uint32_t ar = (R.meta >> 8) & 0xffu, k = b - R.op_begin, cls = (R.meta >> 16) & 3u, op = R.meta & 0xffu;
    const uint32_t s_c = s_c0 + 4 * (R.coord_begin + k * ar);
    const uint32_t ob = R.out_row0 + k * ((uint32_t)LT << cls);
    if (ar == 2) batch_ops<LT, P, HASH, 2>(L, op, s_c, s_w0 + 4 * b, s_k0 + 8 * b, cls, ob, cnt, hacc);
    else if (ar == 1) batch_ops<LT, P, HASH, 1>(L, op, s_c, s_w0 + 4 * b, s_k0 + 8 * b, cls, ob, cnt, hacc);
    else if (ar == 3) batch_ops<LT, P, HASH, 3>(L, op, s_c, s_w0 + 4 * b, s_k0 + 8 * b, cls, ob, cnt, hacc);
    else seg_generic<LT, P, HASH>(L, s_c, s_w0 + 4 * b, s_k0 + 8 * b, R.meta, ob, cnt, hacc);
  }
}

// LATCH stage: tmp = LI[next] & M(w_r); LI[r] = tmp.  One pass is hazard-free
// because every next row is an op row (compiler identity copies; reading R8).
template <int LT, int P, bool HASH>
__device__ __forceinline__ void stage_latch(const LaneP<P>& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t b,
                                            uint32_t e, uint64_t (&hr)[P]) {
  constexpr int U = 4;
#pragma unroll 1
  for (uint32_t j = b; j < e; j += U) {
    uint64_t v[U][P];
    uint32_t cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cc[u] = lds32(s_c + 8 * min(j + u, e - 1));
      gather_raw<P>(L, cc[u], v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u < e) {
        uint64_t x[P];
        gather_fix<P>(L, cc[u], v[u], x);
        const uint64_t m = wmask(lds32(s_w + 4 * (j + u)));
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] &= m;
        const uint32_t rc = lds32(s_c + 8 * (j + u) + 4);
        store_lanes<P>(L, rc >> 30, rc & ROW_MASK, x);
        if constexpr (HASH) {
          const uint64_t k = lds64(s_k + 8 * (j + u));
#pragma unroll
          for (int p = 0; p < P; ++p) hr[p] += x[p] * k;
        }
      }
    }
  }
}

// INJECT stage: LI[in_k] = stimulus & M(w_k) (or the staged value).
template <int LT, int P, bool HASH>
__device__ __forceinline__ void stage_inject(const LaneP<P>& L, uint32_t s_c, uint32_t s_w, uint32_t s_k,
                                             uint32_t first, uint32_t b, uint32_t e, const StepArgs& a, uint32_t lane,
                                             uint64_t cycle, uint64_t (&hacc)[P]) {
#pragma unroll 1
  for (uint32_t j = b; j < e; ++j) {
    const uint32_t k = first + j;
    const uint64_t m = wmask(lds32(s_w + 4 * j));
    uint64_t v[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (a.staged)
        v[p] = lane + p < a.n_lanes
                   ? __ldg(a.stage + ((cycle % a.stage_cap) * a.g.n_inputs + k) * a.n_lanes + lane + p)
                   : 0ull;
      else
        v[p] = d_stimulus(a.seed, k, cycle, a.lane0 + lane + p);
      v[p] &= m;
    }
    const uint32_t c = lds32(s_c + 4 * j);
    store_lanes<P>(L, c >> 30, c & ROW_MASK, v);
    if constexpr (HASH) {
      const uint64_t kk = lds64(s_k + 8 * j);
#pragma unroll
      for (int p = 0; p < P; ++p) hacc[p] += v[p] * kk;
    }
  }
}

// Shared-memory bytes the lane kernel needs beyond its two stage buffers:
// red[2][T*P] + hr[T*P] + hp[T*P] (u64) + lsum[3][32] (u64, cluster partials).
__host__ __device__ constexpr size_t lanes_smem_extra(uint32_t threads) {
  return 4ull * threads * RS_P * 8 + 3ull * 32 * 8;
}

// Level barrier: CTA barrier, or a cluster barrier when one lane tile is
// spread over a thread-block cluster (arrive.release / wait.acquire: the
// state other CTAs of the cluster wrote in this stage is visible after it).
__device__ __forceinline__ void stage_barrier(uint32_t cs) {
  if (cs > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
}

// Generic address of the same shared-memory object in CTA `rank` of the cluster.
__device__ __forceinline__ const uint64_t* dsmem(const uint64_t* p, uint32_t rank) {
  uint32_t a = smem_addr(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  uint64_t out;
  asm volatile("{ .reg .u64 t; cvt.u64.u32 t, %1; cvta.shared::cluster.u64 %0, t; }" : "=l"(out) : "r"(r));
  return reinterpret_cast<const uint64_t*>(out);
}

template <int LT, bool HASH>
__global__ void __launch_bounds__(RS_LANES_MAX_THREADS, 1) k_lanes(const StepArgs a) {
  constexpr int P = RS_P;
  constexpr int LTS = LT / P;  // threads per sub-warp (one op at a time)
  constexpr int LTSL = (LTS == 32) ? 5 : (LTS == 16) ? 4 : (LTS == 8) ? 3 : (LTS == 4) ? 2 : (LTS == 2) ? 1 : 0;
  static_assert(LT % P == 0 && (1 << LTSL) == LTS && LT <= 32, "lane tile / lanes per thread");
  extern __shared__ __align__(128) uint8_t smem[];
  // shared memory: [mbarriers | stage buffer 0 | stage buffer 1 | red[2][T*P] | hr[T*P] | hp[T*P] | lsum[3][32]]
  // red: per-(thread, lane) hash partials of a cycle (double buffered, reduced
  // per lane); hr / hp: register terms of the next / current cycle; lsum: this
  // CTA's per-lane partial of a cycle (two parities) and of the carry, summed
  // across the cluster through distributed shared memory.
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  uint64_t* red = reinterpret_cast<uint64_t*>(smem + 128 + 2 * (size_t)a.stage_bytes);
  uint64_t* hr_s = red + 2 * T * P;
  uint64_t* hp_s = red + 3 * T * P;
  uint64_t* lsum = red + 4 * T * P;

  const uint32_t CS = a.cluster;
  const uint32_t rank = blockIdx.x % CS, tile = blockIdx.x / CS;
  const uint32_t lin = tid & (LTS - 1);
  const uint32_t sub = tid >> LTSL;
  const uint32_t nsub = T >> LTSL;
  const uint32_t gsub = rank * nsub + sub, ngsub = CS * nsub;  // sub-warp index across the cluster
  const uint32_t lane = tile * LT + lin * P;  // first lane of this thread (allocation-relative)
  const LaneP<P> L = make_lanep<P>(a.state + (size_t)tile * a.tile_bytes, lin);

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  if constexpr (HASH) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      hr_s[tid * P + p] = 0;
      hp_s[tid * P + p] = (gsub == 0 && lane + p < a.n_lanes) ? a.hcarry_in[lane + p] : 0ull;
    }
  }
  __syncthreads();
  const uint32_t S = a.n_stages;
  const uint32_t total = a.n_cycles * S;  // host keeps n_cycles * S < 2^31
  if (tid == T - 1 && total) {
    const StageRef r = a.stage_tab[0];
    tma_load_1d(smem + 128, a.stage_blob + r.off, r.bytes, &mbar[0]);
  }
  // thread 0 keeps the reference of the next stage to prefetch in registers,
  // loaded a stage ahead (a global load on the critical path of warp 0 otherwise)
  // The stage prefetch (a ~500-cycle proxy fence + TMA issue) is done by the
  // CTA's LAST thread: work items are dealt from warp 0 up, so the last warp
  // is the least loaded and the issue latency stays off the critical path.
  const uint32_t producer = T - 1;
  StageRef nref{};
  if (tid == producer && total > 1) nref = a.stage_tab[S > 1 ? 1 : 0];
  if (CS > 1) stage_barrier(CS);  // every CTA of the cluster has started (DSMEM use below)

  uint64_t hacc[P];
#pragma unroll
  for (int p = 0; p < P; ++p) hacc[p] = 0;
  uint32_t s = 0, cyc = 0;
  int pend = -1;  // cycle whose cluster-wide hash is still to be summed (CS > 1)
#pragma unroll 1
  for (uint32_t gi = 0; gi < total; ++gi) {
#ifdef RS_TRACE
    // stamps per stage (CTA 0): [0] loop top, [1] after the stage-buffer wait,
    // [2] after the barrier, [3 + w] warp w's work end
    unsigned long long* tr = (blockIdx.x == 0 && gi < 4096) ? a.trace + (size_t)gi * (3 + T / 32) : nullptr;
    if (tr && tid == 0) tr[0] = clock64();
#endif
    const uint32_t bsel = gi & 1u;
    if (tid == producer && gi + 1 < total) {
      tma_load_1d(smem + 128 + (bsel ^ 1u) * a.stage_bytes, a.stage_blob + nref.off, nref.bytes, &mbar[bsel ^ 1u]);
      const uint32_t s2 = (s + 2) % S;  // the stage after the one just requested
      nref = a.stage_tab[s2];
    }
#ifdef RS_TRACE
    if (a.trace && blockIdx.x == 0 && gi < 4096 && tid == producer) a.trace[4096ull * 35 + (size_t)gi * 16 + 0] = clock64();
#endif
    mbar_wait(&mbar[bsel], (gi >> 1) & 1u);
#ifdef RS_TRACE
    if (tr && tid == 0) tr[1] = clock64();
#endif
    const uint8_t* buf = smem + 128 + bsel * a.stage_bytes;
    const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
    const uint32_t type = h->type;
    if (type == ST_OPS) {
      stage_ops<LT, P, HASH>(L, buf, gsub, ngsub, hacc);
    } else if (type == ST_LATCH) {
      uint32_t b, e;
      chunk_of(h->n, gsub, ngsub, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        uint64_t hr[P];
#pragma unroll
        for (int p = 0; p < P; ++p) hr[p] = 0;
        stage_latch<LT, P, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, b, e, hr);
        if constexpr (HASH) {
#pragma unroll
          for (int p = 0; p < P; ++p) hr_s[tid * P + p] += hr[p];
        }
      }
    } else if (type == ST_INJECT) {
      uint32_t b, e;
      chunk_of(h->n, gsub, ngsub, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        stage_inject<LT, P, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, h->first, b, e, a, lane,
                                  a.cycle0 + cyc, hacc);
      }
    } else if (type == ST_WATCH) {
      uint32_t b, e;
      chunk_of(h->n, gsub, ngsub, b, e);
      uint32_t ln[P];
#pragma unroll
      for (int p = 0; p < P; ++p) ln[p] = lin * P + p;
      if (b < e)
        stage_watch<P>(a, a.state + (size_t)tile * a.tile_bytes, reinterpret_cast<const uint32_t*>(buf + h->off_c), b,
                       e, ln, tile, a.cycle0 + cyc);
    }
    const bool eoc = (s + 1 == S);
    if constexpr (HASH) {
      if (eoc) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          red[(cyc & 1u) * T * P + tid * P + p] = hacc[p] + hp_s[tid * P + p];
          hp_s[tid * P + p] = hr_s[tid * P + p];
          hr_s[tid * P + p] = 0;
          hacc[p] = 0;
        }
      }
    }
#ifdef RS_TRACE
    if (tr && (tid & 31) == 0) tr[3 + tid / 32] = clock64();
#endif
    stage_barrier(CS);
#ifdef RS_TRACE
    if (tr && tid == 0) tr[2] = clock64();
#endif
    if constexpr (HASH) {
      if (sub == 0 && a.hashes != nullptr) {
        // the cluster's partials of cycle `pend` were all written before this barrier
        if (pend >= 0 && rank == 0) {
          const uint32_t pb = (uint32_t)pend & 1u;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            uint64_t sum = a.g.const_hash + lsum[pb * 32 + lin * P + p];
            for (uint32_t r = 1; r < CS; ++r) sum += dsmem(lsum, r)[pb * 32 + lin * P + p];
            if (lane + p < a.n_lanes) a.hashes[(size_t)pend * a.n_lanes + lane + p] = sum;
          }
        }
        if (eoc) {
          const uint64_t* rr = red + (cyc & 1u) * T * P + lin * P;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            uint64_t sum = 0;
#pragma unroll 4
            for (uint32_t i = 0; i < nsub; ++i) sum += rr[i * LTS * P + p];
            if (CS == 1) {
              if (lane + p < a.n_lanes) a.hashes[(size_t)cyc * a.n_lanes + lane + p] = sum + a.g.const_hash;
            } else {
              lsum[(cyc & 1u) * 32 + lin * P + p] = sum;
            }
          }
        }
      }
      if (CS > 1) pend = eoc ? (int)cyc : -1;  // any older pending cycle was summed above
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
    if (sub == 0) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        uint64_t sum = 0;
        for (uint32_t i = 0; i < nsub; ++i) sum += hp_s[(i * LTS + lin) * P + p];
        lsum[64 + lin * P + p] = sum;
      }
    }
    stage_barrier(CS);
    if (sub == 0 && rank == 0) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        uint64_t sum = lsum[64 + lin * P + p];
        for (uint32_t r = 1; r < CS; ++r) sum += dsmem(lsum, r)[64 + lin * P + p];
        if (lane + p < a.n_lanes) a.hcarry_out[lane + p] = sum;
        if (pend >= 0 && a.hashes != nullptr) {  // last cycle's cluster-wide hash
          const uint32_t pb = (uint32_t)pend & 1u;
          uint64_t hs = a.g.const_hash + lsum[pb * 32 + lin * P + p];
          for (uint32_t r = 1; r < CS; ++r) hs += dsmem(lsum, r)[pb * 32 + lin * P + p];
          if (lane + p < a.n_lanes) a.hashes[(size_t)pend * a.n_lanes + lane + p] = hs;
        }
      }
    }
    if (CS > 1) stage_barrier(CS);  // keep every CTA's shared memory alive until rank 0 has read it
  }
}

}  // namespace rtlsim
