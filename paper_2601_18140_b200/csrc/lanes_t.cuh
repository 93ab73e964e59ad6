// lanes_t.cuh -- the tile-interleaved lane kernel (k_lanes_t, rs_lane_opts.kernel = 1).
//
// A lane tile is LT = 32 * P lanes; thread t of a warp owns lanes t + 32k
// (k < P) of its tile, so one warp works on ONE op at a time for all LT lanes
// and every row access of the warp is a coalesced 32 * 2^c byte segment per k.
// Because the op is warp-uniform, the width classes of its operands are too:
// the operand gather (eq:split_einsum1) dispatches once per op on
// its class signature through a jump table (gather_brx.cuh) into an arm that
// loads each operand's exact container with P loads at immediate offsets --
// no extraction, no per-operand branches.  The op decode (coordinates,
// parameters, hash weight, addresses) is paid once per thread for P lanes.
//
// Per cycle the CTA walks the same stage schedule as lanes.cuh
// (compiler.hpp build_stages): INJECT | OPS level by level | LATCH, each
// stage's descriptors brought into shared memory by a TMA bulk copy one
// stage ahead, a CTA (or cluster) barrier after every stage = the iterative
// rank I of Cascade 1.  OPS work items (run-aligned batches of one
// (opcode, arity, out class), Format c P:1123-1129) are dealt round-robin to
// the warps of the CTA (or of the cluster sharing the tile).
#pragma once
#include "gather_brx.cuh"
#include "kernels.cuh"

namespace rtlsim {

// Per-thread class bases: tile + (lin << c) - (c << 30), so that base[c] +
// coordinate (class bits included) addresses the thread's lane-0 container.
struct LaneT {
  const uint8_t* p0;
  const uint8_t* p1;
  const uint8_t* p2;
  const uint8_t* p3;
};

__device__ __forceinline__ LaneT make_lanet(uint8_t* tb, uint32_t lin) {
  LaneT L;
  L.p0 = tb + lin;
  L.p1 = tb + 2 * lin - (1ull << 30);
  L.p2 = tb + 4 * lin - (2ull << 30);
  L.p3 = tb + 8 * lin - (3ull << 30);
  return L;
}

template <int A, int P>
__device__ __forceinline__ void gather_t(const LaneT& L, const uint32_t (&c)[A], uint64_t (&x)[A][P]) {
  uint32_t sig = c[0] >> 30;
  if constexpr (A > 1) sig |= (c[1] >> 28) & 0xCu;
  if constexpr (A > 2) sig |= (c[2] >> 26) & 0x30u;
  if constexpr (P == 1) {
    if constexpr (A == 1) gather_sig1_p1(sig, L.p0, L.p1, L.p2, L.p3, c[0], x);
    else if constexpr (A == 2) gather_sig2_p1(sig, L.p0, L.p1, L.p2, L.p3, c[0], c[1], x);
    else gather_sig3_p1(sig, L.p0, L.p1, L.p2, L.p3, c[0], c[1], c[2], x);
  } else if constexpr (P == 2) {
    if constexpr (A == 1) gather_sig1_p2(sig, L.p0, L.p1, L.p2, L.p3, c[0], x);
    else if constexpr (A == 2) gather_sig2_p2(sig, L.p0, L.p1, L.p2, L.p3, c[0], c[1], x);
    else gather_sig3_p2(sig, L.p0, L.p1, L.p2, L.p3, c[0], c[1], c[2], x);
  } else {
    if constexpr (A == 1) gather_sig1_p4(sig, L.p0, L.p1, L.p2, L.p3, c[0], x);
    else if constexpr (A == 2) gather_sig2_p4(sig, L.p0, L.p1, L.p2, L.p3, c[0], c[1], x);
    else gather_sig3_p4(sig, L.p0, L.p1, L.p2, L.p3, c[0], c[1], c[2], x);
  }
}

// One coordinate of runtime class (latch, rare wide folds).
template <int P>
__device__ __forceinline__ void gather1_t(const LaneT& L, uint32_t c, uint64_t (&x)[P]) {
  const uint32_t cc[1] = {c};
  uint64_t t[1][P];
  gather_t<1, P>(L, cc, t);
#pragma unroll
  for (int k = 0; k < P; ++k) x[k] = t[0][k];
}

// Write (LI_{i+1,s} = LO / LO_sel) of the thread's P lanes of a
// row of class cls at coordinate-relative offset (the coordinate itself).
template <int P>
__device__ __forceinline__ void store_t(const LaneT& L, uint32_t c, const uint64_t (&v)[P]) {
  const uint32_t cls = c >> 30;
  if (cls == 0u) {
    uint8_t* q = const_cast<uint8_t*>(L.p0) + c;
#pragma unroll
    for (int k = 0; k < P; ++k) q[32 * k] = (uint8_t)v[k];
  } else if (cls == 1u) {
    uint16_t* q = reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(L.p1) + c);
#pragma unroll
    for (int k = 0; k < P; ++k) q[32 * k] = (uint16_t)v[k];
  } else if (cls == 2u) {
    uint32_t* q = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(L.p2) + c);
#pragma unroll
    for (int k = 0; k < P; ++k) q[32 * k] = (uint32_t)v[k];
  } else {
    uint64_t* q = reinterpret_cast<uint64_t*>(const_cast<uint8_t*>(L.p3) + c);
#pragma unroll
    for (int k = 0; k < P; ++k) q[32 * k] = v[k];
  }
}

// Mask to the out width, hash, store U results of a batch (out class uniform
// over the run; ob = coordinate of the batch's first output row, rows LT << c
// bytes apart).
template <int P, bool HASH, int U>
__device__ __forceinline__ void batch_store_t(const LaneT& L, uint32_t out_cls, uint32_t ob, uint32_t cnt,
                                              uint32_t s_k, const uint32_t (&pw)[U], const uint64_t (&y)[U][P],
                                              uint64_t (&hacc)[P]) {
  constexpr uint32_t LT = 32u * P;
  if (out_cls < 3u) {
    uint32_t v[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t m32 = 0xFFFFFFFFu >> (32u - (pw[u] & 127u));  // w_out <= 32
#pragma unroll
      for (int k = 0; k < P; ++k) v[u][k] = (uint32_t)y[u][k] & m32;
    }
    if constexpr (HASH) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt) {
          const uint64_t K = lds64(s_k + 8 * u);
#pragma unroll
          for (int k = 0; k < P; ++k) hacc[k] += (uint64_t)v[u][k] * K;
        }
    }
    if (out_cls == 0u) {
      uint8_t* q = const_cast<uint8_t*>(L.p0) + ob;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt)
#pragma unroll
          for (int k = 0; k < P; ++k) q[u * LT + 32 * k] = (uint8_t)v[u][k];
    } else if (out_cls == 1u) {
      uint16_t* q = reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(L.p1) + ob);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt)
#pragma unroll
          for (int k = 0; k < P; ++k) q[u * LT + 32 * k] = (uint16_t)v[u][k];
    } else {
      uint32_t* q = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(L.p2) + ob);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((uint32_t)u < cnt)
#pragma unroll
          for (int k = 0; k < P; ++k) q[u * LT + 32 * k] = v[u][k];
    }
  } else {
    uint64_t* q = reinterpret_cast<uint64_t*>(const_cast<uint8_t*>(L.p3) + ob);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((uint32_t)u < cnt) {
        const uint64_t m = wmask(pw[u] & 127u);
        uint64_t K = 0;
        if constexpr (HASH) K = lds64(s_k + 8 * u);
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const uint64_t z = y[u][k] & m;
          if constexpr (HASH) hacc[k] += z * K;
          q[u * LT + 32 * k] = z;
        }
      }
  }
}

// Ops per gather batch: all U ops' operands are in flight before any op is
// computed (the PSU partial S unrolling, used for memory-level
// parallelism); U * A * P values live in registers.
template <int A, int P>
struct BatchU {
#ifndef RS_BATCHU_P4
#define RS_BATCHU_P4 2
#endif
#ifndef RS_BATCHU_P4_A3
#define RS_BATCHU_P4_A3 1  // keeps k_lanes_t<4, 1> at 80 registers without spills (768-thread CTAs)
#endif
  static constexpr int raw = (P == 4) ? (A == 3 ? RS_BATCHU_P4_A3 : RS_BATCHU_P4) : (P == 2 && A == 3) ? 2 : 4;
  static constexpr int value = raw < (int)kBatch ? raw : (int)kBatch;  // a work item has <= kBatch ops
};

// cnt <= U ops of one run: op = opcode, outputs from coordinate ob (rows LT << out_cls apart).
template <int P, bool HASH, int A, int U>
__device__ __forceinline__ void batch_ops_t(const LaneT& L, uint32_t op, uint32_t s_c, uint32_t s_w, uint32_t s_k,
                                            uint32_t out_cls, uint32_t ob, uint32_t cnt, uint64_t (&hacc)[P]) {
  uint64_t x[U][A][P];
  uint32_t pw[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t uu = (uint32_t)u < cnt ? (uint32_t)u : 0u;  // tail slots re-read op 0
    uint32_t c[A];
#pragma unroll
    for (int o = 0; o < A; ++o) c[o] = lds32(s_c + 4 * (uu * A + o));
#ifdef RS_EXPERIMENT_FAKE_GATHER  // diagnostic build only (tools/): every operand read from row 0 of its class
#pragma unroll
    for (int o = 0; o < A; ++o) c[o] &= 0xC0000000u;
#endif
    gather_t<A, P>(L, c, x[u]);
    pw[u] = lds32(s_w + 4 * uu);
  }
  uint64_t y[U][P];
  batch_compute<U, A, P>(op, x, pw, y);
  batch_store_t<P, HASH, U>(L, out_cls, ob, cnt, s_k, pw, y, hacc);
}

// Folds with more than 3 operands (left fold over the O rank; rare).
template <int P, bool HASH>
__device__ __forceinline__ void seg_generic_t(const LaneT& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t meta,
                                              uint32_t ob, uint32_t n, uint64_t (&hacc)[P]) {
  constexpr uint32_t LT = 32u * P;
  const uint32_t op = meta & 0xffu, ar = (meta >> 8) & 0xffu, out_cls = (meta >> 16) & 3u;
#pragma unroll 1
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t c0 = s_c + 4 * j * ar;
    uint64_t r[P], x[P];
    gather1_t<P>(L, lds32(c0), r);
#pragma unroll 1
    for (uint32_t o = 1; o < ar; ++o) {
      gather1_t<P>(L, lds32(c0 + 4 * o), x);
#pragma unroll
      for (int k = 0; k < P; ++k) r[k] = fold_step(op, r[k], x[k]);
    }
    const uint64_t m = wmask(lds32(s_w + 4 * j) & 127u);
#pragma unroll
    for (int k = 0; k < P; ++k) r[k] &= m;
    if constexpr (HASH) {
      const uint64_t K = lds64(s_k + 8 * j);
#pragma unroll
      for (int k = 0; k < P; ++k) hacc[k] += r[k] * K;
    }
    store_t<P>(L, ob + j * (LT << out_cls), r);
  }
}

template <int P, bool HASH>
__device__ __forceinline__ void stage_ops_t(const LaneT& L, const uint8_t* buf, uint32_t w0, uint32_t nw,
                                            uint64_t (&hacc)[P]) {
  constexpr uint32_t LT = 32u * P;
  const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
  const StageRun* runs = reinterpret_cast<const StageRun*>(buf + h->off_runs);
  const uint32_t* items = reinterpret_cast<const uint32_t*>(buf + h->off_items);
  const uint32_t base = smem_addr(buf), n_items = h->n_items;
  const uint32_t s_c0 = base + h->off_c, s_w0 = base + h->off_w, s_k0 = base + h->off_k;
#pragma unroll 1
  for (uint32_t it = w0; it < n_items; it += nw) {
    const uint32_t w = items[it];
    const StageRun R = runs[w >> 16];
    const uint32_t b = w & 0x1FFFu, cnt = ((w >> 13) & 7u) + 1u;
    const uint32_t ar = (R.meta >> 8) & 0xffu, k = b - R.op_begin, cls = (R.meta >> 16) & 3u, op = R.meta & 0xffu;
    const uint32_t s_c = s_c0 + 4 * (R.coord_begin + k * ar);
    // out rows are bound as (class << 30) | byte offset: the coordinate form store_t expects
    const uint32_t ob = ((cls << 30) | R.out_row0) + k * (LT << cls);
    const uint32_t s_w = s_w0 + 4 * b, s_k = s_k0 + 8 * b;
    if (ar == 2) {
      constexpr int U = BatchU<2, P>::value;
#pragma unroll 1
      for (uint32_t j = 0; j < cnt; j += U)
        batch_ops_t<P, HASH, 2, U>(L, op, s_c + 8 * j, s_w + 4 * j, s_k + 8 * j, cls, ob + j * (LT << cls),
                                   min(cnt - j, (uint32_t)U), hacc);
    } else if (ar == 1) {
      constexpr int U = BatchU<1, P>::value;
#pragma unroll 1
      for (uint32_t j = 0; j < cnt; j += U)
        batch_ops_t<P, HASH, 1, U>(L, op, s_c + 4 * j, s_w + 4 * j, s_k + 8 * j, cls, ob + j * (LT << cls),
                                   min(cnt - j, (uint32_t)U), hacc);
    } else if (ar == 3) {
      constexpr int U = BatchU<3, P>::value;
#pragma unroll 1
      for (uint32_t j = 0; j < cnt; j += U)
        batch_ops_t<P, HASH, 3, U>(L, op, s_c + 12 * j, s_w + 4 * j, s_k + 8 * j, cls, ob + j * (LT << cls),
                                   min(cnt - j, (uint32_t)U), hacc);
    } else {
      seg_generic_t<P, HASH>(L, s_c, s_w, s_k, R.meta, ob, cnt, hacc);
    }
  }
}

// LATCH stage: tmp = LI[next] & M(w_r); LI[r] = tmp.  One pass is hazard-free
// because every next row is an op row (compiler identity copies; reading R8).
// UU > 0: registers per batch (their next-value loads in flight together); 0: the default.
template <int P, bool HASH, int UU = 0>
__device__ __forceinline__ void stage_latch_t(const LaneT& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t b,
                                              uint32_t e, uint64_t (&hr)[P]) {
  constexpr int U = UU > 0 ? UU : (P == 4) ? 2 : 4;
#pragma unroll 1
  for (uint32_t j = b; j < e; j += U) {
    uint64_t v[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) gather1_t<P>(L, lds32(s_c + 8 * min(j + u, e - 1)), v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u < e) {
        const uint64_t m = wmask(lds32(s_w + 4 * (j + u)));
#pragma unroll
        for (int k = 0; k < P; ++k) v[u][k] &= m;
        store_t<P>(L, lds32(s_c + 8 * (j + u) + 4), v[u]);
        if constexpr (HASH) {
          const uint64_t K = lds64(s_k + 8 * (j + u));
#pragma unroll
          for (int k = 0; k < P; ++k) hr[k] += v[u][k] * K;
        }
      }
    }
  }
}

// INJECT stage: LI[in_k] = stimulus & M(w_k) (or the staged value); lane =
// allocation-relative index of the thread's lane 0 (its lanes are lane + 32k).
template <int P, bool HASH>
__device__ __forceinline__ void stage_inject_t(const LaneT& L, uint32_t s_c, uint32_t s_w, uint32_t s_k,
                                               uint32_t first, uint32_t b, uint32_t e, const StepArgs& a,
                                               uint32_t lane, uint64_t cycle, uint64_t (&hacc)[P]) {
#pragma unroll 1
  for (uint32_t j = b; j < e; ++j) {
    const uint32_t kk = first + j;
    const uint64_t m = wmask(lds32(s_w + 4 * j));
    uint64_t v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const uint32_t l = lane + 32 * k;
      if (a.staged)
        v[k] = l < a.n_lanes ? __ldg(a.stage + ((cycle % a.stage_cap) * a.g.n_inputs + kk) * a.n_lanes + l) : 0ull;
      else
        v[k] = d_stimulus(a.seed, kk, cycle, a.lane0 + l);
      v[k] &= m;
    }
    store_t<P>(L, lds32(s_c + 4 * j), v);
    if constexpr (HASH) {
      const uint64_t K = lds64(s_k + 8 * j);
#pragma unroll
      for (int k = 0; k < P; ++k) hacc[k] += v[k] * K;
    }
  }
}

// Shared-memory bytes beyond the two stage buffers: red[2][T*P] + hr[T*P] +
// hp[T*P] (u64) + lsum[3][LT] (u64, cluster partials).
__host__ __device__ constexpr size_t lanes_t_smem_extra(uint32_t threads, uint32_t P) {
  return 4ull * threads * P * 8 + 3ull * 32 * P * 8;
}

template <int P, bool HASH>
__global__ void __launch_bounds__(RS_LANES_T_MAX_THREADS, 1) k_lanes_t(const StepArgs a) {
  constexpr uint32_t LT = 32u * P;
  extern __shared__ __align__(128) uint8_t smem[];
  // [mbarriers | stage buffer 0 | stage buffer 1 | red[2][T*P] | hr[T*P] | hp[T*P] | lsum[3][LT]]
  // red: per-(thread, lane) hash partials of a cycle (double buffered); hr /
  // hp: register terms of the next / current cycle; lsum: this CTA's per-lane
  // partial of a cycle (two parities) and of the carry, summed across the
  // cluster through distributed shared memory.  Partial slot of (thread t,
  // k) = t * P + k, for lane (t & 31) + 32k of the tile.
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  uint64_t* red = reinterpret_cast<uint64_t*>(smem + 128 + 2 * (size_t)a.stage_bytes);
  uint64_t* hr_s = red + 2 * T * P;
  uint64_t* hp_s = red + 3 * T * P;
  uint64_t* lsum = red + 4 * T * P;

  const uint32_t CS = a.cluster;
  const uint32_t rank = blockIdx.x % CS, tile = blockIdx.x / CS;
  const uint32_t lin = tid & 31u, warp = tid >> 5, nwarp = T >> 5;
  const uint32_t gw = rank * nwarp + warp, ngw = CS * nwarp;  // warp index across the cluster
  const uint32_t lane = tile * LT + lin;                       // the thread's lane 0 (allocation-relative)
  const LaneT L = make_lanet(a.state + (size_t)tile * a.tile_bytes, lin);

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  if constexpr (HASH) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const uint32_t l = lane + 32 * k;
      hr_s[tid * P + k] = 0;
      hp_s[tid * P + k] = (gw == 0 && l < a.n_lanes) ? a.hcarry_in[l] : 0ull;
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
  for (int k = 0; k < P; ++k) hacc[k] = 0;
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
    mbar_wait(&mbar[bsel], (gi >> 1) & 1u);
#ifdef RS_TRACE
    if (tr && tid == 0) tr[1] = clock64();
#endif
    const uint8_t* buf = smem + 128 + bsel * a.stage_bytes;
    const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
    const uint32_t type = h->type;
    if (type == ST_OPS) {
      stage_ops_t<P, HASH>(L, buf, gw, ngw, hacc);
    } else if (type == ST_LATCH) {
      uint32_t b, e;
      chunk_of(h->n, gw, ngw, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        uint64_t hr[P];
#pragma unroll
        for (int k = 0; k < P; ++k) hr[k] = 0;
        stage_latch_t<P, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, b, e, hr);
        if constexpr (HASH) {
#pragma unroll
          for (int k = 0; k < P; ++k) hr_s[tid * P + k] += hr[k];
        }
      }
    } else if (type == ST_INJECT) {
      uint32_t b, e;
      chunk_of(h->n, gw, ngw, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        stage_inject_t<P, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, h->first, b, e, a, lane,
                                a.cycle0 + cyc, hacc);
      }
    } else if (type == ST_WATCH) {
      uint32_t b, e;
      chunk_of(h->n, gw, ngw, b, e);
      uint32_t ln[P];
#pragma unroll
      for (int k = 0; k < P; ++k) ln[k] = lin + 32 * k;
      if (b < e)
        stage_watch<P>(a, a.state + (size_t)tile * a.tile_bytes, reinterpret_cast<const uint32_t*>(buf + h->off_c), b,
                       e, ln, tile, a.cycle0 + cyc);
    }
    const bool eoc = (s + 1 == S);
    if constexpr (HASH) {
      if (eoc) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
          red[(cyc & 1u) * T * P + tid * P + k] = hacc[k] + hp_s[tid * P + k];
          hp_s[tid * P + k] = hr_s[tid * P + k];
          hr_s[tid * P + k] = 0;
          hacc[k] = 0;
        }
      }
    }
#ifdef RS_TRACE
    if (tr && lin == 0) tr[3 + warp] = clock64();
#endif
    stage_barrier(CS);
#ifdef RS_TRACE
    if (tr && tid == 0) tr[2] = clock64();
#endif
    if constexpr (HASH) {
      if (warp == 0 && a.hashes != nullptr) {
        // the cluster's partials of cycle `pend` were all written before this barrier
        if (pend >= 0 && rank == 0) {
          const uint32_t pb = (uint32_t)pend & 1u;
#pragma unroll
          for (int k = 0; k < P; ++k) {
            const uint32_t li = lin + 32 * k;
            uint64_t sum = a.g.const_hash + lsum[pb * LT + li];
            for (uint32_t r = 1; r < CS; ++r) sum += dsmem(lsum, r)[pb * LT + li];
            if (lane + 32 * k < a.n_lanes) a.hashes[(size_t)pend * a.n_lanes + lane + 32 * k] = sum;
          }
        }
        if (eoc) {
          const uint64_t* rr = red + (cyc & 1u) * T * P + lin * P;
#pragma unroll
          for (int k = 0; k < P; ++k) {
            uint64_t sum = 0;
#pragma unroll 4
            for (uint32_t i = 0; i < nwarp; ++i) sum += rr[i * 32 * P + k];
            if (CS == 1) {
              if (lane + 32 * k < a.n_lanes) a.hashes[(size_t)cyc * a.n_lanes + lane + 32 * k] = sum + a.g.const_hash;
            } else {
              lsum[(cyc & 1u) * LT + lin + 32 * k] = sum;
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
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < P; ++k) {
        uint64_t sum = 0;
        for (uint32_t i = 0; i < nwarp; ++i) sum += hp_s[(i * 32 + lin) * P + k];
        lsum[2 * LT + lin + 32 * k] = sum;
      }
    }
    stage_barrier(CS);
    if (warp == 0 && rank == 0) {
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const uint32_t li = lin + 32 * k, l = lane + 32 * k;
        uint64_t sum = lsum[2 * LT + li];
        for (uint32_t r = 1; r < CS; ++r) sum += dsmem(lsum, r)[2 * LT + li];
        if (l < a.n_lanes) a.hcarry_out[l] = sum;
        if (pend >= 0 && a.hashes != nullptr) {  // last cycle's cluster-wide hash
          const uint32_t pb = (uint32_t)pend & 1u;
          uint64_t hs = a.g.const_hash + lsum[pb * LT + li];
          for (uint32_t r = 1; r < CS; ++r) hs += dsmem(lsum, r)[pb * LT + li];
          if (l < a.n_lanes) a.hashes[(size_t)pend * a.n_lanes + l] = hs;
        }
      }
    }
    if (CS > 1) stage_barrier(CS);  // keep every CTA's shared memory alive until rank 0 has read it
  }
}

}  // namespace rtlsim
