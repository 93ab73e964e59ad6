// lanes_r.cuh -- the record-based tile lane kernel (k_lanes_r, rs_lane_opts.kernel = 7).
//
// Same state layout and tile interleave as lanes_t.cuh (tile = 32 * P lanes, thread t
// owns lanes t + 32k, one warp evaluates one op for all LT lanes, four width classes),
// but the level's op tensor is staged as one 32-byte RECORD per op, prepared at bind
// time (runtime.cu bind_stages_r):
//   {c0, c1, c2, pw, out coordinate, K lo, K hi, sel}
// sel = tail index << 8 (opcode, arity, out class: one specialised compute / mask /
// hash / store tail) | arity << 16 | opcode << 24; the operands are gathered through the
// per-arity class-signature jump tables of gather_brx.cuh.  The warps of the cluster split a stage's ops
// into contiguous ranges; per op a warp issues two shared-memory vector loads, one
// jump into the gather, one into the tail -- no run / work-item decode, no per-op
// address recomputation (the Format-c runs of P:1123-1129 survive as the record order).
// Results <= 32 bits are computed, masked and hashed in 32-bit arithmetic.  The hash
// partials are summed with shared-memory atomics (as lanes_b.cuh).
#pragma once
#include "lanes_b.cuh"

// CTA sizes the register budgets are compiled for: single ops 896 threads (72 registers,
// measured C3 1.148 vs 1.227 ms per cycle at 768), op pairs 768 (80 registers; pairs at
// 896 threads: C4 34.8 vs 31.6 ms)
#ifndef RS_LANES_R_MAX_THREADS
#define RS_LANES_R_MAX_THREADS 896
#endif
#ifndef RS_LANES_R_PAIRS_MAX_THREADS
#define RS_LANES_R_PAIRS_MAX_THREADS 768
#endif
// 32-lane tiles (P = 1, single ops) fit 64 registers: 1,024 threads
#ifndef RS_LANES_R1_MAX_THREADS
#define RS_LANES_R1_MAX_THREADS 1024
#endif

// registers per latch batch in kernel 7 (0: lanes_t.cuh's default, 2 at P = 4).  Measured
// (profiles/r02/kernel7/ab3_latch_u.txt): 4 at P = 4 single ops C3 1.150 -> 1.193 ms per
// cycle (lost), with op pairs C4 634 -> 625 ms per 20 cycles (kept for the pairs kernel)
#ifndef RS_K7_LATCH_U
#define RS_K7_LATCH_U 0
#endif
#ifndef RS_K7_LATCH_U_PAIRS
#define RS_K7_LATCH_U_PAIRS 4
#endif

namespace rtlsim {

constexpr uint32_t kRecBytes = 32;
constexpr uint32_t kTailFold = 84;  // arity > 3: generic left fold

// Dense tail combo index of (opcode, arity); tail = combo * 4 + out class.
__host__ __device__ constexpr int tail_combo(int A, int op) {
  return A == 1 ? (op == RS_OP_NOT ? 0 : op == RS_OP_SHL ? 1 : op == RS_OP_SHR ? 2 : op == RS_OP_BITS ? 3 : 4)
       : A == 2 ? 5 + (op <= RS_OP_MUL ? op - (op > RS_OP_XOR ? 1 : 0) : op == RS_OP_EQ ? 6 : op == RS_OP_LT ? 7 : 8)
                : 14 + (op <= RS_OP_MUL ? op - (op > RS_OP_XOR ? 1 : 0) : 6);
}
// Gather selector of an op with A <= 3 operands of classes cls[0..A).
__host__ __device__ constexpr uint32_t gather_sel(int A, uint32_t c0, uint32_t c1, uint32_t c2) {
  return A == 1 ? c0 : A == 2 ? 4 + c0 + 4 * c1 : 20 + c0 + 4 * c1 + 16 * c2;
}


// One op's tail: compute, mask to w_out, hash, store (out class OC, lanes_t layout).
template <int P, bool HASH, int A, int OP, int OC>
__device__ __forceinline__ void tail_r(const LaneT& L, const uint64_t (&x)[A][P], uint32_t pw, uint32_t oc,
                                       uint64_t K, uint64_t (&hacc)[P]) {
  if constexpr (OC == 3) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      uint64_t xs[A];
#pragma unroll
      for (int o = 0; o < A; ++o) xs[o] = x[o][k];
      const uint64_t v = apply_op<OP, A>(xs, pw);  // masked to w_out
      if constexpr (HASH) hacc[k] += v * K;
      reinterpret_cast<uint64_t*>(const_cast<uint8_t*>(L.p3) + oc)[32 * k] = v;
    }
  } else {
    const uint32_t m = 0xFFFFFFFFu >> (32u - (pw & 127u));  // w_out <= 32
    const uint32_t klo = (uint32_t)K, khi = (uint32_t)(K >> 32);
#pragma unroll
    for (int k = 0; k < P; ++k) {
      uint64_t xs[A];
#pragma unroll
      for (int o = 0; o < A; ++o) xs[o] = x[o][k];
      const uint32_t v = low32<OP, A>(xs, pw) & m;
      if constexpr (HASH) hacc[k] += (uint64_t)v * klo + ((uint64_t)(v * khi) << 32);
      if constexpr (OC == 0) (const_cast<uint8_t*>(L.p0) + oc)[32 * k] = (uint8_t)v;
      else if constexpr (OC == 1) reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(L.p1) + oc)[32 * k] = (uint16_t)v;
      else reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(L.p2) + oc)[32 * k] = v;
    }
  }
}

// Folds with more than 3 operands: c0 = shared-memory address of the coordinate
// list, c1 = arity, opcode in sel bits [31:24].
template <int P, bool HASH>
__device__ __forceinline__ void fold_r(const LaneT& L, uint32_t s_list, uint32_t ar, uint32_t op, uint32_t pw,
                                       uint32_t oc, uint64_t K, uint64_t (&hacc)[P]) {
  uint64_t r[P], x[P];
  gather1_t<P>(L, lds32(s_list), r);
#pragma unroll 1
  for (uint32_t o = 1; o < ar; ++o) {
    gather1_t<P>(L, lds32(s_list + 4 * o), x);
#pragma unroll
    for (int k = 0; k < P; ++k) r[k] = fold_step(op, r[k], x[k]);
  }
  const uint64_t m = wmask(pw & 127u);
#pragma unroll
  for (int k = 0; k < P; ++k) {
    r[k] &= m;
    if constexpr (HASH) hacc[k] += r[k] * K;
  }
  store_t<P>(L, oc, r);
}

// The tail of a 1- or 2-operand op whose operands were gathered two-operand wide.
template <int P, bool HASH>
__device__ __forceinline__ void tail_pair(const LaneT& L, const uint64_t (&x)[2][P], uint32_t pw, uint32_t oc,
                                          uint64_t K, uint32_t t, uint64_t (&hacc)[P]) {
  const uint64_t(&x1)[1][P] = reinterpret_cast<const uint64_t(&)[1][P]>(x);
#define RS_P4(C, AA, XX, OPC)                                                   \
  case 4 * C + 0: tail_r<P, HASH, AA, OPC, 0>(L, XX, pw, oc, K, hacc); break;   \
  case 4 * C + 1: tail_r<P, HASH, AA, OPC, 1>(L, XX, pw, oc, K, hacc); break;   \
  case 4 * C + 2: tail_r<P, HASH, AA, OPC, 2>(L, XX, pw, oc, K, hacc); break;   \
  case 4 * C + 3: tail_r<P, HASH, AA, OPC, 3>(L, XX, pw, oc, K, hacc); break;
  switch (t) {
    RS_P4(0, 1, x1, RS_OP_NOT) RS_P4(1, 1, x1, RS_OP_SHL) RS_P4(2, 1, x1, RS_OP_SHR) RS_P4(3, 1, x1, RS_OP_BITS)
    RS_P4(4, 1, x1, OP_COPY)
    RS_P4(5, 2, x, RS_OP_AND) RS_P4(6, 2, x, RS_OP_OR) RS_P4(7, 2, x, RS_OP_XOR) RS_P4(8, 2, x, RS_OP_ADD)
    RS_P4(9, 2, x, RS_OP_SUB) RS_P4(10, 2, x, RS_OP_MUL) RS_P4(11, 2, x, RS_OP_EQ) RS_P4(12, 2, x, RS_OP_LT)
    RS_P4(13, 2, x, RS_OP_CAT)
    default: break;
  }
#undef RS_P4
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// gather_t with the class signature taken from the record (sel bits 0..7, set at bind
// time) instead of recomputed from the coordinates' class bits -- a few dependent
// instructions off every op's path to its loads (RS_K7_NO_PRESIG: recompute, for A/B).
template <int A, int P>
__device__ __forceinline__ void gather_rs(const LaneT& L, uint32_t sig, const uint32_t (&c)[A], uint64_t (&x)[A][P]) {
#ifdef RS_K7_NO_PRESIG
  gather_t<A, P>(L, c, x);
#else
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
#endif
}

// One op from its record at shared address `rec` (base = the stage buffer, for fold lists).
template <int P, bool HASH>
__device__ __forceinline__ void op_r(const LaneT& L, uint32_t base, uint32_t rec, uint64_t (&hacc)[P]) {
  const uint4 r0 = lds128(rec), r1 = lds128(rec + 16);
  const uint32_t pw = r0.w, oc = r1.x, sel = r1.w, t = (sel >> 8) & 0xffu;
  const uint64_t K = HASH ? ((uint64_t)r1.z << 32 | r1.y) : 0ull;
  if (t == kTailFold) {
    fold_r<P, HASH>(L, base + r0.x, r0.y, sel >> 24, pw, oc, K, hacc);
    return;
  }
  const uint32_t A = (sel >> 16) & 3u;
#define RS_R4(C, AA, OPC)                                                      \
  case 4 * C + 0: tail_r<P, HASH, AA, OPC, 0>(L, x, pw, oc, K, hacc); break;   \
  case 4 * C + 1: tail_r<P, HASH, AA, OPC, 1>(L, x, pw, oc, K, hacc); break;   \
  case 4 * C + 2: tail_r<P, HASH, AA, OPC, 2>(L, x, pw, oc, K, hacc); break;   \
  case 4 * C + 3: tail_r<P, HASH, AA, OPC, 3>(L, x, pw, oc, K, hacc); break;
  // one gather per arity (the class-signature jump tables of gather_brx.cuh), so an op
  // holds only its own operands' registers
  if (A == 2) {
    const uint32_t c[2] = {r0.x, r0.y};
    uint64_t x[2][P];
    gather_rs<2, P>(L, sel & 0xffu, c, x);
    switch (t) {
      RS_R4(5, 2, RS_OP_AND) RS_R4(6, 2, RS_OP_OR) RS_R4(7, 2, RS_OP_XOR) RS_R4(8, 2, RS_OP_ADD)
      RS_R4(9, 2, RS_OP_SUB) RS_R4(10, 2, RS_OP_MUL) RS_R4(11, 2, RS_OP_EQ) RS_R4(12, 2, RS_OP_LT)
      RS_R4(13, 2, RS_OP_CAT)
      default: break;
    }
  } else if (A == 1) {
    const uint32_t c[1] = {r0.x};
    uint64_t x[1][P];
    gather_rs<1, P>(L, sel & 0xffu, c, x);
    switch (t) {
      RS_R4(0, 1, RS_OP_NOT) RS_R4(1, 1, RS_OP_SHL) RS_R4(2, 1, RS_OP_SHR) RS_R4(3, 1, RS_OP_BITS)
      RS_R4(4, 1, OP_COPY)
      default: break;
    }
  } else {
    const uint32_t c[3] = {r0.x, r0.y, r0.z};
    uint64_t x[3][P];
    gather_rs<3, P>(L, sel & 0xffu, c, x);
    switch (t) {
      RS_R4(14, 3, RS_OP_AND) RS_R4(15, 3, RS_OP_OR) RS_R4(16, 3, RS_OP_XOR) RS_R4(17, 3, RS_OP_ADD)
      RS_R4(18, 3, RS_OP_SUB) RS_R4(19, 3, RS_OP_MUL) RS_R4(20, 3, RS_OP_MUX)
      default: break;
    }
  }
#undef RS_R4
}

// Two ops with <= 2 operands from records (a0, a1), (b0, b1): both ops' loads are in flight
// before either is computed (the PSU partial unrolling); a one-operand op is
// gathered as two-operand.
template <int P, bool HASH>
__device__ __forceinline__ void pair_r(const LaneT& L, const uint4& a0, const uint4& a1, const uint4& b0,
                                       const uint4& b1, uint64_t (&hacc)[P]) {
  const uint32_t aA = (a1.w >> 16) & 3u, bA = (b1.w >> 16) & 3u;
  const uint32_t ca[2] = {a0.x, aA == 2u ? a0.y : a0.x}, cb[2] = {b0.x, bA == 2u ? b0.y : b0.x};
  uint64_t xa[2][P], xb[2][P];
  gather_t<2, P>(L, ca, xa);
  gather_t<2, P>(L, cb, xb);
  tail_pair<P, HASH>(L, xa, a0.w, a1.x, HASH ? ((uint64_t)a1.z << 32 | a1.y) : 0ull, (a1.w >> 8) & 0xffu, hacc);
  tail_pair<P, HASH>(L, xb, b0.w, b1.x, HASH ? ((uint64_t)b1.z << 32 | b1.y) : 0ull, (b1.w >> 8) & 0xffu, hacc);
}

__device__ __forceinline__ bool pairable(const uint4& r1) {
  const uint32_t A = (r1.w >> 16) & 3u;
  return A == 1u || A == 2u;  // folds carry arity 0, 3-operand ops 3
}

// OPS stage: records at buf + off_c (h->n of them).
// This warp takes ops j0, j0 + nw, ... -- interleaved across the runs, so every warp gets
// the same mix of cheap and expensive ops and the stage barrier waits for nobody in
// particular (dynamic claiming from a shared-memory counter lost: C3 1.185 vs 1.150 ms
// per cycle, C2 153 vs 125 us).  PAIRS (allocations with many ops per CTA and level;
// measured: C4 37.5 -> 31.6 ms per cycle, C3 1.23 -> 1.29 ms, so C3 stays single): ops
// with <= 2 operands (sorted first in every level) in pairs.
template <int P, bool HASH, bool PAIRS>
__device__ __forceinline__ void stage_ops_r(const LaneT& L, const uint8_t* buf, uint32_t j0, uint32_t nw,
                                            uint64_t (&hacc)[P]) {
  const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
  const uint32_t base = smem_addr(buf), rec0 = base + h->off_c, n = h->n;
  uint32_t j = j0;
#pragma unroll 1
  for (; PAIRS && j + nw < n; j += 2 * nw) {
    const uint4 a0 = lds128(rec0 + kRecBytes * j), a1 = lds128(rec0 + kRecBytes * j + 16);
    const uint4 b0 = lds128(rec0 + kRecBytes * (j + nw)), b1 = lds128(rec0 + kRecBytes * (j + nw) + 16);
    if (!pairable(a1) || !pairable(b1)) break;  // a fold or a 3-operand op: single path
    pair_r<P, HASH>(L, a0, a1, b0, b1, hacc);
  }
#pragma unroll 1
  for (; j < n; j += nw) op_r<P, HASH>(L, base, rec0 + kRecBytes * j, hacc);
}

template <int P, bool HASH, bool PAIRS>
__global__ void __launch_bounds__(PAIRS ? RS_LANES_R_PAIRS_MAX_THREADS
                                        : P == 1 ? RS_LANES_R1_MAX_THREADS : RS_LANES_R_MAX_THREADS, 1)
    k_lanes_r(const StepArgs a) {
  constexpr uint32_t LT = 32u * P;
  extern __shared__ __align__(128) uint8_t smem[];
  // [mbarriers | stage buffer 0 | stage buffer 1 | scyc[4][LT] | sreg[4][LT]] (hash partials as k_lanes_b)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  uint64_t* scyc = reinterpret_cast<uint64_t*>(smem + 128 + 2 * (size_t)a.stage_bytes);
  uint64_t* sreg = scyc + 4 * LT;

  const uint32_t CS = a.cluster;
  const uint32_t rank = blockIdx.x % CS, tile = blockIdx.x / CS;
  const uint32_t lin = tid & 31u, warp = tid >> 5, nwarp = T >> 5;
  const uint32_t gw = rank * nwarp + warp, ngw = CS * nwarp;
  const uint32_t lane = tile * LT + lin;
  const LaneT L = make_lanet(a.state + (size_t)tile * a.tile_bytes, lin);

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  if constexpr (HASH) {
    for (uint32_t i = tid; i < 8 * LT; i += T) {
      const uint32_t l = tile * LT + (i % LT);
      scyc[i] = (i >= 4 * LT && i < 5 * LT && rank == 0 && l < a.n_lanes) ? a.hcarry_in[l] : 0ull;  // sreg[0]
    }
  }
  __syncthreads();
  const uint32_t S = a.n_stages;
  const uint32_t total = a.n_cycles * S;
  if (tid == T - 1 && total) {
    const StageRef r = a.stage_tab[0];
    tma_load_1d(smem + 128, a.stage_blob + r.off, r.bytes, &mbar[0]);
  }
  const uint32_t producer = T - 1;
  StageRef nref{};
  if (tid == producer && total > 1) nref = a.stage_tab[S > 1 ? 1 : 0];
  if (CS > 1) stage_barrier(CS);

  uint64_t hacc[P];
#pragma unroll
  for (int k = 0; k < P; ++k) hacc[k] = 0;
  uint32_t s = 0, cyc = 0;
#pragma unroll 1
  for (uint32_t gi = 0; gi < total; ++gi) {
    const uint32_t bsel = gi & 1u;
    if (tid == producer && gi + 1 < total) {
      tma_load_1d(smem + 128 + (bsel ^ 1u) * a.stage_bytes, a.stage_blob + nref.off, nref.bytes, &mbar[bsel ^ 1u]);
      nref = a.stage_tab[(s + 2) % S];
    }
    mbar_wait(&mbar[bsel], (gi >> 1) & 1u);
    const uint8_t* buf = smem + 128 + bsel * a.stage_bytes;
    const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
    const uint32_t type = h->type;
    uint32_t b, e;
    chunk_of(h->n, gw, ngw, b, e);
    if (type == ST_OPS) {
      stage_ops_r<P, HASH, PAIRS>(L, buf, gw, ngw, hacc);
    } else if (type == ST_LATCH) {
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        uint64_t hr[P];
#pragma unroll
        for (int k = 0; k < P; ++k) hr[k] = 0;
        stage_latch_t<P, HASH, PAIRS ? RS_K7_LATCH_U_PAIRS : RS_K7_LATCH_U>(L, base + h->off_c, base + h->off_w,
                                                                             base + h->off_k, b, e, hr);
        if constexpr (HASH) {
          uint64_t* sr = sreg + ((cyc + 1u) & 3u) * LT;
#pragma unroll
          for (int k = 0; k < P; ++k) atomicAdd((unsigned long long*)&sr[lin + 32 * k], (unsigned long long)hr[k]);
        }
      }
    } else if (type == ST_INJECT) {
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        stage_inject_t<P, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, h->first, b, e, a, lane,
                                a.cycle0 + cyc, hacc);
      }
    } else if (type == ST_WATCH) {
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
        uint64_t* sc = scyc + (cyc & 3u) * LT;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          if (hacc[k]) atomicAdd((unsigned long long*)&sc[lin + 32 * k], (unsigned long long)hacc[k]);
          hacc[k] = 0;
        }
        if (warp == nwarp - 1) {  // clear the slots of cycle c + 2 (read two cycles ago)
#pragma unroll
          for (int k = 0; k < P; ++k) {
            scyc[((cyc + 2u) & 3u) * LT + lin + 32 * k] = 0;
            sreg[((cyc + 2u) & 3u) * LT + lin + 32 * k] = 0;
          }
        }
      }
    }
    stage_barrier(CS);
    if constexpr (HASH) {
      if (eoc && warp == 0 && rank == 0 && a.hashes != nullptr) {
        const uint32_t sl = (cyc & 3u) * LT;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const uint32_t li = lin + 32 * k;
          uint64_t sum = a.g.const_hash + scyc[sl + li] + sreg[sl + li];
          for (uint32_t r = 1; r < CS; ++r) {
            const uint64_t* pc = dsmem(scyc, r);
            sum += pc[sl + li] + pc[4 * LT + sl + li];
          }
          if (lane + 32 * k < a.n_lanes) a.hashes[(size_t)cyc * a.n_lanes + lane + 32 * k] = sum;
        }
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
    stage_barrier(CS);
    if (warp == 0 && rank == 0) {
      const uint32_t sl = (cyc & 3u) * LT;
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const uint32_t li = lin + 32 * k, l = lane + 32 * k;
        uint64_t sum = sreg[sl + li];
        for (uint32_t r = 1; r < CS; ++r) sum += dsmem(sreg, r)[sl + li];
        if (l < a.n_lanes) a.hcarry_out[l] = sum;
      }
    }
    if (CS > 1) stage_barrier(CS);
  }
}

}  // namespace rtlsim
