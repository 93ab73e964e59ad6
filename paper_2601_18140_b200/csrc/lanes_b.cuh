// lanes_b.cuh -- the bit-sliced tile lane kernel (k_lanes_b, rs_lane_opts.kernel = 6;
// SURVEY.md §8(f) NEXT-4, the GPU analog of the paper's specialisation ladder,
// PAPER.md §5.2).
//
// Same tile interleave as lanes_t.cuh (a tile is LT = 32 * P lanes, thread t
// of a warp owns lanes t + 32k, one warp works on one op for all LT lanes),
// but the 1-bit signals -- half of a C3/C4-shaped design -- are stored as bit
// planes: a row is P 32-bit words, word k holding lanes 32k..32k+31.  Then
//   * an op whose result and operands are all 1-bit (compiler run kind 0) is
//     evaluated on words: one logic instruction covers 32 lanes (and / or /
//     xor / not; bit 0 of add / sub is xor, of mul is and; mux is one LOP3);
//   * a 1-bit operand of any other op is one vector load of the row's words
//     (all threads of the warp read the same 4 * P bytes) plus the thread's
//     bit of each word;
//   * a 1-bit result of a wider op (eq, lt, bits, shr, ...) is packed with one
//     warp ballot per word and stored by one thread;
// and the hash of a 1-bit value is a predicated add of the weight.
//
// Bound coordinates (runtime.cu bind_stages_b): byte offset of the row's
// lane-0 container (or first word) inside the tile | class, class 0..3 =
// u8/u16/u32/u64 containers, 4 = bit plane (offsets are multiples of 16).
// Operand gathers dispatch once per op on the class signature through a jump
// table (gather_b.cuh); the op itself is run-uniform (Format c).
#pragma once
#include "gather_b.cuh"
#include "lanes_t.cuh"

#ifndef RS_LANES_B_MAX_THREADS
#define RS_LANES_B_MAX_THREADS 768
#endif

namespace rtlsim {

constexpr uint32_t kClsBit = 4;

struct LaneB {
  const uint8_t* tb;  // tile base
  uint32_t lin;       // thread index in the warp
  uint32_t adj[4];    // (lin << c) - c: coordinate -> byte offset of the thread's lane-0 container
};

__device__ __forceinline__ LaneB make_laneb(const uint8_t* tb, uint32_t lin) {
  LaneB L;
  L.tb = tb;
  L.lin = lin;
#pragma unroll
  for (int c = 0; c < 4; ++c) L.adj[c] = (lin << c) - (uint32_t)c;
  return L;
}

// The P words of a bit-plane row (coordinate c, class 4).
template <int P>
__device__ __forceinline__ void ldwords(const LaneB& L, uint32_t c, uint32_t (&w)[P]) {
  const uint8_t* p = L.tb + (c - kClsBit);
  if constexpr (P == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else if constexpr (P == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    w[0] = v.x; w[1] = v.y;
  } else {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
}
template <int P>
__device__ __forceinline__ void stwords(const LaneB& L, uint32_t c, const uint32_t (&w)[P]) {
  uint8_t* p = const_cast<uint8_t*>(L.tb) + (c - kClsBit);
  if (L.lin != 0u) return;
  if constexpr (P == 4) {
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  } else if constexpr (P == 2) {
    *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  } else {
    *reinterpret_cast<uint32_t*>(p) = w[0];
  }
}

// One operand of runtime class (latch, wide folds): the thread's P lanes.
template <int P>
__device__ __forceinline__ void ldb(const LaneB& L, uint32_t c, uint64_t (&x)[P]) {
  const uint32_t cls = c & 7u;
  if (cls == kClsBit) {
    uint32_t w[P];
    ldwords<P>(L, c, w);
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = (w[k] >> L.lin) & 1u;
    return;
  }
  const uint8_t* p = L.tb + (c + ((L.lin << cls) - cls));
  switch (cls) {
    case 0:
#pragma unroll
      for (int k = 0; k < P; ++k) x[k] = p[32 * k];
      break;
    case 1:
#pragma unroll
      for (int k = 0; k < P; ++k) x[k] = reinterpret_cast<const uint16_t*>(p)[32 * k];
      break;
    case 2:
#pragma unroll
      for (int k = 0; k < P; ++k) x[k] = reinterpret_cast<const uint32_t*>(p)[32 * k];
      break;
    default:
#pragma unroll
      for (int k = 0; k < P; ++k) x[k] = reinterpret_cast<const uint64_t*>(p)[32 * k];
      break;
  }
}

// Store P lanes' values (already masked) to a row of runtime class; a bit-plane
// row is packed with one ballot per word (every thread of the warp takes part).
template <int P>
__device__ __forceinline__ void stb(const LaneB& L, uint32_t c, const uint64_t (&v)[P]) {
  const uint32_t cls = c & 7u;
  if (cls == kClsBit) {
    uint32_t w[P];
#pragma unroll
    for (int k = 0; k < P; ++k) w[k] = __ballot_sync(0xffffffffu, (uint32_t)v[k] & 1u);
    stwords<P>(L, c, w);
    return;
  }
  uint8_t* p = const_cast<uint8_t*>(L.tb) + (c + ((L.lin << cls) - cls));
  switch (cls) {
    case 0:
#pragma unroll
      for (int k = 0; k < P; ++k) p[32 * k] = (uint8_t)v[k];
      break;
    case 1:
#pragma unroll
      for (int k = 0; k < P; ++k) reinterpret_cast<uint16_t*>(p)[32 * k] = (uint16_t)v[k];
      break;
    case 2:
#pragma unroll
      for (int k = 0; k < P; ++k) reinterpret_cast<uint32_t*>(p)[32 * k] = (uint32_t)v[k];
      break;
    default:
#pragma unroll
      for (int k = 0; k < P; ++k) reinterpret_cast<uint64_t*>(p)[32 * k] = v[k];
      break;
  }
}

// hacc += K when bit `lin` of word w is set (a 1-bit value's hash term): one
// predicate and a predicated 64-bit add
__device__ __forceinline__ void hash_bit(uint64_t& hacc, uint32_t w, uint32_t bitmask, uint64_t K) {
  asm("{\n .reg .pred p;\n .reg .u32 t;\n and.b32 t, %1, %2;\n setp.ne.u32 p, t, 0;\n @p add.u64 %0, %0, %3;\n}"
      : "+l"(hacc) : "r"(w), "r"(bitmask), "l"(K));
}

template <int P>
__device__ __forceinline__ void hash_add(uint64_t (&hacc)[P], const uint64_t (&v)[P], uint64_t K) {
#pragma unroll
  for (int k = 0; k < P; ++k) hacc[k] += v[k] * K;
}

template <int A, int P>
__device__ __forceinline__ void gather_b(const LaneB& L, uint32_t sig, const uint32_t (&c)[A], uint64_t (&x)[A][P]) {
  if constexpr (P == 2) {
    if constexpr (A == 1) gatherb_sig1_p2(sig, L.tb, L.lin, L.adj[0], L.adj[1], L.adj[2], L.adj[3], c[0], x);
    else if constexpr (A == 2) gatherb_sig2_p2(sig, L.tb, L.lin, L.adj[0], L.adj[1], L.adj[2], L.adj[3], c[0], c[1], x);
    else gatherb_sig3_p2(sig, L.tb, L.lin, L.adj[0], L.adj[1], L.adj[2], L.adj[3], c[0], c[1], c[2], x);
  } else {
    if constexpr (A == 1) gatherb_sig1_p4(sig, L.tb, L.lin, L.adj[0], L.adj[1], L.adj[2], L.adj[3], c[0], x);
    else if constexpr (A == 2) gatherb_sig2_p4(sig, L.tb, L.lin, L.adj[0], L.adj[1], L.adj[2], L.adj[3], c[0], c[1], x);
    else gatherb_sig3_p4(sig, L.tb, L.lin, L.adj[0], L.adj[1], L.adj[2], L.adj[3], c[0], c[1], c[2], x);
  }
}

// Word evaluation of a kind-0 op (1-bit result of 1-bit operands) on 32 lanes
// per word: the ops' bit-0 semantics (reading R1: every result masked to its
// width; bit 0 of a sum / difference is the xor, of a product the and).
__device__ __forceinline__ uint32_t word_fold(uint32_t op, uint32_t r, uint32_t x) {
  switch (op) {
    case RS_OP_AND: case RS_OP_MUL: return r & x;
    case RS_OP_OR: return r | x;
    default: return r ^ x;  // xor, add, sub
  }
}

template <int P, bool HASH>
__device__ __forceinline__ void word_ops(const LaneB& L, uint32_t op, uint32_t ar, uint32_t s_c, uint32_t s_w,
                                         uint32_t s_k, uint32_t ob, uint32_t cnt, uint64_t (&hacc)[P]) {
#pragma unroll 1
  for (uint32_t j = 0; j < cnt; ++j) {
    const uint32_t cb = s_c + 4 * j * ar;
    uint32_t r[P], x[P];
    ldwords<P>(L, lds32(cb), r);
    if (op == RS_OP_MUX) {
      uint32_t y[P];
      ldwords<P>(L, lds32(cb + 4), x);
      ldwords<P>(L, lds32(cb + 8), y);
#pragma unroll
      for (int k = 0; k < P; ++k) r[k] = (r[k] & x[k]) | (~r[k] & y[k]);
    } else if (ar >= 2) {
      ldwords<P>(L, lds32(cb + 4), x);
      if (op == RS_OP_EQ) {
#pragma unroll
        for (int k = 0; k < P; ++k) r[k] = ~(r[k] ^ x[k]);
      } else if (op == RS_OP_LT) {
#pragma unroll
        for (int k = 0; k < P; ++k) r[k] = ~r[k] & x[k];
      } else if (op == RS_OP_CAT) {
#pragma unroll
        for (int k = 0; k < P; ++k) r[k] = x[k];  // w_b = 1: (x0 << 1 | x1) & 1 = x1
      } else {
#pragma unroll
        for (int k = 0; k < P; ++k) r[k] = word_fold(op, r[k], x[k]);
#pragma unroll 1
        for (uint32_t o = 2; o < ar; ++o) {
          ldwords<P>(L, lds32(cb + 4 * o), x);
#pragma unroll
          for (int k = 0; k < P; ++k) r[k] = word_fold(op, r[k], x[k]);
        }
      }
    } else {
      const uint32_t pw = lds32(s_w + 4 * j), p0 = (pw >> 7) & 127u, p1 = (pw >> 14) & 63u;
      if (op == RS_OP_NOT) {
#pragma unroll
        for (int k = 0; k < P; ++k) r[k] = ~r[k];
      } else if ((op == RS_OP_SHL || op == RS_OP_SHR) ? p0 != 0u : (op == RS_OP_BITS && p1 != 0u)) {
#pragma unroll
        for (int k = 0; k < P; ++k) r[k] = 0u;  // a 1-bit value shifted by >= 1 (or its bit lo >= 1)
      }                                         // else: copy / shift by 0 / bits(x, hi, 0)
    }
    if constexpr (HASH) {
      const uint64_t K = lds64(s_k + 8 * j);
      const uint32_t bm = 1u << L.lin;
#pragma unroll
      for (int k = 0; k < P; ++k) hash_bit(hacc[k], r[k], bm, K);
    }
    stwords<P>(L, ob + 16u * j, r);
  }
}

// Low 32 bits of an op's result (reading R1 semantics before the final mask):
// and / or / xor / add / sub / mul / not / shl / cat / mux / copy need only the
// low 32 bits of their operands (a mux's selector is tested on all 64); eq, lt,
// shr and bits read whole operands.
template <int OP, int A>
__device__ __forceinline__ uint32_t low32(const uint64_t* x, uint32_t pw) {
  const uint32_t p0 = (pw >> 7) & 127u;
  const uint32_t x0 = (uint32_t)x[0], x1 = (uint32_t)x[A > 1 ? 1 : 0], x2 = (uint32_t)x[A > 2 ? 2 : 0];
  if constexpr (OP == RS_OP_AND) return A == 3 ? x0 & x1 & x2 : x0 & x1;
  else if constexpr (OP == RS_OP_OR) return A == 3 ? x0 | x1 | x2 : x0 | x1;
  else if constexpr (OP == RS_OP_XOR) return A == 3 ? x0 ^ x1 ^ x2 : x0 ^ x1;
  else if constexpr (OP == RS_OP_ADD) return A == 3 ? x0 + x1 + x2 : x0 + x1;
  else if constexpr (OP == RS_OP_SUB) return A == 3 ? x0 - x1 - x2 : x0 - x1;
  else if constexpr (OP == RS_OP_MUL) return A == 3 ? x0 * x1 * x2 : x0 * x1;
  else if constexpr (OP == RS_OP_NOT) return ~x0;
  else if constexpr (OP == RS_OP_SHL) return p0 >= 32u ? 0u : x0 << p0;
  else if constexpr (OP == RS_OP_SHR) return p0 >= 64u ? 0u : (uint32_t)(x[0] >> p0);
  else if constexpr (OP == RS_OP_BITS) {
    const uint32_t lo = (pw >> 14) & 63u, n = p0 - lo + 1u;
    return (uint32_t)(x[0] >> lo) & (n >= 32u ? 0xFFFFFFFFu : ((1u << n) - 1u));
  } else if constexpr (OP == RS_OP_CAT) return p0 >= 32u ? x1 : ((x0 << p0) | x1);
  else if constexpr (OP == RS_OP_EQ) return x[0] == x[1 % A] ? 1u : 0u;
  else if constexpr (OP == RS_OP_LT) return x[0] < x[1 % A] ? 1u : 0u;
  else if constexpr (OP == RS_OP_MUX) return x[0] != 0ull ? x1 : x2;
  else return x0;  // OP_COPY
}

enum : uint32_t { OC_BIT = 0, OC_NARROW = 1, OC_WIDE = 2 };

// Compute, mask, hash and store one op (opcode OP, A operands, result kind OC:
// a bit plane, a <= 32-bit container or a 64-bit one) for the thread's P lanes.
template <int P, bool HASH, int A, int OP, int OC>
__device__ __forceinline__ void op_tail(const LaneB& L, const uint64_t (&x)[A][P], uint32_t pw, uint32_t s_k,
                                        uint32_t oc, uint64_t (&hacc)[P]) {
  if constexpr (OC == OC_WIDE) {
    uint64_t v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      uint64_t xs[A];
#pragma unroll
      for (int o = 0; o < A; ++o) xs[o] = x[o][k];
      v[k] = apply_op<OP, A>(xs, pw);  // masked to w_out
    }
    if constexpr (HASH) hash_add<P>(hacc, v, lds64(s_k));
    uint64_t* q = reinterpret_cast<uint64_t*>(const_cast<uint8_t*>(L.tb) + (oc + ((L.lin << 3) - 3u)));
#pragma unroll
    for (int k = 0; k < P; ++k) q[32 * k] = v[k];
  } else {
    uint32_t y[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      uint64_t xs[A];
#pragma unroll
      for (int o = 0; o < A; ++o) xs[o] = x[o][k];
      y[k] = low32<OP, A>(xs, pw);
    }
    if constexpr (OC == OC_BIT) {
      uint32_t w[P];
#pragma unroll
      for (int k = 0; k < P; ++k) w[k] = __ballot_sync(0xffffffffu, y[k] & 1u);
      if constexpr (HASH) {
        const uint64_t K = lds64(s_k);
#pragma unroll
        for (int k = 0; k < P; ++k) hash_bit(hacc[k], y[k], 1u, K);
      }
      stwords<P>(L, oc, w);
    } else {
      const uint32_t m = 0xFFFFFFFFu >> (32u - (pw & 127u));  // w_out <= 32
#pragma unroll
      for (int k = 0; k < P; ++k) y[k] &= m;
      if constexpr (HASH) {
        const uint64_t K = lds64(s_k);
        const uint32_t klo = (uint32_t)K, khi = (uint32_t)(K >> 32);
#pragma unroll
        for (int k = 0; k < P; ++k) hacc[k] += (uint64_t)y[k] * klo + ((uint64_t)(y[k] * khi) << 32);
      }
      const uint32_t cls = oc & 7u;
      uint8_t* q = const_cast<uint8_t*>(L.tb) + (oc + ((L.lin << cls) - cls));
      if (cls == 0u) {
#pragma unroll
        for (int k = 0; k < P; ++k) q[32 * k] = (uint8_t)y[k];
      } else if (cls == 1u) {
#pragma unroll
        for (int k = 0; k < P; ++k) reinterpret_cast<uint16_t*>(q)[32 * k] = (uint16_t)y[k];
      } else {
#pragma unroll
        for (int k = 0; k < P; ++k) reinterpret_cast<uint32_t*>(q)[32 * k] = y[k];
      }
    }
  }
}

// Dense tail index of (opcode, result kind) per arity, written into param word
// bits [31:27] at bind time (runtime.cu bind_stages_b) so the tail dispatch is
// one jump-table branch.
__host__ __device__ constexpr int tail_op_index(int A, int op) {
  return A == 1 ? (op == RS_OP_NOT ? 0 : op == RS_OP_SHL ? 1 : op == RS_OP_SHR ? 2 : op == RS_OP_BITS ? 3 : 4)
       : A == 2 ? (op <= RS_OP_XOR ? op : op <= RS_OP_LT ? op - 1 : 8)  // and or xor | add sub mul eq lt | cat
                : (op <= RS_OP_XOR ? op : op <= RS_OP_MUL ? op - 1 : 6);  // and or xor | add sub mul | mux
}

// cnt ops of one run (kind 1 / 2), gathered op by op through the class
// signature (pw bits [26:20]), then one jump on (opcode, result kind) (pw bits
// [31:27]) into the specialised compute / mask / hash / store tail.
template <int P, bool HASH, int A>
__device__ __forceinline__ void lane_ops(const LaneB& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t ob,
                                         uint32_t ostride, uint32_t cnt, uint64_t (&hacc)[P]) {
#pragma unroll 1
  for (uint32_t j = 0; j < cnt; ++j) {
    uint32_t c[A];
#pragma unroll
    for (int o = 0; o < A; ++o) c[o] = lds32(s_c + 4 * (j * A + o));
    const uint32_t pw = lds32(s_w + 4 * j);
    uint64_t x[A][P];
    gather_b<A, P>(L, (pw >> 20) & 127u, c, x);
    const uint32_t oc = ob + ostride * j, sk = s_k + 8 * j;
#define RS_T(I, OPC)                                                                              \
  case 3 * I + OC_BIT: op_tail<P, HASH, A, OPC, OC_BIT>(L, x, pw, sk, oc, hacc); break;             \
  case 3 * I + OC_NARROW: op_tail<P, HASH, A, OPC, OC_NARROW>(L, x, pw, sk, oc, hacc); break;       \
  case 3 * I + OC_WIDE: op_tail<P, HASH, A, OPC, OC_WIDE>(L, x, pw, sk, oc, hacc); break;
    if constexpr (A == 1) {
      switch (pw >> 27) {
        RS_T(0, RS_OP_NOT) RS_T(1, RS_OP_SHL) RS_T(2, RS_OP_SHR) RS_T(3, RS_OP_BITS) RS_T(4, OP_COPY)
        default: break;
      }
    } else if constexpr (A == 2) {
      switch (pw >> 27) {
        RS_T(0, RS_OP_AND) RS_T(1, RS_OP_OR) RS_T(2, RS_OP_XOR) RS_T(3, RS_OP_ADD) RS_T(4, RS_OP_SUB)
        RS_T(5, RS_OP_MUL) RS_T(6, RS_OP_EQ) RS_T(7, RS_OP_LT) RS_T(8, RS_OP_CAT)
        default: break;
      }
    } else {
      switch (pw >> 27) {
        RS_T(0, RS_OP_AND) RS_T(1, RS_OP_OR) RS_T(2, RS_OP_XOR) RS_T(3, RS_OP_ADD) RS_T(4, RS_OP_SUB)
        RS_T(5, RS_OP_MUL) RS_T(6, RS_OP_MUX)
        default: break;
      }
    }
#undef RS_T
  }
}

// Folds with more than 3 operands (kind 1 / 2; left fold over the O rank; rare).
template <int P, bool HASH>
__device__ __forceinline__ void fold_ops(const LaneB& L, uint32_t op, uint32_t ar, uint32_t s_c, uint32_t s_w,
                                         uint32_t s_k, uint32_t ob, uint32_t ostride, uint32_t cnt,
                                         uint64_t (&hacc)[P]) {
#pragma unroll 1
  for (uint32_t j = 0; j < cnt; ++j) {
    const uint32_t cb = s_c + 4 * j * ar;
    uint64_t r[P], x[P];
    ldb<P>(L, lds32(cb), r);
#pragma unroll 1
    for (uint32_t o = 1; o < ar; ++o) {
      ldb<P>(L, lds32(cb + 4 * o), x);
#pragma unroll
      for (int k = 0; k < P; ++k) r[k] = fold_step(op, r[k], x[k]);
    }
    const uint64_t m = wmask(lds32(s_w + 4 * j) & 127u);
#pragma unroll
    for (int k = 0; k < P; ++k) r[k] &= m;
    if constexpr (HASH) hash_add<P>(hacc, r, lds64(s_k + 8 * j));
    stb<P>(L, ob + ostride * j, r);
  }
}

// Prefetch into L1 the operand rows of work item `it` (this warp's next item):
// thread t touches 128-byte line t of each row segment of the tile, so the
// gathers of that item hit L1 instead of waiting on L2 / HBM (memory-level
// parallelism across items without holding values in registers).
template <int P>
__device__ __forceinline__ void prefetch_item(const LaneB& L, const uint32_t* items, const StageRun* runs,
                                              uint32_t s_c0, uint32_t it) {
  const uint32_t w = items[it];
  const StageRun R = runs[w >> 16];
  const uint32_t b = w & 0x1FFFu, cnt = ((w >> 13) & 7u) + 1u, ar = (R.meta >> 8) & 0xffu;
  const uint32_t n = min(cnt * ar, 12u);
  const uint32_t s_c = s_c0 + 4 * (R.coord_begin + (b - R.op_begin) * ar);
#pragma unroll 1
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t c = lds32(s_c + 4 * i), cls = c & 7u;
    const uint32_t lines = cls == kClsBit ? 1u : max(1u, (uint32_t)(P << cls) >> 2);  // (32 * P << cls) / 128
    if (L.lin < lines) {
      const uint8_t* p = L.tb + ((c & ~15u) + 128u * L.lin);
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
    }
  }
}

template <int P, bool HASH>
__device__ __forceinline__ void stage_ops_b(const LaneB& L, const uint8_t* buf, uint32_t w0, uint32_t nw,
                                            uint64_t (&hacc)[P]) {
  constexpr uint32_t LT = 32u * P;
  const StageHdr* h = reinterpret_cast<const StageHdr*>(buf);
  const StageRun* runs = reinterpret_cast<const StageRun*>(buf + h->off_runs);
  const uint32_t* items = reinterpret_cast<const uint32_t*>(buf + h->off_items);
  const uint32_t base = smem_addr(buf), n_items = h->n_items;
  const uint32_t s_c0 = base + h->off_c, s_w0 = base + h->off_w, s_k0 = base + h->off_k;
#ifndef RS_NO_PREFETCH
  if (w0 < n_items) prefetch_item<P>(L, items, runs, s_c0, w0);
#endif
#pragma unroll 1
  for (uint32_t it = w0; it < n_items; it += nw) {
#ifndef RS_NO_PREFETCH
    if (it + nw < n_items) prefetch_item<P>(L, items, runs, s_c0, it + nw);
#endif
    const uint32_t w = items[it];
    const StageRun R = runs[w >> 16];
    const uint32_t b = w & 0x1FFFu, cnt = ((w >> 13) & 7u) + 1u;
    const uint32_t op = R.meta & 0xffu, ar = (R.meta >> 8) & 0xffu, kind = (R.meta >> 18) & 3u, k = b - R.op_begin;
    // out_row0 is bound to the first output's coordinate (offset | class)
    const uint32_t ocls = R.out_row0 & 7u;
    const uint32_t ostride = ocls == kClsBit ? 16u : (LT << ocls);
    const uint32_t ob = R.out_row0 + k * ostride;
    const uint32_t s_c = s_c0 + 4 * (R.coord_begin + k * ar), s_w = s_w0 + 4 * b, s_k = s_k0 + 8 * b;
    if (kind == 0u) {
      word_ops<P, HASH>(L, op, ar, s_c, s_w, s_k, ob, cnt, hacc);
    } else if (ar == 2) {
      lane_ops<P, HASH, 2>(L, s_c, s_w, s_k, ob, ostride, cnt, hacc);
    } else if (ar == 1) {
      lane_ops<P, HASH, 1>(L, s_c, s_w, s_k, ob, ostride, cnt, hacc);
    } else if (ar == 3) {
      lane_ops<P, HASH, 3>(L, s_c, s_w, s_k, ob, ostride, cnt, hacc);
    } else {
      fold_ops<P, HASH>(L, op, ar, s_c, s_w, s_k, ob, ostride, cnt, hacc);
    }
  }
}

// LATCH stage: tmp = LI[next] & M(w_r); LI[r] = tmp (one pass: every next row is an op row).
template <int P, bool HASH>
__device__ __forceinline__ void stage_latch_b(const LaneB& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t b,
                                              uint32_t e, uint64_t (&hr)[P]) {
#pragma unroll 1
  for (uint32_t j = b; j < e; ++j) {
    uint64_t v[P];
    ldb<P>(L, lds32(s_c + 8 * j), v);
    const uint64_t m = wmask(lds32(s_w + 4 * j));
#pragma unroll
    for (int k = 0; k < P; ++k) v[k] &= m;
    stb<P>(L, lds32(s_c + 8 * j + 4), v);
    if constexpr (HASH) hash_add<P>(hr, v, lds64(s_k + 8 * j));
  }
}

// INJECT stage: LI[in_k] = stimulus & M(w_k) (or the staged value).
template <int P, bool HASH>
__device__ __forceinline__ void stage_inject_b(const LaneB& L, uint32_t s_c, uint32_t s_w, uint32_t s_k, uint32_t first,
                                               uint32_t b, uint32_t e, const StepArgs& a, uint32_t lane,
                                               uint64_t cycle, uint64_t (&hacc)[P]) {
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
    stb<P>(L, lds32(s_c + 4 * j), v);
    if constexpr (HASH) hash_add<P>(hacc, v, lds64(s_k + 8 * j));
  }
}

// WATCH stage (rs_watch) on a bit-sliced tile: as stage_watch (kernels.cuh).
template <int P>
__device__ __forceinline__ void stage_watch_b(const StepArgs& a, const LaneB& L, const uint32_t* coords, uint32_t b,
                                              uint32_t e, uint32_t tile, uint64_t cycle) {
  const size_t lanes_pad = (size_t)gridDim.x / a.cluster * a.LT;
#pragma unroll 1
  for (uint32_t j = b; j < e; ++j) {
    uint64_t v[P];
    ldb<P>(L, coords[j], v);
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const uint32_t l = tile * a.LT + L.lin + 32 * k;  // allocation lane
      uint64_t* prev = a.wave_prev + (size_t)j * lanes_pad + l;
      const bool rec = l < a.n_lanes && (cycle == a.wave_first || *prev != v[k]);
      *prev = v[k];
      const uint32_t m = __ballot_sync(0xffffffffu, rec);
      if (m == 0u) continue;
      const uint32_t leader = __ffs(m) - 1;
      unsigned long long base = 0;
      if (L.lin == leader) base = atomicAdd(a.wave_count, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (rec) {
        const unsigned long long i = base + __popc(m & ((1u << L.lin) - 1u));
        if (i < a.wave_cap) {
          uint64_t* r = a.wave_rec + 4 * i;
          r[0] = cycle;
          r[1] = a.lane0 + l;
          r[2] = j;
          r[3] = v[k];
        }
      }
    }
  }
}

// Shared-memory bytes beyond the two stage buffers: per-lane hash partials,
// scyc[4][LT] (the CTA's op / input terms of a cycle, by cycle mod 4) and
// sreg[4][LT] (its register terms), summed with shared-memory atomics -- no
// per-thread partial arrays, so the CTA can run 1,024 threads.
__host__ __device__ constexpr size_t lanes_b_smem_extra(uint32_t P) { return 2ull * 4 * 32 * P * 8; }

template <int P, bool HASH>
__global__ void __launch_bounds__(RS_LANES_B_MAX_THREADS, 1) k_lanes_b(const StepArgs a) {
  constexpr uint32_t LT = 32u * P;
  extern __shared__ __align__(128) uint8_t smem[];
  // [mbarriers | stage buffer 0 | stage buffer 1 | scyc[4][LT] | sreg[4][LT]]
  // Hash of cycle c (reading R12) = const + sum over the cluster's CTAs of
  // scyc[c % 4] (ops and inputs of cycle c) + sreg[c % 4] (registers committed
  // by the latch of cycle c - 1; slot 0 starts from the carry).  Every thread
  // adds its partials with atomics at the cycle's last stage; after that
  // stage's barrier the cluster's rank 0 sums the slots of all its CTAs
  // (distributed shared memory); slot (c + 2) % 4 is cleared at cycle c.
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  uint64_t* scyc = reinterpret_cast<uint64_t*>(smem + 128 + 2 * (size_t)a.stage_bytes);
  uint64_t* sreg = scyc + 4 * LT;

  const uint32_t CS = a.cluster;
  const uint32_t rank = blockIdx.x % CS, tile = blockIdx.x / CS;
  const uint32_t lin = tid & 31u, warp = tid >> 5, nwarp = T >> 5;
  const uint32_t gw = rank * nwarp + warp, ngw = CS * nwarp;
  const uint32_t lane = tile * LT + lin;
  const LaneB L = make_laneb(a.state + (size_t)tile * a.tile_bytes, lin);

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  if constexpr (HASH) {
    for (uint32_t i = tid; i < 8 * LT; i += T) {
      const uint32_t l = tile * LT + (i % LT);
      scyc[i] = (i == 4 * LT + (i % LT) && rank == 0 && l < a.n_lanes) ? a.hcarry_in[l] : 0ull;  // sreg[0]
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
    if (type == ST_OPS) {
      stage_ops_b<P, HASH>(L, buf, gw, ngw, hacc);
    } else if (type == ST_LATCH) {
      uint32_t b, e;
      chunk_of(h->n, gw, ngw, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        uint64_t hr[P];
#pragma unroll
        for (int k = 0; k < P; ++k) hr[k] = 0;
        stage_latch_b<P, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, b, e, hr);
        if constexpr (HASH) {
          uint64_t* sr = sreg + ((cyc + 1u) & 3u) * LT;
#pragma unroll
          for (int k = 0; k < P; ++k) atomicAdd((unsigned long long*)&sr[lin + 32 * k], (unsigned long long)hr[k]);
        }
      }
    } else if (type == ST_INJECT) {
      uint32_t b, e;
      chunk_of(h->n, gw, ngw, b, e);
      if (b < e) {
        const uint32_t base = smem_addr(buf);
        stage_inject_b<P, HASH>(L, base + h->off_c, base + h->off_w, base + h->off_k, h->first, b, e, a, lane,
                                a.cycle0 + cyc, hacc);
      }
    } else if (type == ST_WATCH) {
      uint32_t b, e;
      chunk_of(h->n, gw, ngw, b, e);
      if (b < e)
        stage_watch_b<P>(a, L, reinterpret_cast<const uint32_t*>(buf + h->off_c), b, e, tile, a.cycle0 + cyc);
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
    // register term of the next cycle: sreg[cyc % 4] over the cluster
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
    if (CS > 1) stage_barrier(CS);  // keep every CTA's shared memory alive until rank 0 has read it
  }
}

}  // namespace rtlsim
