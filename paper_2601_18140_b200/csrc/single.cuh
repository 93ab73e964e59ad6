// single.cuh -- single-lane step kernel (RS_MODE_SINGLE; configs C1, C5).
//
// One lane has no lane parallelism; the parallel axis is the ops of a level
// (the S rank of Cascade 1).  A persistent grid of G CTAs (cooperative launch:
// all co-resident) walks the cycle; CTA g owns a fixed contiguous chunk of
// every level's ops, registers and inputs, whose descriptors (param words,
// operand coordinates, output run pieces) it copies into shared memory once per
// launch (compiler.hpp build_single_slices) -- the per-level critical path is
// then one state gather (L2) plus one grid barrier.  The grid barrier is a
// release-add / acquire-poll on one counter; with G == 1 it is __syncthreads
// and the state is read through L1.
#pragma once
#include "kernels.cuh"

namespace rtlsim {

struct SingleArgs {
  StepArgs a;
  const uint8_t* slice_blob;
  const uint64_t* slice_off;
  uint32_t slice_max;    // bytes of the largest slice (128-aligned; dynamic shared memory)
  uint32_t state_smem;   // single-CTA launches: bytes of signal state kept in shared memory (0 = off)
  // level cut (compiler.hpp SliceHdr): slices [k*gp, (k+1)*gp)
  // run partition k on replica rep[k]; partition k publishes "absolute cycle c
  // done" as *flag[k] = c + 1.  On one device every partition is a CTA group of
  // one cooperative launch (part_base = 0); across devices (rs_ipc_connect) each
  // process launches its own partition's gp CTAs (part_base = rank * gp), rep[m]
  // and flag[m] of the other partitions are peer-mapped device memory, and the
  // flags and fences are system scope (sys = 1).  parts == 1: plain single-lane.
  uint32_t parts, gp;
  uint32_t tail_global;  // slice tails (push / latch / inject lists) read from global memory
  uint32_t part_base;    // slice index of this launch's CTA 0
  uint32_t sys;          // partitions on other devices: .sys-scope flags and fences
  unsigned long long* flag[kMaxParts];
  uint8_t* rep[kMaxParts];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Grid barrier; before it, each warp's lane 0 has put the warp's hash partial
// in wsum[warp] (or 0): the CTA's sum is added to *hsum (relaxed atomic) by
// thread 0 on the way in.
template <bool GRID>
__device__ __forceinline__ void single_barrier(unsigned long long* bar, unsigned long long& target, uint32_t nctas,
                                               uint64_t* wsum, unsigned long long* hsum) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (hsum) {
      uint64_t s = 0;
      for (uint32_t w = 0; w < (blockDim.x + 31) / 32; ++w) s += wsum[w];
      atomicAdd(hsum, (unsigned long long)s);
    }
    if constexpr (GRID) {
      target += nctas;
      red_release_add(bar, 1ull);
      while (ld_acquire(bar) < target) {
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void warp_partial(uint64_t v, uint64_t* wsum) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
}

template <bool GRID>
struct SState {
  uint8_t* base;
  uint64_t r1, r2, r3;  // class region offsets (class 0 region starts at 0 after rebasing)
  __device__ __forceinline__ uint8_t* addr(uint32_t c) const {
    const uint32_t cls = c >> 30;
    const uint64_t reg = cls == 0 ? 0 : cls == 1 ? r1 : cls == 2 ? r2 : r3;
    return base + reg + ((uint64_t)(c & ROW_MASK) << cls);
  }
  // Branch-free gather (threads of a warp hold different ops, so a per-class
  // switch would diverge and serialize the warp's loads): load the aligned
  // 64-bit word holding the container, then shift and mask it.
  __device__ __forceinline__ uint64_t word(uint32_t c) const {
    const uintptr_t p = reinterpret_cast<uintptr_t>(addr(c));
    const uint64_t* q = reinterpret_cast<const uint64_t*>(p & ~(uintptr_t)7);
    if constexpr (GRID) return __ldcg(q);
    else return *q;
  }
  __device__ __forceinline__ uint64_t fix(uint32_t c, uint64_t w) const {
    const uint32_t cls = c >> 30;
    const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(addr(c)) & 7u) * 8u;
    const uint64_t v = w >> sh;
    return cls == 3u ? w : (v & (0xFFFFFFFFull >> (32u - (8u << min(cls, 2u)))));
  }
  __device__ __forceinline__ uint64_t ld(uint32_t c) const {
    const uint8_t* p = addr(c);
    if constexpr (GRID) {
      switch (c >> 30) {
        case 0: return __ldcg(p);
        case 1: return __ldcg(reinterpret_cast<const uint16_t*>(p));
        case 2: return __ldcg(reinterpret_cast<const uint32_t*>(p));
        default: return __ldcg(reinterpret_cast<const uint64_t*>(p));
      }
    } else {
      switch (c >> 30) {
        case 0: return *p;
        case 1: return *reinterpret_cast<const uint16_t*>(p);
        case 2: return *reinterpret_cast<const uint32_t*>(p);
        default: return *reinterpret_cast<const uint64_t*>(p);
      }
    }
  }
  __device__ __forceinline__ void st(uint32_t c, uint64_t v) const {
    uint8_t* p = addr(c);
    switch (c >> 30) {
      case 0: *p = (uint8_t)v; break;
      case 1: *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; break;
      case 2: *reinterpret_cast<uint32_t*>(p) = (uint32_t)v; break;
      default: *reinterpret_cast<uint64_t*>(p) = v; break;
    }
  }
};

// One op of a level chunk: gather (eq:split_einsum1), op_u / op_r / op_s.
template <bool GRID>
__device__ __forceinline__ uint64_t single_eval(const SState<GRID>& S, uint32_t pw, const uint32_t* cp) {
  const uint32_t op = (pw >> 22) & 15u, n = pw >> 26, p0 = (pw >> 7) & 127u;
  // all operand loads first (convergent, predicated by arity), then the fix-ups
  const uint32_t c0 = cp[0], c1 = n >= 2 ? cp[1] : c0, c2 = n >= 3 ? cp[2] : c0;
  const uint64_t w0 = S.word(c0), w1 = S.word(c1), w2 = S.word(c2);
  const uint64_t x0 = S.fix(c0, w0), x1 = S.fix(c1, w1), x2 = S.fix(c2, w2);
  uint64_t r;
  switch (op) {
    case RS_OP_AND: r = x0 & x1; if (n >= 3) r &= x2; break;
    case RS_OP_OR: r = x0 | x1; if (n >= 3) r |= x2; break;
    case RS_OP_XOR: r = x0 ^ x1; if (n >= 3) r ^= x2; break;
    case RS_OP_ADD: r = x0 + x1; if (n >= 3) r += x2; break;
    case RS_OP_SUB: r = x0 - x1; if (n >= 3) r -= x2; break;
    case RS_OP_MUL: r = x0 * x1; if (n >= 3) r *= x2; break;
    case RS_OP_EQ: r = x0 == x1 ? 1ull : 0ull; break;
    case RS_OP_LT: r = x0 < x1 ? 1ull : 0ull; break;
    case RS_OP_NOT: r = ~x0; break;
    case RS_OP_SHL: r = p0 >= 64 ? 0ull : (x0 << p0); break;
    case RS_OP_SHR: r = p0 >= 64 ? 0ull : (x0 >> p0); break;
    case RS_OP_BITS: {
      const uint32_t lo = (pw >> 14) & 63u;
      r = (x0 >> lo) & wmask(p0 - lo + 1u);
      break;
    }
    case RS_OP_CAT: r = p0 >= 64 ? x1 : ((x0 << p0) | x1); break;
    case RS_OP_MUX: r = x0 != 0 ? x1 : x2; break;
    default: r = x0; break;  // OP_COPY
  }
  if (n > 3 && op <= RS_OP_MUL)  // rare long folds (left fold over the O rank)
    for (uint32_t o = 3; o < n; ++o) r = fold_step(op, r, S.ld(cp[o]));
  return r & wmask(pw & 127u);
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool GRID, bool HASH>
__global__ void __launch_bounds__(1024, 1) k_single2(const SingleArgs sa) {
  const StepArgs& a = sa.a;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t wsum[32];
  const uint32_t tid = threadIdx.x, T = blockDim.x;
  {  // this CTA's slice of the graph, resident for the whole launch
    const uint8_t* src = sa.slice_blob + sa.slice_off[sa.part_base + blockIdx.x];
    const SliceHdr* sh = reinterpret_cast<const SliceHdr*>(src);
    const uint32_t bytes = sa.tail_global ? sh->head_bytes : sh->bytes;
    for (uint32_t i = tid * 16; i < bytes; i += T * 16)
      *reinterpret_cast<uint4*>(smem + i) = __ldg(reinterpret_cast<const uint4*>(src + i));
  }
  if (tid < 32) wsum[tid] = 0;
  __syncthreads();
  const SliceHdr* h = reinterpret_cast<const SliceHdr*>(smem);
  const SliceLvl* lvl = reinterpret_cast<const SliceLvl*>(smem + h->off_lvl);
  const SliceSeg* seg = reinterpret_cast<const SliceSeg*>(smem + h->off_seg);
  const uint32_t* pws = reinterpret_cast<const uint32_t*>(smem + h->off_pw);
  const uint32_t* crd = reinterpret_cast<const uint32_t*>(smem + h->off_coord);
  const uint8_t* tail = sa.tail_global ? sa.slice_blob + sa.slice_off[sa.part_base + blockIdx.x] : smem;
  const uint32_t* lat = reinterpret_cast<const uint32_t*>(tail + h->off_latch);
  const uint32_t* inj = reinterpret_cast<const uint32_t*>(tail + h->off_inj);
  const uint32_t* psh = reinterpret_cast<const uint32_t*>(tail + h->off_push);
  const uint32_t part = h->part, P = sa.parts;
  const bool lead = blockIdx.x == 0;               // adds this launch's carry (its registers' hash term)
  const bool lead0 = lead && sa.part_base == 0;    // ... and the constants' term, once over all partitions
  unsigned long long* bar = a.bar + 4 * part;      // partition-local grid barrier

  // single CTA with a small state: the whole signal state lives in shared memory
  uint8_t* st_base = P > 1 ? sa.rep[part] : a.state;
  if (!GRID && sa.state_smem) {
    st_base = smem + sa.slice_max;
    for (uint32_t i = tid * 16; i < sa.state_smem; i += T * 16)
      *reinterpret_cast<uint4*>(st_base + i) = *reinterpret_cast<const uint4*>(a.state + i);
    __syncthreads();
  }
  SState<GRID> S;
  S.base = st_base + a.region[0];
  S.r1 = a.region[1] - a.region[0];
  S.r2 = a.region[2] - a.region[0];
  S.r3 = a.region[3] - a.region[0];
  // the same signal in replica m (level cut): same offset from the replica base
  auto peer = [&](uint32_t c, uint32_t m) -> uint8_t* { return sa.rep[m] + (S.addr(c) - st_base); };
  auto peer_st = [&](uint32_t c, uint32_t m, uint64_t v) {
    uint8_t* q = peer(c, m);
    switch (c >> 30) {
      case 0: *q = (uint8_t)v; break;
      case 1: *reinterpret_cast<uint16_t*>(q) = (uint16_t)v; break;
      case 2: *reinterpret_cast<uint32_t*>(q) = (uint32_t)v; break;
      default: *reinterpret_cast<uint64_t*>(q) = v; break;
    }
  };
  unsigned long long target = 0;
  uint64_t hacc = (HASH && lead && tid == 0) ? a.hcarry_in[0] + (lead0 ? a.g.const_hash : 0ull) : 0ull;

  // inputs are injected into every replica; partition 0 hashes them
  const bool hin_on = HASH && part == 0;
  const uint64_t kinj = (hin_on && tid < h->n_inj) ? __ldg(a.g.in_k + h->inj_first + tid) : 0ull;
  auto inject = [&](uint64_t cyc) -> uint64_t {
    uint64_t hh = 0;
    for (uint32_t i = tid; i < h->n_inj; i += T) {
      const uint32_t k = h->inj_first + i;
      uint64_t v = a.staged ? __ldg(a.stage + (size_t)(cyc % a.stage_cap) * a.g.n_inputs + k)
                            : d_stimulus(a.seed, k, cyc, a.lane0);
      v &= wmask(inj[2 * i + 1]);
      S.st(inj[2 * i], v);
      if (hin_on) hh += v * (i == tid ? kinj : __ldg(a.g.in_k + k));
    }
    return hh;
  };
  if (a.n_cycles == 0) return;
  hacc += inject(a.cycle0);
  single_barrier<GRID>(bar, target, sa.gp, wsum, nullptr);
  uint64_t hr = 0;
  // op slot of this thread: ops are dealt to warps first (op t -> warp t % W,
  // lane t / W), so a level with few ops puts one op per warp -- the warps run
  // their ops' code paths in parallel instead of one warp diverging over them
  const uint32_t W = (T + 31) / 32;
  const uint32_t top_w = (tid & 31u) * W + (tid >> 5);
  // ...but a level with more than two ops per warp is dealt densely (op t ->
  // thread t): consecutive ops share a run (opcode, arity, class), so a warp's
  // threads mostly take one code path, and far fewer warp instructions issue
  auto slot = [&](uint32_t n) -> uint32_t { return n > 2 * W ? tid : top_w; };
  // hash weights are software-pipelined one level ahead: with few warps per
  // SM an exposed global load per level would dominate the level's latency
  auto kload = [&](uint32_t l) -> uint64_t {
    if (!HASH || l >= h->n_levels) return 0ull;
    const SliceLvl& L = lvl[l];
    const uint32_t t0 = slot(L.n);
    return t0 < L.n ? __ldg(a.g.opk + L.op_begin + t0) : 0ull;
  };
  uint64_t knext = kload(0);
  const uint64_t klat = (HASH && tid < h->n_latch && (lat[4 * tid + 2] & 128u)) ? __ldg(a.g.reg_k + lat[4 * tid + 3]) : 0ull;
#pragma unroll 1
  for (uint32_t cyc = 0; cyc < a.n_cycles; ++cyc) {
    if (P > 1) {  // token ring: partition k runs cycle c after k-1 finished it; 0 after P-1 finished c-1
      if (tid == 0) {
        const unsigned long long* f = sa.flag[part == 0 ? P - 1 : part - 1];
        const unsigned long long want = part == 0 ? a.cycle0 + cyc : a.cycle0 + cyc + 1;
        if (sa.sys) {  // bounded: a peer that never arrives must not hang the device (results then differ)
          for (uint32_t spin = 0; ld_acquire_sys(f) < want && spin < (1u << 26); ++spin) {
          }
        } else {
          for (uint32_t spin = 0; ld_acquire(f) < want && spin < (1u << 26); ++spin) {
          }
        }
      }
      __syncthreads();
    }
#pragma unroll 1
    for (uint32_t l = 0; l < h->n_levels; ++l) {
      const SliceLvl L = lvl[l];
      const uint64_t kcur = knext;
      knext = kload(l + 1 < h->n_levels ? l + 1 : 0);
      const uint32_t top = slot(L.n);
#pragma unroll 1
      for (uint32_t t = top; t < L.n; t += T) {
        const uint64_t k = !HASH ? 0ull : (t == top ? kcur : __ldg(a.g.opk + L.op_begin + t));
        const uint32_t pw = pws[L.pw_base + t];
        uint32_t lo = L.seg_begin, hi = L.seg_begin + L.n_seg - 1;  // last piece with first <= t
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (seg[mid].first <= t) lo = mid; else hi = mid - 1;
        }
        const SliceSeg G_ = seg[lo];
        const uint64_t y = single_eval<GRID>(S, pw, crd + L.coord_base + G_.coord0 + (t - G_.first) * (pw >> 26));
        S.st(G_.out_coord0 + (t - G_.first), y);
        if (HASH) hacc += y * k;
      }
      single_barrier<GRID>(bar, target, sa.gp, wsum, nullptr);
#ifdef RS_TRACE
      if (blockIdx.x == 0 && tid == 0 && a.trace && cyc < 8 && l < 60) a.trace[cyc * 64 + l] = clock64();
#endif
    }
    if (a.n_watch) {  // waveform (rs_watch): the snapshot the hash covers, before the commit
#pragma unroll 1
      for (uint32_t i = blockIdx.x * T + tid; i < a.n_watch; i += gridDim.x * T)
        watch_single(a, i, S.ld(a.watch_ent[i]), a.cycle0 + cyc);
      single_barrier<GRID>(bar, target, sa.gp, wsum, nullptr);  // no latch before every watched value is read
    }
    hr = 0;
#pragma unroll 1
    for (uint32_t i = tid; i < h->n_latch; i += T) {
      const uint32_t wf = lat[4 * i + 2];
      // differential exchange: a register other partitions read is sent to
      // their replicas only when its value changed -- every replica already holds the
      // value it had (each change was sent); the first cycle of a launch sends all, so
      // host writes between launches (rs_write_registers) cannot leave replicas apart
      const bool diff = (wf >> 8) != 0u && cyc > 0;
      const uint64_t old = diff ? S.ld(lat[4 * i + 1]) : 0ull;
      const uint64_t x = S.ld(lat[4 * i]) & wmask(wf & 127u);
      S.st(lat[4 * i + 1], x);
      if (wf & 128u) {  // own register: hash it; publish it to the replicas that finished the cycle
        if (HASH) hr += x * (i == tid ? klat : __ldg(a.g.reg_k + lat[4 * i + 3]));
        if (!diff || x != old)
          for (uint32_t m = wf >> 8; m; m &= m - 1) peer_st(lat[4 * i + 1], __ffs(m) - 1, x);
      }
    }
    if (P > 1) {  // cut signals to the later partitions that read them
#pragma unroll 1
      for (uint32_t i = tid; i < h->n_push; i += T) {
        const uint32_t c = psh[2 * i];
        const uint64_t v = S.ld(c);
        for (uint32_t m = psh[2 * i + 1]; m; m &= m - 1) peer_st(c, __ffs(m) - 1, v);
      }
    }
    uint64_t hin = 0;
    if (cyc + 1 < a.n_cycles) hin = inject(a.cycle0 + cyc + 1);
    if (HASH) {
      warp_partial(hacc, wsum);
      hacc = hr + hin + ((lead0 && tid == 0) ? a.g.const_hash : 0ull);
    }
#ifdef RS_TRACE
    if (blockIdx.x == 0 && tid == 0 && a.trace && cyc < 8) a.trace[cyc * 64 + 60] = clock64();
#endif
    if (sa.sys) __threadfence_system();  // this CTA's peer stores, visible system-wide before the flag
    single_barrier<GRID>(bar, target, sa.gp, wsum, (HASH && a.hashes) ? (unsigned long long*)(a.hashes + cyc) : nullptr);
    if (P > 1 && tid == 0 && blockIdx.x + sa.part_base == part * sa.gp) {
      if (sa.sys) st_release_sys(sa.flag[part], a.cycle0 + cyc + 1);
      else st_release(sa.flag[part], a.cycle0 + cyc + 1);
    }
#ifdef RS_TRACE
    if (blockIdx.x == 0 && tid == 0 && a.trace && cyc < 8) a.trace[cyc * 64 + 61] = clock64();
#endif
  }
  if (HASH) {
    warp_partial(hr, wsum);
    __syncthreads();
    if (tid == 0) {
      uint64_t s = 0;
      for (uint32_t w = 0; w < (T + 31) / 32; ++w) s += wsum[w];
      atomicAdd((unsigned long long*)a.hcarry_out, (unsigned long long)s);
    }
  }
  if (!GRID && sa.state_smem) {  // write the state back
    __syncthreads();
    for (uint32_t i = tid * 16; i < sa.state_smem; i += T * 16)
      *reinterpret_cast<uint4*>(a.state + i) = *reinterpret_cast<const uint4*>(st_base + i);
  }
}

}  // namespace rtlsim
