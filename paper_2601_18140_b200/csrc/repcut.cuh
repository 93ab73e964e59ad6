// repcut.cuh -- replicated-cut single-lane kernels (rs_lane_opts.repcut; the
// single-lane auto choice with one partition when a design fits one SM).
//
// The RepCut cascade (App. C, Cascade 2 P:2021-2078; SURVEY.md §8(f)
// NEXT-2): partition p = CTA p of a cooperative launch owns a block of the
// registers and evaluates the combinational cone of their next values
// (compiler.hpp build_repcut: shared logic replicated) on its OWN copy of the
// state, so the levels of a cycle need only CTA barriers -- no grid barrier
// per level as in single.cuh.  After the register commit, the Register Update
// Map (Cascade 2's last Einsum, LI_{c+1} = LI_{c,I} . RUM) delivers every
// register's new value to the partitions that read it.  Hash terms (reading
// R12) are added by the one partition that owns each op.
//   k_repcut      -- state replicas in global memory; RUM as a push between two
//                    grid barriers (inputs hashed by partition 0);
//   k_repcut_smem -- working set in shared memory; RUM as a pull through a
//                    mailbox after one grid barrier (inputs hashed by their
//                    lowest reader).
#pragma once
#include "kernels.cuh"

namespace rtlsim {

struct RepArgs {
  StepArgs a;
  const uint32_t* lvl_begin;   // [P][n_levels + 1]
  const uint32_t* ops;         // op index | owned << 31
  const uint32_t* reg_begin;   // [P + 1]
  const uint32_t* regs;
  const uint32_t* push_begin;  // [P + 1]
  const uint32_t* push;        // (register, reader partition) pairs
  uint8_t* chg;                // [n_regs]: the register's committed value changed this cycle
};

template <bool HASH>
__global__ void __launch_bounds__(1024, 1) k_repcut(const RepArgs ra) {
  const StepArgs& a = ra.a;
  __shared__ uint64_t wsum[32];
  const uint32_t p = blockIdx.x, tid = threadIdx.x, T = blockDim.x, NL = a.g.n_levels;
  const TileP<1> t = tile_ptrs<1>(a, p, 0);  // this partition's replica (replica p = tile p)
  const uint32_t* lb = ra.lvl_begin + (size_t)p * (NL + 1);
  unsigned long long target = 0;
#pragma unroll 1
  for (uint32_t cyc = 0; cyc < a.n_cycles; ++cyc) {
    const uint64_t cycle = a.cycle0 + cyc;
    uint64_t hacc = 0;
    // input injection into every replica (partition 0 hashes the inputs)
#pragma unroll 1
    for (uint32_t k = tid; k < a.g.n_inputs; k += T) {
      uint64_t v = a.staged ? __ldg(a.stage + (size_t)(cycle % a.stage_cap) * a.g.n_inputs + k)
                            : d_stimulus(a.seed, k, cycle, a.lane0);
      v &= wmask(__ldg(a.g.in_w + k));
      t.stc(__ldg(a.g.in_coord + k), v);
      if (HASH && p == 0) hacc += v * __ldg(a.g.in_k + k);
    }
    __syncthreads();
    // the partition's cone, level by level, CTA barriers only
#pragma unroll 1
    for (uint32_t l = 0; l < NL; ++l) {
#pragma unroll 1
      for (uint32_t i = lb[l] + tid; i < lb[l + 1]; i += T) {
        const uint32_t e = __ldg(ra.ops + i), j = e & 0x7FFFFFFFu;
        const uint64_t y = single_op<false>(a, t, j);
        t.stc(__ldg(a.g.out_coord + j), y);
        if (HASH && (e >> 31)) hacc += y * __ldg(a.g.opk + j);
      }
      __syncthreads();
    }
    // commit of the partition's registers (their pre-commit values are this cycle's hash terms)
#pragma unroll 1
    for (uint32_t k = ra.reg_begin[p] + tid; k < ra.reg_begin[p + 1]; k += T) {
      const uint32_t r = __ldg(ra.regs + k), rc = __ldg(a.g.reg_coord + r);
      const uint64_t old = t.ld(rc), nv = t.ld(__ldg(a.g.reg_next_coord + r)) & wmask(__ldg(a.g.reg_w + r));
      if (HASH) hacc += old * __ldg(a.g.reg_k + r);
      t.stc(rc, nv);
      if (ra.chg) ra.chg[r] = nv != old ? 1 : 0;
    }
    if (HASH) {
      const uint64_t s = block_sum(hacc, wsum) + (p == 0 ? a.g.const_hash : 0ull);
      if (tid == 0 && a.hashes) atomicAdd((unsigned long long*)(a.hashes + cyc), (unsigned long long)s);
    }
    grid_barrier(a.bar, target);  // every partition has finished reading this cycle's register values
    // Register Update Map: new register values into the replicas that read them -- with
    // differential exchange only the registers whose value changed: every
    // reader replica already holds the previous value (each change was pushed), and the
    // first cycle of a launch pushes all (host writes between launches)
#pragma unroll 1
    for (uint32_t k = ra.push_begin[p] + tid; k < ra.push_begin[p + 1]; k += T) {
      const uint32_t r = __ldg(ra.push + 2 * k), q = __ldg(ra.push + 2 * k + 1), rc = __ldg(a.g.reg_coord + r);
      if (cyc == 0 || !ra.chg || ra.chg[r]) tile_ptrs<1>(a, q, 0).stc(rc, t.ld(rc));
    }
    grid_barrier(a.bar, target);  // pushes visible before the next cycle's reads
  }
}

// ---------------------------------------------------------------------------
// k_repcut_smem: the same cascade with each partition's working set resident
// in its SM (compiler.hpp RepSliceHdr): the op descriptors and a compact local
// copy of the signals it touches live in shared memory for the whole launch,
// so a level is shared-memory loads + ALU + one CTA barrier.  Registers cross
// partitions through a global mailbox indexed by register (double-buffered by
// cycle parity): owners post at the commit, readers pull after the single
// grid barrier of the cycle -- the Register Update Map as a pull.  The local
// state is loaded from / written back to replica p at launch start / end, so
// read-back, checkpoint and the aux kernels see the usual replicas.
struct RepSmemArgs {
  StepArgs a;
  const uint8_t* blob;
  const uint64_t* slice_off;
  const uint64_t* op_k;   // per-partition op hash weights in slice op order (0: not owned)
  uint64_t* mail;         // [2][n_regs]
};

template <bool WIDE>
struct LocalState {
  uint8_t* s;
  uint32_t sa;          // shared-window address of s
  uint32_t b1, b2, b3;
  // width class of a local offset: the u64 region comes first, then u32, u16, u8
  __device__ __forceinline__ uint32_t cls(uint32_t o) const {
    return (uint32_t)(o < b1) + (uint32_t)(o < b2) + (uint32_t)(o < b3);
  }
  // branch-free gather and store: one predicated ld/st.shared per width class,
  // exactly one of which is on (a switch compiles to an indirect branch that
  // splits a warp whose operands have several widths)
  __device__ __forceinline__ uint64_t ld(uint32_t o) const {
    uint64_t v;
    if constexpr (WIDE) {  // every signal in an 8-byte slot
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sa + o) : "memory");
      return v;
    }
    asm volatile(
        "{\n\t.reg .pred q1, q2, q3, p16, p32;\n\t.reg .u32 t;\n\t"
        "setp.lt.u32 q3, %1, %2;\n\tsetp.lt.u32 q2, %1, %3;\n\tsetp.lt.u32 q1, %1, %4;\n\t"
        "xor.pred p16, q1, q2;\n\txor.pred p32, q2, q3;\n\tmov.u32 t, 0;\n\t"
        "@!q1 ld.shared.u8 t, [%5];\n\t@p16 ld.shared.u16 t, [%5];\n\t@p32 ld.shared.u32 t, [%5];\n\t"
        "cvt.u64.u32 %0, t;\n\t@q3 ld.shared.u64 %0, [%5];\n\t}"
        : "=l"(v) : "r"(o), "r"(b1), "r"(b2), "r"(b3), "r"(sa + o) : "memory");
    return v;
  }
  __device__ __forceinline__ void st(uint32_t o, uint64_t v) const {
    if constexpr (WIDE) {
      asm volatile("st.shared.u64 [%0], %1;" ::"r"(sa + o), "l"(v) : "memory");
      return;
    }
    const uint32_t c = cls(o), a = sa + o;
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
        "setp.eq.u32 q0, %2, 0;\n\tsetp.eq.u32 q1, %2, 1;\n\tsetp.eq.u32 q2, %2, 2;\n\tsetp.eq.u32 q3, %2, 3;\n\t"
        "@q0 st.shared.u8 [%0], %1;\n\t@q1 st.shared.u16 [%0], %1;\n\t"
        "@q2 st.shared.u32 [%0], %1;\n\t@q3 st.shared.u64 [%0], %1;\n\t}"
        :: "r"(a), "l"(v), "r"(c) : "memory");
  }
};

// One op (kernels.cuh select_op: branch-free; on the 16-core design a switch
// cost 2,240 cycles per level, a 14-deep select chain 1,275, the selection
// tree 1,186 -- a partition's level mixes many opcodes).
template <bool WIDE>
__device__ __forceinline__ uint64_t rep_eval(const LocalState<WIDE>& S, uint32_t pw, uint2 cw, const uint16_t* ovf) {
  const uint32_t op = (pw >> 22) & 15u, n = pw >> 26;
  const uint32_t c0 = cw.x >> 16, c1 = cw.y & 0xFFFFu, c2 = n > 3 ? c0 : cw.y >> 16;
  const uint64_t x0 = S.ld(c0), x1 = S.ld(c1), x2 = S.ld(c2);
  uint64_t r = select_op(pw, x0, x1, x2);
  if (n > 3) {  // rare long folds (op <= RS_OP_MUL): operands 2.. in the overflow list
    r = fold_step(op, x0, x1);
    for (uint32_t o = 2; o < n; ++o) r = fold_step(op, r, S.ld(ovf[(cw.y >> 16) + o - 2]));
  }
  return r & wmask(pw & 127u);
}

template <bool HASH, bool ONE, bool WIDE>
__global__ void __launch_bounds__(1024, 1) k_repcut_smem(const RepSmemArgs ra) {
  const StepArgs& a = ra.a;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t wsum[32];
  const uint32_t p = blockIdx.x, tid = threadIdx.x, T = blockDim.x, R = a.g.n_regs;
  const uint8_t* src = ra.blob + ra.slice_off[p];
  {
    const uint32_t sb = reinterpret_cast<const RepSliceHdr*>(src)->smem_bytes;
    for (uint32_t i = tid * 16; i < sb; i += T * 16)
      *reinterpret_cast<uint4*>(smem + i) = __ldg(reinterpret_cast<const uint4*>(src + i));
  }
  __syncthreads();
  const RepSliceHdr& h = *reinterpret_cast<const RepSliceHdr*>(smem);
  const uint32_t* lvl = reinterpret_cast<const uint32_t*>(smem + h.off_lvl);
  const uint32_t* pws = reinterpret_cast<const uint32_t*>(smem + h.off_pw);
  const uint2* cws = reinterpret_cast<const uint2*>(smem + h.off_cw);
  const uint16_t* ovf = reinterpret_cast<const uint16_t*>(smem + h.off_ovf);
  const uint32_t* com = reinterpret_cast<const uint32_t*>(smem + h.off_commit);
  const uint32_t* pul = reinterpret_cast<const uint32_t*>(smem + h.off_pull);
  const uint32_t* inj = reinterpret_cast<const uint32_t*>(smem + h.off_inj);
  const uint32_t* map = reinterpret_cast<const uint32_t*>(src + h.off_map);
  const uint64_t* opk = ra.op_k + h.k_base;
  LocalState<WIDE> S{smem + h.state_off, (uint32_t)__cvta_generic_to_shared(smem + h.state_off), h.b1, h.b2, h.b3};
  const TileP<1> t = tile_ptrs<1>(a, p, 0);
  for (uint32_t i = tid; i < h.n_map; i += T) S.st(map[2 * i], t.ld(map[2 * i + 1]));
  if (a.n_cycles == 0) return;
  const uint32_t NL = h.n_levels;
  // op hash weights, loaded two levels ahead for the thread's (first) op of
  // the level: from shared memory when they fit in the slice, else from global
  // memory (an exposed L2 load per level would dominate a level's work)
  const bool ksm = h.kop_smem != 0;
  const uint64_t* kop = ksm ? reinterpret_cast<const uint64_t*>(smem + h.off_kop) : opk;
  auto kload = [&](uint32_t l) -> uint64_t {
    if (!HASH || l >= NL) return 0ull;
    const uint32_t i = lvl[l] + tid;
    return i < lvl[l + 1] ? (ksm ? kop[i] : __ldg(opk + i)) : 0ull;
  };
  unsigned long long target = 0;
  uint64_t hacc = 0;
  __syncthreads();
#pragma unroll 1
  for (uint32_t cyc = 0; cyc < a.n_cycles; ++cyc) {
    const uint64_t cycle = a.cycle0 + cyc;
    uint64_t k0 = kload(0), k1 = kload(1);
#pragma unroll 1
    for (uint32_t i = tid; i < h.n_inj; i += T) {
      const uint4 e = *reinterpret_cast<const uint4*>(inj + 4 * i);
      uint64_t v = a.staged ? __ldg(a.stage + (size_t)(cycle % a.stage_cap) * a.g.n_inputs + e.y)
                            : d_stimulus(a.seed, e.y, cycle, a.lane0);
      v &= wmask((e.x >> 16) & 127u);
      S.st(e.x & 0xFFFFu, v);
      if (HASH) hacc += v * (((uint64_t)e.w << 32) | e.z);
    }
    __syncthreads();
    uint32_t b = NL ? lvl[0] : 0u, e = NL ? lvl[1] : 0u;  // level bounds, loaded a level ahead
#pragma unroll 1
    for (uint32_t l = 0; l < NL; ++l) {
      const uint32_t en = lvl[l + 2 <= NL ? l + 2 : NL];
      const uint64_t kcur = k0;
      k0 = k1;
      k1 = kload(l + 2);
      const auto do_op = [&](uint32_t i, uint64_t k) {
        const uint64_t y = rep_eval(S, pws[i], cws[i], ovf);
        S.st(cws[i].x & 0xFFFFu, y);
        if (HASH) hacc += y * k;
      };
      if (ONE) {  // the launch has a thread for every op of every level
        if (b + tid < e) do_op(b + tid, kcur);
      } else {
        if (b + tid < e) do_op(b + tid, kcur);
#pragma unroll 1
        for (uint32_t i = b + tid + T; i < e; i += T) do_op(i, HASH ? (ksm ? kop[i] : __ldg(opk + i)) : 0ull);
      }
      __syncthreads();
#ifdef RS_TRACE
      if (p == 0 && tid == 0 && a.trace && cyc < 8 && l < 60) a.trace[cyc * 64 + l] = clock64();
#endif
      b = e;
      e = en;
    }
    if (a.n_watch) {  // waveform (rs_watch): this partition's watched signals, before the commit
#pragma unroll 1
      for (uint32_t i = a.watch_begin[p] + tid; i < a.watch_begin[p + 1]; i += T)
        watch_single(a, a.watch_ent[2 * i + 1], S.ld(a.watch_ent[2 * i]), cycle);
      __syncthreads();
    }
    // commit: the pre-commit values are this cycle's register hash terms
    uint64_t* mail = ra.mail + (size_t)(cyc & 1u) * R;
#pragma unroll 1
    for (uint32_t i = tid; i < h.n_commit; i += T) {
      const uint4 e = *reinterpret_cast<const uint4*>(com + 4 * i);
      const uint32_t r = e.y & 0xFFFFFFu;
      const uint64_t nv = S.ld(e.x >> 16) & wmask(e.y >> 24);
      if (HASH) hacc += S.ld(e.x & 0xFFFFu) * (((uint64_t)e.w << 32) | e.z);
      S.st(e.x & 0xFFFFu, nv);
      if (gridDim.x > 1) mail[r] = nv;  // one partition: nobody pulls
    }
    if (HASH) {
      const uint64_t s = block_sum(hacc, wsum) + (p == 0 ? a.g.const_hash : 0ull);
      if (tid == 0 && a.hashes) atomicAdd((unsigned long long*)(a.hashes + cyc), (unsigned long long)s);
      hacc = 0;
    }
#ifdef RS_TRACE
    if (p == 0 && tid == 0 && a.trace && cyc < 8) a.trace[cyc * 64 + 60] = clock64();
#endif
    grid_barrier(a.bar, target);
#ifdef RS_TRACE
    if (p == 0 && tid == 0 && a.trace && cyc < 8) a.trace[cyc * 64 + 61] = clock64();
#endif
    // Register Update Map: pull the new values of the registers this partition reads
#pragma unroll 1
    for (uint32_t i = tid; i < h.n_pull; i += T) S.st(pul[2 * i], __ldcg(mail + pul[2 * i + 1]));
#ifdef RS_TRACE
    __syncthreads();
    if (p == 0 && tid == 0 && a.trace && cyc < 8) a.trace[cyc * 64 + 62] = clock64();
#endif
  }
  __syncthreads();
  for (uint32_t i = tid; i < h.n_map; i += T) {
    const uint32_t c = map[2 * i + 1];
    t.stc(c, S.ld(map[2 * i]));
  }
}

}  // namespace rtlsim
