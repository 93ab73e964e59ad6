// runtime.cu -- C ABI (include/rtlsim.h): device graph replicas, lane state,
// staged-input ring, launches.  No host fallback: every simulated cycle runs
// in the kernels of kernels.cuh.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // NVTX ranges around the ABI's device work (header-only; no-ops without a tool)

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rtlsim.h"
#include "codegen.hpp"
#include "compiler.hpp"
#include "kernels.cuh"
#include "lanes.cuh"
#include "lanes_t.cuh"
#include "lanes_b.cuh"
#include "lanes_r.cuh"
#include "single.cuh"
#include "repcut.cuh"

using namespace rtlsim;

namespace {
thread_local std::string g_err = "no error";

struct NvtxRange {  // an NVTX range for the scope (nsys / ncu --nvtx timelines)
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

rs_status set_err(rs_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      return set_err(e_ == cudaErrorMemoryAllocation ? RS_E_OOM : RS_E_CUDA, "%s: %s (%s:%d)", #call, \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                                  \
    }                                                                                              \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
};

template <class T>
size_t bytes_of(const std::vector<T>& v) { return v.size() * sizeof(T); }

}  // namespace

struct rs_graph {
  int device = 0;
  CompiledGraph cg;
  void* dmem = nullptr;   // one allocation holding every device array
  size_t dbytes = 0;
  GraphDev gd{};
  // device copies for read/write kernels
  uint32_t* d_sig_coord = nullptr;
  int sm_count = 148;
  int live_lanes = 0;
  // lane mode stage schedule (compiler.hpp build_stages)
  // (host copy; every allocation binds it to its own layout, see bind_stages)
  // lane-mode stage schedules, by work-item size: [0] kBatch ops (built at
  // load), [1] kBatchWide ops (built on first use)
  std::vector<uint8_t> stage_blob[2];
  std::vector<StageRef> stage_tab[2];
  bool stages_built[2] = {false, false};
  uint32_t stage_bytes = 0;
  // kernel 8 (codegen.hpp): the design's specialised kernel, compiled once (rs_specialize)
  bool su_built = false;
  std::string su_ptx;
  uint32_t su_threads = 32;
  cudaLibrary_t su_lib = nullptr;
  cudaKernel_t su_fn = nullptr;
};

struct rs_lanes {
  rs_graph* g = nullptr;
  uint32_t n_lanes = 0, LT = 1, n_tiles = 1, threads = 1024, ctas = 1, cluster = 1, variant = 1;
  uint64_t lane0 = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool counted = false;       // counted in g->live_lanes (a fully built allocation)
  void* dwatch = nullptr;      // single-lane watch entries (device)
  const uint32_t* watch_ent = nullptr;
  const uint32_t* watch_begin = nullptr;
  void* state_mem = nullptr;       // [n_tiles][tile_bytes]
  size_t state_bytes = 0;
  uint64_t tile_bytes = 0;
  uint64_t region[4] = {0, 0, 0, 0};
  uint64_t region_b = 0;           // kernel 6: bit-plane region (1-bit rows) inside a tile
  void* dstages = nullptr;         // bound stage schedule: blob, then table
  const uint8_t* stage_blob = nullptr;
  const StageRef* stage_tab = nullptr;
  uint32_t n_stages = 0;
  uint64_t* hcarry = nullptr;       // [2][n_lanes_pad]
  int hc_cur = 0;
  bool hc_valid = true;
  uint64_t cycle = 0;
  int staged = 0;
  uint64_t seed = 0;
  uint64_t* stage = nullptr;
  uint32_t stage_cap = 0;
  uint64_t st_lo = 0, st_hi = 0;    // staged window [st_lo, st_hi)
  uint32_t batch_idx = 0;           // rs_graph stage schedule in use (work-item size)
  uint32_t op_pairs = 0;            // rs_lane_opts.op_pairs (kernel 7: 0 auto, 1 single ops, 2 pairs)
  // staged-input copies run on their own stream so the next chunk's transfer
  // overlaps the current chunk's step: a copy waits for the last launch that
  // read the ring slots it overwrites; a step waits for the copies before it
  cudaStream_t cstream = nullptr;
  struct CycleRec { uint64_t c0 = 0, c1 = 0; cudaEvent_t ev = nullptr; };
  CycleRec lrec[4];                 // the last 4 launches (cycles read)
  uint64_t lrec_n = 0;
  CycleRec crec[4];                 // the last 4 copies (cycles written)
  uint64_t crec_n = 0;
  uint64_t crec_waited = 0;         // copies [0, crec_waited) are ordered before the lanes' stream
  cudaEvent_t ev_order = nullptr;   // device-to-device staging follows the lanes' stream
  uint64_t* hbuf = nullptr;         // device hash temp for host outputs
  size_t hbuf_cap = 0;
  unsigned long long* bar = nullptr;
  uint64_t launches = 0;
  unsigned long long* trace = nullptr;  // RS_TRACE builds only
  // single-lane mode: per-CTA graph slices resident in shared memory (single.cuh)
  void* dslices = nullptr;               // blob, then u64 offsets per CTA
  const uint8_t* slice_blob = nullptr;
  const uint64_t* slice_off = nullptr;
  uint32_t slice_max = 0;
  // level cut: parts partitions x gp CTAs, replica k = tile k of state_mem
  uint32_t parts = 1, gp = 1;
  // level cut across processes (rs_lane_opts.part_world): this rank's partition, its own
  // replica (state_mem) with the cycle flag after it, the peers' mapped replicas / flags
  uint32_t part_world = 0, part_rank = 0;
  bool connected = false;
  uint32_t l2_policy = 0;           // rs_lane_opts.l2_policy
  bool state_owned = true;          // false: the caller's buffer (rs_lanes_bind_state)
  size_t flag_bytes = 0;            // level cut across processes: the cycle flag after the replica
  size_t l2_persist_max = 0;        // cudaDevAttrMaxPersistingL2CacheSize
  uint8_t* peer_rep[kMaxParts] = {};
  unsigned long long* peer_flag[kMaxParts] = {};
  bool tail_global = false;
  std::vector<uint8_t> sig_part;         // canonical id -> partition whose replica holds it
  size_t total_bytes = 0;
  // RepCut (rs_lane_opts.repcut): device plan arrays
  bool repcut = false;
  void* drep = nullptr;
  RepArgs rep{};
  bool rep_smem = false;      // k_repcut_smem (partition-local shared-memory slices)
  void* rep_mail = nullptr;   // [2][n_regs] register mailbox
  bool rep_one = false;       // threads >= every partition level: one op per thread
  bool rep_wide = false;      // slices with 8-byte signal slots
  RepSmemArgs reps{};
  uint32_t rep_smem_bytes = 0;
  size_t sched_bytes = 0;                // device bytes of the bound stage schedule
  // waveform capture (rs_watch)
  std::vector<uint32_t> watch;           // canonical ids
  uint64_t* wave_prev = nullptr;         // [n_watch][lanes_pad]
  uint64_t* wave_rec = nullptr;          // [wave_cap][4]
  unsigned long long* wave_count = nullptr;
  uint64_t wave_cap = 0;
  uint64_t wave_first = 0;
};

namespace {

// kernel 7 stage buffers: a C3 level's op records (~1,650 x 32 B) fit one stage
constexpr uint32_t kStageBytesR = 96 * 1024;
constexpr size_t kBarBytes = 1024;      // partition k's grid barrier at u64 [4k]; level-cut flags at [kFlagOffset + k]
constexpr size_t kFlagOffset = 64;

bool k7_pairs(const rs_lanes* s);

StepArgs base_args(const rs_lanes* s) {
  StepArgs a{};
  a.g = s->g->gd;
  a.state = (uint8_t*)s->state_mem;
  a.tile_bytes = s->tile_bytes;
  for (int c = 0; c < 4; ++c) {
    a.region[c] = s->region[c];
    a.rows[c] = s->g->cg.rows[c];
  }
  a.LT = s->LT;
  a.n_lanes = s->n_lanes;
  a.lane0 = s->lane0;
  a.seed = s->seed;
  a.staged = s->staged;
  a.stage = s->stage;
  a.stage_cap = s->stage_cap;
  a.bar = s->bar;
  a.stage_blob = s->stage_blob;
  a.stage_tab = s->stage_tab;
  a.n_stages = s->n_stages;
  a.stage_bytes = s->variant == 7 ? kStageBytesR : s->g->stage_bytes;
  a.trace = s->trace;
  a.cluster = s->cluster;
  a.wave_prev = s->wave_prev;
  a.wave_rec = s->wave_rec;
  a.wave_count = s->wave_count;
  a.wave_cap = s->wave_cap;
  a.wave_first = s->wave_first;
  a.watch_ent = s->watch_ent;
  a.watch_begin = s->watch_begin;
  a.n_watch = s->g->cg.mode == RS_MODE_SINGLE ? (uint32_t)s->watch.size() : 0u;
  a.bitplane = s->variant == 6 ? 1u : 0u;
  a.pairs = (s->variant == 7 && k7_pairs(s)) ? 1u : 0u;  // k_lanes_r<.., true>
  a.rows_bit = s->g->cg.rows_bit;
  a.region_b = s->region_b;
  return a;
}

// Bind the graph's stage schedule to one allocation's layout: every state
// coordinate (class << 30 | row) becomes (class << 30 | byte offset of the
// row's lane 0 inside a tile); run out rows become byte offsets.  Requires
// tile_bytes < 2^30.
void bind_stages(const rs_graph* g, uint32_t bi, uint32_t LT, const uint64_t* region, std::vector<uint8_t>* out) {
  *out = g->stage_blob[bi];
  auto bind = [&](uint32_t c) -> uint32_t {
    const uint32_t cls = c >> 30, row = c & ROW_MASK;
    return (cls << 30) | (uint32_t)(region[cls] + ((uint64_t)row * LT << cls));
  };
  for (const StageRef& r : g->stage_tab[bi]) {
    uint8_t* p = out->data() + r.off;
    StageHdr h;
    std::memcpy(&h, p, sizeof h);
    uint32_t* c = reinterpret_cast<uint32_t*>(p + h.off_c);
    for (uint32_t i = 0; i < h.n_coords; ++i) c[i] = bind(c[i]);
    StageRun* runs = reinterpret_cast<StageRun*>(p + h.off_runs);
    for (uint32_t i = 0; i < h.n_runs; ++i) {
      const uint32_t cls = (runs[i].meta >> 16) & 3u;
      runs[i].out_row0 = bind((cls << 30) | runs[i].out_row0) & ROW_MASK;
    }
  }
}

// Bit-sliced allocations (kernel 6, lanes_b.cuh): coordinate -> tile byte offset
// of the row's lane-0 container | class (0..3), or of its first word | 4 for the
// 1-bit rows (bit planes, 16 bytes per row).
uint32_t bind_b(const rs_lanes* s, uint32_t c) {
  const uint32_t cls = c >> 30, row = c & ROW_MASK;
  if (cls == 0 && row < s->g->cg.rows_bit) return (uint32_t)(s->region_b + 16ull * row) | kClsBit;
  return (uint32_t)(s->region[cls] + ((uint64_t)row * s->LT << cls)) | cls;
}

void bind_stages_b(const rs_lanes* s, std::vector<uint8_t>* out) {
  const rs_graph* g = s->g;
  *out = g->stage_blob[s->batch_idx];
  for (const StageRef& r : g->stage_tab[s->batch_idx]) {
    uint8_t* p = out->data() + r.off;
    StageHdr h;
    std::memcpy(&h, p, sizeof h);
    uint32_t* c = reinterpret_cast<uint32_t*>(p + h.off_c);
    if (h.type == ST_OPS) {
      // param words get the operand class signature sum_o class(o) * 5^o in bits [26:20]
      uint32_t* w = reinterpret_cast<uint32_t*>(p + h.off_w);
      const StageRun* runs = reinterpret_cast<const StageRun*>(p + h.off_runs);
      for (uint32_t i = 0; i < h.n_runs; ++i) {
        const uint32_t ar = (runs[i].meta >> 8) & 0xffu;
        for (uint32_t j = 0; j < runs[i].count; ++j) {
          uint32_t sig = 0, m = 1;
          for (uint32_t o = 0; o < ar && o < 3; ++o, m *= 5) sig += (bind_b(s, c[runs[i].coord_begin + j * ar + o]) & 7u) * m;
          // bits [31:27]: dense (opcode, result kind) tail index (lanes_b.cuh tail_op_index)
          const uint32_t op = runs[i].meta & 0xffu, ocls = (runs[i].meta >> 16) & 3u;
          const uint32_t kind = ((runs[i].meta >> 18) & 3u) < 2u ? OC_BIT : ocls == 3u ? OC_WIDE : OC_NARROW;
          const uint32_t tail = ar <= 3 ? 3u * (uint32_t)tail_op_index((int)ar, (int)op) + kind : 0u;
          uint32_t& pw = w[runs[i].op_begin + j];
          pw = (pw & 0xFFFFFu) | ((ar <= 3 ? sig : 0u) << 20) | (tail << 27);
        }
      }
    }
    for (uint32_t i = 0; i < h.n_coords; ++i) c[i] = bind_b(s, c[i]);
    StageRun* runs = reinterpret_cast<StageRun*>(p + h.off_runs);
    for (uint32_t i = 0; i < h.n_runs; ++i) {
      const uint32_t cls = (runs[i].meta >> 16) & 3u;
      runs[i].out_row0 = bind_b(s, (cls << 30) | runs[i].out_row0);
    }
  }
}

// Record-based allocations (kernel 7, lanes_r.cuh): the kernel-1 bound schedule
// with every OPS stage rewritten as 32-byte op records {c0, c1, c2, pw, out
// coordinate, K, sel} (split into several stages when the records outgrow a
// stage buffer; an extra barrier is harmless).  Other stages are kept as bound.
void bind_stages_r(const rs_lanes* s, std::vector<uint8_t>* out, std::vector<StageRef>* tab) {
  const rs_graph* g = s->g;
  std::vector<uint8_t> k1;
  bind_stages(g, s->batch_idx, s->LT, s->region, &k1);
  out->clear();
  tab->clear();
  auto emit = [&](const uint8_t* src, uint32_t bytes, uint32_t type) {
    const size_t at = (out->size() + 15) & ~(size_t)15;
    out->resize(at + bytes, 0);
    std::memcpy(out->data() + at, src, bytes);
    tab->push_back({at, bytes, type});
  };
  const uint32_t cap = kStageBytesR;
  struct Rec { uint32_t v[8]; std::vector<uint32_t> fold; };
  std::vector<Rec> recs;   // the current level's records (kernel-1 OPS stages of one level merged)
  uint32_t rec_level = 0, rec_first = 0;
  auto flush = [&]() {
    // ops with <= 2 operands first: the kernel evaluates them in pairs (lanes_r.cuh);
    // every record carries its own output coordinate, so the order is free
    std::stable_partition(recs.begin(), recs.end(), [](const Rec& r) {
      const uint32_t ar = (r.v[7] >> 16) & 3u;
      return ((r.v[7] >> 8) & 0xffu) != kTailFold && ar >= 1u && ar <= 2u;
    });
    uint32_t i = 0;
    const uint32_t total_n = (uint32_t)recs.size();
    while (i < total_n) {  // pack records (+ fold lists) into stages of at most `cap` bytes
      const uint32_t off_rec = (uint32_t)((sizeof(StageHdr) + 15) & ~(size_t)15);
      uint32_t n = 0, nfold = 0;
      while (i + n < total_n) {
        const uint32_t nf = nfold + (uint32_t)recs[i + n].fold.size();
        if (off_rec + kRecBytes * (n + 1) + 4 * nf > cap && n > 0) break;
        nfold = nf;
        ++n;
      }
      StageHdr q{};
      q.type = ST_OPS;
      q.n = n;
      q.first = rec_first + i;
      q.level = rec_level;
      q.off_c = off_rec;
      q.bytes = (off_rec + kRecBytes * n + 4 * nfold + 15) & ~15u;
      std::vector<uint8_t> blk(q.bytes, 0);
      std::memcpy(blk.data(), &q, sizeof q);
      uint32_t fo = off_rec + kRecBytes * n;
      for (uint32_t m = 0; m < n; ++m) {
        Rec& rr = recs[i + m];
        if (!rr.fold.empty()) {
          rr.v[0] = fo;  // stage-relative byte offset of the coordinate list
          std::memcpy(blk.data() + fo, rr.fold.data(), 4 * rr.fold.size());
          fo += 4 * (uint32_t)rr.fold.size();
        }
        std::memcpy(blk.data() + off_rec + kRecBytes * m, rr.v, kRecBytes);
      }
      emit(blk.data(), q.bytes, ST_OPS);
      i += n;
    }
    recs.clear();
  };
  for (const StageRef& r : g->stage_tab[s->batch_idx]) {
    const uint8_t* p = k1.data() + r.off;
    StageHdr h;
    std::memcpy(&h, p, sizeof h);
    if (h.type != ST_OPS || (!recs.empty() && h.level != rec_level)) flush();
    if (h.type != ST_OPS) {
      emit(p, r.bytes, r.type);
      continue;
    }
    if (recs.empty()) {
      rec_level = h.level;
      rec_first = h.first;
    }
    const uint32_t* w = reinterpret_cast<const uint32_t*>(p + h.off_w);
    const uint64_t* kk = reinterpret_cast<const uint64_t*>(p + h.off_k);
    const uint32_t* c = reinterpret_cast<const uint32_t*>(p + h.off_c);
    const StageRun* runs = reinterpret_cast<const StageRun*>(p + h.off_runs);
    // records (and fold coordinate lists) per op, in stage order
    const size_t rb = recs.size();
    recs.resize(rb + h.n);
    for (uint32_t ri = 0; ri < h.n_runs; ++ri) {
      const StageRun& R = runs[ri];
      const uint32_t op = R.meta & 0xffu, ar = (R.meta >> 8) & 0xffu, cls = (R.meta >> 16) & 3u;
      for (uint32_t k = 0; k < R.count; ++k) {
        Rec& q = recs[rb + R.op_begin + k];
        const uint32_t* cc = c + R.coord_begin + k * ar;
        const uint32_t j = R.op_begin + k;
        q.v[3] = w[j];
        q.v[4] = ((cls << 30) | R.out_row0) + k * (s->LT << cls);
        q.v[5] = (uint32_t)kk[j];
        q.v[6] = (uint32_t)(kk[j] >> 32);
        if (ar <= 3) {
          q.v[0] = cc[0];
          q.v[1] = ar > 1 ? cc[1] : 0u;
          q.v[2] = ar > 2 ? cc[2] : 0u;
          q.v[7] = ((uint32_t)(4 * tail_combo((int)ar, (int)op)) + cls) << 8 | ar << 16 | op << 24;
          // bits 0..7: the operands' class signature (the gather's jump index, lanes_r.cuh op_r)
          for (uint32_t o = 0; o < ar; ++o) q.v[7] |= (cc[o] >> 30) << (2 * o);
        } else {
          q.fold.assign(cc, cc + ar);
          q.v[1] = ar;
          q.v[2] = 0;
          q.v[7] = kTailFold << 8 | op << 24;
        }
      }
    }
  }
  flush();
}

// Bind the graph's schedule to the allocation and upload it; with watched
// signals (rs_watch) a WATCH stage is spliced in before the register commit.
rs_status upload_schedule(rs_lanes* s) {
  const rs_graph* g = s->g;
  std::vector<uint8_t> bound;
  std::vector<StageRef> tab = g->stage_tab[s->batch_idx];
  if (s->variant == 6)
    bind_stages_b(s, &bound);
  else if (s->variant == 7)
    bind_stages_r(s, &bound, &tab);
  else
    bind_stages(g, s->batch_idx, s->LT, s->region, &bound);
  if (!s->watch.empty()) {
    StageHdr h{};
    h.type = ST_WATCH;
    h.n = h.n_coords = (uint32_t)s->watch.size();
    h.off_c = (uint32_t)((sizeof(StageHdr) + 15) & ~(size_t)15);
    h.bytes = (uint32_t)((h.off_c + 4ull * h.n + 15) & ~15ull);
    const size_t base = (bound.size() + 15) & ~(size_t)15;
    bound.resize(base + h.bytes, 0);
    std::memcpy(bound.data() + base, &h, sizeof h);
    uint32_t* c = reinterpret_cast<uint32_t*>(bound.data() + base + h.off_c);
    for (uint32_t i = 0; i < h.n; ++i) {
      const uint32_t co = g->cg.sig_coord[s->watch[i]], cls = co >> 30;
      c[i] = s->variant == 6 ? bind_b(s, co)
                             : (cls << 30) | (uint32_t)(s->region[cls] + ((uint64_t)(co & ROW_MASK) * s->LT << cls));
    }
    size_t at = 0;
    while (at < tab.size() && tab[at].type != ST_LATCH) ++at;
    tab.insert(tab.begin() + at, StageRef{base, h.bytes, ST_WATCH});
  }
  const size_t tab_off = (bound.size() + 255) & ~(size_t)255;
  const size_t nbytes = tab_off + tab.size() * sizeof(StageRef);
  if (s->dstages) {
    CU(cudaStreamSynchronize(s->stream));
    cudaFree(s->dstages);
    s->dstages = nullptr;
    s->total_bytes -= s->sched_bytes;
  }
  cudaError_t e = cudaMalloc(&s->dstages, nbytes);
  if (e == cudaSuccess) e = cudaMemcpy(s->dstages, bound.data(), bound.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy((uint8_t*)s->dstages + tab_off, tab.data(), tab.size() * sizeof(StageRef), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_err(RS_E_OOM, "stage schedule (%zu B): %s", nbytes, cudaGetErrorString(e));
  s->stage_blob = (const uint8_t*)s->dstages;
  s->stage_tab = (const StageRef*)((const uint8_t*)s->dstages + tab_off);
  s->n_stages = (uint32_t)tab.size();
  s->sched_bytes = nbytes;
  s->total_bytes += nbytes;
  return RS_OK;
}

rs_status set_device(const rs_graph* g) {
  CU(cudaSetDevice(g->device));
  (void)cudaGetLastError();  // a stale non-sticky error of an unrelated earlier call must not surface here
  return RS_OK;
}

template <class T>
void put(std::vector<uint8_t>& blob, size_t& off, const std::vector<T>& v, size_t* where) {
  off = (off + 255) & ~(size_t)255;
  *where = off;
  if (!v.empty()) {
    if (blob.size() < off + bytes_of(v)) blob.resize(off + bytes_of(v));
    std::memcpy(blob.data() + off, v.data(), bytes_of(v));
  }
  off += bytes_of(v);
}

// Shared-memory bytes of one stage buffer (two buffers per CTA: the stage in
// use and the one being prefetched by TMA).
constexpr uint32_t kStageBytes = 48 * 1024;

size_t lanes_smem(uint32_t stage_bytes, uint32_t threads) {
  return 128 + 2ull * stage_bytes + lanes_smem_extra(threads);
}

// Lane tile and cluster size: the widest tile (most lanes per warp instruction)
// spread over the fewest CTAs of a cluster (at most 4) that keeps >= 80% of the
// SMs busy; 8-CTA clusters only when no tile reaches that with 4.  Measured on
// B200 (profiles/r02/sweep_shapes): the best C3-shaped shapes at 4096 / 2048 /
// 1024 / 512 lanes are 128x4 (kernel 1), 64x4 (kernel 1), 32x4 and 16x4
// (kernel 2) -- 8-CTA clusters lost everywhere (e.g. 2048 lanes: 128x8 took
// 1.44 ms per cycle, 64x4 0.93 ms).  Kernel 1 tiles are 32 * P lanes (P = 1, 2,
// 4 lanes per thread), kernel 2 tiles 8, 16 or 32 lanes, kernel 6 64 or 128.
void choose_tiling(uint32_t kernel, uint32_t n_lanes, int sms, uint32_t want_lt, uint32_t want_cs, uint32_t* lt,
                   uint32_t* cs) {
  const uint32_t k1[3] = {128u, 64u, 32u}, k2[3] = {32u, 16u, 8u}, k6[2] = {128u, 64u};
  const uint32_t* cand = (kernel == 1 || kernel == 7) ? k1 : kernel == 6 ? k6 : k2;
  const int nc = kernel == 6 ? 2 : 3;
  const uint32_t smallest = cand[nc - 1];
  for (const uint32_t cmax : {4u, 8u}) {
    for (int i = 0; i < nc; ++i) {
      const uint32_t t = cand[i];
      if (want_lt && t != want_lt) continue;
      const uint64_t tiles = (n_lanes + t - 1) / t;
      for (uint32_t c : {1u, 2u, 4u, 8u}) {
        if (c > cmax || (want_cs && c != want_cs)) continue;
        if (tiles * c * 10 >= (uint64_t)sms * 8 || (want_lt && want_cs)) {
          *lt = t;
          *cs = c;
          return;
        }
      }
    }
  }
  *lt = want_lt ? want_lt : smallest;
  *cs = want_cs ? want_cs : 8;
}


// Lane-mode step kernel of an allocation (variant, tile, hash, pairs) and its
// dynamic shared memory; the shared-memory cap is a per-device function attribute,
// raised once per device to the largest size any allocation there has needed.
const void* const kLaneFns[] = {
    (const void*)k_lanes<32, true>,        (const void*)k_lanes<32, false>,
    (const void*)k_lanes<16, true>,        (const void*)k_lanes<16, false>,
    (const void*)k_lanes<8, true>,         (const void*)k_lanes<8, false>,
    (const void*)k_lanes_t<1, true>,       (const void*)k_lanes_t<1, false>,
    (const void*)k_lanes_t<2, true>,       (const void*)k_lanes_t<2, false>,
    (const void*)k_lanes_t<4, true>,       (const void*)k_lanes_t<4, false>,
    (const void*)k_lanes_b<2, true>,       (const void*)k_lanes_b<2, false>,
    (const void*)k_lanes_b<4, true>,       (const void*)k_lanes_b<4, false>,
    (const void*)k_lanes_r<2, true, false>, (const void*)k_lanes_r<2, false, false>,
    (const void*)k_lanes_r<4, true, false>, (const void*)k_lanes_r<4, false, false>,
    (const void*)k_lanes_r<2, true, true>,  (const void*)k_lanes_r<2, false, true>,
    (const void*)k_lanes_r<4, true, true>,  (const void*)k_lanes_r<4, false, true>,
    (const void*)k_lanes_r<1, true, false>, (const void*)k_lanes_r<1, false, false>,
    (const void*)k_lanes_r<1, true, true>,  (const void*)k_lanes_r<1, false, true>};

// >= 2,048 ops per CTA and level: kBatchWide work items (kernels 1 / 6) and op pairs (kernel 7)
bool wide_items(const rs_graph* g, uint32_t cluster) {
  const uint64_t ops_per_cta_level =
      g->cg.n_levels ? (uint64_t)g->cg.n_ops_total() / g->cg.n_levels / std::max<uint32_t>(1, cluster) : 0;
  return ops_per_cta_level >= 2048;
}
// kernel 7 evaluates ops in pairs (rs_lane_opts.op_pairs; auto: >= 2,048 ops per CTA and level)
bool k7_pairs(const rs_lanes* s) { return s->op_pairs ? s->op_pairs == 2u : wide_items(s->g, s->cluster); }
uint32_t k7_max_threads(const rs_lanes* s) {
  return k7_pairs(s)     ? (uint32_t)RS_LANES_R_PAIRS_MAX_THREADS
         : s->LT == 32u ? (uint32_t)RS_LANES_R1_MAX_THREADS
                        : (uint32_t)RS_LANES_R_MAX_THREADS;
}

const void* lane_kernel_fn(const rs_lanes* s, bool hash) {
  const int fi = (s->variant == 1   ? 6 + (s->LT == 32 ? 0 : s->LT == 64 ? 2 : 4)
                  : s->variant == 6 ? 12 + (s->LT == 64 ? 0 : 2)
                  : s->variant == 7 ? (s->LT == 32 ? 24 + (k7_pairs(s) ? 2 : 0) : 16 + (s->LT == 64 ? 0 : 2) + (k7_pairs(s) ? 4 : 0))
                                    : (s->LT == 32 ? 0 : s->LT == 16 ? 2 : 4)) + (hash ? 0 : 1);
  return kLaneFns[fi];
}

size_t lane_smem_bytes(const rs_lanes* s) {
  return s->variant == 7   ? 128 + 2ull * kStageBytesR + lanes_b_smem_extra(s->LT / 32)
         : s->variant == 6 ? 128 + 2ull * s->g->stage_bytes + lanes_b_smem_extra(s->LT / 32)
         : s->variant == 1 ? 128 + 2ull * s->g->stage_bytes + lanes_t_smem_extra(s->threads, s->LT / 32)
                           : lanes_smem(s->g->stage_bytes, s->threads);
}

cudaError_t raise_smem_attr(int device, size_t smem) {
  static thread_local size_t attr_set[64] = {};
  size_t& have = attr_set[device & 63];
  if (have >= smem) return cudaSuccess;
  if (have == 0) {
    // 16-CTA clusters (kernel 7 only) are a non-portable cluster size
    for (const void* f : kLaneFns) {
      const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
  }
  for (const void* f : kLaneFns) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  have = smem;
  return cudaSuccess;
}

// Clusters of this allocation's launch shape that fit the device at once.  A launch
// with more clusters runs them in waves -- which the measured "8-CTA clusters are slow"
// (2,048 C3 lanes: 16 clusters of 8 took 1.44 ms per cycle, 8 clusters of 8 ran fine)
// turned out to be.
int co_resident_clusters(const rs_lanes* s) {
  const size_t smem = lane_smem_bytes(s);
  if (raise_smem_attr(s->g->device, smem) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(s->n_tiles * s->cluster);
  cfg.blockDim = dim3(s->threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = s->cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, lane_kernel_fn(s, true), &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    return -1;  // unknown
  }
  return n;
}

}  // namespace

extern "C" {

static rs_status init_state(rs_lanes* s);

const char* rs_version(void) { return "rtlsim-b200 0.1 (sm_100a)"; }
const char* rs_last_error(void) { return g_err.c_str(); }

rs_status rs_load_graph(const rs_graph_desc* desc, int device, uint32_t mode, rs_graph** out) {
  if (!desc || !out) return set_err(RS_E_INVALID_ARG, "NULL desc/out");
  *out = nullptr;
  if (device != RS_DEVICE_NONE) {
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return set_err(RS_E_INVALID_ARG, "device %d out of range (%d devices)", device, ndev);
  }
  rs_graph* g = new (std::nothrow) rs_graph();
  if (!g) return set_err(RS_E_OOM, "host allocation failed");
  g->device = device;
  std::string err;
  rs_status st = compile_graph(desc, mode, &g->cg, &err);
  if (st != RS_OK) {
    delete g;
    return set_err(st, "%s", err.c_str());
  }
  CompiledGraph& cg = g->cg;
  // out coords per op (single-lane mode and diagnostics)
  std::vector<uint32_t> out_coord(cg.n_ops_total());
  for (const DevRun& r : cg.runs)
    for (uint32_t k = 0; k < r.count; ++k) out_coord[r.op_begin + k] = make_coord((r.meta >> 16) & 3u, r.out_row0 + k);
  std::vector<uint8_t> blob;
  size_t off = 0, o_runs, o_lrb, o_lob, o_opw, o_opk, o_coff, o_coord, o_outc, o_inc, o_inw, o_ink, o_rc, o_rn, o_rw,
         o_rk, o_sig;
  put(blob, off, cg.runs, &o_runs);
  put(blob, off, cg.level_run_begin, &o_lrb);
  put(blob, off, cg.level_op_begin, &o_lob);
  put(blob, off, cg.opw, &o_opw);
  put(blob, off, cg.opk, &o_opk);
  put(blob, off, cg.coord_off, &o_coff);
  put(blob, off, cg.coord, &o_coord);
  put(blob, off, out_coord, &o_outc);
  put(blob, off, cg.in_coord, &o_inc);
  put(blob, off, cg.in_w, &o_inw);
  put(blob, off, cg.in_k, &o_ink);
  put(blob, off, cg.reg_coord, &o_rc);
  put(blob, off, cg.reg_next_coord, &o_rn);
  put(blob, off, cg.reg_w, &o_rw);
  put(blob, off, cg.reg_k, &o_rk);
  put(blob, off, cg.sig_coord, &o_sig);
  blob.resize(std::max<size_t>(off, 256));
  if (device == RS_DEVICE_NONE) {  // compile-only handle
    g->dbytes = blob.size();
    *out = g;
    return RS_OK;
  }
  if ((st = set_device(g)) != RS_OK) { delete g; return st; }
  cudaError_t e = cudaMalloc(&g->dmem, blob.size());
  if (e != cudaSuccess) { delete g; return set_err(RS_E_OOM, "cudaMalloc graph (%zu B): %s", blob.size(), cudaGetErrorString(e)); }
  g->dbytes = blob.size();
  e = cudaMemcpy(g->dmem, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(g->dmem); delete g; return set_err(RS_E_CUDA, "graph H2D: %s", cudaGetErrorString(e)); }
  auto P = [&](size_t o) { return (const void*)((const uint8_t*)g->dmem + o); };
  GraphDev& d = g->gd;
  d.runs = (const DevRun*)P(o_runs);
  d.level_run_begin = (const uint32_t*)P(o_lrb);
  d.level_op_begin = (const uint32_t*)P(o_lob);
  d.opw = (const uint32_t*)P(o_opw);
  d.opk = (const uint64_t*)P(o_opk);
  d.coord_off = (const uint32_t*)P(o_coff);
  d.coord = (const uint32_t*)P(o_coord);
  d.out_coord = (const uint32_t*)P(o_outc);
  d.in_coord = (const uint32_t*)P(o_inc);
  d.in_w = (const uint32_t*)P(o_inw);
  d.in_k = (const uint64_t*)P(o_ink);
  d.reg_coord = (const uint32_t*)P(o_rc);
  d.reg_next_coord = (const uint32_t*)P(o_rn);
  d.reg_w = (const uint32_t*)P(o_rw);
  d.reg_k = (const uint64_t*)P(o_rk);
  d.n_levels = cg.n_levels;
  d.n_inputs = cg.n_inputs;
  d.n_regs = cg.n_regs;
  d.n_ops_total = cg.n_ops_total();
  d.const_hash = cg.const_hash;
  g->d_sig_coord = (uint32_t*)P(o_sig);
  cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cg.mode == RS_MODE_LANES) {  // (mode may carry RS_LOAD_PASSES)
    g->stage_bytes = kStageBytes;
    build_stages(cg, g->stage_bytes, kBatch, &g->stage_blob[0], &g->stage_tab[0]);
    g->stages_built[0] = true;
  }
  *out = g;
  return RS_OK;
}

rs_status rs_graph_info_get(const rs_graph* g, rs_graph_info* o) {
  if (!g || !o) return set_err(RS_E_INVALID_ARG, "NULL graph/out");
  const CompiledGraph& cg = g->cg;
  std::memset(o, 0, sizeof *o);
  o->mode = cg.mode;
  o->n_levels = cg.n_levels;
  o->n_ops = cg.n_ops;
  o->n_copy_ops = cg.n_copy;
  o->n_runs = (uint32_t)cg.runs.size();
  o->n_coords = (uint32_t)cg.coord.size();
  for (int c = 0; c < 4; ++c) o->rows[c] = cg.rows[c];
  o->state_bytes_per_lane = cg.state_bytes_per_lane();
  o->graph_device_bytes = g->dbytes;
  o->graph_alg_bytes = cg.graph_alg_bytes;
  o->alg_bytes_per_lane_cycle = cg.alg_bytes_per_lane_cycle;
  o->identity_ops_naive = cg.identity_ops_naive;
  o->rows_bit = cg.rows_bit;
  o->n_alias = cg.n_alias;
  o->n_folded = cg.n_folded;
  o->n_mux_chain = cg.n_mux_chain;
  return RS_OK;
}

rs_status rs_graph_export(const rs_graph* g, uint32_t what, void* out, uint64_t* count) {
  if (!g || !count) return set_err(RS_E_INVALID_ARG, "NULL graph/count");
  const CompiledGraph& cg = g->cg;
  const void* src = nullptr;
  size_t n = 0, esz = 4;
  switch (what) {
    case RS_EXPORT_RUNS: src = cg.runs.data(); n = cg.runs.size() * 5; break;
    case RS_EXPORT_LEVEL_RUN_BEGIN: src = cg.level_run_begin.data(); n = cg.level_run_begin.size(); break;
    case RS_EXPORT_LEVEL_OP_BEGIN: src = cg.level_op_begin.data(); n = cg.level_op_begin.size(); break;
    case RS_EXPORT_OPW: src = cg.opw.data(); n = cg.opw.size(); break;
    case RS_EXPORT_OPK: src = cg.opk.data(); n = cg.opk.size(); esz = 8; break;
    case RS_EXPORT_COORD_OFF: src = cg.coord_off.data(); n = cg.coord_off.size(); break;
    case RS_EXPORT_COORD: src = cg.coord.data(); n = cg.coord.size(); break;
    case RS_EXPORT_SIG_COORD: src = cg.sig_coord.data(); n = cg.sig_coord.size(); break;
    case RS_EXPORT_REG_COORD: src = cg.reg_coord.data(); n = cg.reg_coord.size(); break;
    case RS_EXPORT_REG_NEXT_COORD: src = cg.reg_next_coord.data(); n = cg.reg_next_coord.size(); break;
    case RS_EXPORT_IN_COORD: src = cg.in_coord.data(); n = cg.in_coord.size(); break;
    default: return set_err(RS_E_INVALID_ARG, "unknown export %u", what);
  }
  *count = n;
  if (out && n) std::memcpy(out, src, n * esz);
  return RS_OK;
}

rs_status rs_repcut_stats(const rs_graph* g, uint32_t P, uint64_t* ops_total, uint32_t* max_ops, uint64_t* push) {
  if (!g) return set_err(RS_E_INVALID_ARG, "NULL graph");
  RepCutPlan plan;
  std::string err;
  if (!build_repcut(g->cg, P, &plan, &err)) return set_err(RS_E_INVALID_ARG, "%s", err.c_str());
  if (ops_total) *ops_total = plan.ops_total;
  if (max_ops) *max_ops = plan.max_ops;
  if (push) *push = plan.push.size() / 2;
  return RS_OK;
}

rs_status rs_level_cut(const rs_graph* g, uint32_t parts, uint32_t* cut) {
  if (!g || !cut) return set_err(RS_E_INVALID_ARG, "NULL argument");
  if (parts == 0 || parts > kMaxParts || parts > std::max<uint32_t>(1, g->cg.n_levels))
    return set_err(RS_E_INVALID_ARG, "parts = %u: must be in [1, min(%u, n_levels = %u)]", parts, kMaxParts,
                   g->cg.n_levels);
  const std::vector<uint32_t> c = level_cut(g->cg, parts);
  std::memcpy(cut, c.data(), c.size() * 4);
  return RS_OK;
}

rs_status rs_specialize(rs_graph* g) {
  NvtxRange nvtx_range("rs_specialize");
  if (!g) return set_err(RS_E_INVALID_ARG, "NULL graph");
  if (!g->su_built) {
    if (g->cg.n_ops_total() > kSuMaxOps)
      return set_err(RS_E_CAPACITY, "kernel 8 (specialised) is capped at %u ops (graph has %u)", kSuMaxOps,
                     g->cg.n_ops_total());
    g->su_ptx = su_ptx(g->cg, &g->su_threads);
    g->su_built = true;
  }
  if (g->dmem && !g->su_fn) {
    rs_status st = set_device(g);
    if (st != RS_OK) return st;
    // the driver JIT-compiles the PTX for this device (ptxas)
    cudaError_t e = cudaLibraryLoadData(&g->su_lib, g->su_ptx.c_str(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&g->su_fn, g->su_lib, "rs_su");
    if (e != cudaSuccess) {
      g->su_fn = nullptr;
      return set_err(RS_E_CUDA, "kernel 8 load (PTX JIT): %s", cudaGetErrorString(e));
    }
  }
  return RS_OK;
}

rs_status rs_specialized_ptx(const rs_graph* g, char* buf, uint64_t cap, uint64_t* len) {
  if (!g) return set_err(RS_E_INVALID_ARG, "NULL graph");
  if (!g->su_built) return set_err(RS_E_STATE, "rs_specialize first");
  if (len) *len = g->su_ptx.size();
  if (buf && cap) {
    const size_t n = (size_t)std::min<uint64_t>(cap - 1, g->su_ptx.size());
    std::memcpy(buf, g->su_ptx.data(), n);
    buf[n] = 0;
  }
  return RS_OK;
}

void rs_free_graph(rs_graph* g) {
  if (!g) return;
  if (g->dmem) {
    cudaSetDevice(g->device);
    cudaFree(g->dmem);
  }
  if (g->su_lib) cudaLibraryUnload(g->su_lib);
  delete g;
}

// dynamic shared memory a RepCut slice may take (227 KiB less k_repcut_smem's static shared memory)
constexpr uint32_t kRepSmemMax = 227u * 1024u - 2048u;

rs_status rs_alloc_lanes(rs_graph* g, uint32_t n_lanes, const rs_lane_opts* opts, rs_lanes** out) {
  NvtxRange nvtx_range("rs_alloc_lanes");
  if (!g || !out) return set_err(RS_E_INVALID_ARG, "NULL graph/out");
  *out = nullptr;
  if (n_lanes == 0) return set_err(RS_E_INVALID_ARG, "n_lanes must be >= 1");
  if (!g->dmem) return set_err(RS_E_STATE, "graph was loaded with RS_DEVICE_NONE (compile only)");
  if (g->cg.mode == RS_MODE_SINGLE && n_lanes != 1)
    return set_err(RS_E_INVALID_ARG, "RS_MODE_SINGLE simulates exactly one lane (got %u)", n_lanes);
  rs_lane_opts o{};
  if (opts) o = *opts;
  rs_status st = set_device(g);
  if (st != RS_OK) return st;
  rs_lanes* s = new (std::nothrow) rs_lanes();
  if (!s) return set_err(RS_E_OOM, "host allocation failed");
  s->g = g;
  s->n_lanes = n_lanes;
  s->lane0 = o.lane0;
  if (g->cg.mode == RS_MODE_SINGLE && o.kernel && o.kernel != 3 && o.kernel != 4 && o.kernel != 5 && o.kernel != 8) {
    rs_free_lanes(s);
    return set_err(RS_E_INVALID_ARG, "single-lane kernel must be 0 (auto), 3 (RepCut, shared memory), 4 (RepCut, "
                                     "global replicas), 5 (level-synchronous grid) or 8 (specialised)");
  }
  if (o.kernel == 8) {  // the design's own straight-line kernel (codegen.hpp): one thread per lane
    if (o.parts > 1 || o.repcut || o.part_world) {
      rs_free_lanes(s);
      return set_err(RS_E_INVALID_ARG, "kernel 8 (specialised) excludes parts / repcut / part_world");
    }
    if (o.lane_tile && o.lane_tile != 32 && o.lane_tile != 64 && o.lane_tile != 128) {
      rs_free_lanes(s);
      return set_err(RS_E_INVALID_ARG, "kernel 8: lane_tile must be 0, 32, 64 or 128");
    }
    rs_status st8 = rs_specialize(g);
    if (st8 != RS_OK) {
      rs_free_lanes(s);
      return st8;
    }
    s->variant = 8;
    s->LT = g->cg.mode == RS_MODE_SINGLE ? 1u : (o.lane_tile ? o.lane_tile : 32u);
    s->n_tiles = (n_lanes + s->LT - 1) / s->LT;
    s->parts = 1;
    s->threads = g->su_threads;
    s->ctas = (n_lanes + s->threads - 1) / s->threads;
  }
  if (g->cg.mode == RS_MODE_SINGLE && (o.kernel == 3 || o.kernel == 4) && !o.repcut) o.repcut = 1;
  if (g->cg.mode == RS_MODE_SINGLE && o.kernel == 4) o.repcut_global = 1;
  if (o.repcut_global > 2) {
    rs_free_lanes(s);
    return set_err(RS_E_INVALID_ARG, "repcut_global must be 0, 1 or 2");
  }
  if (o.l2_policy > 2) {
    rs_free_lanes(s);
    return set_err(RS_E_INVALID_ARG, "l2_policy must be 0, 1 or 2");
  }
  s->l2_policy = g->cg.mode == RS_MODE_LANES ? o.l2_policy : 0u;
  if (s->l2_policy) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, g->device);
    s->l2_persist_max = (size_t)std::max(0, v);
    // the persisting carve-out is a device-wide limit: raise it to the maximum once
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur < s->l2_persist_max) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, s->l2_persist_max);
    (void)cudaGetLastError();
  }
  if (o.part_world == 1) o.part_world = 0;
  if (o.part_world && (g->cg.mode != RS_MODE_SINGLE || o.part_world > kMaxParts || o.part_rank >= o.part_world ||
                       o.parts > 1 || o.repcut || (o.kernel && o.kernel != 5) ||
                       o.part_world > std::max<uint32_t>(1, g->cg.n_levels))) {
    rs_free_lanes(s);
    return set_err(RS_E_INVALID_ARG, "part_world = %u / part_rank = %u: a single-lane level cut of 2..%u partitions "
                   "(<= n_levels), without parts / repcut", o.part_world, o.part_rank, kMaxParts);
  }
  if (o.part_world && o.defer_state) {
    rs_free_lanes(s);
    return set_err(RS_E_INVALID_ARG, "defer_state: a level cut across processes owns its state (CUDA IPC)");
  }
  if (o.part_world) {
    o.parts = o.part_world;
    o.kernel = 5;
    s->part_world = o.part_world;
    s->part_rank = o.part_rank;
  }
  if (g->cg.mode == RS_MODE_SINGLE && o.kernel == 5 && o.repcut) {
    rs_free_lanes(s);
    return set_err(RS_E_INVALID_ARG, "kernel 5 (level-synchronous) excludes repcut");
  }
  // auto: a design whose whole working set fits one SM's shared memory runs as
  // RepCut with one partition (one CTA, CTA barriers only; C1: 4.9 vs 17 us per
  // cycle on the level-synchronous grid)
  if (g->cg.mode == RS_MODE_SINGLE && o.kernel == 0 && o.repcut == 0 && o.parts <= 1 &&
      (size_t)g->cg.n_ops_total() * 12 < kRepSmemMax && g->cg.n_regs >= 1) {
    RepCutPlan plan;
    std::string err;
    std::vector<uint8_t> b1, b2;
    std::vector<uint64_t> b3, b4;
    if (build_repcut(g->cg, 1, &plan, &err) &&
        build_repcut_slices(g->cg, plan, kRepSmemMax, false, &b1, &b3, &b4, &b2, &err))
      o.repcut = 1;
  }
  if (s->variant == 8) {
    // shape set above (one thread per lane, LT-lane tiles of the usual layout)
  } else if (g->cg.mode == RS_MODE_SINGLE && o.repcut >= 1) {
    if (o.parts > 1 || o.repcut > (uint32_t)g->sm_count) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "repcut = %u: must be <= %d SMs and not combined with parts (level cut)", o.repcut,
                     g->sm_count);
    }
    s->LT = 1;
    s->repcut = true;
    s->parts = o.repcut;   // one state replica per partition: the aux kernels' replica machinery
    s->n_tiles = o.repcut;
  } else if (g->cg.mode == RS_MODE_SINGLE) {
    s->LT = 1;
    s->parts = std::max<uint32_t>(1, o.parts);
    if (s->parts > kMaxParts || s->parts > std::max<uint32_t>(1, g->cg.n_levels)) {
      const uint32_t p = s->parts;
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "parts = %u: must be <= %u and <= n_levels (%u)", p, kMaxParts, g->cg.n_levels);
    }
    s->n_tiles = s->part_world ? 1u : s->parts;  // one state replica per partition (lane index = replica in the
                                                 // aux kernels); across processes: this rank's replica only
  } else {
    if (o.parts > 1) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "parts (level cut) applies to RS_MODE_SINGLE only");
    }
    // auto: lane-poor allocations (< 2048 lanes: per-level work per SM is a few
    // hundred lane-ops, latency-bound) take kernel 2's 8..32-lane tiles; lane-rich
    // ones kernel 1's 32 * P-lane tiles (P = 4 amortizes the per-op decode).
    // (kernel 7, the record-based tile kernel, measured fastest at >= 2048 lanes: C3 1.23 vs
    // 1.30 ms per cycle for kernel 1, C4 31.6 vs 34.8 ms; profiles/r02)
    // Designs with few ops per level (<= 1,024: C2's 500) are latency-bound at every lane
    // count; there kernel 7's 32-lane tiles at 1,024 threads beat kernel 2 where their
    // clusters are co-resident with >= 64 CTAs or the lanes are few (profiles/r02/k7low:
    // C2 at 1,024 / 256 / 128 lanes 123.6 / 90.6 / 90.6 vs 130.6 / 104.7 / 103.1 us per
    // cycle), not at 512 lanes (120.7 vs 100.7: the 8-CTA clusters it needs are not
    // co-resident) nor for C3 / C4-sized levels at < 2,048 lanes (C3 1,024 lanes 689 vs 626).
    const uint32_t opl = g->cg.n_levels ? g->cg.n_ops_total() / g->cg.n_levels : 0;
    const bool k7_low = opl <= 1024u && (n_lanes >= 1024u || n_lanes <= 256u);
    const uint32_t kern = o.kernel ? o.kernel : (n_lanes >= 2048u || k7_low) ? 7u : 2u;
    if (o.lane_tile && (kern == 2   ? (o.lane_tile != 8 && o.lane_tile != 16 && o.lane_tile != 32)
                        : kern == 6 ? (o.lane_tile != 64 && o.lane_tile != 128)
                                    : (o.lane_tile != 32 && o.lane_tile != 64 && o.lane_tile != 128))) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "lane_tile must be 32, 64 or 128 (kernels 1 and 7), 8, 16 or 32 (kernel 2) "
                                       "or 64 or 128 (kernel 6)");
    }
    if (o.cluster && o.cluster != 1 && o.cluster != 2 && o.cluster != 4 && o.cluster != 8 &&
        !(o.cluster == 16 && kern == 7)) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "cluster must be 1, 2, 4 or 8 (or 16 for kernel 7)");
    }
    if (o.kernel > 2 && o.kernel != 6 && o.kernel != 7) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "lane kernel must be 0, 1, 2, 6 or 7");
    }
    if (o.op_pairs > 2) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "op_pairs must be 0, 1 or 2");
    }
    s->op_pairs = o.op_pairs;
    s->variant = kern;
    uint32_t lt, cs;
    choose_tiling(kern, n_lanes, g->sm_count, o.lane_tile, o.cluster, &lt, &cs);
    s->LT = lt;
    s->cluster = cs;
    s->n_tiles = (n_lanes + lt - 1) / lt;
  }
  // launch shape
  if (s->variant == 8) {
    // set with the kernel choice
  } else if (o.threads) {
    const uint32_t tmax = g->cg.mode == RS_MODE_SINGLE ? 1024u
                          : s->variant == 1            ? (uint32_t)RS_LANES_T_MAX_THREADS
                          : s->variant == 6            ? (uint32_t)RS_LANES_B_MAX_THREADS
                          : s->variant == 7            ? k7_max_threads(s)
                                                       : (uint32_t)RS_LANES_MAX_THREADS;
    if (o.threads % 32 || o.threads > tmax || o.threads < (s->variant != 2 ? 32u : s->LT)) {
      rs_free_lanes(s);
      return set_err(RS_E_INVALID_ARG, "threads must be a multiple of 32 in [32, %u] for this kernel", tmax);
    }
    s->threads = o.threads;
  } else if (g->cg.mode == RS_MODE_SINGLE) {
    s->threads = 1024;
  } else {
    const uint32_t per_sm = (s->n_tiles * s->cluster + g->sm_count - 1) / g->sm_count;
    const uint32_t tmax = s->variant == 1   ? (uint32_t)RS_LANES_T_MAX_THREADS
                          : s->variant == 6 ? (uint32_t)RS_LANES_B_MAX_THREADS
                          : s->variant == 7 ? k7_max_threads(s)
                                            : (uint32_t)RS_LANES_MAX_THREADS;
    uint32_t th = tmax / std::max<uint32_t>(1, per_sm);
    th = std::max<uint32_t>(64, th & ~31u);
    s->threads = th;
  }
  // lane mode: every cluster of the launch must be co-resident, else the launch runs in
  // waves; an automatic shape halves its cluster until it fits (fewer CTAs, one wave)
  if (g->cg.mode == RS_MODE_LANES && !o.cluster && s->variant != 8) {
    s->batch_idx = 0;  // not chosen yet; it only picks a kernel-7 variant of the same shared memory
    int fit = co_resident_clusters(s);
    while (fit >= 0 && (uint32_t)fit < s->n_tiles && s->cluster > 1) {
      s->cluster /= 2;
      fit = co_resident_clusters(s);
    }
  }
  if (g->cg.mode == RS_MODE_LANES && s->variant == 7 && s->threads > k7_max_threads(s)) {
    if (o.threads) {
      rs_free_lanes(s);
      return set_err(RS_E_INVALID_ARG, "threads > %u for kernel 7 at this shape", k7_max_threads(s));
    }
    s->threads = k7_max_threads(s);
  }
  if (s->repcut) {
    RepCutPlan plan;
    std::string err;
    if (!build_repcut(g->cg, s->parts, &plan, &err)) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_INVALID_ARG, "%s", err.c_str());
    }
    s->threads = o.threads ? o.threads : 1024;
    s->ctas = s->parts;
    s->sig_part = plan.sig_owner;
    std::vector<uint8_t> blob;
    size_t off = 0, o_lb, o_ops, o_rb, o_regs, o_pb, o_push;
    std::vector<uint8_t> sblob, in_owner;
    std::vector<uint64_t> sl_off, op_k;
    bool fits = false;
    if (o.repcut_global != 1) {  // 8-byte slots if every partition still fits, else width-packed
      fits = o.repcut_global != 2 &&
             build_repcut_slices(g->cg, plan, kRepSmemMax, true, &sblob, &sl_off, &op_k, &in_owner, &err);
      if (fits) s->rep_wide = true;
      else fits = build_repcut_slices(g->cg, plan, kRepSmemMax, false, &sblob, &sl_off, &op_k, &in_owner, &err);
    }
    if (fits) {
      s->rep_smem = true;
      uint32_t max_level = 0;
      for (uint32_t p = 0; p < s->parts; ++p) {
        const RepSliceHdr* h = reinterpret_cast<const RepSliceHdr*>(sblob.data() + sl_off[p]);
        s->rep_smem_bytes = std::max(s->rep_smem_bytes, h->smem_bytes + h->state_bytes);
        max_level = std::max(max_level, h->max_level);
      }
      // one op per thread per level where possible (the hash weights are prefetched for one)
      if (!o.threads) s->threads = std::min<uint32_t>(1024, std::max<uint32_t>(128, (max_level + 31) / 32 * 32));
      s->rep_one = s->threads >= max_level;
      size_t o_bl;
      put(blob, off, sblob, &o_bl);
      size_t o_so, o_k;
      put(blob, off, sl_off, &o_so);
      put(blob, off, op_k, &o_k);
      s->reps.blob = (const uint8_t*)(uintptr_t)o_bl;
      s->reps.slice_off = (const uint64_t*)(uintptr_t)o_so;
      s->reps.op_k = (const uint64_t*)(uintptr_t)o_k;
      // inputs read back from the replica of the partition that injects and hashes them
      for (uint32_t sg = 0; sg < g->cg.n_signals; ++sg)
        if (g->cg.sig_kind[sg] == 0) {
          const uint32_t c = g->cg.sig_coord[sg];
          for (uint32_t k = 0; k < g->cg.n_inputs; ++k)
            if (g->cg.in_coord[k] == c) {
              s->sig_part[sg] = in_owner[k];
              break;
            }
        }
    }
    put(blob, off, plan.lvl_begin, &o_lb);
    put(blob, off, plan.ops, &o_ops);
    put(blob, off, plan.reg_begin, &o_rb);
    put(blob, off, plan.regs, &o_regs);
    put(blob, off, plan.push_begin, &o_pb);
    put(blob, off, plan.push, &o_push);
    size_t o_chg = 0;  // k_repcut's per-register "changed" flags (differential exchange; RTLSIM_REPCUT_DIFFX=0: off)
    const char* dx = std::getenv("RTLSIM_REPCUT_DIFFX");
    const bool diffx = !(dx && dx[0] == '0');
    put(blob, off, std::vector<uint8_t>(diffx ? std::max<uint32_t>(1, g->cg.n_regs) : 0), &o_chg);
    blob.resize(std::max<size_t>(off, 256));
    cudaError_t e2 = cudaMalloc(&s->drep, blob.size());
    if (e2 == cudaSuccess) e2 = cudaMemcpy(s->drep, blob.data(), blob.size(), cudaMemcpyHostToDevice);
    if (e2 != cudaSuccess) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_OOM, "repcut plan: %s", cudaGetErrorString(e2));
    }
    const uint8_t* b = (const uint8_t*)s->drep;
    s->rep.lvl_begin = (const uint32_t*)(b + o_lb);
    s->rep.ops = (const uint32_t*)(b + o_ops);
    s->rep.reg_begin = (const uint32_t*)(b + o_rb);
    s->rep.regs = (const uint32_t*)(b + o_regs);
    s->rep.push_begin = (const uint32_t*)(b + o_pb);
    s->rep.push = (const uint32_t*)(b + o_push);
    s->rep.chg = diffx ? (uint8_t*)s->drep + o_chg : nullptr;
    s->total_bytes += blob.size();
    if (s->rep_smem) {
      s->reps.blob = b + (uintptr_t)s->reps.blob;
      s->reps.slice_off = (const uint64_t*)(b + (uintptr_t)s->reps.slice_off);
      s->reps.op_k = (const uint64_t*)(b + (uintptr_t)s->reps.op_k);
      e2 = cudaMalloc(&s->rep_mail, std::max<size_t>(16, 16ull * g->cg.n_regs));
      if (e2 != cudaSuccess) {
        s->rep_mail = nullptr;
        rs_free_lanes(s);  // partially built: frees what exists (drep included)
        return set_err(RS_E_OOM, "repcut mailbox: %s", cudaGetErrorString(e2));
      }
      s->reps.mail = (uint64_t*)s->rep_mail;
      s->total_bytes += 16ull * g->cg.n_regs;
      const void* fns[] = {(const void*)k_repcut_smem<true, true, true>,   (const void*)k_repcut_smem<true, false, true>,
                           (const void*)k_repcut_smem<false, true, true>,  (const void*)k_repcut_smem<false, false, true>,
                           (const void*)k_repcut_smem<true, true, false>,  (const void*)k_repcut_smem<true, false, false>,
                           (const void*)k_repcut_smem<false, true, false>, (const void*)k_repcut_smem<false, false, false>};
      // the dynamic shared-memory cap is a per-function attribute (process-wide):
      // checked here, and set again before every launch (rs_step_cycles), so a later
      // allocation with smaller slices cannot lower it under this one
      for (const void* f : fns)
        if (e2 == cudaSuccess)
          e2 = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->rep_smem_bytes);
      if (e2 != cudaSuccess) {
        rs_free_lanes(s);  // partially built: frees what exists (drep, rep_mail included)
        return set_err(RS_E_CUDA, "repcut smem attribute: %s", cudaGetErrorString(e2));
      }
    }
  } else if (s->variant == 8) {
    // shape set with the kernel choice
  } else if (g->cg.mode == RS_MODE_SINGLE) {
    const uint32_t work = std::max<uint32_t>(1, std::max(g->cg.n_inputs, g->cg.n_regs));
    uint32_t maxops = 0;
    for (uint32_t l = 0; l < g->cg.n_levels; ++l)
      maxops = std::max(maxops, g->cg.level_op_begin[l + 1] - g->cg.level_op_begin[l]);
    // resident-slice kernel (single.cuh): fewest CTAs whose graph slices fit in shared memory
    const CompiledGraph& cg = g->cg;
    const uint64_t est = 4ull * cg.n_ops_total() + 4ull * cg.coord.size() + 12ull * cg.n_regs + 8ull * cg.n_inputs;
    const uint32_t kMaxSlice = 212 * 1024;  // + static shared memory stays below the 227 KB per-CTA limit
    const uint32_t P = s->parts, maxG = (uint32_t)g->sm_count / (s->part_world ? 1u : P);
    uint32_t G = (uint32_t)std::max<uint64_t>({1, (est + kMaxSlice / 2) / (kMaxSlice * 3 / 4) / P, (maxops + 1023) / 1024});
    G = std::min<uint32_t>(G, maxG);
    std::vector<uint8_t> sblob;
    std::vector<uint64_t> soff;
    bool ok = false;
    while (true) {  // G = CTAs per partition
      ok = build_single_slices(cg, P, G, kMaxSlice, &sblob, &soff);
      if (ok || G >= maxG) break;
      G = std::min<uint32_t>(maxG, G + std::max<uint32_t>(1, G / 4));
    }
    if (!ok && P > 1) {
      rs_free_lanes(s);  // partially built: frees what exists
      return set_err(RS_E_CAPACITY, "level cut: %u partitions' slices do not fit %u co-resident CTAs", P, maxG * P);
    }
    if (ok && !o.threads) {
      const uint32_t chunk = std::max<uint32_t>(1, (maxops + G - 1) / G);
      s->threads = std::min<uint32_t>(1024, 32u * chunk);  // up to one op per warp (single.cuh op slots)
    }
    if (ok && P > 1) {
      std::vector<uint8_t> owner[4];
      row_owner(cg, level_cut(cg, P), owner);
      s->sig_part.assign(cg.n_signals, 0);
      for (uint32_t id = 0; id < cg.n_signals; ++id)
        if (cg.sig_kind[id] == 3) s->sig_part[id] = owner[cg.sig_coord[id] >> 30][cg.sig_coord[id] & ROW_MASK];
    }
    if (ok) {
      s->gp = G;
      G *= P;
      uint32_t smax = 0, hmax = 0;
      for (uint32_t i = 0; i < G; ++i) {
        const SliceHdr* sh = reinterpret_cast<const SliceHdr*>(sblob.data() + soff[i]);
        smax = std::max(smax, sh->bytes);
        hmax = std::max(hmax, sh->head_bytes);
      }
      // tails (latch / push / inject lists) stay in global memory unless every slice fits whole
      s->tail_global = smax > kMaxSlice;
      if (s->tail_global) smax = hmax;
      const size_t off_off = (sblob.size() + 255) & ~(size_t)255;
      cudaError_t e2 = cudaMalloc(&s->dslices, off_off + G * 8);
      if (e2 == cudaSuccess) e2 = cudaMemcpy(s->dslices, sblob.data(), sblob.size(), cudaMemcpyHostToDevice);
      if (e2 == cudaSuccess) e2 = cudaMemcpy((uint8_t*)s->dslices + off_off, soff.data(), G * 8, cudaMemcpyHostToDevice);
      if (e2 != cudaSuccess) {
        rs_free_lanes(s);  // partially built: frees what exists
        return set_err(RS_E_OOM, "single-lane slices: %s", cudaGetErrorString(e2));
      }
      s->slice_blob = (const uint8_t*)s->dslices;
      s->slice_off = (const uint64_t*)((const uint8_t*)s->dslices + off_off);
      s->slice_max = smax;
      s->ctas = s->part_world ? s->gp : G;  // across processes: this rank's partition only
      s->total_bytes += off_off + G * 8;
    } else {  // graph too large for resident slices: descriptors streamed from global memory
      const uint32_t need = std::max(work, maxops);
      uint32_t ctas = (need + s->threads - 1) / s->threads;
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_single<true>, s->threads, 0);
      const uint32_t maxc = (uint32_t)std::max(1, occ) * g->sm_count;
      s->ctas = std::max<uint32_t>(1, std::min(ctas, maxc));
    }
  } else {
    s->ctas = s->n_tiles * s->cluster;
  }
  // state: [n_tiles][class 0 rows x LT | class 1 | class 2 | class 3], regions 128-B aligned
  uint64_t off = 0;
  if (s->variant == 6) {
    // bit-sliced tile: [bit planes: rows_bit x 16 B | u8 rows [rows_bit, rows[0]) | u16 | u32 | u64];
    // region[0] is biased so region[0] + row * LT addresses u8 row `row` (>= rows_bit)
    const uint32_t nb = g->cg.rows_bit;
    s->region_b = 0;
    off = 16ull * nb;
    off = (off + 127) & ~(uint64_t)127;
    s->region[0] = off - (uint64_t)nb * s->LT;
    off += (uint64_t)(g->cg.rows[0] - nb) * s->LT;
    for (int c = 1; c < 4; ++c) {
      off = (off + 127) & ~(uint64_t)127;
      s->region[c] = off;
      off += (uint64_t)g->cg.rows[c] * s->LT * (1u << c);
    }
  } else {
    for (int c = 0; c < 4; ++c) {
      off = (off + 127) & ~(uint64_t)127;
      s->region[c] = off;
      off += (uint64_t)g->cg.rows[c] * s->LT * (1u << c);
    }
  }
  s->tile_bytes = std::max<uint64_t>((off + 127) & ~(uint64_t)127, 128);
  if (g->cg.mode == RS_MODE_LANES && s->tile_bytes >= (s->variant == 6 ? (1ull << 32) : (1ull << 30))) {
    rs_free_lanes(s);  // partially built: frees what exists
    return set_err(RS_E_CAPACITY, "a lane tile needs %llu B of state (limit 2^30); use a smaller lane_tile",
                   (unsigned long long)s->tile_bytes);
  }
  s->state_bytes = (size_t)s->tile_bytes * s->n_tiles;
  cudaError_t e;
  // across processes the cycle flag follows the replica in the same allocation (one IPC handle)
  const size_t flag_bytes = s->part_world ? 256 : 0;
  if (!o.defer_state && (e = cudaMalloc(&s->state_mem, s->state_bytes + flag_bytes)) != cudaSuccess) {
    rs_free_lanes(s);  // partially built: frees what exists
    return set_err(RS_E_OOM, "cudaMalloc state (%zu B): %s", s->state_bytes, cudaGetErrorString(e));
  }
  if (g->cg.mode == RS_MODE_LANES && s->variant != 8) {
    // work items: kernel 1 takes kBatchWide-op items when its CTAs have many ops
    // per level (C4: ~6,700; fewer, longer items cut the per-item decode), else
    // kBatch-op items (more items to deal when a level is short: C3 ~470)
    s->batch_idx = (s->variant != 2 && wide_items(g, s->cluster)) ? 1u : 0u;
    if (!g->stages_built[s->batch_idx]) {
      build_stages(g->cg, g->stage_bytes, s->batch_idx ? kBatchWide : kBatch, &g->stage_blob[s->batch_idx],
                   &g->stage_tab[s->batch_idx]);
      g->stages_built[s->batch_idx] = true;
    }
    if ((st = upload_schedule(s)) != RS_OK) {
      rs_free_lanes(s);
      return st;
    }
  }
  const size_t lanes_pad = (size_t)s->n_tiles * s->LT;
  if ((e = cudaMalloc(&s->hcarry, 2 * lanes_pad * sizeof(uint64_t))) != cudaSuccess ||
      (e = cudaMalloc(&s->bar, kBarBytes)) != cudaSuccess) {
    rs_free_lanes(s);
    return set_err(RS_E_OOM, "cudaMalloc: %s", cudaGetErrorString(e));
  }
  if (o.stage_cycles) {
    const size_t sb = (size_t)o.stage_cycles * std::max<uint32_t>(1, g->cg.n_inputs) * n_lanes * sizeof(uint64_t);
    if ((e = cudaMalloc(&s->stage, sb)) != cudaSuccess) {
      rs_free_lanes(s);
      return set_err(RS_E_OOM, "cudaMalloc stage ring (%zu B): %s", sb, cudaGetErrorString(e));
    }
    s->stage_cap = o.stage_cycles;
  }
  s->total_bytes += (o.defer_state ? 0 : s->state_bytes) + 2 * lanes_pad * 8 + kBarBytes +
                   (size_t)s->stage_cap * std::max<uint32_t>(1, g->cg.n_inputs) * n_lanes * 8;
  if (o.stream) {
    s->stream = (cudaStream_t)o.stream;
  } else {
    if ((e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking)) != cudaSuccess) {
      rs_free_lanes(s);
      return set_err(RS_E_CUDA, "stream: %s", cudaGetErrorString(e));
    }
    s->own_stream = true;
  }
  s->flag_bytes = flag_bytes;
  g->live_lanes++;
  s->counted = true;
  if (o.defer_state) {  // the caller binds its own device buffer (rs_lanes_bind_state)
    *out = s;
    return RS_OK;
  }
  if ((st = init_state(s)) != RS_OK) {
    rs_free_lanes(s);
    return st;
  }
  *out = s;
  return RS_OK;
}

// Initial state: zero, constants, register init, hash carry.
static rs_status init_state(rs_lanes* s) {
  rs_graph* g = s->g;
  const size_t lanes_pad = (size_t)s->n_tiles * s->LT;
  StepArgs a = base_args(s);
  cudaError_t e = cudaMemsetAsync(s->state_mem, 0, s->state_bytes + s->flag_bytes, s->stream);
  std::vector<uint32_t> coords;
  std::vector<uint64_t> vals;
  coords.insert(coords.end(), g->cg.const_coord.begin(), g->cg.const_coord.end());
  vals.insert(vals.end(), g->cg.const_val.begin(), g->cg.const_val.end());
  coords.insert(coords.end(), g->cg.reg_coord.begin(), g->cg.reg_coord.end());
  vals.insert(vals.end(), g->cg.reg_init.begin(), g->cg.reg_init.end());
  if (e == cudaSuccess && !coords.empty()) {
    void* tmp = nullptr;
    const size_t nb = coords.size() * 4, vb = vals.size() * 8;
    e = cudaMalloc(&tmp, nb + vb + 8);
    if (e == cudaSuccess) {
      cudaMemcpyAsync(tmp, coords.data(), nb, cudaMemcpyHostToDevice, s->stream);
      uint64_t* dv = (uint64_t*)((uint8_t*)tmp + ((nb + 7) & ~(size_t)7));
      cudaMemcpyAsync(dv, vals.data(), vb, cudaMemcpyHostToDevice, s->stream);
      k_broadcast<<<std::min<uint64_t>(4096, (coords.size() * lanes_pad + 255) / 256), 256, 0, s->stream>>>(
          a, (uint32_t)lanes_pad, (const uint32_t*)tmp, dv, (uint32_t)coords.size());
      e = cudaStreamSynchronize(s->stream);
      cudaFree(tmp);
      s->launches++;
    }
  }
  if (e == cudaSuccess) {
    // across processes each partition carries its own registers' term: all of it on rank 0 at first
    std::vector<uint64_t> hc(lanes_pad, (s->part_world && s->part_rank != 0) ? 0ull : g->cg.init_reg_hash);
    e = cudaMemcpy(s->hcarry, hc.data(), lanes_pad * 8, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) return set_err(RS_E_CUDA, "state init: %s", cudaGetErrorString(e));
  return RS_OK;
}

uint64_t rs_lanes_state_bytes(const rs_lanes* s) { return s ? (uint64_t)(s->state_bytes + s->flag_bytes) : 0; }

rs_status rs_lanes_bind_state(rs_lanes* s, void* state, uint64_t bytes) {
  if (!s || !state) return set_err(RS_E_INVALID_ARG, "NULL argument");
  if (s->state_mem) return set_err(RS_E_STATE, "the allocation already has its state");
  if (s->part_world) return set_err(RS_E_UNSUPPORTED, "a level cut across processes owns its state (CUDA IPC)");
  if (bytes < s->state_bytes + s->flag_bytes)
    return set_err(RS_E_CAPACITY, "state buffer of %llu B; needs %llu B (rs_lanes_state_bytes)",
                   (unsigned long long)bytes, (unsigned long long)(s->state_bytes + s->flag_bytes));
  if ((uintptr_t)state % 256) return set_err(RS_E_INVALID_ARG, "state buffer must be 256-byte aligned");
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, state) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
      pa.device != s->g->device) {
    (void)cudaGetLastError();
    return set_err(RS_E_INVALID_ARG, "state buffer is not device memory of device %d", s->g->device);
  }
  s->state_mem = state;
  s->state_owned = false;
  return init_state(s);
}

void rs_free_lanes(rs_lanes* s) {
  if (!s) return;
  cudaSetDevice(s->g->device);
  if (s->stream) cudaStreamSynchronize(s->stream);  // no launch may still use a peer mapping
  if (s->connected)
    for (uint32_t k = 0; k < s->part_world; ++k)
      if (k != s->part_rank && s->peer_rep[k]) cudaIpcCloseMemHandle(s->peer_rep[k]);
  if (s->state_mem && s->state_owned) cudaFree(s->state_mem);
  if (s->dstages) cudaFree(s->dstages);
  if (s->dslices) cudaFree(s->dslices);
  if (s->hcarry) cudaFree(s->hcarry);
  if (s->bar) cudaFree(s->bar);
  if (s->stage) cudaFree(s->stage);
  if (s->hbuf) cudaFree(s->hbuf);
  if (s->wave_prev) cudaFree(s->wave_prev);
  if (s->wave_rec) cudaFree(s->wave_rec);
  if (s->wave_count) cudaFree(s->wave_count);
  if (s->drep) cudaFree(s->drep);
  if (s->rep_mail) cudaFree(s->rep_mail);
  if (s->dwatch) cudaFree(s->dwatch);
  if (s->cstream) {
    cudaStreamSynchronize(s->cstream);
    cudaStreamDestroy(s->cstream);
  }
  for (auto& r : s->lrec)
    if (r.ev) cudaEventDestroy(r.ev);
  for (auto& r : s->crec)
    if (r.ev) cudaEventDestroy(r.ev);
  if (s->ev_order) cudaEventDestroy(s->ev_order);
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  if (s->g && s->counted) s->g->live_lanes--;
  delete s;
}

uint64_t rs_lanes_bytes(const rs_lanes* s) { return s ? s->total_bytes : 0; }

rs_status rs_set_input_seed(rs_lanes* s, uint64_t seed) {
  if (!s) return set_err(RS_E_INVALID_ARG, "NULL lanes");
  s->seed = seed;
  s->staged = 0;
  return RS_OK;
}

rs_status rs_set_inputs(rs_lanes* s, uint64_t first_cycle, uint32_t n_cycles, const uint64_t* values, int on_device) {
  NvtxRange nvtx_range("rs_set_inputs");
  if (!s) return set_err(RS_E_INVALID_ARG, "NULL lanes");
  if (!s->stage_cap) return set_err(RS_E_STATE, "no staged-input ring (rs_lane_opts.stage_cycles = 0)");
  if (n_cycles > s->stage_cap) return set_err(RS_E_RANGE, "n_cycles %u > stage_cycles %u", n_cycles, s->stage_cap);
  if (n_cycles && !values) return set_err(RS_E_INVALID_ARG, "NULL values");
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  const uint32_t NI = s->g->cg.n_inputs;
  const size_t per = (size_t)NI * s->n_lanes;
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (!s->cstream) CU(cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking));
  if (n_cycles && per) {
    // the ring slots of cycles [first_cycle, +n_cycles) may still be read by a
    // recorded launch: wait for the latest launch whose cycles share a slot
    // (launches run in order on the lanes' stream); launches evicted from the
    // record ring are older than its oldest entry, which then stands for them
    const uint64_t cap = s->stage_cap;
    auto shares_slot = [&](uint64_t a0, uint64_t la, uint64_t b0, uint64_t lb) {
      if (!la || !lb) return false;
      if (la >= cap || lb >= cap) return true;
      a0 %= cap;
      b0 %= cap;
      return (b0 + cap - a0) % cap < la || (a0 + cap - b0) % cap < lb;
    };
    const uint64_t kept = std::min<uint64_t>(s->lrec_n, 4);
    cudaEvent_t wait = nullptr;
    for (uint64_t j = 0; j < kept && !wait; ++j) {  // newest first
      const auto& r = s->lrec[(s->lrec_n - 1 - j) % 4];
      if (shares_slot(r.c0, r.c1 - r.c0, first_cycle, n_cycles)) wait = r.ev;
    }
    if (!wait && s->lrec_n > 4) wait = s->lrec[(s->lrec_n - kept) % 4].ev;
    if (wait) CU(cudaStreamWaitEvent(s->cstream, wait, 0));
    if (on_device) {
      // device values may be produced by work queued on the lanes' stream
      // (the caller's): the copy follows everything queued there so far
      if (!s->ev_order) CU(cudaEventCreateWithFlags(&s->ev_order, cudaEventDisableTiming));
      CU(cudaEventRecord(s->ev_order, s->stream));
      CU(cudaStreamWaitEvent(s->cstream, s->ev_order, 0));
    }
  }
  uint32_t done = 0;
  while (done < n_cycles && per) {
    const uint64_t c = first_cycle + done;
    const uint32_t slot = (uint32_t)(c % s->stage_cap);
    const uint32_t n = std::min<uint32_t>(n_cycles - done, s->stage_cap - slot);
    CU(cudaMemcpyAsync(s->stage + (size_t)slot * per, values + (size_t)done * per, (size_t)n * per * 8, kind,
                       s->cstream));
    done += n;
  }
  if (n_cycles && per) {
    auto& r = s->crec[s->crec_n % 4];
    if (s->crec_n >= 4 && s->crec_waited < s->crec_n - 3) {
      // the record about to be reused was never waited for: order it now
      CU(cudaStreamWaitEvent(s->stream, r.ev, 0));
      s->crec_waited = s->crec_n - 3;
    }
    if (!r.ev) CU(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming));
    r.c0 = first_cycle;
    r.c1 = first_cycle + n_cycles;
    CU(cudaEventRecord(r.ev, s->cstream));
    s->crec_n++;
  }
  // staged window
  if (s->staged && first_cycle <= s->st_hi && first_cycle >= s->st_lo) {
    s->st_hi = std::max<uint64_t>(s->st_hi, first_cycle + n_cycles);
  } else {
    s->st_lo = first_cycle;
    s->st_hi = first_cycle + n_cycles;
  }
  if (s->st_hi - s->st_lo > s->stage_cap) s->st_lo = s->st_hi - s->stage_cap;
  s->staged = 1;
  return RS_OK;
}

static rs_status refresh_hcarry(rs_lanes* s) {
  if (s->hc_valid) return RS_OK;
  if (s->part_world)
    return set_err(RS_E_UNSUPPORTED, "level cut across processes: a hashed step after a hash-off step");
  StepArgs a = base_args(s);
  k_reg_hash<<<std::max<uint32_t>(1, (s->n_lanes + 127) / 128), 128, 0, s->stream>>>(
      a, s->n_lanes, s->hcarry + s->hc_cur * (size_t)s->n_tiles * s->LT);
  s->launches++;
  CU(cudaGetLastError());
  s->hc_valid = true;
  return RS_OK;
}

rs_status rs_step_cycles(rs_lanes* s, uint32_t n_cycles, uint64_t* hashes, int hashes_mem) {
  NvtxRange nvtx_range("rs_step_cycles");
  if (!s) return set_err(RS_E_INVALID_ARG, "NULL lanes");
  if (!s->state_mem) return set_err(RS_E_STATE, "no state bound (rs_lanes_bind_state)");
  if (hashes_mem != RS_MEM_NONE && hashes_mem != RS_MEM_HOST && hashes_mem != RS_MEM_DEVICE)
    return set_err(RS_E_INVALID_ARG, "bad hashes_mem %d", hashes_mem);
  if (hashes_mem != RS_MEM_NONE && !hashes && n_cycles) return set_err(RS_E_INVALID_ARG, "NULL hashes");
  if (n_cycles == 0) return RS_OK;
  if (s->g->cg.mode == RS_MODE_LANES && (uint64_t)n_cycles * s->n_stages >= (1ull << 31)) {
    // the kernel counts stages in 32 bits: split very long runs
    const uint32_t chunk = (uint32_t)((1ull << 31) / s->n_stages) - 1;
    for (uint32_t done = 0; done < n_cycles;) {
      const uint32_t n = std::min(chunk, n_cycles - done);
      rs_status st = rs_step_cycles(s, n, hashes ? hashes + (size_t)done * s->n_lanes : nullptr, hashes_mem);
      if (st != RS_OK) return st;
      done += n;
    }
    return RS_OK;
  }
  if (s->staged && (s->cycle < s->st_lo || s->cycle + n_cycles > s->st_hi))
    return set_err(RS_E_STATE, "cycles [%llu, %llu) are not staged (window [%llu, %llu))",
                   (unsigned long long)s->cycle, (unsigned long long)(s->cycle + n_cycles),
                   (unsigned long long)s->st_lo, (unsigned long long)s->st_hi);
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  const bool hash = hashes_mem != RS_MEM_NONE;
  if (hash && (st = refresh_hcarry(s)) != RS_OK) return st;
  uint64_t* hout = nullptr;
  const size_t hn = (size_t)n_cycles * s->n_lanes;
  if (hashes_mem == RS_MEM_DEVICE) {
    hout = hashes;
  } else if (hashes_mem == RS_MEM_HOST) {
    if (s->hbuf_cap < hn) {
      if (s->hbuf) cudaFree(s->hbuf);
      s->hbuf = nullptr;
      s->hbuf_cap = 0;
      CU(cudaMalloc(&s->hbuf, hn * 8));
      s->hbuf_cap = hn;
    }
    hout = s->hbuf;
  }
  (void)cudaGetLastError();  // clear a stale non-sticky error of an unrelated earlier call
  if (s->staged && s->crec_waited < s->crec_n) {
    // the newest copy that wrote any of this launch's cycles must come first
    // (copies run in order on the copy stream, so it stands for older ones);
    // copies of later cycles (the next chunk) keep running beside the launch
    const uint64_t c0 = s->cycle, c1 = s->cycle + n_cycles;
    for (uint64_t j = s->crec_n; j > s->crec_waited; --j) {
      const auto& r = s->crec[(j - 1) % 4];
      if (r.c0 < c1 && c0 < r.c1) {
        CU(cudaStreamWaitEvent(s->stream, r.ev, 0));
        s->crec_waited = j;
        break;
      }
    }
  }
  StepArgs a = base_args(s);
  a.cycle0 = s->cycle;
  a.n_cycles = n_cycles;
  a.hashes = hout;
  const size_t lanes_pad = (size_t)s->n_tiles * s->LT;
  a.hcarry_in = s->hcarry + s->hc_cur * lanes_pad;
  if (s->variant == 8) {  // the design's specialised kernel (codegen.hpp)
    SuArgs u{};
    u.state = a.state;
    u.tile_bytes = a.tile_bytes;
    for (int c = 0; c < 4; ++c) u.region[c] = a.region[c];
    u.LT = s->LT;
    u.n_lanes = s->n_lanes;
    u.lane0 = s->lane0;
    u.cycle0 = a.cycle0;
    u.n_cycles = n_cycles;
    u.staged = a.staged ? 1u : 0u;
    u.seed = a.seed;
    u.stage = a.stage;
    u.stage_cap = a.stage_cap;
    u.hashes = hout;
    u.hcarry = a.hcarry_in;
    void* args[] = {&u};
    cudaError_t e = cudaLaunchKernel((const void*)s->g->su_fn, dim3(s->ctas), dim3(s->threads), args, 0, s->stream);
    if (e != cudaSuccess) return set_err(RS_E_CUDA, "kernel 8 launch: %s", cudaGetErrorString(e));
  } else if (s->g->cg.mode == RS_MODE_SINGLE) {
    a.hcarry_out = s->hcarry + (1 - s->hc_cur) * lanes_pad;
    if (hash) {
      CU(cudaMemsetAsync(a.hcarry_out, 0, 8, s->stream));
      if (hout) CU(cudaMemsetAsync(hout, 0, hn * 8, s->stream));
    }
    // grid-barrier counters only: level-cut cycle flags hold absolute cycles and persist
    CU(cudaMemsetAsync(s->bar, 0, kFlagOffset * 8, s->stream));
    if (s->part_world && !s->connected) return set_err(RS_E_STATE, "level cut across processes: rs_ipc_connect first");
    cudaError_t e;
    if (s->repcut && s->rep_smem) {
      RepSmemArgs ra = s->reps;
      ra.a = a;
      void* args[] = {&ra};
      const void* fns[] = {(const void*)k_repcut_smem<true, true, true>,   (const void*)k_repcut_smem<true, false, true>,
                           (const void*)k_repcut_smem<false, true, true>,  (const void*)k_repcut_smem<false, false, true>,
                           (const void*)k_repcut_smem<true, true, false>,  (const void*)k_repcut_smem<true, false, false>,
                           (const void*)k_repcut_smem<false, true, false>, (const void*)k_repcut_smem<false, false, false>};
      const void* fn = fns[(s->rep_wide ? 0 : 4) + (hash ? 0 : 2) + (s->rep_one ? 0 : 1)];
      CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->rep_smem_bytes));
      e = cudaLaunchCooperativeKernel(fn, s->ctas, s->threads, args, s->rep_smem_bytes, s->stream);
    } else if (s->repcut) {
      RepArgs ra = s->rep;
      ra.a = a;
      void* args[] = {&ra};
      e = cudaLaunchCooperativeKernel(hash ? (const void*)k_repcut<true> : (const void*)k_repcut<false>, s->ctas,
                                      s->threads, args, 0, s->stream);
    } else if (s->slice_blob) {
      const bool grid = s->ctas > 1;
      const uint32_t smax = (s->slice_max + 127u) & ~127u;
      const uint32_t st_smem =
          (!grid && smax + s->tile_bytes <= 200u * 1024u) ? (uint32_t)s->tile_bytes : 0u;
      SingleArgs sa{};
      sa.a = a;
      sa.slice_blob = s->slice_blob;
      sa.slice_off = s->slice_off;
      sa.slice_max = smax;
      sa.state_smem = s->parts > 1 ? 0u : st_smem;
      sa.parts = s->parts;
      sa.tail_global = s->tail_global ? 1u : 0u;
      sa.gp = s->gp;
      if (s->part_world) {  // this rank's partition; the others through peer-mapped memory
        sa.part_base = s->part_rank * s->gp;
        sa.sys = 1;
        for (uint32_t k = 0; k < s->parts; ++k) {
          sa.rep[k] = s->peer_rep[k];
          sa.flag[k] = s->peer_flag[k];
        }
      } else {
        for (uint32_t k = 0; k < s->parts; ++k) {
          sa.rep[k] = (uint8_t*)s->state_mem + (size_t)k * s->tile_bytes;
          sa.flag[k] = s->bar + kFlagOffset + k;
        }
      }
      void* args[] = {&sa};
      const void* fn = grid ? (hash ? (const void*)k_single2<true, true> : (const void*)k_single2<true, false>)
                            : (hash ? (const void*)k_single2<false, true> : (const void*)k_single2<false, false>);
      CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smax + st_smem)));
      e = cudaLaunchCooperativeKernel(fn, s->ctas, s->threads, args, smax + st_smem, s->stream);
    } else {
      void* args[] = {&a};
      e = hash ? cudaLaunchCooperativeKernel((const void*)k_single<true>, s->ctas, s->threads, args, 0, s->stream)
               : cudaLaunchCooperativeKernel((const void*)k_single<false>, s->ctas, s->threads, args, 0, s->stream);
    }
    if (e != cudaSuccess) return set_err(RS_E_CUDA, "k_single launch: %s", cudaGetErrorString(e));
    if (hash) s->hc_cur = 1 - s->hc_cur;
  } else {
    a.hcarry_out = a.hcarry_in;
    const size_t smem = lane_smem_bytes(s);
    const void* fn = lane_kernel_fn(s, hash);
    CU(raise_smem_attr(s->g->device, smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(s->n_tiles * s->cluster);
    cfg.blockDim = dim3(s->threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = s->cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (s->l2_policy && s->l2_persist_max) {  // L2-residency policy: one access-policy window per launch
      cudaAccessPolicyWindow& w = attr[1].val.accessPolicyWindow;
      attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
      const size_t bytes = s->l2_policy == 1 ? s->sched_bytes : s->state_bytes;
      w.base_ptr = s->l2_policy == 1 ? s->dstages : s->state_mem;
      w.num_bytes = std::min(bytes, s->l2_persist_max);
      w.hitRatio = s->l2_policy == 1 ? 1.0f : (float)std::min(1.0, (double)s->l2_persist_max / (double)std::max<size_t>(1, bytes));
      w.hitProp = cudaAccessPropertyPersisting;
      w.missProp = cudaAccessPropertyStreaming;
      cfg.numAttrs = 2;
    }
    void* args[] = {&a};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return set_err(RS_E_CUDA, "k_lanes launch: %s", cudaGetErrorString(e));
  }
  s->launches++;
  if (s->staged) {  // which cycles (ring slots) this launch reads, for later rs_set_inputs
    auto& r = s->lrec[s->lrec_n % 4];
    if (!r.ev) CU(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming));
    r.c0 = s->cycle;
    r.c1 = s->cycle + n_cycles;
    CU(cudaEventRecord(r.ev, s->stream));
    s->lrec_n++;
  }
  if (!hash) s->hc_valid = false;
  s->cycle += n_cycles;
  if (hashes_mem == RS_MEM_HOST) {
    CU(cudaMemcpyAsync(hashes, hout, hn * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
  }
  return RS_OK;
}

rs_status rs_read_signals(rs_lanes* s, const uint32_t* ids, uint32_t n_ids, uint32_t lane_begin, uint32_t n_lanes,
                          uint64_t* out) {
  NvtxRange nvtx_range("rs_read_signals");
  if (!s || (n_ids && (!ids || !out))) return set_err(RS_E_INVALID_ARG, "NULL argument");
  if (!s->state_mem) return set_err(RS_E_STATE, "no state bound (rs_lanes_bind_state)");
  if ((uint64_t)lane_begin + n_lanes > s->n_lanes) return set_err(RS_E_RANGE, "lanes [%u, %u) out of range (%u lanes)", lane_begin, lane_begin + n_lanes, s->n_lanes);
  if (n_ids == 0 || n_lanes == 0) return RS_OK;
  std::vector<uint32_t> coords(n_ids);
  for (uint32_t i = 0; i < n_ids; ++i) {
    if (ids[i] >= s->g->cg.n_signals) return set_err(RS_E_RANGE, "signal id %u out of range", ids[i]);
    coords[i] = s->g->cg.sig_coord[ids[i]];
  }
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  // level cut: read every replica (the aux kernels see replica k as lane k), keep the producer's
  const uint32_t P = s->parts;
  const uint32_t rb = P > 1 ? 0 : lane_begin, rn = P > 1 ? P : n_lanes;
  const size_t n = (size_t)n_ids * rn;
  void* tmp = nullptr;
  CU(cudaMalloc(&tmp, n * 8 + n_ids * 4 + 8));
  uint64_t* dout = (uint64_t*)tmp;
  uint32_t* dco = (uint32_t*)(dout + n);
  std::vector<uint64_t> all(P > 1 ? n : 0);
  const char* what = "ids H2D";
  cudaError_t e = cudaMemcpyAsync(dco, coords.data(), n_ids * 4, cudaMemcpyHostToDevice, s->stream);
  if (e == cudaSuccess) {
    StepArgs a = base_args(s);
    what = "k_read launch";
    k_read<<<(unsigned)std::min<size_t>(8192, (n + 255) / 256), 256, 0, s->stream>>>(a, dco, n_ids, rb, rn, dout);
    s->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    what = "D2H";
    e = cudaMemcpyAsync(P > 1 ? all.data() : out, dout, n * 8, cudaMemcpyDeviceToHost, s->stream);
  }
  if (e == cudaSuccess) {
    what = "sync";
    e = cudaStreamSynchronize(s->stream);
  }
  cudaFree(tmp);
  if (e != cudaSuccess) return set_err(RS_E_CUDA, "read_signals (%s): %s", what, cudaGetErrorString(e));
  if (P > 1)
    for (uint32_t i = 0; i < n_ids; ++i) out[i] = all[(size_t)i * P + s->sig_part[ids[i]]];
  return RS_OK;
}

rs_status rs_write_registers(rs_lanes* s, const uint32_t* reg_ids, uint32_t n, uint32_t lane_begin, uint32_t n_lanes,
                             const uint64_t* values) {
  if (!s || (n && (!reg_ids || !values))) return set_err(RS_E_INVALID_ARG, "NULL argument");
  if ((uint64_t)lane_begin + n_lanes > s->n_lanes) return set_err(RS_E_RANGE, "lanes out of range");
  if (n == 0 || n_lanes == 0) return RS_OK;
  std::vector<uint32_t> cw(2 * (size_t)n);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t id = reg_ids[i];
    if (id >= s->g->cg.n_signals || s->g->cg.sig_kind[id] != 1 || s->g->cg.sig_rep[id] != id)
      return set_err(RS_E_RANGE, "signal %u is not a register", id);
    cw[i] = s->g->cg.sig_coord[id];
    cw[n + i] = s->g->cg.reg_w[s->g->cg.sig_reg_index[id]];
  }
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  // level cut: every replica holds every register
  const uint32_t P = s->parts;
  const uint32_t wb = P > 1 ? 0 : lane_begin, wn = P > 1 ? P : n_lanes;
  std::vector<uint64_t> rv;
  if (P > 1) {
    rv.resize((size_t)n * P);
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t k = 0; k < P; ++k) rv[(size_t)i * P + k] = values[i];
    values = rv.data();
  }
  const size_t nv = (size_t)n * wn;
  void* tmp = nullptr;
  CU(cudaMalloc(&tmp, nv * 8 + cw.size() * 4 + 8));
  uint64_t* dv = (uint64_t*)tmp;
  uint32_t* dc = (uint32_t*)(dv + nv);
  cudaError_t e = cudaMemcpyAsync(dv, values, nv * 8, cudaMemcpyHostToDevice, s->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dc, cw.data(), cw.size() * 4, cudaMemcpyHostToDevice, s->stream);
  if (e == cudaSuccess) {
    StepArgs a = base_args(s);
    k_write<<<(unsigned)std::min<size_t>(8192, (nv + 255) / 256), 256, 0, s->stream>>>(a, dc, dc + n, n, wb, wn, dv);
    s->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  cudaFree(tmp);
  if (e != cudaSuccess) return set_err(RS_E_CUDA, "write_registers: %s", cudaGetErrorString(e));
  s->hc_valid = false;
  return refresh_hcarry(s);
}

rs_status rs_get_cycle(const rs_lanes* s, uint64_t* cycle) {
  if (!s || !cycle) return set_err(RS_E_INVALID_ARG, "NULL argument");
  *cycle = s->cycle;
  return RS_OK;
}

rs_status rs_set_cycle(rs_lanes* s, uint64_t cycle) {
  if (!s) return set_err(RS_E_INVALID_ARG, "NULL lanes");
  if (s->parts > 1 && cycle != s->cycle) {
    // level-cut flags hold absolute cycles ("partition k finished cycle c - 1" = c):
    // restart them as if every partition had just finished cycle - 1
    rs_status st = set_device(s->g);
    if (st != RS_OK) return st;
    const std::vector<unsigned long long> f(kMaxParts, (unsigned long long)cycle);
    CU(cudaStreamSynchronize(s->stream));
    if (s->part_world)
      CU(cudaMemcpy((uint8_t*)s->state_mem + s->state_bytes, f.data(), 8, cudaMemcpyHostToDevice));
    else
      CU(cudaMemcpy(s->bar + kFlagOffset, f.data(), 8 * kMaxParts, cudaMemcpyHostToDevice));
  }
  s->cycle = cycle;
  return RS_OK;
}

rs_status rs_ipc_handle(rs_lanes* s, void* handle) {
  if (!s || !handle) return set_err(RS_E_INVALID_ARG, "NULL argument");
  if (!s->part_world) return set_err(RS_E_STATE, "not a level-cut-across-processes allocation (part_world)");
  static_assert(sizeof(cudaIpcMemHandle_t) <= RS_IPC_HANDLE_BYTES, "IPC handle size");
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, s->state_mem));
  std::memset(handle, 0, RS_IPC_HANDLE_BYTES);
  std::memcpy(handle, &h, sizeof h);
  return RS_OK;
}

rs_status rs_ipc_connect(rs_lanes* s, const void* handles) {
  if (!s || !handles) return set_err(RS_E_INVALID_ARG, "NULL argument");
  if (!s->part_world) return set_err(RS_E_STATE, "not a level-cut-across-processes allocation (part_world)");
  if (s->connected) return set_err(RS_E_STATE, "already connected");
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  for (uint32_t k = 0; k < s->part_world; ++k) {
    if (k == s->part_rank) {
      s->peer_rep[k] = (uint8_t*)s->state_mem;
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, (const uint8_t*)handles + (size_t)k * RS_IPC_HANDLE_BYTES, sizeof h);
      void* p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (uint32_t m = 0; m < k; ++m)
          if (m != s->part_rank && s->peer_rep[m]) cudaIpcCloseMemHandle(s->peer_rep[m]);
        return set_err(RS_E_CUDA, "cudaIpcOpenMemHandle(rank %u): %s", k, cudaGetErrorString(e));
      }
      s->peer_rep[k] = (uint8_t*)p;
    }
    // every replica has the same layout: the flag follows tile_bytes of state
    s->peer_flag[k] = reinterpret_cast<unsigned long long*>(s->peer_rep[k] + s->state_bytes);
  }
  s->connected = true;
  return RS_OK;
}

uint64_t rs_launch_count(const rs_lanes* s) { return s ? s->launches : 0; }

rs_status rs_debug_trace(rs_lanes* s, uint64_t* out, uint64_t n) {
#ifdef RS_TRACE
  if (!s || !out) return set_err(RS_E_INVALID_ARG, "NULL argument");
  const uint64_t cap = 4096ull * (3 + 1024 / 32) + 4096ull * 16;  // stage stamps + extra stamps
  if (!s->trace) {
    CU(cudaMalloc(&s->trace, cap * 8));
    CU(cudaMemset(s->trace, 0, cap * 8));
    return RS_OK;  // first call arms the buffer; step, then call again to read
  }
  CU(cudaStreamSynchronize(s->stream));
  CU(cudaMemcpy(out, s->trace, std::min(n, cap) * 8, cudaMemcpyDeviceToHost));
  return RS_OK;
#else
  (void)s; (void)out; (void)n;
  return set_err(RS_E_UNSUPPORTED, "built without RS_TRACE");
#endif
}

rs_status rs_watch(rs_lanes* s, const uint32_t* ids, uint32_t n_ids, uint64_t capacity) {
  if (!s || (n_ids && !ids)) return set_err(RS_E_INVALID_ARG, "NULL argument");
  const bool single = s->g->cg.mode == RS_MODE_SINGLE;
  if (s->variant == 8) return set_err(RS_E_UNSUPPORTED, "waveform capture is not built into kernel 8 (specialised)");
  if (single && (s->parts > 1 && !s->repcut))
    return set_err(RS_E_UNSUPPORTED, "waveform capture with a level cut (parts > 1) is not supported");
  if (single && s->repcut && !s->rep_smem)
    return set_err(RS_E_UNSUPPORTED, "waveform capture needs the shared-memory RepCut kernel (not repcut_global)");
  if (n_ids > 8192u) return set_err(RS_E_INVALID_ARG, "at most 8192 watched signals (got %u)", n_ids);
  if (n_ids && capacity == 0) return set_err(RS_E_INVALID_ARG, "capacity must be >= 1");
  for (uint32_t i = 0; i < n_ids; ++i)
    if (ids[i] >= s->g->cg.n_signals) return set_err(RS_E_RANGE, "signal id %u out of range", ids[i]);
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  CU(cudaStreamSynchronize(s->stream));
  if (s->wave_prev) cudaFree(s->wave_prev);
  if (s->wave_rec) cudaFree(s->wave_rec);
  if (s->wave_count) cudaFree(s->wave_count);
  s->wave_prev = nullptr;
  s->wave_rec = nullptr;
  s->wave_count = nullptr;
  s->wave_cap = 0;
  s->watch.assign(ids, ids + n_ids);
  if (n_ids) {
    const size_t lanes_pad = (size_t)s->n_tiles * s->LT;
    CU(cudaMalloc(&s->wave_prev, (size_t)n_ids * lanes_pad * 8));
    CU(cudaMalloc(&s->wave_rec, capacity * 32));
    CU(cudaMalloc(&s->wave_count, 8));
    // on the lanes' stream (non-blocking: a legacy-stream memset would not be ordered with the steps)
    CU(cudaMemsetAsync(s->wave_count, 0, 8, s->stream));
    s->wave_cap = capacity;
    s->wave_first = s->cycle;
  }
  if (!single) return upload_schedule(s);
  // single lane: k_single2 reads the watched signals' coordinates; a RepCut
  // partition reads its own watched signals (those whose value its replica
  // holds, sig_part) from its local state: their local offsets come from the
  // partition's (local, coord) map, sorted by coord, in the device slice blob
  if (s->dwatch) cudaFree(s->dwatch);
  s->dwatch = nullptr;
  s->watch_ent = s->watch_begin = nullptr;
  if (!n_ids) return RS_OK;
  std::vector<uint32_t> ent, begin;
  if (!s->repcut) {
    for (uint32_t i = 0; i < n_ids; ++i) ent.push_back(s->g->cg.sig_coord[ids[i]]);
  } else {
    const uint32_t P = s->parts;
    std::vector<uint64_t> soff(P);
    CU(cudaMemcpy(soff.data(), s->reps.slice_off, P * 8, cudaMemcpyDeviceToHost));
    begin.assign(P + 1, 0);
    for (uint32_t p = 0; p < P; ++p) {
      begin[p] = (uint32_t)(ent.size() / 2);
      RepSliceHdr h;
      CU(cudaMemcpy(&h, s->reps.blob + soff[p], sizeof h, cudaMemcpyDeviceToHost));
      std::vector<uint32_t> map(2ull * h.n_map);
      if (h.n_map) CU(cudaMemcpy(map.data(), s->reps.blob + soff[p] + h.off_map, map.size() * 4, cudaMemcpyDeviceToHost));
      for (uint32_t j = 0; j < n_ids; ++j) {
        const uint32_t sig = ids[j];
        if ((s->sig_part.empty() ? 0u : s->sig_part[sig]) != p) continue;
        const uint32_t c = s->g->cg.sig_coord[sig];
        uint32_t lo = 0, hi = h.n_map;  // first map entry with coord >= c
        while (lo < hi) {
          const uint32_t mid = (lo + hi) / 2;
          if (map[2 * mid + 1] < c) lo = mid + 1; else hi = mid;
        }
        if (lo == h.n_map || map[2 * lo + 1] != c)
          return set_err(RS_E_STATE, "signal %u is not in its partition's local state", sig);
        ent.push_back(map[2 * lo]);
        ent.push_back(j);
      }
    }
    begin[P] = (uint32_t)(ent.size() / 2);
  }
  const size_t eb = ent.size() * 4, off_b = (eb + 255) & ~(size_t)255;
  CU(cudaMalloc(&s->dwatch, off_b + std::max<size_t>(4, begin.size() * 4)));
  if (eb) CU(cudaMemcpy(s->dwatch, ent.data(), eb, cudaMemcpyHostToDevice));
  if (!begin.empty()) CU(cudaMemcpy((uint8_t*)s->dwatch + off_b, begin.data(), begin.size() * 4, cudaMemcpyHostToDevice));
  s->watch_ent = (const uint32_t*)s->dwatch;
  s->watch_begin = begin.empty() ? nullptr : (const uint32_t*)((uint8_t*)s->dwatch + off_b);
  return RS_OK;
}

rs_status rs_wave_read(rs_lanes* s, rs_change* out, uint64_t cap, uint64_t* n_out, uint64_t* dropped) {
  if (!s || (cap && !out)) return set_err(RS_E_INVALID_ARG, "NULL argument");
  if (n_out) *n_out = 0;
  if (dropped) *dropped = 0;
  if (!s->wave_count) return RS_OK;
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  unsigned long long cnt = 0;
  CU(cudaMemcpyAsync(&cnt, s->wave_count, 8, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  const uint64_t have = std::min<uint64_t>(cnt, s->wave_cap), n = std::min<uint64_t>(have, cap);
  if (n) CU(cudaMemcpyAsync(out, s->wave_rec, n * 32, cudaMemcpyDeviceToHost, s->stream));
  // reset on the lanes' stream, ordered before the next step's records
  CU(cudaMemsetAsync(s->wave_count, 0, 8, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  if (n_out) *n_out = n;
  if (dropped) *dropped = cnt - n;
  return RS_OK;
}

uint32_t rs_lanes_kernel(const rs_lanes* s) {
  if (!s) return 0u;
  if (s->g->cg.mode == RS_MODE_LANES || s->variant == 8) return s->variant;
  return s->repcut ? (s->rep_smem ? 3u : 4u) : 5u;
}

rs_status rs_launch_shape(const rs_lanes* s, uint32_t* lt, uint32_t* threads, uint32_t* ctas, uint32_t* cluster) {
  if (s && cluster) *cluster = s->cluster;
  if (!s) return set_err(RS_E_INVALID_ARG, "NULL lanes");
  if (lt) *lt = s->LT;
  if (threads) *threads = s->threads;
  if (ctas) *ctas = s->ctas;
  return RS_OK;
}

rs_status rs_sync(rs_lanes* s) {
  if (!s) return set_err(RS_E_INVALID_ARG, "NULL lanes");
  rs_status st = set_device(s->g);
  if (st != RS_OK) return st;
  if (s->cstream) CU(cudaStreamSynchronize(s->cstream));
  CU(cudaStreamSynchronize(s->stream));
  return RS_OK;
}

}  // extern "C"
