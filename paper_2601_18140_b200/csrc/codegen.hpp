// codegen.hpp -- per-design specialised step kernel (rs_lane_opts.kernel = 8; SURVEY.md
// §8(f) NEXT-4, the GPU analog of the paper's SU mode: "S fully unrolled; OIM embedded in
// the binary", §5.2, Tables 4-6).
//
// The compiled graph (after the optional passes) is emitted as PTX: one thread per lane
// runs the whole cycle as straight-line code -- every op a few register instructions with
// its operand signals, widths, parameters and hash weight baked in as immediates, the
// design's registers held in registers across cycles, signals of <= 32 bits in 32-bit
// registers.  The driver JIT-compiles it (cudaLibraryLoadData) at rs_specialize /
// rs_alloc_lanes time -- no NVVM pass over a huge straight-line function (which takes
// minutes at a few thousand ops), ptxas only.  There is no op tensor left to read: the
// trade is instruction-cache footprint for data traffic (the paper's SU vs TI / NU trade),
// which pays for small designs (C1) and is capped at kSuMaxOps ops.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "compiler.hpp"

namespace rtlsim {

// Kernel parameter of the generated kernel `rs_su` (one struct by value; all fields
// 8 bytes, offsets fixed: the PTX reads them at 8 * field index).
struct SuArgs {
  uint8_t* state;          // [n_tiles][tile_bytes], the allocation's state layout
  uint64_t tile_bytes;
  uint64_t region[4];      // byte offset of class c's rows inside a tile
  uint64_t LT;             // lanes per tile (1 in single-lane mode)
  uint64_t n_lanes;
  uint64_t lane0;          // global id of lane 0 (stimulus)
  uint64_t cycle0;         // absolute cycle of the first stepped cycle
  uint64_t n_cycles;
  uint64_t staged;         // 0: seeded stimulus, 1: staged ring
  uint64_t seed;
  const uint64_t* stage;   // [stage_cap][n_inputs][n_lanes]
  uint64_t stage_cap;
  uint64_t* hashes;        // [n_cycles][n_lanes] or null
  uint64_t* hcarry;        // per-lane register term of the hash after the last cycle
};
static_assert(sizeof(SuArgs) == 17 * 8, "SuArgs: 17 eight-byte fields");

constexpr uint32_t kSuMaxOps = 4096;  // ptxas time: C1 256 ops 0.4 s, C2 20k ops 25 min

// PTX of the specialised kernel for `cg` (.entry rs_su(SuArgs)), for sm_100a; *threads =
// the CTA size it is written for (single lane: 32 per warp of the multi-warp split; lanes: 128).
std::string su_ptx(const CompiledGraph& cg, uint32_t* threads);

}  // namespace rtlsim
