// Certified brute-force nearest-neighbour search (the hot loop of
// optimize_grasp: match_surface_to_pool grasp.cpp:92-106 /
// collision_loss_and_gradients grasp.cpp:68-84 / final ranking
// grasp.cpp:263-281, replacing the kd-tree of spatial_index.cpp:14-105).
//
// FP32 filter, FP64 decision (nn.cu):
//   * forward / final: CTA work items (particle, <= 1024 queries, candidate
//     split); the split is staged whole into shared memory by TMA bulk copies
//     and read with broadcast LDS.128; the number of splits adapts on the
//     device to the number of particles that match in the iteration;
//   * reverse: warp work items (particle, <= 32 colliding points) against the
//     particle's contact surface read through L1;
//   * a (query, candidate) pair is 3 FFMA in the expansion form
//     d = |b|^2 - 2 a.b plus a min; each query keeps a running top-3 of
//     32-candidate subtile minima;
//   * the reference's answer (min FP64 (p - q).squaredNorm(), ties -> lowest
//     position, spatial_index.cpp:70,83) provably lies in {d <= b1 + margin};
//     a window of one is certified, larger windows are decided in FP64 with
//     the reference formula, overflowing windows by a full FP64 rescan.
#pragma once

#include <cstdint>

namespace asicp {

constexpr int kNnThreads = 128;
constexpr int kNnQ = 8;                         // queries per thread
constexpr int kNnQB = kNnThreads * kNnQ;        // queries per work item
constexpr int kNnTile = 256;                    // candidates per TMA tile (4 KB)
constexpr int kNnStages = 8;                    // whole chunk resident: rescans read shared memory
constexpr int kNnMaxChunk = kNnStages * kNnTile; // candidates per work item (2048, 32 KB)
constexpr int kNnL = 4;                         // window list entries per query
constexpr int kRevWQ = 64;                      // reverse: queries per warp item (two per lane)

// One NN work item: a block of <= kNnQB queries against a contiguous
// candidate chunk.
struct NnItem {
  const float4* q;   // queries (x, y, z, margin), re-centred FP32
  const float4* c;   // candidates (-2x, -2y, -2z, |b|^2)
  int nq;
  int nc;
  int c_base;        // position of c[0] in the full candidate set
  int kind;          // 0 forward, 1 reverse, 2 final
  int owner;         // particle index
  int q_first;       // index of q[0] in the kind's query numbering
  int chunk;         // chunk index (0..S-1)
  int nchunks;       // S
  int slot;          // forward: global query-block index (partials are [slot][chunk][query])
};

// Per (query, split) partial result: the split's best FP32 value and its
// position; the top bit of `pos` flags an ambiguous window (another candidate
// within the certification margin, or an overflowing top-3).
struct NnPartial {
  float b1;
  int pos;
};
constexpr int kAmbiguous = static_cast<int>(0x80000000u);
constexpr int kNoBlock = 0x7fffffff;  // ambiguous without a member list (pool exhausted)
constexpr int kWinCap = 8;            // members per ambiguous-window list

}  // namespace asicp
