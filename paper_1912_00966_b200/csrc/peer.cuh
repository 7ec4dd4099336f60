// peer.cuh -- edge-partitioned single query with an in-kernel exchange over
// peer memory (NEXT-2; the fused alternative to partition.cu's
// per-round NCCL min-allreduce of the whole e[]).
//
// Partition p owns the out-types of internal vertices [lo_p, hi_p) and one
// "exchange block" in its GPU's memory: a full e[] replica (authoritative on
// the owned range), inbox lists and dedup flags.  A relaxation that lowers a
// vertex v owned elsewhere applies atomicMin directly to the owner's e[v]
// (NVLink peer atomic, system scope) and, if that improved it, appends v to
// the owner's inbox -- no host round trip, no dense collective.  Partitions
// run local sweeps to quiescence, then meet at a cross-partition barrier
// (system-scope atomics in partition 0's block); a round in which nobody sent
// a message ends the query (the fixpoint is unique).
//
// Deployments: one process per GPU, blocks mapped with CUDA IPC handles
// (eat_peer_export / eat_peer_connect), one CTA group per launch; or all P
// partitions as P CTA groups of a single launch on one device (loopback: the
// same code with same-device pointers, used by the tests).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace eat {

constexpr uint32_t kMaxPeerParts = 16;

// Partition p's exchange block as seen from the launching device.
struct PeerPart {
    uint32_t *arr;        // [n] e[] replica (authoritative on [lo, hi))
    uint32_t *inflag;     // [2][own] inbox dedup flags by round parity
    uint32_t *inbox;      // [2][own] owned vertices lowered by other partitions, by round parity
    uint32_t *inbox_cnt;  // [2]
    uint32_t lo, hi;
};

struct PeerCtx {
    PeerPart part[kMaxPeerParts];
    uint32_t P;              // partitions of the query
    uint32_t part0;          // partition of this launch's first CTA group
    uint32_t groups;         // CTA groups (= partitions) in this launch
    uint32_t ctas_per_group;
    uint32_t *gctl;          // partition 0's control words: [0] arrivals, [1] generation, [2..4] messages per round % 3
};

// Per partition run by this launch (memory of the launching device).
struct PeerLocal {
    uint32_t *q0, *q1, *stamp;  // [n] local frontier worklists + dedup stamps
    uint32_t *ctl;              // [kCtlWords]: 0-2 frontier counters, 8 sweeps, 9 rounds, 10 round base, kBarWord group barrier
};

// Bytes of one exchange block (offsets below are identical on every rank).
size_t peer_block_bytes(uint32_t n, uint32_t own);
// PeerPart view of a block at `base` (any address space mapping of it).
PeerPart peer_part_view(void *base, uint32_t n, uint32_t lo, uint32_t hi);
// Control words live at the end of partition 0's block.
uint32_t *peer_gctl(void *base0, uint32_t n, uint32_t own0);

cudaError_t peer_local_alloc(PeerLocal &l, uint32_t n);
// Resident CTAs per SM of the peer kernel (capped by EAT_GRID_CTAS_PER_SM).
int peer_ctas_per_sm();
void peer_local_free(PeerLocal &l);

// One query: a cooperative launch of ctx.groups CTA groups (d_ix[g] is group
// g's index slice, d_ctx / d_loc device copies), then the caller-ordered
// gather of the owners' e[] into d_out.  Collective across all partitions.
cudaError_t peer_query(const DevIndex *d_ix, const PeerCtx &ctx, const PeerCtx *d_ctx, const PeerLocal *h_loc,
                       PeerLocal *d_loc, const uint32_t *d_perm, uint32_t n, int subwarp, uint32_t s, uint32_t t_s,
                       uint32_t *d_out, cudaStream_t st);

}  // namespace eat
