// eat_internal.h -- internal layout shared by the host compressor (build.cpp),
// the CUDA kernels (kernels.cu) and the C ABI (api.cu).  Product code only;
// nothing here is shared with oracle/.
//
// Packed index (the paper's CT[]/CL[]/AP[] of
// PAPER.md:382-390 redesigned for 32-byte sectors):
//
//   type_ptr[x]..type_ptr[x+1]   connection types whose source is
//                                internal vertex x, sorted by (v, lambda): the
//                                types of one edge (u,v) are contiguous (Edge-
//                                version grouping).
//   type_rec[t] (32 B)           {v, lambda, first_dep, last_dep, crec_base,
//                                 c_first, u, 0}; first/last serve the early
//                                termination tests of PAPER.md:411-416.
//   crec[r] (32 B)               one record per hour cluster k in
//                                [c_first, c_last] of a type:
//                                {next_min, item0..item6}; next_min is the first
//                                departure of the next non-empty cluster
//                                (reading R4), EAT_INF if none.
//                                More than 7 items: {next_min, SPILL, off, cnt}.
//   item (u32)                   one arithmetic progression (PAPER.md:142,
//                                Algorithm 6): bits 0-11 first-term offset inside
//                                the cluster, 12-23 difference, 24-31 count-1.
//                                Singletons are count 1.
//
// Lookup for bound b = e[u] (PAPER.md:305-306 + Algorithm 6):
//   b > last -> none;  b <= first -> first;
//   else k = b / cs, r = crec_base + k - c_first, scan r's items for the
//   smallest term >= b (ceil-div per item), else next_min.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#ifdef __CUDACC__
#define EAT_HD __host__ __device__
#else
#define EAT_HD
#endif

namespace eat {

constexpr uint32_t kInf = 0x7FFFFFFFu;
constexpr uint32_t kItemEmpty = 0xFFFFFFFFu;
constexpr uint32_t kItemSpill = 0xFFFFFFFEu;
constexpr uint32_t kMaxClusterSeconds = 4096;   // 12-bit offsets/differences
constexpr uint32_t kMaxRunTerms = 256;          // 8-bit count-1
constexpr int kInlineItems = 7;
constexpr int kTypeWords = 8;
constexpr int kCrecWords = 8;

EAT_HD inline uint32_t item_pack(uint32_t off, uint32_t stride, uint32_t count) {
    return (off & 0xFFFu) | ((stride & 0xFFFu) << 12) | ((count - 1u) << 24);
}

struct HostIndex {
    uint32_t n = 0;               // |V|
    uint64_t m = 0;               // |C|
    uint32_t cs = 3600;           // cluster seconds
    uint32_t num_clusters = 24;
    uint32_t max_dep = 0;
    std::vector<uint32_t> perm;   // caller id -> internal id
    std::vector<uint32_t> inv;    // internal id -> caller id
    std::vector<uint32_t> type_ptr;  // n + 1
    std::vector<uint32_t> type_rec;  // 8 * T
    std::vector<uint32_t> crec;      // 8 * R
    std::vector<uint32_t> pool;      // spilled items
    uint64_t num_types = 0, num_edges = 0, num_crec = 0, num_items = 0;
    uint32_t dense_nc = 0;           // > 0: dense cluster directory, record (t, k) at t*dense_nc + k
    double build_ms = 0.0;
};

struct BuildParams {
    uint32_t cs = 3600;
    uint32_t renumber = 0;
    uint32_t dense = 0;   // cluster directory: 0 auto, 1 dense, 2 compact
};

struct SubtripStats {
    uint64_t trips = 0, chained = 0, shortcuts = 0;
    uint32_t r_global = 0;
};

// Sub-trip shortcuts: U/V/D/L = the input connections
// followed by one shortcut per sub-trip.  Returns 0 or an eat_status code.
int make_subtrips(uint64_t m, const uint32_t *u, const uint32_t *v, const uint32_t *dep, const uint32_t *dur,
                  const uint32_t *trip, uint32_t scheme, std::vector<uint32_t> &U, std::vector<uint32_t> &V,
                  std::vector<uint32_t> &D, std::vector<uint32_t> &L, SubtripStats &st, std::string &msg);

// Host compressor (build.cpp).  Returns 0 or an eat_status code; msg set on error.
int build_host_index(uint32_t n, uint64_t m, const uint32_t *u, const uint32_t *v, const uint32_t *dep,
                     const uint32_t *dur, const float *xy, const BuildParams &p, HostIndex &out,
                     std::string &msg);

// Vertex range [lo, hi) of partition `rank` of `count` (balanced by out-type count).
void partition_range(const HostIndex &ix, uint32_t rank, uint32_t count, uint32_t &lo, uint32_t &hi);

}  // namespace eat
