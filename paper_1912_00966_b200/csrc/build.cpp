// build.cpp -- host-side timetable compressor (north-star subsystem 1).
//
// Raw connections (u, v, t, lambda) ->
//   1. validation (ids, dep + dur < EAT_INF);
//   2. CSR by source vertex (Edge-version preprocessing);
//   3. connection types = equal (u, v, lambda) (relation R),
//      departures sorted ("sorted according to their departure
//      time in pre-processing time");
//   4. locality renumbering of vertices (ours; Morton on coordinates or BFS);
//   5. per type, hour clusters k = floor(t / cs),
//      each covered greedily by arithmetic progressions,
//      packed into 32-byte cluster records with the next-non-empty-cluster
//      fallback precomputed (reading R4).
// Untimed preprocessing, like the paper's.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>

#include "eat.h"
#include "eat_internal.h"

namespace eat {
namespace {

unsigned num_threads() {
    unsigned t = std::thread::hardware_concurrency();
    return t == 0 ? 1 : std::min(t, 64u);
}

// Run f(chunk_lo, chunk_hi) over [0, n) split into ~4 chunks per thread.
template <class F>
void parallel_chunks(uint64_t n, F f) {
    unsigned nt = num_threads();
    if (n < 4096 || nt == 1) {
        f(uint64_t(0), n);
        return;
    }
    uint64_t nchunks = std::min<uint64_t>(n, uint64_t(nt) * 4);
    std::atomic<uint64_t> next(0);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (;;) {
                uint64_t c = next.fetch_add(1);
                if (c >= nchunks) break;
                f(n * c / nchunks, n * (c + 1) / nchunks);
            }
        });
    for (auto &x : th) x.join();
}

struct Rec {  // one connection inside its source's segment
    uint32_t v, dur, dep;
};

// ---------------------------------------------------------------- renumbering
uint32_t spread16(uint32_t x) {
    x &= 0xFFFF;
    x = (x | (x << 8)) & 0x00FF00FF;
    x = (x | (x << 4)) & 0x0F0F0F0F;
    x = (x | (x << 2)) & 0x33333333;
    x = (x | (x << 1)) & 0x55555555;
    return x;
}

void renumber_morton(uint32_t n, const float *xy, std::vector<uint32_t> &inv) {
    float xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    for (uint32_t i = 0; i < n; ++i) {
        xmin = std::min(xmin, xy[2 * i]);
        xmax = std::max(xmax, xy[2 * i]);
        ymin = std::min(ymin, xy[2 * i + 1]);
        ymax = std::max(ymax, xy[2 * i + 1]);
    }
    double sx = xmax > xmin ? 65535.0 / (xmax - xmin) : 0.0, sy = ymax > ymin ? 65535.0 / (ymax - ymin) : 0.0;
    std::vector<uint64_t> key(n);
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t qx = std::isfinite(xy[2 * i]) ? uint32_t((xy[2 * i] - xmin) * sx) : 0;
        uint32_t qy = std::isfinite(xy[2 * i + 1]) ? uint32_t((xy[2 * i + 1] - ymin) * sy) : 0;
        key[i] = (uint64_t(spread16(qx) | (spread16(qy) << 1)) << 32) | i;
    }
    std::sort(key.begin(), key.end());
    inv.resize(n);
    for (uint32_t i = 0; i < n; ++i) inv[i] = uint32_t(key[i] & 0xFFFFFFFFu);
}

// BFS order over the undirected edge graph; unvisited components in id order.
void renumber_bfs(uint32_t n, const std::vector<uint64_t> &seg, const std::vector<Rec> &recs,
                  std::vector<uint32_t> &inv) {
    // undirected adjacency from distinct (u, v)
    std::vector<uint64_t> deg(n + 1, 0);
    for (uint32_t x = 0; x < n; ++x)
        for (uint64_t i = seg[x]; i < seg[x + 1]; ++i)
            if (i == seg[x] || recs[i].v != recs[i - 1].v) {
                deg[x + 1]++;
                deg[recs[i].v + 1]++;
            }
    for (uint32_t x = 0; x < n; ++x) deg[x + 1] += deg[x];
    std::vector<uint32_t> adj(deg[n]);
    std::vector<uint64_t> fill(deg.begin(), deg.end() - 1);
    for (uint32_t x = 0; x < n; ++x)
        for (uint64_t i = seg[x]; i < seg[x + 1]; ++i)
            if (i == seg[x] || recs[i].v != recs[i - 1].v) {
                adj[fill[x]++] = recs[i].v;
                adj[fill[recs[i].v]++] = x;
            }
    inv.clear();
    inv.reserve(n);
    std::vector<uint8_t> seen(n, 0);
    for (uint32_t r = 0; r < n; ++r) {
        if (seen[r]) continue;
        size_t head = inv.size();
        inv.push_back(r);
        seen[r] = 1;
        while (head < inv.size()) {
            uint32_t x = inv[head++];
            for (uint64_t i = deg[x]; i < deg[x + 1]; ++i)
                if (!seen[adj[i]]) {
                    seen[adj[i]] = 1;
                    inv.push_back(adj[i]);
                }
        }
    }
}

// ---------------------------------------------------------------- AP cover
// Greedy arithmetic-progression cover of one cluster: take the
// smallest uncovered offset a; among progressions a, a+d, a+2d, ... whose
// terms are all uncovered departures, pick the one covering the most (ties:
// smallest d; candidates d = b - a for the next 32 uncovered b); mark its
// terms covered; repeat.  Runs are capped at 256 terms (8-bit count); the
// remainder is covered by later steps.  Duplicate departures become extra
// singleton items so that decoding reproduces the exact multiset.
struct ClusterCoder {
    uint64_t bits[kMaxClusterSeconds / 64 + 1];
    uint32_t words = 0;

    bool test(uint32_t i) const { return (bits[i >> 6] >> (i & 63)) & 1u; }
    void clear(uint32_t i) { bits[i >> 6] &= ~(uint64_t(1) << (i & 63)); }
    int next_set(uint32_t from) const {  // first set bit >= from, or -1
        uint32_t w = from >> 6;
        if (w >= words) return -1;
        uint64_t cur = bits[w] & (~uint64_t(0) << (from & 63));
        for (;;) {
            if (cur) return int(w * 64 + __builtin_ctzll(cur));
            if (++w >= words) return -1;
            cur = bits[w];
        }
    }

    void encode(const uint32_t *deps, size_t cnt, uint32_t base, uint32_t cs, std::vector<uint32_t> &items) {
        words = (cs + 63) / 64;
        std::memset(bits, 0, sizeof(uint64_t) * words);
        size_t first_item = items.size();
        for (size_t i = 0; i < cnt; ++i) {
            uint32_t off = deps[i] - base;
            if (test(off))
                items.push_back(item_pack(off, 0, 1));  // duplicate occurrence
            else
                bits[off >> 6] |= uint64_t(1) << (off & 63);
        }
        for (int a = next_set(0); a >= 0; a = next_set(uint32_t(a))) {
            uint32_t best_d = 0, best_c = 1;
            int b = next_set(uint32_t(a) + 1);
            for (int cand = 0; cand < 32 && b >= 0; ++cand, b = next_set(uint32_t(b) + 1)) {
                uint32_t d = uint32_t(b - a), c = 2;
                while (c < kMaxRunTerms && uint32_t(a) + c * d < cs && test(uint32_t(a) + c * d)) ++c;
                if (c > best_c) {
                    best_c = c;
                    best_d = d;
                }
            }
            for (uint32_t i = 0; i < best_c; ++i) clear(uint32_t(a) + i * best_d);
            items.push_back(item_pack(uint32_t(a), best_c > 1 ? best_d : 0, best_c));
        }
        std::sort(items.begin() + first_item, items.end(), [](uint32_t x, uint32_t y) {
            return (x & 0xFFFu) != (y & 0xFFFu) ? (x & 0xFFFu) < (y & 0xFFFu) : x < y;
        });
    }
};

struct Chunk {
    std::vector<uint32_t> type_rec, crec, pool;
    uint64_t edges = 0, items = 0;
};

}  // namespace

// ---------------------------------------------------------------- sub-trips
// Data enhancement of PAPER.md:342-354 (Sec. II-G): every trip, a sequence of
// connections (v_1,v_2,t_1,l_1), ..., (v_k,v_{k+1},t_k,l_k) with
// t_i + l_i <= t_{i+1}, is cut into consecutive, non-overlapping
// sub-trips of r connections (the last one k % r); a sub-trip
// (v_i..v_{j+1}) adds the shortcut (v_i, v_{j+1}, t_i, t_j + l_j - t_i).
// A shortcut's arrival is the arrival of the vehicle itself, so earliest
// arrival times are unchanged; paths get fewer hops, so sweeps drop.
// scheme 1: r = round(sqrt(k)) per trip; scheme 2: r =
// round(sqrt(average trip length)); scheme >= 3: r = scheme.
// Connections of a trip are ordered by departure (ties: input order); a trip
// that does not chain (v_i != u_{i+1} or t_i + l_i > t_{i+1}) gets no shortcut.
int make_subtrips(uint64_t m, const uint32_t *u, const uint32_t *v, const uint32_t *dep, const uint32_t *dur,
                  const uint32_t *trip, uint32_t scheme, std::vector<uint32_t> &U, std::vector<uint32_t> &V,
                  std::vector<uint32_t> &D, std::vector<uint32_t> &L, SubtripStats &st, std::string &msg) {
    st = SubtripStats{};
    if (!trip) {
        msg = "sub-trips need the timetable's trip ids (eat_timetable.trip)";
        return EAT_EINVAL;
    }
    // order connections by (trip, dep, input index): counting sort by trip id
    // when ids are dense, else a comparison sort
    uint32_t tmax = 0;
    for (uint64_t i = 0; i < m; ++i) tmax = std::max(tmax, trip[i]);
    std::vector<uint64_t> order(m);
    std::vector<uint64_t> tptr;
    if (m && uint64_t(tmax) <= 4 * m + 16) {
        tptr.assign(uint64_t(tmax) + 2, 0);
        for (uint64_t i = 0; i < m; ++i) tptr[trip[i] + 1]++;
        for (uint64_t t = 0; t <= tmax; ++t) tptr[t + 1] += tptr[t];
        std::vector<uint64_t> fill(tptr.begin(), tptr.end() - 1);
        for (uint64_t i = 0; i < m; ++i) order[fill[trip[i]]++] = i;
    } else {
        std::iota(order.begin(), order.end(), uint64_t(0));
        std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return trip[a] < trip[b]; });
        tptr.push_back(0);
        for (uint64_t i = 1; i <= m; ++i)
            if (i == m || trip[order[i]] != trip[order[i - 1]]) tptr.push_back(i);
    }
    const uint64_t ntrips = tptr.size() - 1;
    // per trip: stable sort by departure, chain check
    std::vector<uint8_t> ok(ntrips, 0);
    std::atomic<uint64_t> sum_len(0), n_ok(0);
    parallel_chunks(ntrips, [&](uint64_t lo, uint64_t hi) {
        uint64_t sl = 0, no = 0;
        for (uint64_t t = lo; t < hi; ++t) {
            const uint64_t a = tptr[t], b = tptr[t + 1];
            if (b - a < 2) continue;
            std::stable_sort(order.begin() + a, order.begin() + b, [&](uint64_t x, uint64_t y) { return dep[x] < dep[y]; });
            bool good = true;
            for (uint64_t i = a; i + 1 < b && good; ++i) {
                const uint64_t c = order[i], d = order[i + 1];
                good = v[c] == u[d] && uint64_t(dep[c]) + dur[c] <= dep[d];
            }
            if (good) {
                ok[t] = 1;
                sl += b - a;
                ++no;
            }
        }
        sum_len += sl;
        n_ok += no;
    });
    st.trips = ntrips;
    st.chained = n_ok.load();
    const double avg = st.chained ? double(sum_len.load()) / double(st.chained) : 0.0;
    // scheme >= EAT_SUBTRIPS_HIER: hierarchical blocks of r, r^2, ... (ours)
    const bool hier = scheme >= EAT_SUBTRIPS_HIER;
    const uint32_t r_global = hier ? scheme - EAT_SUBTRIPS_HIER
                              : scheme == 2 ? uint32_t(std::lround(std::sqrt(avg))) : (scheme >= 3 ? scheme : 0);
    st.r_global = r_global;
    auto r_of = [&](uint64_t k) -> uint64_t { return scheme == 1 ? uint64_t(std::llround(std::sqrt(double(k)))) : r_global; };
    // Blocks [i, j] of one trip of k connections that get a shortcut: aligned
    // blocks of r; hierarchical: also of r^2, r^3, ... up to the
    // first size covering the trip, skipping blocks equal to a smaller level's.
    auto for_blocks = [&](uint64_t k, auto &&emit) {
        const uint64_t r = r_of(k);
        if (r < 2) return;
        uint64_t prev = 1;
        for (uint64_t B = r;; prev = B, B *= r) {
            for (uint64_t i = 0; i < k; i += B) {
                const uint64_t j = std::min(k, i + B) - 1;
                if (j > i && j - i + 1 > prev) emit(i, j);
            }
            if (!hier || B >= k) break;
        }
    };
    // emit shortcuts (count first, then fill, in trip order)
    std::vector<uint64_t> cnt(ntrips + 1, 0);
    parallel_chunks(ntrips, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t t = lo; t < hi; ++t) {
            if (!ok[t]) continue;
            uint64_t c = 0;
            for_blocks(tptr[t + 1] - tptr[t], [&](uint64_t, uint64_t) { ++c; });
            cnt[t + 1] = c;
        }
    });
    for (uint64_t t = 0; t < ntrips; ++t) cnt[t + 1] += cnt[t];
    const uint64_t S = cnt[ntrips];
    st.shortcuts = S;
    U.resize(m + S);
    V.resize(m + S);
    D.resize(m + S);
    L.resize(m + S);
    std::copy(u, u + m, U.begin());
    std::copy(v, v + m, V.begin());
    std::copy(dep, dep + m, D.begin());
    std::copy(dur, dur + m, L.begin());
    parallel_chunks(ntrips, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t t = lo; t < hi; ++t) {
            if (!ok[t] || cnt[t + 1] == cnt[t]) continue;
            const uint64_t a = tptr[t], k = tptr[t + 1] - a;
            uint64_t o = m + cnt[t];
            for_blocks(k, [&](uint64_t i, uint64_t j) {  // sub-trip = connections i..j
                const uint64_t ci = order[a + i], cj = order[a + j];
                U[o] = u[ci];
                V[o] = v[cj];
                D[o] = dep[ci];
                L[o] = dep[cj] + dur[cj] - dep[ci];
                ++o;
            });
        }
    });
    return EAT_OK;
}

void partition_range(const HostIndex &ix, uint32_t rank, uint32_t count, uint32_t &lo, uint32_t &hi) {
    uint64_t T = ix.num_types;
    auto cut = [&](uint32_t r) -> uint32_t {
        if (r == 0) return 0;
        if (r >= count) return ix.n;
        uint64_t target = T * r / count;
        // first vertex x with type_ptr[x] >= target
        return uint32_t(std::lower_bound(ix.type_ptr.begin(), ix.type_ptr.end() - 1, uint32_t(target)) -
                        ix.type_ptr.begin());
    };
    lo = cut(rank);
    hi = cut(rank + 1);
    if (hi < lo) hi = lo;
}

int build_host_index(uint32_t n, uint64_t m, const uint32_t *u, const uint32_t *v, const uint32_t *dep,
                     const uint32_t *dur, const float *xy, const BuildParams &p, HostIndex &ix,
                     std::string &msg) {
    auto t0 = std::chrono::steady_clock::now();
    if (n == 0) {
        msg = "num_vertices must be >= 1";
        return EAT_EINVAL;
    }
    if (m > 0 && (!u || !v || !dep || !dur)) {
        msg = "u, v, dep, dur must be non-NULL when num_connections > 0";
        return EAT_EINVAL;
    }
    if (p.cs == 0 || p.cs > kMaxClusterSeconds) {
        msg = "cluster_seconds must be in 1..4096";
        return EAT_EINVAL;
    }
    if (m > 0xFFFFFFFFull * 4) {
        msg = "too many connections";
        return EAT_EINVAL;
    }
    // 1. validation (a1)
    std::atomic<int> bad(0);
    std::atomic<uint32_t> maxdep(0);
    parallel_chunks(m, [&](uint64_t lo, uint64_t hi) {
        uint32_t md = 0;
        for (uint64_t i = lo; i < hi; ++i) {
            if (u[i] >= n || v[i] >= n) bad.store(1);
            else if (uint64_t(dep[i]) + dur[i] >= kInf) bad.store(bad.load() ? bad.load() : 2);
            md = std::max(md, dep[i]);
        }
        uint32_t cur = maxdep.load();
        while (md > cur && !maxdep.compare_exchange_weak(cur, md)) {
        }
    });
    if (bad.load() == 1) {
        msg = "connection endpoint >= num_vertices";
        return EAT_EINVAL;
    }
    if (bad.load() == 2) {
        msg = "dep + dur >= EAT_INF";
        return EAT_ERANGE;
    }
    ix.n = n;
    ix.m = m;
    ix.cs = p.cs;
    ix.max_dep = maxdep.load();
    ix.num_clusters = std::max<uint32_t>(24, uint32_t((uint64_t(ix.max_dep) + p.cs) / p.cs));

    // 2. counting sort by source (a3)
    std::vector<uint64_t> seg(uint64_t(n) + 1, 0);
    for (uint64_t i = 0; i < m; ++i) seg[u[i] + 1]++;
    for (uint32_t x = 0; x < n; ++x) seg[x + 1] += seg[x];
    std::vector<Rec> recs(m);
    {
        std::vector<uint64_t> fill(seg.begin(), seg.end() - 1);
        for (uint64_t i = 0; i < m; ++i) recs[fill[u[i]]++] = Rec{v[i], dur[i], dep[i]};
    }
    // 3. types: sort each segment by (v, lambda, dep) (a4)
    parallel_chunks(n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t x = lo; x < hi; ++x)
            std::sort(recs.begin() + seg[x], recs.begin() + seg[x + 1], [](const Rec &a, const Rec &b) {
                if (a.v != b.v) return a.v < b.v;
                if (a.dur != b.dur) return a.dur < b.dur;
                return a.dep < b.dep;
            });
    });

    // 4. renumbering (a2)
    uint32_t mode = p.renumber;
    if (mode == EAT_RENUMBER_AUTO) mode = xy ? EAT_RENUMBER_MORTON : EAT_RENUMBER_BFS;
    if (mode == EAT_RENUMBER_MORTON && !xy) {
        msg = "EAT_RENUMBER_MORTON needs xy";
        return EAT_EINVAL;
    }
    if (mode == EAT_RENUMBER_MORTON)
        renumber_morton(n, xy, ix.inv);
    else if (mode == EAT_RENUMBER_BFS)
        renumber_bfs(n, seg, recs, ix.inv);
    else if (mode == EAT_RENUMBER_NONE) {
        ix.inv.resize(n);
        std::iota(ix.inv.begin(), ix.inv.end(), 0u);
    } else {
        msg = "unknown renumber mode";
        return EAT_EINVAL;
    }
    ix.perm.assign(n, 0);
    for (uint32_t i = 0; i < n; ++i) ix.perm[ix.inv[i]] = i;

    // 5. types per internal vertex -> type_ptr
    std::vector<uint32_t> ntypes(n, 0);
    parallel_chunks(n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t x = lo; x < hi; ++x) {
            uint32_t o = ix.inv[x], c = 0;
            for (uint64_t i = seg[o]; i < seg[o + 1]; ++i)
                if (i == seg[o] || recs[i].v != recs[i - 1].v || recs[i].dur != recs[i - 1].dur) ++c;
            ntypes[x] = c;
        }
    });
    ix.type_ptr.assign(uint64_t(n) + 1, 0);
    uint64_t T = 0;
    for (uint32_t x = 0; x < n; ++x) {
        ix.type_ptr[x] = uint32_t(T);
        T += ntypes[x];
        if (T > 0xFFFFFFF0ull) {
            msg = "too many connection types";
            return EAT_EUNSUPPORTED;
        }
    }
    ix.type_ptr[n] = uint32_t(T);
    ix.num_types = T;

    // 6. clusters + AP cover per type, in chunks of internal vertices (a5, a6)
    const uint32_t cs = p.cs;
    unsigned nt = num_threads();
    uint64_t nchunks = n < 4096 ? 1 : std::min<uint64_t>(n, uint64_t(nt) * 8);
    std::vector<Chunk> chunks(nchunks);
    std::atomic<uint64_t> next(0);
    auto work = [&] {
        ClusterCoder coder;
        std::vector<uint32_t> items, deps;
        for (;;) {
            uint64_t c = next.fetch_add(1);
            if (c >= nchunks) break;
            Chunk &ch = chunks[c];
            uint64_t xlo = uint64_t(n) * c / nchunks, xhi = uint64_t(n) * (c + 1) / nchunks;
            for (uint64_t x = xlo; x < xhi; ++x) {
                uint32_t o = ix.inv[x];
                uint64_t i = seg[o], e = seg[o + 1];
                while (i < e) {
                    uint64_t j = i;
                    while (j < e && recs[j].v == recs[i].v && recs[j].dur == recs[i].dur) ++j;
                    if (i == seg[o] || recs[i].v != recs[i - 1].v) ch.edges++;
                    // type [i, j): departures sorted ascending
                    uint32_t first = recs[i].dep, last = recs[j - 1].dep;
                    uint32_t cf = first / cs, cl = last / cs;
                    uint64_t crec_base = ch.crec.size() / kCrecWords;
                    ch.type_rec.insert(ch.type_rec.end(),
                                       {ix.perm[recs[i].v], recs[i].dur, first, last, uint32_t(crec_base), cf,
                                        uint32_t(x), 0u});
                    ch.crec.resize(ch.crec.size() + uint64_t(cl - cf + 1) * kCrecWords);
                    uint32_t *rec0 = ch.crec.data() + crec_base * kCrecWords;
                    uint32_t next_min = kInf;
                    uint64_t hiidx = j;  // deps of clusters > k are in [.., hiidx)
                    for (uint32_t k = cl + 1; k-- > cf;) {
                        uint64_t loidx = hiidx;
                        while (loidx > i && recs[loidx - 1].dep / cs == k) --loidx;
                        uint32_t *r = rec0 + uint64_t(k - cf) * kCrecWords;
                        r[0] = next_min;
                        items.clear();
                        if (loidx < hiidx) {
                            deps.resize(hiidx - loidx);
                            for (uint64_t q = loidx; q < hiidx; ++q) deps[q - loidx] = recs[q].dep;
                            coder.encode(deps.data(), deps.size(), k * cs, cs, items);
                            next_min = recs[loidx].dep;
                        }
                        ch.items += items.size();
                        if (items.size() <= size_t(kInlineItems)) {
                            for (int s = 0; s < kInlineItems; ++s)
                                r[1 + s] = s < int(items.size()) ? items[s] : kItemEmpty;
                        } else {
                            r[1] = kItemSpill;
                            r[2] = uint32_t(ch.pool.size());
                            r[3] = uint32_t(items.size());
                            for (int s = 4; s < kCrecWords; ++s) r[s] = kItemEmpty;
                            ch.pool.insert(ch.pool.end(), items.begin(), items.end());
                        }
                        hiidx = loidx;
                    }
                    i = j;
                }
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < std::min<uint64_t>(nt, nchunks); ++t) th.emplace_back(work);
        for (auto &x : th) x.join();
    }
    // 7. concatenate chunks, rebasing crec / pool offsets
    uint64_t R = 0, P = 0;
    for (auto &ch : chunks) {
        R += ch.crec.size() / kCrecWords;
        P += ch.pool.size();
    }
    if (R > 0xFFFFFFF0ull || P > 0xFFFFFFF0ull) {
        msg = "index too large for 32-bit offsets";
        return EAT_EUNSUPPORTED;
    }
    ix.type_rec.resize(T * kTypeWords);
    ix.crec.resize(R * kCrecWords);
    ix.pool.resize(P);
    uint64_t to = 0, ro = 0, po = 0;
    ix.num_edges = 0;
    ix.num_items = 0;
    for (auto &ch : chunks) {
        uint64_t nt_c = ch.type_rec.size() / kTypeWords, nr_c = ch.crec.size() / kCrecWords;
        for (uint64_t t = 0; t < nt_c; ++t) ch.type_rec[t * kTypeWords + 4] += uint32_t(ro);
        for (uint64_t r = 0; r < nr_c; ++r)
            if (ch.crec[r * kCrecWords + 1] == kItemSpill) ch.crec[r * kCrecWords + 2] += uint32_t(po);
        std::copy(ch.type_rec.begin(), ch.type_rec.end(), ix.type_rec.begin() + to * kTypeWords);
        std::copy(ch.crec.begin(), ch.crec.end(), ix.crec.begin() + ro * kCrecWords);
        std::copy(ch.pool.begin(), ch.pool.end(), ix.pool.begin() + po);
        to += nt_c;
        ro += nr_c;
        po += ch.pool.size();
        ix.num_edges += ch.edges;
        ix.num_items += ch.items;
        std::vector<uint32_t>().swap(ch.type_rec);
        std::vector<uint32_t>().swap(ch.crec);
        std::vector<uint32_t>().swap(ch.pool);
    }
    ix.num_crec = R;
    // 8. dense cluster directory (the paper's CL[y*i + j] addressing,
    // PAPER.md:386-390): record of (type t, cluster k) at t*NC + k, so a
    // kernel can fetch it from (t, e[u]) alone, in parallel with the type
    // record -- one dependent load less per relaxation.  Used when it costs at
    // most ~3x the compact layout; records outside [c_first, c_last] are never
    // read (the lookup only reaches a cluster record when first < e[u] <= last).
    const uint64_t NC = uint64_t(ix.max_dep) / cs + 1;
    const uint64_t dense_recs = T * NC;
    bool dense = p.dense == 1;
    // auto: only graphs too large for the shared-memory (CTA) kernels, which
    // run the latency-bound grid kernels (measured: metro -5 %, city batch +14 %
    // slower with dense because of the speculative record loads)
    if (p.dense == 0)
        dense = n > 52000 && dense_recs * kCrecWords * 4 <= 3 * R * kCrecWords * 4;
    if (dense && T && dense_recs < 0xFFFFFFF0ull) {
        std::vector<uint32_t> dcrec(dense_recs * kCrecWords, 0u);
        parallel_chunks(T, [&](uint64_t lo, uint64_t hi) {
            for (uint64_t t = lo; t < hi; ++t) {
                uint32_t *tr = ix.type_rec.data() + t * kTypeWords;
                const uint32_t cf = tr[5], cl = tr[3] / cs;
                std::copy(ix.crec.begin() + uint64_t(tr[4]) * kCrecWords,
                          ix.crec.begin() + (uint64_t(tr[4]) + (cl - cf + 1)) * kCrecWords,
                          dcrec.begin() + (t * NC + cf) * kCrecWords);
                tr[4] = uint32_t(t * NC);  // crec_base
                tr[5] = 0;                 // c_first: record index = crec_base + k
            }
        });
        ix.crec.swap(dcrec);
        ix.num_crec = dense_recs;
        ix.dense_nc = uint32_t(NC);
    }
    ix.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return EAT_OK;
}

}  // namespace eat
