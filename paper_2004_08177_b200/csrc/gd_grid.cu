// gd_grid.cu -- K2+K3: the (app x clock) grid path.
//
// Replaces ModelPredictorState::build + 2x models::predict
// (scheduler.cpp:329-370) and decide()'s selection (scheduler.cpp:54-100,
// 187-234): candidate rows are never materialised, both ensembles are
// evaluated for every catalog clock of an app, and the deadline-masked
// selection runs in the epilogue.
//
// Partial evaluation.  For one app every candidate row is identical except
// the sm_clock / mem_clock columns, so every non-clock node test has the same
// outcome for all C clocks.  A tree therefore contributes, per app, either a
// constant (its row-only walk ends on a leaf) or a small clock-only residue
// (the walk stops at a clock node; below it, row-only walks again end on
// leaves or further clock nodes).  The leaf each candidate reaches is exactly
// predict_row's leaf (models.cpp:71-78), so the ordered sums are bit-exact.
//
// Three kernels per app batch:
//
//   grid_rank_kernel      exact 16-bit ranks of every (app, feature) against
//       each model's sorted thresholds (x <= thr_k <=> rank(x) <= k), in the
//       walk kernel's tile layout.
//   K2a grid_walk_kernel  (tree-major, shared-memory latency bound)
//       persistent CTAs, tiles of 512 apps (lane = app); trees (8-byte rank-
//       form WNodes) stream into shared memory by TMA bulk copies through a
//       full/empty mbarrier ring; every warp walks every staged tree for its
//       32 apps, four walks in flight per lane.  Walks that stop at a clock
//       node are resolved from per-warp job queues with full warps.  Each
//       (app, tree) becomes one 16-byte TreeRec: CONST (leaf), SM / MEM (one
//       clock test between two leaves), TABLE (balanced depth-2/3 residue,
//       128-byte side record) or FULL (deeper: per-clock traversal).
//   K2b grid_acc_kernel   (app-major, FP64-add / issue bound)
//       a warp PAIR per app (energy warp, time warp), lane l owning CPL
//       catalog clocks that share one memory clock (one in-order accumulator
//       per clock).  Records stream through a cp.async ring (32 trees per
//       stage; leaf values / tables one stage behind) and become CPL
//       __dadd_rn's each, in tree order.  The energy warp then runs the
//       selection epilogue (K3) on the pair's E/T values.  Small batches use
//       grid_acc_sliced_kernel (a pair per (app, 32-clock slice)).
//
// Clock packing.  Each owned clock is one register ck = sm << 16 | mem
// (1 <= sm, mem <= 65535, validated on the host).  A test `(double)sm <= thr`
// is `ck <= ((clamp(floor(thr), 0, 65535) << 16) | 0xffff)` (unsigned); a test
// `(double)mem <= thr` is `(ck & 0xffff) <= clamp(floor(thr), 0, 65535)`.
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include "gd_common.cuh"

#ifndef GD_TABLE_KEYS
#define GD_TABLE_KEYS 1  // 1: per-lane compare keys for depth-2/3 tables on memory-uniform lanes
#endif
#ifndef GD_WALK_LATE_LEAF
#define GD_WALK_LATE_LEAF 1  // 1: a root walk's leaf index is formed after its loop, not per step
#endif


namespace gd {
#ifdef GD_WALK_TRACE
__device__ unsigned long long g_wtrace[4096][8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define WTRACE(k) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_wtrace[blockIdx.x][k] = gtime(); } while (0)
#else
#define WTRACE(k) do {} while (0)
#endif
namespace {

using namespace dev;

// ---------------------------------------------------------------------------
// The walk -> accumulate hand-off.
// ---------------------------------------------------------------------------
enum : uint32_t { kRecConst = 0, kRecSm = 1, kRecMem = 2, kRecTable = 3, kRecFull = 4, kRecTable4 = 5, kRecTable5 = 6 };

// One (app, tree) record.  info = kind | t16 << 16 (SM / MEM keys); leaves
// are referenced by packed (grid) index and their values fetched by the
// accumulate kernel's prefetch stage.
//   CONST: ref = the leaf.                 SM/MEM: ref / ref2 = left / right leaf.
//   TABLE: ref = residue-table index.      FULL:   ref = first clock node.
struct __align__(16) TreeRec {
    uint32_t info;
    int32_t ref;
    int32_t ref2;
    uint32_t pad;
};
static_assert(sizeof(TreeRec) == 16, "TreeRec is 16 bytes");

// A residue table: the clock-only residue of one (app, tree) as a balanced
// tree of depth D (2 or 3).  Test k is node k (children 2k+1, 2k+2); a clock
// goes right iff (ck & mask) > key (always-left = {0, 0}).  Leaves are stored
// in depth-3 slots whatever D is: the leaf a depth-D walk ends on (node
// 2^D - 1 + l) is leaf[l << (3 - D)].  A leaf found at level k < D sits under
// always-left tests, so it is read through its leftmost slot only.
struct __align__(16) RTRec {
    uint2 test[7];
    uint32_t depth;
    uint32_t pad;
    double leaf[8];
};
static_assert(sizeof(RTRec) == 128, "RTRec is 128 bytes");

// A depth-4 residue (two consecutive pool slots, record kind kRecTable4):
// tests 0..14 in heap order, leaf l (node 15 + l) at leaf[l].
struct __align__(16) RTRec4 {
    uint2 test[15];
    uint32_t pad[2];
    double leaf[16];
};
static_assert(sizeof(RTRec4) == 256, "RTRec4 is two pool slots");

// A depth-5 residue (four consecutive pool slots, record kind kRecTable5):
// tests 0..30 in heap order, leaf l (node 31 + l) at leaf[l].  Trained
// ensembles split on the two clock columns in turn near their roots: 1.5 %
// of a trained time model's residues have 5 test levels (per-clock traversal
// from global memory otherwise).
struct __align__(16) RTRec5 {
    uint2 test[31];
    uint32_t pad[2];
    double leaf[32];
};
static_assert(sizeof(RTRec5) == 512, "RTRec5 is four pool slots");


// Records of tree t for batch-local app la: pairs of trees are interleaved
// per app so a lane of the walk kernel stores 32 contiguous bytes.
__host__ __device__ __forceinline__ int64_t rec_index(int32_t t, int64_t la, int64_t n_apps) {
    return ((static_cast<int64_t>(t >> 1) * n_apps + la) << 1) | (t & 1);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct AccParams {
    const PNode* nodes[2];
    int32_t n_trees[2];
    double base[2], lr[2];
    const TreeRec* rec[2];
    const RTRec* pool;
    const double* rows;
    const double* cat_t;
    const int32_t* cat_cols;
    const int32_t* sm;
    const int32_t* mem;
    const double* budgets;
    gd_decision* out;
    double* e_out;
    double* t_out;
    int64_t a0;
    int32_t n_apps;
    int32_t n_cols, n_cat, n_clocks;
    int32_t mode, objective, best_effort;
    int64_t out_stride;  // row stride of e_out / t_out
    // Sliced mode (small batches): per-app E/T staging and arrival counters.
    double* et;          // [n_apps][2][n_clocks]
    uint32_t* arrive;    // [n_apps], zeroed
};

struct WalkParams {
    const WNode* wnodes[2];
    const int32_t* wroots[2];  // n_trees + 1 entries, walk-node units
    const int32_t* roots[2];   // grid roots, n_trees + 1 entries
    const int32_t* wint[2];    // per tree: loadable walk-node prefix (window size when it fits)
    const PNode* gnodes[2];    // grid nodes (leaf values)
    int32_t n_trees[2];
    const unsigned char* ranks;  // [2][tile][n_cols][tile_apps] ranks of RB bytes for the batch
    int32_t n_apps;            // apps in the batch
    int32_t n_cols;
    int32_t tile_apps;         // apps per work item = 32 * groups
    int32_t splits;            // tree-pair ranges per model
    int32_t tiles;             // app tiles in the batch
    int32_t n_items;           // 2 * splits * tiles
    int32_t split_major;       // item order: (model, split, tile) if set, else (tile, model, split)
    int32_t chunk;             // consecutive items per fetch
    uint32_t* item_next;       // chunk counter (zeroed per batch)
    int32_t win_nodes;         // per-tree window staged in shared memory (BFS prefix, even)
    int32_t stage_nodes;       // capacity of one stage buffer (walk nodes)
    int32_t n_bufs;            // stage buffers in the ring (2..4)
    int32_t n_subs;            // warps per 32-app group (1: a warp walks every tree; 2: even / odd)
    TreeRec* rec[2];
    RTRec* pool;
    uint32_t* pool_count;
    uint32_t pool_cap;
    int32_t res_levels;        // test levels a residue table may hold (3 or 4; deeper: FULL)
    int32_t job_run;           // queued jobs that start a run (<= kJobCap - 32)
};

// ---------------------------------------------------------------------------
// K2a: walks.
//
// Persistent CTAs, each owning a contiguous range of work items (app tile x
// model x tree-pair range).  A stage is a run of consecutive tree pairs whose
// top-level windows (the first win_nodes walk nodes of each tree: its top
// levels, trees being laid out breadth-first) fit one shared-memory buffer;
// thread 0 streams the next stage in with TMA bulk copies (cp.async.bulk +
// mbarrier) while the CTA walks the current one.  Rows are staged as 16-bit
// feature ranks, transposed ([col][app]) so lane-per-app reads are
// conflict-free; walks compare ranks with threshold indices (WNode).
// ---------------------------------------------------------------------------

struct Walk {
    int32_t n;    // byte offset of the current node within its tree (walk nodes)
    int32_t key;
    int32_t fc;   // feat << 16 | child
};

__device__ __forceinline__ int32_t wfeat(int32_t fc) { return fc >> 19; }
__device__ __forceinline__ int32_t wchild(int32_t fc) { return fc & 0x7fff8; }  // byte offset of the left child
// fc of a leaf synthesized from its parent's flags (feat = kFeatLeaf).
constexpr int32_t kLeafFc = static_cast<int32_t>(0xfff80000u);

// Where one tree's walk nodes live during a stage.
struct TreeSrc {
    int32_t wroot;    // walk-node index of the root
    int32_t groot;    // grid index of the root
    uint32_t win;     // nodes [0, win) of the tree are in shared memory ...
    uint32_t saddr;   // ... at this shared address
};

struct WalkCtx {
    const WNode* __restrict__ wnodes;  // global walk nodes of the model
    const PNode* __restrict__ gnodes;  // grid nodes (leaf values)
    uint32_t row_saddr;                // shared address of this lane's app in the staged ranks
    int32_t row_stride;                // bytes between consecutive columns
};

template <bool kAllSmem>
__device__ __forceinline__ void load_wnode(const WalkCtx& c, const TreeSrc& s, Walk& w) {
    if (kAllSmem || static_cast<uint32_t>(w.n) < 8u * s.win) {
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];"
                     : "=r"(w.key), "=r"(w.fc)
                     : "r"(s.saddr + static_cast<uint32_t>(w.n)));
    } else {
        const int2 q = __ldg(reinterpret_cast<const int2*>(reinterpret_cast<const char*>(c.wnodes + s.wroot) + w.n));
        w.key = q.x;
        w.fc = q.y;
    }
}

// The rank of feature wfeat(fc) for the app whose ranks start at shared
// address `row` (RB = bytes per rank: 1 when every feature of both models has
// at most 255 distinct thresholds, else 2).
template <int RB>
__device__ __forceinline__ int32_t rank_at(uint32_t row, int32_t stride, int32_t fc) {
    const uint32_t a = row + static_cast<uint32_t>(wfeat(fc) * stride);
    uint32_t x;
    if constexpr (RB == 1) {
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(x) : "r"(a));
    } else {
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(a));
    }
    return static_cast<int32_t>(x);
}
template <int RB>
__device__ __forceinline__ int32_t rank_value(const WalkCtx& c, int32_t fc) {
    return rank_at<RB>(c.row_saddr, c.row_stride, fc);
}

// N independent row-only walks advanced in lockstep until each reaches a leaf
// or a clock node (feat < 0, i.e. fc < 0).  Walks enter LOADED (key / fc
// describe node n).  A step whose child is a leaf (the parent's flag bits)
// synthesizes it -- {leaf position, packed index = grid root + position,
// kLeafFc} -- instead of loading it; lanes that do not advance reload the
// root (always in the window) so the loop stays branch-free.
template <bool kAllSmem, int RB, int N>
__device__ __forceinline__ void walkn(const WalkCtx& c, const uint32_t (&ra)[N], const TreeSrc (&s)[N],
                                      const bool (&v)[N], Walk (&w)[N]) {
    bool g[N];
    bool any = false;
#pragma unroll
    for (int h = 0; h < N; ++h) {
        g[h] = v[h] && w[h].fc >= 0;
        any |= g[h];
    }
    while (any) {
        int32_t x[N];
#pragma unroll
        for (int h = 0; h < N; ++h) x[h] = rank_at<RB>(ra[h], c.row_stride, g[h] ? w[h].fc : 0);
        any = false;
#pragma unroll
        for (int h = 0; h < N; ++h) {
            const int right = x[h] <= w[h].key ? 0 : 1;
            const int32_t nn = wchild(w[h].fc) + 8 * right;
            const bool lf = (w[h].fc >> right) & 1;
            Walk t{g[h] && !lf ? nn : 0, 0, 0};
            load_wnode<kAllSmem>(c, s[h], t);
            if (g[h]) {
                w[h].n = nn;
#if GD_WALK_LATE_LEAF
                w[h].key = t.key;  // a leaf's packed index is filled in after the loop
#else
                w[h].key = lf ? s[h].groot + (nn >> 3) : t.key;
#endif
                w[h].fc = lf ? kLeafFc : t.fc;
            }
            g[h] = g[h] && w[h].fc >= 0;
            any |= g[h];
        }
    }
#if GD_WALK_LATE_LEAF
#pragma unroll
    for (int h = 0; h < N; ++h) {
        if (v[h] && w[h].fc == kLeafFc) w[h].key = s[h].groot + (w[h].n >> 3);
    }
#endif
}

// Compare key of a clock node's test (see the header comment).
__device__ __forceinline__ uint2 test_mk(const Walk& w) {
    const uint32_t t = static_cast<uint32_t>(w.key);
    return wfeat(w.fc) == kFeatMem ? make_uint2(0xffffu, t) : make_uint2(0xffffffffu, (t << 16) | 0xffffu);
}


// Child `side` of node w, loaded (or synthesized when the parent flags it a leaf).
template <bool kAllSmem>
__device__ __forceinline__ Walk child_walk(const WalkCtx& c, const TreeSrc& s, const Walk& w, int side) {
    const int32_t nn = wchild(w.fc) + 8 * side;
    if ((w.fc >> side) & 1) return Walk{nn, s.groot + (nn >> 3), kLeafFc};
    Walk t{nn, 0, 0};
    load_wnode<kAllSmem>(c, s, t);
    return t;
}

// Records are written once and read once by the accumulate kernel: stream
// them past L2 (evict-first) so the models' nodes stay L2-resident.
__device__ __forceinline__ void store_rec(TreeRec* dst, const TreeRec& r) {
    __stcs(reinterpret_cast<int4*>(dst), make_int4(static_cast<int>(r.info), r.ref, r.ref2, static_cast<int>(r.pad)));
}

// Residue-table pool: the first 3/4 are per-CTA shares -- CTA b allocates
// from [b * R / grid, (b + 1) * R / grid) with a shared-memory counter (no
// global atomics) -- and a CTA whose share is used up takes from the last
// quarter through one global counter (CTAs' shares fill unevenly when the
// work items are few, e.g. the configs[4] 64-app batches).  Tables that fit
// in neither become FULL records.
struct PoolRegion {
    uint32_t* next;      // shared
    uint32_t end;
    uint32_t* ovf_next;  // global, zeroed per batch
    uint32_t ovf_base, cap;
};
__device__ __forceinline__ uint32_t pool_take(const PoolRegion& r, uint32_t n) {
    uint32_t idx = atomicAdd(r.next, n);
    if (idx + n <= r.end) return idx;
    idx = r.ovf_base + atomicAdd(r.ovf_next, n);
    return idx + n <= r.cap ? idx : 0xffffffffu;
}

__device__ __forceinline__ TreeSrc tree_src(const int4& te, bool all_smem) {
    TreeSrc s;
    s.wroot = te.x;
    s.groot = te.y;
    s.win = all_smem ? 0xffffffffu : static_cast<uint32_t>(te.z);
    s.saddr = static_cast<uint32_t>(te.w);
    return s;
}

// A root walk that stopped at a clock node, queued for resolution so the
// (divergent) residue walks run with full warps.
struct Job {
    int32_t n;   // the clock node (byte offset within the tree)
    int32_t t;   // tree
    int32_t e;   // the tree's entry in the stage table (roots, window, shared address)
    int32_t li;  // app within the tile
};
#ifndef GD_JOB_PAIR
#define GD_JOB_PAIR 0
#endif
#ifndef GD_JOB_CAP
#define GD_JOB_CAP 128
#endif
// Queued jobs per warp; a run starts once WalkParams::job_run (<= cap - 32)
// are queued, and at the end of a stage.
constexpr int kJobCap = GD_JOB_CAP;

// Resolve the queued jobs, one lane per job, depth-first: the clock node's
// children are walked row-only to their next event (leaf or clock node); a
// clock node at level < 4 adds a test (its right child is pushed, the left
// one walked next), a leaf is stored in its depth-4 slot.  One test between
// two leaves -> SM / MEM (no table); tests on up to 3 levels -> TABLE (the
// depth-4 layout compacted into one 128-byte slot); 4 levels -> TABLE4 (two
// slots); deeper -> FULL (ref = the first clock node, per-clock traversal in
// the accumulate kernel).  The walks between events run as an inner loop, so
// the warp's lanes (each on its own job) handle their events together, and
// a lane that finishes its job takes the next queued one at once: the run
// costs about the longest lane's SUM of jobs, not the sum over rounds of the
// longest job of each round of 32.  Out of line: reached from every
// walk-group width and the drain, one copy keeps the kernel in the I-cache.
template <bool kAllSmem, int RB>
__device__ __noinline__ void run_jobs(const WalkParams& p, const WalkCtx& c0, const int4* table, Job* jobs,
                                      int& count, int lane, TreeRec* out, int64_t tile0, const PoolRegion& region) {
    const int n_jobs = count;
    const unsigned lt = (1u << lane) - 1u;
    int next = min(32, n_jobs);  // jobs handed out (warp-uniform)
    int k = lane;
    bool has = k < n_jobs;
    WalkCtx c = c0;
    TreeSrc s{0, 0, 0u, 0u};
    Job jb{0, 0, 0, 0};
    Walk w0{0, 0, 0}, cur{0, 0, 0};
    uint2 t0 = make_uint2(0u, 0u);
    // Pending right children, a stack of at most 5: (byte offset << 8) | leaf << 7 | heap position.
    uint32_t st0 = 0, st1 = 0, st2 = 0, st3 = 0, st4 = 0, P = 1;
    int nst = 0;
    // The table is built in the 128-byte RTRec form, moved to the two-slot
    // RTRec4 form when a fourth test level appears and to a new four-slot
    // RTRec5 when a fifth does (both rare); L = the form's leaf depth.
    RTRec4* q = nullptr;
    uint32_t L = 3;
    uint32_t tmask = 1u, idx = 0;
    int maxlev = 0;
    int32_t lleaf = -1;
    // One leaf store in flight: its value load overlaps the next walk.
    double* pend_dst = nullptr;
    double pend_v = 0.0;
    auto put_leaf = [&](uint32_t pos, int32_t leaf_idx) {
        if (pend_dst) *pend_dst = pend_v;
        const uint32_t lev = 31u - __clz(pos + 1u);
        const uint32_t path = pos + 1u - (1u << lev);
        pend_dst = L == 4u   ? &q->leaf[path << (4u - lev)]
                   : L == 3u ? &reinterpret_cast<RTRec*>(q)->leaf[path << (3u - lev)]
                             : &reinterpret_cast<RTRec5*>(q)->leaf[path << (5u - lev)];
        pend_v = __ldg(&c.gnodes[leaf_idx].v);
    };
    auto start = [&]() {  // job k: its clock node, then the left child's walk
        jb = jobs[k];
        c.row_saddr = c0.row_saddr + static_cast<uint32_t>(jb.li * RB);
        s = tree_src(table[jb.e], kAllSmem);
        w0 = Walk{jb.n, 0, 0};
        load_wnode<kAllSmem>(c, s, w0);
        t0 = test_mk(w0);
#if GD_JOB_PAIR
        // Both children walked side by side to their next events: the right
        // one's walk is pushed standing on its event.
        Walk ab[2] = {child_walk<kAllSmem>(c, s, w0, 0), child_walk<kAllSmem>(c, s, w0, 1)};
        {
            const uint32_t ra[2] = {c.row_saddr, c.row_saddr};
            const TreeSrc ss[2] = {s, s};
            const bool vv[2] = {true, true};
            walkn<kAllSmem, RB, 2>(c, ra, ss, vv, ab);
        }
        st0 = (static_cast<uint32_t>(ab[1].n) << 8) | (wfeat(ab[1].fc) == kFeatLeaf ? 1u << 7 : 0u) | 2u;
        cur = ab[0];
#else
        st0 = (static_cast<uint32_t>(wchild(w0.fc) + 8) << 8) | (static_cast<uint32_t>((w0.fc >> 1) & 1) << 7) | 2u;
        cur = child_walk<kAllSmem>(c, s, w0, 0);
#endif
        nst = 1;
        P = 1u;
        q = nullptr;
        L = 3u;
        tmask = 1u;
        maxlev = 0;
        lleaf = -1;
    };
    if (has) start();
    while (__any_sync(kFull, has)) {
        bool fin = false;
        TreeRec r{0u, 0, 0, 0u};
        if (has) {
            while (cur.fc >= 0) {  // row-only steps to the next event
                const int32_t x = rank_value<RB>(c, cur.fc);
                const int right = x <= cur.key ? 0 : 1;
                const int32_t nn = wchild(cur.fc) + 8 * right;
                if ((cur.fc >> right) & 1) {
                    cur = Walk{nn, s.groot + (nn >> 3), kLeafFc};
                } else {
                    cur.n = nn;
                    load_wnode<kAllSmem>(c, s, cur);
                }
            }
            if (wfeat(cur.fc) == kFeatLeaf) {
                if (!q) {
                    if (P == 1u) {
                        lleaf = cur.key;
                    } else {  // P == 2 with no table: one test between two leaves
                        r.info = (wfeat(w0.fc) == kFeatMem ? kRecMem : kRecSm) | (static_cast<uint32_t>(w0.key) << 16);
                        r.ref = lleaf;
                        r.ref2 = cur.key;
                        fin = true;
                    }
                } else {
                    put_leaf(P, cur.key);
                }
                if (!fin) {
                    if (nst == 0) {  // the residue is complete: its table
                        const uint32_t D = static_cast<uint32_t>(maxlev) + 1u;  // 2 .. 5
                        // Leaves above the last level sit under always-left tests.
#pragma unroll
                        for (uint32_t z = 1; z < 31; ++z) {
                            if (z + 1u < (1u << D) && !((tmask >> z) & 1u))
                                reinterpret_cast<RTRec5*>(q)->test[z] = make_uint2(0u, 0u);
                            if ((z == 6 && D < 4) || (z == 14 && D < 5)) break;
                        }
                        r.ref = static_cast<int32_t>(idx);
                        if (L == 5u) {
                            r.info = kRecTable5;
                        } else if (L == 4u) {
                            r.info = kRecTable4;
                        } else {
                            reinterpret_cast<RTRec*>(q)->depth = D;
                            r.info = kRecTable;
                        }
                        fin = true;
                    } else {
                        const uint32_t e = st0;
                        st0 = st1;
                        st1 = st2;
                        st2 = st3;
                        st3 = st4;
                        --nst;
                        P = e & 127u;
                        const int32_t n = static_cast<int32_t>(e >> 8);
                        if ((e >> 7) & 1u) {
                            cur = Walk{n, s.groot + (n >> 3), kLeafFc};
                        } else {
                            cur = Walk{n, 0, 0};
                            load_wnode<kAllSmem>(c, s, cur);
                        }
                    }
                }
            } else {  // a clock node at heap position P
                const int lev = 31 - __clz(static_cast<int>(P) + 1);
                uint32_t idx5 = 0;
                if (lev >= p.res_levels || (!q && (idx = pool_take(region, 2u)) == 0xffffffffu) ||
                    (lev == 4 && L == 4u && (idx5 = pool_take(region, 4u)) == 0xffffffffu)) {
                    r.info = kRecFull;
                    r.ref = s.groot + (w0.n >> 3);
                    fin = true;
                } else {
                    if (!q) {
                        q = reinterpret_cast<RTRec4*>(p.pool + idx);
                        q->test[0] = t0;
                        if (lleaf >= 0) put_leaf(1u, lleaf);
                    }
                    if (lev == 3 && L == 3u) {  // fourth level: depth-3 leaf slot k becomes depth-4 slot 2k
                        if (pend_dst) *pend_dst = pend_v;
                        pend_dst = nullptr;
                        RTRec* t = reinterpret_cast<RTRec*>(q);
                        double lv[8];
#pragma unroll
                        for (int z = 0; z < 8; ++z) lv[z] = t->leaf[z];
#pragma unroll
                        for (int z = 0; z < 8; ++z) q->leaf[2 * z] = lv[z];
                        L = 4u;
                    }
                    if (lev == 4 && L == 4u) {  // fifth level: move to four new slots, leaf k -> 2k
                        if (pend_dst) *pend_dst = pend_v;
                        pend_dst = nullptr;
                        RTRec5* u = reinterpret_cast<RTRec5*>(p.pool + idx5);
#pragma unroll
                        for (int z = 0; z < 15; ++z) u->test[z] = q->test[z];
#pragma unroll
                        for (int z = 0; z < 16; ++z) u->leaf[2 * z] = q->leaf[z];
                        q = reinterpret_cast<RTRec4*>(u);
                        idx = idx5;
                        L = 5u;
                    }
                    reinterpret_cast<RTRec5*>(q)->test[P] = test_mk(cur);
                    tmask |= 1u << P;
                    maxlev = max(maxlev, lev);
                    st4 = st3;
                    st3 = st2;
                    st2 = st1;
                    st1 = st0;
                    st0 = (static_cast<uint32_t>(wchild(cur.fc) + 8) << 8) |
                          (static_cast<uint32_t>((cur.fc >> 1) & 1) << 7) | (2u * P + 2u);
                    ++nst;
                    cur = child_walk<kAllSmem>(c, s, cur, 0);
                    P = 2u * P + 1u;
                }
            }
            if (fin) store_rec(out + rec_index(jb.t, tile0 + jb.li, p.n_apps), r);
        }
        // Lanes that finished a job take the next queued ones.
        const unsigned fm = __ballot_sync(kFull, fin);
        if (fm) {
            if (fin) {
                k = next + __popc(fm & lt);
                has = k < n_jobs;
                if (has) start();
            }
            next += __popc(fm);
        }
    }
    if (pend_dst) *pend_dst = pend_v;
    __syncwarp();
    count = 0;
}

// Queue the walk of one tree if it stopped at a clock node, else store its
// constant record; run a round of jobs once 32 are pending.
template <bool kAllSmem, int RB>
__device__ __forceinline__ void finish_walk(const WalkParams& p, const WalkCtx& c0, const int4* table, Job* jobs,
                                            int& count, int lane, bool v, const Walk& w, int32_t t, int32_t e,
                                            int li, TreeRec* out, int64_t tile0, const PoolRegion& region) {
    const bool job = v && wfeat(w.fc) != kFeatLeaf;
    if (v && !job) store_rec(out + rec_index(t, tile0 + li, p.n_apps), TreeRec{kRecConst, w.key, 0, 0u});
    const unsigned m = __ballot_sync(kFull, job);
    if (job) jobs[count + __popc(m & ((1u << lane) - 1u))] = Job{w.n, t, e, li};
    count += __popc(m);
    __syncwarp();
    if (count >= p.job_run) run_jobs<kAllSmem, RB>(p, c0, table, jobs, count, lane, out, tile0, region);
}

constexpr int kStageTrees = 128;  // trees per stage (table entries per buffer)
constexpr int kMaxTileApps = 512;  // apps per walk tile (16 groups of 32)
#ifndef GD_WALK_NW
#define GD_WALK_NW 4  // independent walks per lane in the root-walk loop
#endif
#ifndef GD_WALK_ADAPT
#define GD_WALK_ADAPT 1  // narrower walk groups for a stage's last trees
#endif

// One stage of the CTA's schedule.
struct Stage {
    int32_t item, q0, q1, valid;
};

struct ItemInfo {
    int32_t tile, model, p0, p1;
};

// Items are handed out in chunks of consecutive items by one global counter,
// so no CTA idles while others still have work (trained ensembles' items
// differ widely in cost).  Default order (model, split, tile), one item per
// fetch: the CTAs in flight at any moment work on a few consecutive tree
// ranges (megabytes: L2-resident even for models larger than L2, so each
// range is read from HBM about once per batch, not once per tile); the
// alternative (tile, model, split) order lets a chunk's items share their
// tile's staged ranks.
__device__ __forceinline__ ItemInfo item_info(const WalkParams& p, int32_t it) {
    ItemInfo r;
    int32_t split;
    if (p.split_major) {
        const int32_t k = it / p.tiles;
        r.tile = it - k * p.tiles;
        r.model = k / p.splits;
        split = k - r.model * p.splits;
    } else {
        const int32_t per_tile = 2 * p.splits;
        r.tile = it / per_tile;
        const int32_t k = it - r.tile * per_tile;
        r.model = k / p.splits;
        split = k - r.model * p.splits;
    }
    const int64_t pairs = (p.n_trees[r.model] + 1) >> 1;
    r.p0 = static_cast<int32_t>(pairs * split / p.splits);
    r.p1 = static_cast<int32_t>(pairs * (split + 1) / p.splits);
    return r;
}


__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Bounded spin: a barrier that never completes is a bug -- trap (the launch
// fails) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    for (uint32_t spins = 0;; ++spins) {
        uint32_t done;
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
        if (spins > (1u << 26)) __trap();
    }
}
// Non-blocking probe of a barrier phase.
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Warp 0 (all lanes, uniform result): plan the next stage after cursor (it,
// q), advancing the cursor, and start loading it into buffer `buf_saddr`.
// Lane l sizes pair q + l; a stage is the longest prefix of up to 32 pairs
// whose windows fit one buffer (at least one pair).  The same loads give the
// stage's tree table -- lane l fills the entries {walk root, grid root, window
// nodes, shared address} of trees 2(q+l) and 2(q+l)+1 -- so planning and
// issuing cost one round trip.  Whole trees are contiguous, so with kAllSmem
// the stage is one bulk copy; otherwise each window is copied on its own.
// Arms the buffer's barrier (or arrives on it for an invalid stage).
template <bool kAllSmem>
__device__ void plan_stage(const WalkParams& p, int32_t it_end, int32_t& it, int32_t& chunk_end, int32_t& q, int lane,
                           uint32_t buf_saddr, uint32_t bar, int4* table, Stage* desc) {
    while (it < it_end) {
        const ItemInfo ii = item_info(p, it);
        if (q < ii.p0) q = ii.p0;
        if (q >= ii.p1) {
            if (++it >= chunk_end) {  // next chunk
                uint32_t nx = 0;
                if (lane == 0) nx = gridDim.x + atomicAdd(p.item_next, 1u);  // chunks past the first wave
                it = static_cast<int32_t>(__shfl_sync(kFull, nx, 0)) * p.chunk;
                chunk_end = min(it + p.chunk, it_end);
            }
            q = -1;
            continue;
        }
        const int32_t nt = p.n_trees[ii.model];
        const int32_t* wroots = p.wroots[ii.model];
        const int32_t* roots = p.roots[ii.model];
        const int32_t* wint = p.wint[ii.model];
        const int32_t pr = q + lane;
        int32_t w = 1 << 20;  // > any stage; 32 of them cannot overflow
        int32_t r0 = 0, r1 = 0, g0 = 0, g1 = 0, wa = 0, wb = 0;
        if (pr < ii.p1) {
            r0 = __ldg(wroots + 2 * pr);
            r1 = __ldg(wroots + min(2 * pr + 1, nt));
            g0 = __ldg(roots + 2 * pr);
            g1 = 2 * pr + 1 < nt ? __ldg(roots + 2 * pr + 1) : 0;
            wa = min(__ldg(wint + 2 * pr), p.win_nodes);
            wb = 2 * pr + 1 < nt ? min(__ldg(wint + 2 * pr + 1), p.win_nodes) : 0;
            w = wa + wb;
        }
        int32_t incl = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t o = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += o;
        }
        const bool fits = lane == 0 || (incl <= p.stage_nodes && 2 * (lane + 1) <= kStageTrees);
        const int n = __popc(__ballot_sync(kFull, fits));
        const Stage st{it, q, q + n, 1};
        q += n;
        const WNode* nodes = p.wnodes[ii.model];
        if (lane < n) {
            const uint32_t off = 8u * static_cast<uint32_t>(incl - w);
            const int k = 2 * lane;  // table index of tree 2 * pr
            table[k] = make_int4(r0, g0, wa, static_cast<int>(buf_saddr + off));
            if (2 * pr + 1 < nt) table[k + 1] = make_int4(r1, g1, wb, static_cast<int>(buf_saddr + off + 8u * wa));
            // Each tree's window is its own bulk copy (windows are prefixes).
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_g2s(buf_saddr + off, nodes + r0, 8u * static_cast<uint32_t>(wa), bar);
            if (2 * pr + 1 < nt && wb > 0) bulk_g2s(buf_saddr + off + 8u * wa, nodes + r1, 8u * static_cast<uint32_t>(wb), bar);
        }
        const uint32_t total = 8u * static_cast<uint32_t>(__shfl_sync(kFull, incl, n - 1));
        __syncwarp();  // the table entries are visible before lane 0's arrive releases them
        if (lane == 0) {
            *desc = st;  // published by the barrier's phase completion
            mbar_expect_tx(bar, total);
        }
        return;
    }
    if (lane == 0) {
        *desc = Stage{0, 0, 0, 0};
        mbar_arrive(bar);
    }
}

// Shared layout: barriers + stage descriptors | buffer 0 | buffer 1 | ranks
// [n_cols][tile_apps] u16 | per-warp job queues | stage tree tables.
__host__ __device__ constexpr size_t walk_jobs_bytes(int warps) {
    return static_cast<size_t>(warps) * kJobCap * sizeof(Job);
}
__host__ __device__ constexpr size_t walk_rank_bytes(int n_cols, int tile_apps, int rb) {
    return (static_cast<size_t>(n_cols) * tile_apps * rb + 15) & ~static_cast<size_t>(15);
}

// Grid: persistent CTAs; blockDim = 64 * groups (two warps per group of 32
// apps, taking the even / odd trees of every stage).
//
// RB = 1 (every feature of both models has <= 255 distinct thresholds):
// 8-bit ranks, tiles of 1024 apps -- each warp walks two blocks of 32 apps
// (lane = apps li and li + 512), so a stage's trees are staged once per 1024
// apps and a lane has twice the walks in flight.
//
// kLazy: warp 0 refills a released buffer between its own walk groups rather
// than waiting for the slowest warp before it walks (stages of many trees).
template <bool kAllSmem, int RB, bool kLazy>
__global__ void __launch_bounds__(512, 1) grid_walk_kernel(const __grid_constant__ WalkParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TA = p.tile_apps, groups = TA >> 5, NSUB = p.n_subs;
    const int group = warp % groups, sub = warp / groups;
    const size_t buf_bytes = static_cast<size_t>(p.stage_nodes) * 8;
    const int NB = p.n_bufs;
    // Header: full[b] at bar0 + 8b, empty[b] at bar0 + 32 + 8b, stage
    // descriptors at +64 (NB <= 4).
    Stage* desc = reinterpret_cast<Stage*>(smem + 64);
    const uint32_t bar0 = smem_addr(smem), bufs0 = smem_addr(smem + 128);
    unsigned char* srank = smem + 128 + NB * buf_bytes;
    unsigned char* after_ranks = smem + 128 + NB * buf_bytes + walk_rank_bytes(p.n_cols, TA, RB);
    Job* jobs = reinterpret_cast<Job*>(after_ranks) + warp * kJobCap;
    int4* tables = reinterpret_cast<int4*>(after_ranks + walk_jobs_bytes(blockDim.x >> 5));
    uint32_t* pool_next = reinterpret_cast<uint32_t*>(tables + NB * kStageTrees);
    PoolRegion region;
    region.next = pool_next;
    const uint32_t shared_cap = p.pool_cap / 4 * 3;
    region.end = static_cast<uint32_t>(static_cast<uint64_t>(blockIdx.x + 1) * shared_cap / gridDim.x);
    region.ovf_next = p.pool_count;
    region.ovf_base = shared_cap;
    region.cap = p.pool_cap;
    WTRACE(0);
    const int32_t it_end = p.n_items;
    int32_t* first_item = reinterpret_cast<int32_t*>(pool_next + 1);

    // full[b]: thread 0's arrive + the stage's TMA bytes; empty[b]: one arrive
    // per warp once done with the stage.  Warps run decoupled; thread 0
    // refills a buffer (NB - 1 stages ahead) only after every warp released it.
    const int nwarps = blockDim.x >> 5;
    int32_t cur_it = 0, cur_end = 0, cur_q = -1;  // warp 0's schedule cursor (item, end of its chunk, pair)
    auto produce = [&](int j) {  // warp 0: plan stage j into buffer j % NB
        const int b = j % NB;
        plan_stage<kAllSmem>(p, it_end, cur_it, cur_end, cur_q, lane, bufs0 + static_cast<uint32_t>(b * buf_bytes), bar0 + 8 * b,
                             tables + b * kStageTrees, desc + b);
    };
    if (threadIdx.x == 0) {
        *pool_next = static_cast<uint32_t>(static_cast<uint64_t>(blockIdx.x) * shared_cap / gridDim.x);
        *first_item = static_cast<int32_t>(blockIdx.x) * p.chunk;  // the first chunk is static: no atomic on the way in
        for (int b = 0; b < NB; ++b) {
            mbar_init(bar0 + 8 * b, 1);
            mbar_init(bar0 + 32 + 8 * b, nwarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int32_t it_begin = *first_item;
    cur_it = it_begin;
    cur_end = min(it_begin + p.chunk, it_end);
    if (warp == 0) {
        for (int j = 0; j + 1 < NB; ++j) produce(j);
    }
    int32_t row_tile = -1, row_model = -1;
    // The tile's ranks ([col][app], already in that layout in global memory:
    // a contiguous, coalesced 16-byte copy) by threads [t0, blockDim.x).
    auto stage_ranks = [&](int32_t tile, int32_t model, int t0) {
        const int64_t tiles = (p.n_apps + TA - 1) / TA;
        const int4* src = reinterpret_cast<const int4*>(
            p.ranks + ((static_cast<int64_t>(model) * tiles + tile) * p.n_cols) * TA * RB);
        const uint32_t dst = smem_addr(srank);
        const int n16 = p.n_cols * TA * RB / 16;
        // cp.async: every 16-byte piece in flight at once (a load -> store
        // loop would serialise one L2 round trip per iteration).
        for (int i = static_cast<int>(threadIdx.x) - t0; i >= 0 && i < n16; i += blockDim.x - t0) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * static_cast<uint32_t>(i)),
                         "l"(src + i)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        row_tile = tile;
        row_model = model;
    };
    WTRACE(1);
    if (it_begin < it_end) {
        // The first item's ranks load while its first stage is planned and in
        // flight: warp 0 is busy planning, so the other warps copy them.
        const ItemInfo i0 = item_info(p, it_begin);
        stage_ranks(i0.tile, i0.model, nwarps > 1 ? 32 : 0);
        __syncthreads();
    }
    for (int k = 0;; ++k) {
        const int buf = k % NB;
        // Warp 0 refills the buffer of stage k - 1 with stage k + NB - 1 once
        // every warp released it.  kLazy: it probes that barrier between its
        // own walk groups of stage k (blocking only after them), so it is not
        // held back by the slowest warp of stage k - 1; otherwise it waits
        // before walking.
        if (warp == 0 && (!kLazy || k == 0)) {
            if (k >= 1) mbar_wait(bar0 + 32 + 8 * ((k - 1) % NB), static_cast<uint32_t>((k - 1) / NB) & 1u);
            produce(k + NB - 1);
            __syncwarp();
        }
        bool produced = !(kLazy && warp == 0 && k >= 1);
        auto poll_produce = [&](bool block) {
            if (!kLazy || produced) return;
            const uint32_t eb = bar0 + 32 + 8 * ((k - 1) % NB), ep = static_cast<uint32_t>((k - 1) / NB) & 1u;
            if (block) mbar_wait(eb, ep);
            else if (!mbar_test(eb, ep)) return;
            produce(k + NB - 1);
            __syncwarp();
            produced = true;
        };
        if (k == 0) WTRACE(2);
        mbar_wait(bar0 + 8 * buf, static_cast<uint32_t>(k / NB) & 1u);
        if (k == 0) WTRACE(3);
        const Stage s = desc[buf];
        if (!s.valid) break;  // every later stage is invalid too; no warp waits on one
        const ItemInfo ii = item_info(p, s.item);
        const int64_t tile0 = static_cast<int64_t>(ii.tile) * TA;
        const int n_here = static_cast<int>(min(static_cast<int64_t>(TA), p.n_apps - tile0));
        if (ii.tile != row_tile || ii.model != row_model) {
            __syncthreads();  // every warp is done with the previous tile's ranks
            stage_ranks(ii.tile, ii.model, 0);
            __syncthreads();
        }

        // Lane apps: li (and li + 512 with 1024-app tiles).
        constexpr int APL = RB == 1 ? 2 : 1;
        const int li = group * 32 + lane;
        WalkCtx c0;  // rank base of the tile (jobs add their own app)
        c0.wnodes = p.wnodes[ii.model];
        c0.gnodes = p.gnodes[ii.model];
        c0.row_saddr = smem_addr(srank);
        c0.row_stride = TA * RB;
        const int32_t nt = p.n_trees[ii.model];
        TreeRec* out = p.rec[ii.model];
        int count = 0;
        // This warp walks the stage's trees t = 2*q0 + sub + NSUB*k, up to
        // NW side by side; a stage with fewer trees left (e.g. one pair of
        // configs[3]'s depth-12 trees) takes a narrower group so no walk
        // slot idles.
        const int4* table = tables + buf * kStageTrees;
        constexpr int NW = GD_WALK_NW / APL;  // trees per group
        const int32_t t_last = min(2 * s.q1, nt) - 1;
        // One group: trees t0, t0 + NSUB, ... (G / APL of them) for each of
        // the lane's APL apps -- G independent walks.
        auto group = [&](int32_t t0, auto nw_tag) {
            constexpr int G = decltype(nw_tag)::value * APL;
            TreeSrc src[G];
            uint32_t ra[G];
            int32_t tt[G];
            int la[G];
            bool vv[G];
            Walk w[G];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                tt[h] = t0 + NSUB * (h / APL);
                la[h] = li + 512 * (h % APL);
                vv[h] = la[h] < n_here && tt[h] <= t_last;
                ra[h] = c0.row_saddr + static_cast<uint32_t>((vv[h] ? la[h] : 0) * RB);
                const int4 e = table[min(tt[h], t_last) - 2 * s.q0];
                src[h].wroot = e.x;
                src[h].groot = e.y;
                src[h].win = kAllSmem ? 0xffffffffu : static_cast<uint32_t>(e.z);
                src[h].saddr = static_cast<uint32_t>(e.w);
                w[h] = Walk{0, 0, 0};
                load_wnode<kAllSmem>(c0, src[h], w[h]);
            }
            walkn<kAllSmem, RB, G>(c0, ra, src, vv, w);
#pragma unroll
            for (int h = 0; h < G; ++h)
                finish_walk<kAllSmem, RB>(p, c0, table, jobs, count, lane, vv[h], w[h], tt[h],
                                          min(tt[h], t_last) - 2 * s.q0, la[h], out, tile0, region);
        };
        int32_t t0 = 2 * s.q0 + sub;
#if GD_WALK_ADAPT
        for (; t0 + NSUB * (NW - 1) <= t_last; t0 += NW * NSUB) {
            group(t0, std::integral_constant<int, NW>{});
            poll_produce(false);
        }
#else
        for (; t0 <= t_last; t0 += NW * NSUB) group(t0, std::integral_constant<int, NW>{});
#endif
        const int32_t rest = t0 <= t_last ? (t_last - t0) / NSUB + 1 : 0;  // warp-uniform
        if (rest > 2) group(t0, std::integral_constant<int, NW>{});
        else if (rest == 2) group(t0, std::integral_constant<int, (NW < 2 ? NW : 2)>{});
        else if (rest == 1) group(t0, std::integral_constant<int, 1>{});
        if (k == 0) WTRACE(4);
        poll_produce(false);
        if (count > 0) run_jobs<kAllSmem, RB>(p, c0, table, jobs, count, lane, out, tile0, region);
        poll_produce(true);
        if (k == 0) WTRACE(5);
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 32 + 8 * buf);  // this warp is done with buffer `buf`
    }
}

// Ranks of the batch's rows for both models, laid out as the walk kernel
// stages them: ranks[m][tile][f][app in tile] (tile = TA apps), value =
// #{thresholds of model m on feature f that are < x} (NaN: their count); the
// time model sees the time-encoded categorical columns.  grid_rank_kernel:
// consecutive threads take consecutive apps of one (m, tile, f), so the stores
// are coalesced.  Both rank kernels also zero `zero[0, n_zero)` (the batch's
// walk / accumulate counters).
//
// Small batches (latency mode): a warp per rank, 32-ary search -- each round
// samples the last threshold of 32 equal chunks and keeps the chunk holding
// the boundary, so ~3 dependent loads replace ~13 of the binary search.
template <class RT>
__global__ void __launch_bounds__(256) grid_rank_warp_kernel(
    const double* __restrict__ rows, const double* __restrict__ cat_t, const int32_t* __restrict__ cat_cols,
    int32_t n_cat, int64_t a0, int32_t n_apps, int32_t F, int32_t TA, const double* __restrict__ thr_e,
    const int32_t* __restrict__ off_e, const double* __restrict__ thr_t, const int32_t* __restrict__ off_t,
    RT* __restrict__ ranks, uint32_t* __restrict__ zero, int32_t n_zero) {
    const int lane = threadIdx.x & 31;
    for (int64_t z = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; z < n_zero;
         z += static_cast<int64_t>(gridDim.x) * blockDim.x)
        zero[z] = 0u;
    const int64_t tiles = (n_apps + TA - 1) / TA;
    const int64_t total = 2LL * tiles * F * TA;
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (i >= total) return;
    const int64_t plane = i / TA;
    const int64_t la = (plane / F % tiles) * TA + (i - plane * TA);
    if (la >= n_apps) return;
    const int f = static_cast<int>(plane % F);
    const int m = static_cast<int>(plane / (F * tiles));
    double x = __ldg(rows + (a0 + la) * F + f);
    if (m == 1) {
        for (int k = 0; k < n_cat; ++k)
            if (__ldg(cat_cols + k) == f) x = __ldg(cat_t + (a0 + la) * n_cat + k);
    }
    const double* thr = m ? thr_t : thr_e;
    const int32_t* off = m ? off_t : off_e;
    const int32_t o = __ldg(off + f);
    int lo = 0, hi = __ldg(off + f + 1) - o;  // answer in [lo, hi]
    if (x != x) lo = hi;
    while (lo < hi) {
        const int len = hi - lo;
        const int step = (len + 31) >> 5;
        const int last = min(lo + (lane + 1) * step, hi) - 1;  // last index of chunk `lane`
        const bool in = lo + lane * step < hi;
        const unsigned below = __ballot_sync(kFull, in && __ldg(thr + o + last) < x);
        const int c = __popc(below);  // chunks entirely below x (a prefix: thresholds sorted)
        lo = min(lo + c * step, hi);
        hi = min(hi, lo + step);
        if (step == 1) break;  // chunks of one: lo is the count
    }
    if (lane == 0) ranks[i] = static_cast<RT>(lo);
}

// Large batches: a block per (model, tile, feature, 256 apps).  The block
// stages 256 evenly spaced samples of the feature's sorted thresholds (or all
// of them when there are at most 256) in shared memory; a rank is then 8
// shared-memory steps plus a short global binary search inside the bracketing
// sample interval (~5 dependent loads instead of ~13).  Same count as rank_of.
constexpr int kRankSamples = 256;
template <class RT>
__global__ void __launch_bounds__(256) grid_rank_sampled_kernel(
    const double* __restrict__ rows, const double* __restrict__ cat_t, const int32_t* __restrict__ cat_cols,
    int32_t n_cat, int64_t a0, int32_t n_apps, int32_t F, int32_t TA, const double* __restrict__ thr_e,
    const int32_t* __restrict__ off_e, const double* __restrict__ thr_t, const int32_t* __restrict__ off_t,
    RT* __restrict__ ranks, uint32_t* __restrict__ zero, int32_t n_zero) {
    __shared__ double sample[kRankSamples];
    if (blockIdx.x == 0) {
        for (int z = threadIdx.x; z < n_zero; z += blockDim.x) zero[z] = 0u;
    }
    const int halves = TA / 256;
    const int64_t tiles = (n_apps + TA - 1) / TA;
    const int64_t unit = blockIdx.x;  // ((m * tiles + tile) * F + f) * halves + h
    const int h = static_cast<int>(unit % halves);
    const int64_t plane = unit / halves;  // (m * tiles + tile) * F + f
    const int f = static_cast<int>(plane % F);
    const int64_t tile = plane / F % tiles;
    const int m = static_cast<int>(plane / (F * tiles));
    const double* thr = m ? thr_t : thr_e;
    const int32_t* off = m ? off_t : off_e;
    const int32_t o = __ldg(off + f), n = __ldg(off + f + 1) - o;
    const bool all = n <= kRankSamples;
    const int ns = all ? n : kRankSamples;
    // sample k = thr[q_k], q_k = (k + 1) * n / (kRankSamples + 1) (strictly increasing for n > kRankSamples)
    for (int k = threadIdx.x; k < ns; k += blockDim.x) {
        const int32_t q = all ? k : static_cast<int32_t>((static_cast<int64_t>(k) + 1) * n / (kRankSamples + 1));
        sample[k] = __ldg(thr + o + q);
    }
    __syncthreads();
    const int64_t la = tile * TA + static_cast<int64_t>(h) * 256 + threadIdx.x;
    if (la >= n_apps) return;
    double x = __ldg(rows + (a0 + la) * F + f);
    if (m == 1) {
        for (int k = 0; k < n_cat; ++k)
            if (__ldg(cat_cols + k) == f) x = __ldg(cat_t + (a0 + la) * n_cat + k);
    }
    int r;
    if (x != x) {
        r = n;
    } else {
        int lo = 0, hi = ns;  // c = #{samples < x}
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sample[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        if (all) {
            r = lo;
        } else {
            const int c = lo;
            const int32_t b0 = c == 0 ? 0 : static_cast<int32_t>(static_cast<int64_t>(c) * n / (kRankSamples + 1)) + 1;
            const int32_t b1 = c == kRankSamples ? n
                                                 : static_cast<int32_t>((static_cast<int64_t>(c) + 1) * n / (kRankSamples + 1));
            r = b0 + rank_of(thr + o + b0, b1 - b0, x);
        }
    }
    ranks[plane * TA + static_cast<int64_t>(h) * 256 + threadIdx.x] = static_cast<RT>(r);
}

template <class RT>
__global__ void grid_rank_kernel(const double* __restrict__ rows, const double* __restrict__ cat_t,
                                 const int32_t* __restrict__ cat_cols, int32_t n_cat, int64_t a0, int32_t n_apps,
                                 int32_t F, int32_t TA, const double* __restrict__ thr_e,
                                 const int32_t* __restrict__ off_e, const double* __restrict__ thr_t,
                                 const int32_t* __restrict__ off_t, RT* __restrict__ ranks, uint32_t* __restrict__ zero, int32_t n_zero) {
    for (int64_t z = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; z < n_zero;
         z += static_cast<int64_t>(gridDim.x) * blockDim.x)
        zero[z] = 0u;
    const int64_t tiles = (n_apps + TA - 1) / TA;
    const int64_t total = 2LL * tiles * F * TA;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t plane = i / TA;  // (m * tiles + tile) * F + f
        const int64_t la = (plane / F % tiles) * TA + (i - plane * TA);
        if (la >= n_apps) continue;
        const int f = static_cast<int>(plane % F);
        const int m = static_cast<int>(plane / (F * tiles));
        double x = __ldg(rows + (a0 + la) * F + f);
        if (m == 1) {
            for (int k = 0; k < n_cat; ++k)
                if (__ldg(cat_cols + k) == f) x = __ldg(cat_t + (a0 + la) * n_cat + k);
        }
        const double* thr = m ? thr_t : thr_e;
        const int32_t* off = m ? off_t : off_e;
        const int32_t o = __ldg(off + f);
        ranks[i] = static_cast<RT>(rank_of(thr + o, __ldg(off + f + 1) - o, x));
    }
}

// ---------------------------------------------------------------------------
// K2b: accumulate + select.
// ---------------------------------------------------------------------------

// Resident CTAs per SM the accumulate kernel is compiled for (register cap
// 65536 / (128 * N)).
#ifndef GD_ACC_MIN_BLOCKS
#define GD_ACC_MIN_BLOCKS 6
#endif
constexpr int64_t kRankWarpLimit = 1 << 16;  // ranks per batch below which a warp takes each
#ifndef GD_ACC_WARPS
#define GD_ACC_WARPS 4
#endif
constexpr int kAccWarps = GD_ACC_WARPS;  // 2 warp pairs = 2 apps in flight per CTA
constexpr int kAccThreads = kAccWarps * 32;

// Per-warp shared region of the two-stage prefetch ring: record slots
// [RR+1][32] | leaf values [RS+1][32] | right leaf values [RS+1][32] |
// residue-table slots [RS+1][kSide] | overflow slot | row.  Records are
// fetched RR groups ahead, what they point at RS groups ahead (RS < RR), as
// one cp.async commit group per iteration; an iteration waits only for the
// group that carries its own side data and the records the next side fetch
// reads, so kWait younger groups stay in flight.
#ifndef GD_SIDE_SLOTS
#define GD_SIDE_SLOTS 8
#endif
constexpr int kSide = GD_SIDE_SLOTS;  // residue tables staged per group (more: copied on demand)
template <int RR, int RS>
struct RingT {
    static_assert(RS >= 1 && RR > RS, "records must run ahead of the side data");
    static constexpr int kRecAhead = RR;
    static constexpr int kSideAhead = RS;
    static constexpr int kWait = (RS - 1) < (RR - RS - 1) ? (RS - 1) : (RR - RS - 1);
    static constexpr int kMeta = 0;
    static constexpr int kVal = kMeta + (RR + 1) * 32 * 16;
    static constexpr int kRv = kVal + (RS + 1) * 32 * 8;
    static constexpr int kSideOff = kRv + (RS + 1) * 32 * 8;
    static constexpr int kOvf = kSideOff + (RS + 1) * kSide * 128;
    static constexpr int kRow = kOvf + 512;
    __host__ __device__ static constexpr int rs(int g) { return g % (RR + 1); }  // record slot
    __host__ __device__ static constexpr int ss(int g) { return g % (RS + 1); }  // side slot
};
#ifndef GD_ACC_RR
#define GD_ACC_RR 2
#endif
#ifndef GD_ACC_RS
#define GD_ACC_RS 1
#endif
#ifndef GD_SLICED_RING
#define GD_SLICED_RING 8, 4
#endif
using AccRing = RingT<GD_ACC_RR, GD_ACC_RS>;  // main kernel (shared memory bound)
using SlicedRing = RingT<GD_SLICED_RING>;  // latency mode (few warps: deep prefetch)
template <class RG>
__host__ __device__ constexpr size_t acc_smem_per_warp(int n_cols) {
    return static_cast<size_t>(RG::kRow) + static_cast<size_t>((n_cols + 1) & ~1) * 8;
}
__host__ __device__ constexpr size_t acc_smem_per_pair(int cpl) { return 32 * static_cast<size_t>(cpl) * 8; }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

struct AccModel {
    const PNode* nodes;
    const TreeRec* rec;
    int32_t n_trees;
};

// Full per-candidate traversal from node n (grid nodes) with a packed clock:
// predict_row on the substituted row (models.cpp:71-78).  (Walking all CPL
// clocks in lockstep, inline or out of line, costs the hot loop registers:
// spills, +40 % accumulate time at configs[3].)
__device__ __forceinline__ double eval_full_packed(const PNode* __restrict__ nodes, int32_t n, const double* row,
                                                   unsigned ck) {
    const double sm = static_cast<double>(ck >> 16), mem = static_cast<double>(ck & 0xffffu);
    double v;
    int32_t feat, aux;
    while (true) {
        load_node(nodes, n, v, feat, aux);
        if (feat == kFeatLeaf) return v;
        const double x = feat >= 0 ? row[feat] : (feat == kFeatSm ? sm : mem);
        n = (x <= v) ? aux : aux + 1;
    }
}

// Stage 1 of the ring: the record of tree g*32 + lane.
template <class RG>
__device__ __forceinline__ void issue_rec(const AccModel& m, int64_t la, int64_t n_apps, int g, int lane,
                                          uint32_t ws) {
    const int32_t t = g * 32 + lane;
    if (t < m.n_trees) {
        cp_async16(ws + RG::kMeta + static_cast<uint32_t>((RG::rs(g) * 32 + lane) * 16),
                   m.rec + rec_index(t, la, n_apps));
    }
}

// Stage 2: what the record points at -- leaf values (CONST, SM / MEM) or the
// residue table (staged into slot = rank among the group's tables).
template <class RG>
__device__ __forceinline__ void issue_side(const AccModel& m, const RTRec* __restrict__ pool, int g, int lane,
                                           uint32_t ws) {
    const int32_t t = g * 32 + lane;
    uint32_t kind = kRecFull, ref = 0, ref2 = 0;
    if (t < m.n_trees) {
        const uint32_t a = ws + RG::kMeta + static_cast<uint32_t>((RG::rs(g) * 32 + lane) * 16);
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(kind), "=r"(ref) : "r"(a));
        ref2 = lds_u32(a + 8u);
        kind &= 7u;
    }
    const unsigned tm = __ballot_sync(kFull, kind == kRecTable);
    const uint32_t vslot = static_cast<uint32_t>((RG::ss(g) * 32 + lane) * 8);
    if (kind == kRecConst || kind == kRecSm || kind == kRecMem) {
        cp_async8(ws + RG::kVal + vslot, &m.nodes[static_cast<int32_t>(ref)].v);
        if (kind != kRecConst) cp_async8(ws + RG::kRv + vslot, &m.nodes[static_cast<int32_t>(ref2)].v);
    } else if (kind == kRecTable) {
        const int slot = __popc(tm & ((1u << lane) - 1u));
        if (slot < kSide) {
            const unsigned char* src = reinterpret_cast<const unsigned char*>(pool + ref);
            const uint32_t dst = ws + RG::kSideOff + static_cast<uint32_t>((RG::ss(g) * kSide + slot) * 128);
#pragma unroll
            for (int k = 0; k < 8; ++k) cp_async16(dst + 16 * k, src + 16 * k);
        }
    }
}

template <int CPL>
__device__ __forceinline__ void add_const(double (&acc)[CPL], double v) {
#pragma unroll
    for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], v);
}

// Residue table at shared address sb, depth D (2 or 3).
template <int CPL, int D>
__device__ __forceinline__ void add_table(double (&acc)[CPL], const unsigned (&ck)[CPL], uint32_t sb) {
    const uint2 t0 = lds_u2(sb);
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
        uint32_t n = 1u + ((ck[i] & t0.x) > t0.y ? 1u : 0u);
#pragma unroll
        for (int d = 1; d < D; ++d) {
            const uint2 t = lds_u2(sb + n * 8u);
            n = 2u * n + 1u + ((ck[i] & t.x) > t.y ? 1u : 0u);
        }
        acc[i] = __dadd_rn(acc[i], lds_f64(sb + 64u + ((n - ((1u << D) - 1u)) << (3 - D)) * 8u));
    }
}

#if GD_TABLE_KEYS
// Lanes whose clocks share one memory clock (mem_l): every test of a table
// becomes one unsigned compare `ck > K` -- a core-clock test keeps its key,
// a memory-clock or always-left test has one outcome for the whole lane and
// becomes K = 0 (right: ck >= 1 << 16) or K = ~0 (left).  Per clock the path
// is compares and selects of per-lane keys, no per-clock test loads.
__device__ __forceinline__ uint32_t lane_key(uint2 t, unsigned mem_l) {
    return t.x == 0xffffffffu ? t.y : (((mem_l & t.x) > t.y) ? 0u : 0xffffffffu);
}
template <int CPL, int D>
__device__ __forceinline__ void add_table_keys(double (&acc)[CPL], const unsigned (&ck)[CPL], uint32_t sb,
                                               unsigned mem_l) {
    const uint32_t K0 = lane_key(lds_u2(sb), mem_l), K1 = lane_key(lds_u2(sb + 8u), mem_l),
                   K2 = lane_key(lds_u2(sb + 16u), mem_l);
    if constexpr (D == 2) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const bool b0 = ck[i] > K0;
            const bool b1 = ck[i] > (b0 ? K2 : K1);
            acc[i] = __dadd_rn(acc[i], lds_f64(sb + 64u + (b0 ? 32u : 0u) + (b1 ? 16u : 0u)));
        }
    } else {
        const uint32_t K3 = lane_key(lds_u2(sb + 24u), mem_l), K4 = lane_key(lds_u2(sb + 32u), mem_l),
                       K5 = lane_key(lds_u2(sb + 40u), mem_l), K6 = lane_key(lds_u2(sb + 48u), mem_l);
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const bool b0 = ck[i] > K0;
            const bool b1 = ck[i] > (b0 ? K2 : K1);
            const uint32_t Kl = b1 ? K4 : K3, Kr = b1 ? K6 : K5;
            const bool b2 = ck[i] > (b0 ? Kr : Kl);
            acc[i] = __dadd_rn(acc[i], lds_f64(sb + 64u + (b0 ? 32u : 0u) + (b1 ? 16u : 0u) + (b2 ? 8u : 0u)));
        }
    }
}
#endif

// Depth-2 table when every clock of this lane has memory clock mem_l: a test
// whose mask has no core-clock bits (a memory test, or the always-left
// filler) has one outcome for the whole lane, so it is resolved once per lane
// and at most one test remains per clock.  The test kinds are the table's
// (the same for every lane), so the branches are uniform.
template <int CPL>
__device__ __forceinline__ void add_table2_mem_uniform(double (&acc)[CPL], const unsigned (&ck)[CPL], uint32_t sb,
                                                       unsigned mem_l) {
    const uint2 t0 = lds_u2(sb);
    if (t0.x != 0xffffffffu) {  // root resolved per lane: child n, then one test per clock
        const uint32_t n = 1u + ((mem_l & t0.x) > t0.y ? 1u : 0u);
        const uint2 tc = lds_u2(sb + n * 8u);
        const double lv = lds_f64(sb + 64u + (2u * n - 2u) * 16u), rv = lds_f64(sb + 64u + (2u * n - 1u) * 16u);
#if GD_TABLE_KEYS
        const uint32_t kc = lane_key(tc, mem_l);  // one unsigned compare per clock
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], ck[i] > kc ? rv : lv);
#else
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], (ck[i] & tc.x) > tc.y ? rv : lv);
#endif
        return;
    }
    const uint2 t1 = lds_u2(sb + 8u), t2 = lds_u2(sb + 16u);
    if (t1.x != 0xffffffffu && t2.x != 0xffffffffu) {  // both children resolved per lane: one test per clock
        const double lv = lds_f64(sb + 64u + ((mem_l & t1.x) > t1.y ? 16u : 0u));
        const double rv = lds_f64(sb + 96u + ((mem_l & t2.x) > t2.y ? 16u : 0u));
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], ck[i] > t0.y ? rv : lv);
        return;
    }
#if GD_TABLE_KEYS
    add_table_keys<CPL, 2>(acc, ck, sb, mem_l);
#else
    add_table<CPL, 2>(acc, ck, sb);
#endif
}

// The group's per-kind tree masks (ballots: warp-uniform, so the per-tree
// dispatch below is uniform branching).
struct GroupMasks {
    unsigned nc, sm, mem, tab;
};

// One non-constant tree j of the group being processed.
template <int CPL, class RG>
__device__ __forceinline__ void add_residue(const AccModel& m, const RTRec* __restrict__ pool, uint32_t ws, int g,
                                            int j, const GroupMasks& gm, const double* row,
                                            const unsigned (&ck)[CPL], bool mem_uniform, unsigned mem_l, int lane,
                                            double (&acc)[CPL]) {
    const uint32_t slotb = static_cast<uint32_t>((RG::rs(g) * 32 + j) * 16);
    const uint32_t vslot = static_cast<uint32_t>((RG::ss(g) * 32 + j) * 8);
    const unsigned bit = 1u << j;
    if (gm.sm & bit) {
        const uint32_t info = lds_u32(ws + RG::kMeta + slotb);
        const double lv = lds_f64(ws + RG::kVal + vslot);
        const double rv = lds_f64(ws + RG::kRv + vslot);
        const unsigned key = (info & 0xffff0000u) | 0xffffu;
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], ck[i] <= key ? lv : rv);
    } else if (gm.mem & bit) {
        const uint32_t info = lds_u32(ws + RG::kMeta + slotb);
        const double lv = lds_f64(ws + RG::kVal + vslot);
        const double rv = lds_f64(ws + RG::kRv + vslot);
        const unsigned key = info >> 16;
        if (mem_uniform) {  // all of this lane's clocks share one memory clock
            add_const<CPL>(acc, mem_l <= key ? lv : rv);
        } else {
#pragma unroll
            for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], (ck[i] & 0xffffu) <= key ? lv : rv);
        }
    } else if (gm.tab & bit) {
        const int slot = __popc(gm.tab & (bit - 1u));
        uint32_t sb;
        if (slot < kSide) {
            sb = ws + RG::kSideOff + static_cast<uint32_t>((RG::ss(g) * kSide + slot) * 128);
        } else {  // more tables in this group than staged slots: copy it now
            const uint32_t ref = lds_u32(ws + RG::kMeta + slotb + 4);
            sb = ws + RG::kOvf;
            __syncwarp();
            if (lane < 8) {
                const int4 x = __ldg(reinterpret_cast<const int4*>(pool + ref) + lane);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sb + 16u * lane), "r"(x.x), "r"(x.y),
                             "r"(x.z), "r"(x.w)
                             : "memory");
            }
            __syncwarp();
        }
        if (lds_u32(sb + 56u) == 2u) {
            if (mem_uniform) add_table2_mem_uniform<CPL>(acc, ck, sb, mem_l);
            else add_table<CPL, 2>(acc, ck, sb);
        } else {
#if GD_TABLE_KEYS
            if (mem_uniform) add_table_keys<CPL, 3>(acc, ck, sb, mem_l);
            else add_table<CPL, 3>(acc, ck, sb);
#else
            add_table<CPL, 3>(acc, ck, sb);
#endif
        }
    } else {
        const uint32_t info = lds_u32(ws + RG::kMeta + slotb);
        const int32_t ref = static_cast<int32_t>(lds_u32(ws + RG::kMeta + slotb + 4));
        if ((info & 7u) == kRecTable5) {  // rarer still: copied on demand (four pool slots)
            const uint32_t sb = ws + RG::kOvf;
            __syncwarp();
            {
                const int4 x = __ldg(reinterpret_cast<const int4*>(pool + ref) + lane);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sb + 16u * lane), "r"(x.x), "r"(x.y),
                             "r"(x.z), "r"(x.w)
                             : "memory");
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                uint32_t n = 0;
#pragma unroll
                for (int d = 0; d < 5; ++d) {
                    const uint2 t = lds_u2(sb + n * 8u);
                    n = 2u * n + 1u + ((ck[i] & t.x) > t.y ? 1u : 0u);
                }
                acc[i] = __dadd_rn(acc[i], lds_f64(sb + 256u + (n - 31u) * 8u));
            }
        } else if ((info & 7u) == kRecTable4) {  // rare: copied on demand (two pool slots)
            const uint32_t sb = ws + RG::kOvf;
            __syncwarp();
            if (lane < 16) {
                const int4 x = __ldg(reinterpret_cast<const int4*>(pool + ref) + lane);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sb + 16u * lane), "r"(x.x), "r"(x.y),
                             "r"(x.z), "r"(x.w)
                             : "memory");
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                uint32_t n = 0;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const uint2 t = lds_u2(sb + n * 8u);
                    n = 2u * n + 1u + ((ck[i] & t.x) > t.y ? 1u : 0u);
                }
                acc[i] = __dadd_rn(acc[i], lds_f64(sb + 128u + (n - 15u) * 8u));
            }
        } else {
#pragma unroll
            for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], eval_full_packed(m.nodes, ref, row, ck[i]));
        }
    }
}

template <int CPL, class RG>
__device__ __forceinline__ void accumulate_model(const AccModel& m, const RTRec* __restrict__ pool, int64_t la,
                                                 int64_t n_apps, const double* row, uint32_t ws,
                                                 const unsigned (&ck)[CPL], bool mem_uniform, unsigned mem_l,
                                                 int lane, double (&acc)[CPL]) {
    const int ng = (m.n_trees + 31) >> 5;
    if (ng == 0) return;
    __syncwarp();
    constexpr int RR = RG::kRecAhead, RS = RG::kSideAhead;
    // Prologue: records of groups 0 .. RR-1, then the side data of 0 .. RS-1
    // (one commit group each, so group g of the loop's wait arithmetic holds
    // side(g)).
    for (int j = 0; j < RR && j < ng; ++j) issue_rec<RG>(m, la, n_apps, j, lane, ws);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
#pragma unroll
    for (int j = 0; j < RS; ++j) {
        if (j < ng) issue_side<RG>(m, pool, j, lane, ws);
        cp_async_commit();
    }
    for (int g = 0; g < ng; ++g) {
        // Complete: side(g) (group g) and rec(g + RS) (group g + 2RS - RR).
        cp_async_wait<RG::kWait>();
        __syncwarp();
        if (g + RS < ng) issue_side<RG>(m, pool, g + RS, lane, ws);
        if (g + RR < ng) issue_rec<RG>(m, la, n_apps, g + RR, lane, ws);
        cp_async_commit();

        const int nth = min(32, m.n_trees - g * 32);
        const uint32_t vals = ws + RG::kVal + static_cast<uint32_t>(RG::ss(g) * 32 * 8);
        const uint32_t kind_l = lane < nth ? (lds_u32(ws + RG::kMeta + static_cast<uint32_t>((RG::rs(g) * 32 + lane) * 16)) & 7u)
                                           : kRecConst;
        GroupMasks gm;
        gm.nc = __ballot_sync(kFull, kind_l != kRecConst);
        gm.sm = __ballot_sync(kFull, kind_l == kRecSm);
        gm.mem = __ballot_sync(kFull, kind_l == kRecMem);
        gm.tab = __ballot_sync(kFull, kind_l == kRecTable);
        // Runs of constant trees between residue trees (uniform control flow).
        unsigned rest = gm.nc;
        int j = 0;
        while (true) {
            const int r = rest ? __ffs(rest) - 1 : nth;
            int k = j;
            for (; k + 4 <= r; k += 4) {
                const double v0 = lds_f64(vals + static_cast<uint32_t>(k * 8));
                const double v1 = lds_f64(vals + static_cast<uint32_t>(k * 8 + 8));
                const double v2 = lds_f64(vals + static_cast<uint32_t>(k * 8 + 16));
                const double v3 = lds_f64(vals + static_cast<uint32_t>(k * 8 + 24));
                add_const<CPL>(acc, v0);
                add_const<CPL>(acc, v1);
                add_const<CPL>(acc, v2);
                add_const<CPL>(acc, v3);
            }
            if (k + 2 <= r) {
                const double v0 = lds_f64(vals + static_cast<uint32_t>(k * 8));
                const double v1 = lds_f64(vals + static_cast<uint32_t>(k * 8 + 8));
                add_const<CPL>(acc, v0);
                add_const<CPL>(acc, v1);
                k += 2;
            }
            if (k < r) add_const<CPL>(acc, lds_f64(vals + static_cast<uint32_t>(k * 8)));
            if (r >= nth) break;
            add_residue<CPL, RG>(m, pool, ws, g, r, gm, row, ck, mem_uniform, mem_l, lane, acc);
            rest &= rest - 1u;
            j = r + 1;
        }
    }
}

// One clock per lane (the sliced latency kernel): CONST, SM and MEM records
// all reduce to one select per tree -- pass ? left : right, with pass forced
// for CONST -- so the per-tree work is branch-free and the only uniform
// branch is the rare TABLE / FULL record.  (With one DADD per tree, the run
// structure of accumulate_model costs more than it saves.)
template <class RG>
__device__ __forceinline__ void accumulate_lane(const AccModel& m, const RTRec* __restrict__ pool, int64_t la,
                                                int64_t n_apps, const double* row, uint32_t ws, unsigned ck, int lane,
                                                double& acc) {
    constexpr int RR = RG::kRecAhead, RS = RG::kSideAhead;
    const int ng = (m.n_trees + 31) >> 5;
    if (ng == 0) return;
    const unsigned mem_l = ck & 0xffffu;
    const unsigned ck1[1] = {ck};
    double acc1[1];
    __syncwarp();
    for (int j = 0; j < RR && j < ng; ++j) issue_rec<RG>(m, la, n_apps, j, lane, ws);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
#pragma unroll
    for (int j = 0; j < RS; ++j) {
        if (j < ng) issue_side<RG>(m, pool, j, lane, ws);
        cp_async_commit();
    }
    for (int g = 0; g < ng; ++g) {
        cp_async_wait<RG::kWait>();
        __syncwarp();
        if (g + RS < ng) issue_side<RG>(m, pool, g + RS, lane, ws);
        if (g + RR < ng) issue_rec<RG>(m, la, n_apps, g + RR, lane, ws);
        cp_async_commit();

        const int nth = min(32, m.n_trees - g * 32);
        const uint32_t meta = ws + RG::kMeta + static_cast<uint32_t>(RG::rs(g) * 32 * 16);
        const uint32_t vals = ws + RG::kVal + static_cast<uint32_t>(RG::ss(g) * 32 * 8);
        const uint32_t rvs = ws + RG::kRv + static_cast<uint32_t>(RG::ss(g) * 32 * 8);
        // Lane t turns tree t's record into a clock test (mask, key):
        // (ck & mask) <= key picks the left leaf -- CONST (0, 0) always, SM
        // (0xffff0000, t16 << 16 | 0xffff) iff sm <= t16, MEM (0xffff, t16) iff
        // mem <= t16 -- written over the record's ref2 / pad words, which the
        // side fetch has already consumed.
        uint32_t kind_l = kRecConst;
        if (lane < nth) {
            const uint32_t info = lds_u32(meta + static_cast<uint32_t>(lane * 16));
            kind_l = info & 7u;
            const uint32_t t16 = info >> 16;
            if (kind_l <= kRecMem) {
                const uint32_t mask = kind_l == kRecSm ? 0xffff0000u : (kind_l == kRecMem ? 0xffffu : 0u);
                const uint32_t key = kind_l == kRecSm ? ((t16 << 16) | 0xffffu) : (kind_l == kRecMem ? t16 : 0u);
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(meta + static_cast<uint32_t>(lane * 16 + 8)),
                             "r"(mask), "r"(key)
                             : "memory");
            }
        }
        __syncwarp();
        GroupMasks gm{0u, 0u, 0u, __ballot_sync(kFull, kind_l == kRecTable)};
        const unsigned slow = __ballot_sync(kFull, kind_l >= kRecTable);
        // Blocks of 8 trees: the loads and selects are independent and only
        // the 8 adds chain (a lone warp per slice has no other latency
        // hiding).  Software-pipelined: block j's values are formed while
        // block j-8's adds retire.
        auto values = [&](int j, double (&v)[8]) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // slots past nth / slow records: unused values
                const uint2 mk = lds_u2(meta + static_cast<uint32_t>((j + k) * 16 + 8));
                const double lv = lds_f64(vals + static_cast<uint32_t>((j + k) * 8));
                const double rv = lds_f64(rvs + static_cast<uint32_t>((j + k) * 8));
                v[k] = (ck & mk.x) <= mk.y ? lv : rv;
            }
            // TABLE / FULL trees of the block: their value for this lane's
            // clock, computed into a -0.0-seeded temporary (exact).
            for (unsigned b = (slow >> j) & 0xffu; b; b &= b - 1u) {
                const int k = __ffs(b) - 1;
                acc1[0] = -0.0;
                add_residue<1, RG>(m, pool, ws, g, j + k, gm, row, ck1, true, mem_l, lane, acc1);
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = q == k ? acc1[0] : v[q];
            }
        };
        auto chain = [&](int j, const double (&v)[8]) {
            if (j + 8 <= nth) {
#pragma unroll
                for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, v[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (j + k < nth) acc = __dadd_rn(acc, v[k]);
                }
            }
        };
        double va[8];
        values(0, va);
        int j = 8;
        for (; j < nth; j += 8) {
            chain(j - 8, va);  // independent of the next block's loads and selects
            values(j, va);
        }
        chain(j - 8, va);
    }
}

// Named barrier for one warp pair (ids are immediates: a register id makes
// ptxas reserve all 16 named barriers per CTA).
template <int kId>
__device__ __forceinline__ void pair_sync() {
    __syncwarp();
    asm volatile("barrier.sync %0, 64;" ::"n"(kId) : "memory");
}
__device__ __forceinline__ void pair_sync_a(int pair) {
    switch (pair) {
        case 0: pair_sync<1>(); break;
        case 1: pair_sync<3>(); break;
        case 2: pair_sync<5>(); break;
        default: pair_sync<7>(); break;
    }
}
__device__ __forceinline__ void pair_sync_b(int pair) {
    switch (pair) {
        case 0: pair_sync<2>(); break;
        case 1: pair_sync<4>(); break;
        case 2: pair_sync<6>(); break;
        default: pair_sync<8>(); break;
    }
}
static_assert(kAccWarps / 2 <= 4, "pair barriers cover four warp pairs");

// The catalog -> (lane, slot) map, built by one warp into map[slot * 32 +
// lane] (catalog index or -1).  Preferred: every lane's clocks lie in ONE run
// of equal memory clocks (catalog order groups them: mem asc, sm asc), so a
// memory-clock test is one compare per lane; runs take consecutive lanes,
// slots in catalog order, so lane-major slot order is still catalog order.
// If the runs need more than 32 lanes, lane l owns clocks l*cpl .. l*cpl+cpl-1.
// Returns 1 for the per-lane-uniform memory clock layout.
__device__ int build_clock_map(const int32_t* __restrict__ mem, int C, int cpl, int16_t* map, int lane) {
    constexpr int K = 16;  // clocks per lane (C <= 512)
    for (int i = 0; i < cpl; ++i) map[i * 32 + lane] = -1;
    const int c0 = lane * K;
    // Run starts in my chunk.
    unsigned starts = 0;
    int prev = c0 > 0 && c0 < C ? __ldg(mem + c0 - 1) : 0;
    for (int k = 0; k < K; ++k) {
        const int c = c0 + k;
        if (c >= C) break;
        const int mv = __ldg(mem + c);
        if (c == 0 || mv != prev) starts |= 1u << k;
        prev = mv;
    }
    // Last start at or before my chunk (max-scan) and first start after it (min-scan).
    int last_in = starts ? c0 + 31 - __clz(static_cast<int>(starts)) : -1;
    int first_in = starts ? c0 + __ffs(starts) - 1 : C;
    int carry_last = last_in, carry_first = first_in;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(kFull, carry_last, d);
        const int b = __shfl_down_sync(kFull, carry_first, d);
        if (lane >= d) carry_last = max(carry_last, a);
        if (lane + d < 32) carry_first = min(carry_first, b);
    }
    int before_last = __shfl_up_sync(kFull, carry_last, 1);    // last start before my chunk
    int after_first = __shfl_down_sync(kFull, carry_first, 1);  // first start after my chunk
    if (lane == 0) before_last = -1;
    if (lane == 31) after_first = C;
    // Lanes used by the runs that START in my chunk, then an exclusive scan.
    int mine = 0;
    for (int k = 0; k < K; ++k) {
        if (!((starts >> k) & 1u)) continue;
        const unsigned later = starts & ~((2u << k) - 1u);
        const int end = later ? c0 + __ffs(later) - 1 : after_first;
        mine += (end - (c0 + k) + cpl - 1) / cpl;
    }
    int incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += a;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const int uniform = total <= 32;
    __syncwarp();
    // Base lane of the run in progress at c0 (it started before my chunk).
    int run_start = before_last, base = incl - mine;
    if (run_start >= 0) {
        const int end = starts ? c0 + __ffs(starts) - 1 : after_first;
        base -= (end - run_start + cpl - 1) / cpl;
    }
    for (int k = 0; k < K; ++k) {
        const int c = c0 + k;
        if (c >= C) break;
        if ((starts >> k) & 1u) {
            if (run_start >= 0 && run_start >= c0) {
                // previous run started in my chunk: advance the base past it
                base += (c - run_start + cpl - 1) / cpl;
            } else if (run_start >= 0) {
                base += (c - run_start + cpl - 1) / cpl;
            }
            run_start = c;
        }
        if (uniform) {
            const int off = c - run_start;
            map[(off % cpl) * 32 + base + off / cpl] = static_cast<int16_t>(c);
        } else {
            map[(c % cpl) * 32 + c / cpl] = static_cast<int16_t>(c);
        }
    }
    __syncwarp();
    return uniform;
}

template <int CPL>
__global__ void __launch_bounds__(kAccThreads, (CPL >= 12 ? 4 : GD_ACC_MIN_BLOCKS)) grid_acc_kernel(const __grid_constant__ AccParams p) {
    using RING = AccRing;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = warp >> 1;
    const int model = warp & 1;  // 0 energy, 1 time
    const int F = p.n_cols;
    unsigned char* wsp = smem + acc_smem_per_warp<RING>(F) * warp;
    const uint32_t ws = smem_addr(wsp);
    double* row = reinterpret_cast<double*>(wsp + RING::kRow);
    double* tbuf = reinterpret_cast<double*>(smem + acc_smem_per_warp<RING>(F) * kAccWarps + acc_smem_per_pair(CPL) * pair);
    int16_t* map = reinterpret_cast<int16_t*>(smem + acc_smem_per_warp<RING>(F) * kAccWarps +
                                              acc_smem_per_pair(CPL) * (kAccWarps / 2));
    int* flag = reinterpret_cast<int*>(map + 32 * CPL);
    if (warp == 0) {
        const int u = build_clock_map(p.mem, p.n_clocks, CPL, map, lane);
        if (lane == 0) *flag = u;
    }
    __syncthreads();
    const bool mem_uniform = *flag != 0;

    unsigned ck[CPL];
    unsigned mem_l = 0;
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
        const int c = map[i * 32 + lane];
        ck[i] = c >= 0 ? ((static_cast<unsigned>(__ldg(p.sm + c)) << 16) | static_cast<unsigned>(__ldg(p.mem + c))) : 0u;
        if (i == 0) mem_l = ck[0] & 0xffffu;
    }
    AccModel m;
    m.nodes = model ? p.nodes[1] : p.nodes[0];
    m.rec = model ? p.rec[1] : p.rec[0];
    m.n_trees = model ? p.n_trees[1] : p.n_trees[0];

    for (int64_t la = static_cast<int64_t>(blockIdx.x) * (kAccWarps / 2) + pair; la < p.n_apps;
         la += static_cast<int64_t>(gridDim.x) * (kAccWarps / 2)) {
        const int64_t a = p.a0 + la;
        double acc[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = 0.0;
        // The row is only read by FULL records (rare); staging it is cheap.
        __syncwarp();
        const double* src = p.rows + a * F;
        for (int j = lane; j < F; j += 32) row[j] = __ldg(src + j);
        __syncwarp();
        if (model == 1) {
            for (int k = lane; k < p.n_cat; k += 32) row[__ldg(p.cat_cols + k)] = __ldg(p.cat_t + a * p.n_cat + k);
            __syncwarp();
        }
        accumulate_model<CPL, RING>(m, p.pool, la, p.n_apps, row, ws, ck, mem_uniform, mem_l, lane, acc);
        if (model == 1) {
            pair_sync_a(pair);  // the energy warp is done reading the previous app's times
#pragma unroll
            for (int i = 0; i < CPL; ++i) tbuf[lane * CPL + i] = finish(p.base[1], p.lr[1], acc[i]);
            pair_sync_b(pair);
        } else {
            double E[CPL], T[CPL];
            int smv[CPL], cidx[CPL];
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                E[i] = clamp_energy(finish(p.base[0], p.lr[0], acc[i]));
                smv[i] = static_cast<int>(ck[i] >> 16);
            }
            pair_sync_a(pair);
            pair_sync_b(pair);
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                T[i] = tbuf[lane * CPL + i];
                const int c = map[i * 32 + lane];
                cidx[i] = c;
                if (c >= 0) {
                    if (p.e_out) p.e_out[a * p.out_stride + c] = E[i];
                    if (p.t_out) p.t_out[a * p.out_stride + c] = T[i];
                }
            }
            select_epilogue<CPL>(E, T, smv, cidx, lane, __ldg(p.budgets + a), p.mode, p.objective, p.best_effort,
                                 p.out + a);
        }
    }
}

// ---------------------------------------------------------------------------
// K2b, sliced (latency mode for small batches, e.g. the configs[4] stream):
// a warp pair per (app, 32-clock slice), lane l owning clock 32*slice + l
// (one clock per lane, so every memory-clock test is per lane).  Slices
// publish E/T to a staging row; the last slice to arrive (threadfence +
// atomic counter) gathers the app's full row and runs the selection.
// ---------------------------------------------------------------------------
template <int CPLF>
__global__ void __launch_bounds__(kAccThreads) grid_acc_sliced_kernel(const __grid_constant__ AccParams p) {
    using RING = SlicedRing;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = warp >> 1;
    const int model = warp & 1;
    const int F = p.n_cols, C = p.n_clocks;
    unsigned char* wsp = smem + acc_smem_per_warp<RING>(F) * warp;
    const uint32_t ws = smem_addr(wsp);
    double* row = reinterpret_cast<double*>(wsp + RING::kRow);
    AccModel m;
    m.nodes = model ? p.nodes[1] : p.nodes[0];
    m.rec = model ? p.rec[1] : p.rec[0];
    m.n_trees = model ? p.n_trees[1] : p.n_trees[0];
    const int S = (C + 31) >> 5;
    const int64_t units = static_cast<int64_t>(p.n_apps) * S;
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * (kAccWarps / 2) + pair; u < units;
         u += static_cast<int64_t>(gridDim.x) * (kAccWarps / 2)) {
        const int64_t la = u / S;
        const int sl = static_cast<int>(u - la * S);
        const int64_t a = p.a0 + la;
        const int c = sl * 32 + lane;
        const unsigned ck[1] = {c < C ? ((static_cast<unsigned>(__ldg(p.sm + c)) << 16) |
                                         static_cast<unsigned>(__ldg(p.mem + c)))
                                      : 0u};
        double acc[1] = {0.0};
        __syncwarp();
        const double* src = p.rows + a * F;
        for (int j = lane; j < F; j += 32) row[j] = __ldg(src + j);
        __syncwarp();
        if (model == 1) {
            for (int k = lane; k < p.n_cat; k += 32) row[__ldg(p.cat_cols + k)] = __ldg(p.cat_t + a * p.n_cat + k);
            __syncwarp();
        }
#ifdef GD_SLICED_RUNS
        accumulate_model<1, RING>(m, p.pool, la, p.n_apps, row, ws, ck, true, ck[0] & 0xffffu, lane, acc);
#else
        accumulate_lane<RING>(m, p.pool, la, p.n_apps, row, ws, ck[0], lane, acc[0]);
#endif
        double* et = p.et + la * 2 * C;
        if (model == 1) {
            const double t = finish(p.base[1], p.lr[1], acc[0]);
            if (c < C) {
                et[C + c] = t;
                if (p.t_out) p.t_out[a * p.out_stride + c] = t;
            }
            __threadfence();
            pair_sync_a(pair);  // both warps of the pair have published their slice
            pair_sync_b(pair);  // the energy warp has read last_flag
        } else {
            const double e = clamp_energy(finish(p.base[0], p.lr[0], acc[0]));
            if (c < C) {
                et[c] = e;
                if (p.e_out) p.e_out[a * p.out_stride + c] = e;
            }
            __threadfence();
            pair_sync_a(pair);
            int last = 0;
            if (lane == 0) last = atomicAdd(p.arrive + la, 1u) == static_cast<unsigned>(S - 1);
            last = __shfl_sync(kFull, last, 0);
            pair_sync_b(pair);
            if (last) {
                __threadfence();
                double E[CPLF], T[CPLF];
                int smv[CPLF], cidx[CPLF];
                contiguous_cidx<CPLF>(lane, C, cidx);
#pragma unroll
                for (int i = 0; i < CPLF; ++i) {
                    const int cc = cidx[i];
                    E[i] = cc >= 0 ? __ldcg(et + cc) : 0.0;
                    T[i] = cc >= 0 ? __ldcg(et + C + cc) : 0.0;
                    smv[i] = cc >= 0 ? __ldg(p.sm + cc) : 0;
                }
                select_epilogue<CPLF>(E, T, smv, cidx, lane, __ldg(p.budgets + a), p.mode, p.objective,
                                      p.best_effort, p.out + a);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Rows genuinely differ per clock (nearest-record substitution from several
// profiled records, scheduler.cpp:341-359): full traversal per candidate.
// ---------------------------------------------------------------------------
template <int CPL>
__global__ void __launch_bounds__(256) grid_general_kernel(const __grid_constant__ GridParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    int smv[CPL], memv[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
        const int c = lane * CPL + i;
        smv[i] = c < p.n_clocks ? __ldg(p.sm + c) : 0;
        memv[i] = c < p.n_clocks ? __ldg(p.mem + c) : 0;
    }
    const int F = p.n_cols;
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * wpb + warp; a < p.n_apps;
         a += static_cast<int64_t>(gridDim.x) * wpb) {
        double accE[CPL], accT[CPL];
        const double* rE[CPL];
        const double* rT[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            accE[i] = accT[i] = 0.0;
            const int c = lane * CPL + i;
            const int64_t rec = c < p.n_clocks ? (p.rec_of_clock ? __ldg(p.rec_of_clock + a * p.out_stride + c) : a) : 0;
            rE[i] = p.rows + rec * F;
            rT[i] = p.rows_t + rec * F;
        }
        for (int32_t t = 0; t < p.e_trees; ++t) {
            const int32_t root = __ldg(p.e_roots + t);
#pragma unroll
            for (int i = 0; i < CPL; ++i)
                accE[i] = __dadd_rn(accE[i], eval_full(p.e_nodes, root, rE[i], p.sm_col, p.mem_col, smv[i], memv[i]));
        }
        for (int32_t t = 0; t < p.t_trees; ++t) {
            const int32_t root = __ldg(p.t_roots + t);
#pragma unroll
            for (int i = 0; i < CPL; ++i)
                accT[i] = __dadd_rn(accT[i], eval_full(p.t_nodes, root, rT[i], p.sm_col, p.mem_col, smv[i], memv[i]));
        }
        double E[CPL], T[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            E[i] = clamp_energy(finish(p.e_base, p.e_lr, accE[i]));
            T[i] = finish(p.t_base, p.t_lr, accT[i]);
            const int c = lane * CPL + i;
            if (c < p.n_clocks) {
                if (p.e_out) p.e_out[a * p.out_stride + c] = E[i];
                if (p.t_out) p.t_out[a * p.out_stride + c] = T[i];
            }
        }
        int cidx[CPL];
        contiguous_cidx<CPL>(lane, p.n_clocks, cidx);
        select_epilogue<CPL>(E, T, smv, cidx, lane, __ldg(p.budgets + a), p.mode, p.objective, p.best_effort,
                             p.out + a);
    }
}

// Resident CTAs per SM for (kernel, threads, dynamic smem), raising the
// kernel's dynamic shared memory limit first when needed.  Cached per device:
// the attribute call and the occupancy query cost microseconds of host time
// on every launch otherwise, which the latency stream pays in full.
int occupancy(const void* fn, int threads, size_t smem) {
    struct Entry {
        const void* fn;
        int device, threads;
        size_t smem;
        int per_sm;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int device = 0;
    cudaGetDevice(&device);
    {
        std::lock_guard<std::mutex> lock(mu);
        for (const Entry& e : cache) {
            if (e.fn == fn && e.device == device && e.threads == threads && e.smem == smem) return e.per_sm;
        }
    }
    std::lock_guard<std::mutex> lock(mu);
    // The limit only ever rises (a cached launch with a larger size must stay
    // valid after a smaller one was configured).
    size_t limit = 48 * 1024;
    for (const Entry& e : cache) {
        if (e.fn == fn && e.device == device && e.smem > limit) limit = e.smem;
    }
    if (smem > limit &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess) {
        return -1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) return -1;
    cache.push_back(Entry{fn, device, threads, smem, per_sm});
    return per_sm;
}

template <int CPL>
int launch_general(const GridParams& p, int sm_count, cudaStream_t stream) {
    const int per_sm = occupancy(reinterpret_cast<const void*>(grid_general_kernel<CPL>), 256, 0);
    if (per_sm < 0) return cudaErrorInvalidConfiguration;
    const int blocks = grid_blocks(8, p.n_apps, sm_count, per_sm);
    grid_general_kernel<CPL><<<blocks, 256, 0, stream>>>(p);
    return cudaGetLastError();
}

template <int CPL>
int launch_acc(const AccParams& p, int sm_count, cudaStream_t stream) {
    const size_t smem = acc_smem_per_warp<AccRing>(p.n_cols) * kAccWarps + acc_smem_per_pair(CPL) * (kAccWarps / 2) +
                        32 * CPL * sizeof(int16_t) + 16;
    auto kern = grid_acc_kernel<CPL>;
    const int per_sm = occupancy(reinterpret_cast<const void*>(kern), kAccThreads, smem);
    if (per_sm < 0) return cudaErrorInvalidConfiguration;
    const int blocks = grid_blocks(kAccWarps / 2, p.n_apps, sm_count, per_sm);
    kern<<<blocks, kAccThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

template <int CPLF>
int launch_acc_sliced(const AccParams& p, int sm_count, cudaStream_t stream) {
    const size_t smem = acc_smem_per_warp<SlicedRing>(p.n_cols) * kAccWarps + acc_smem_per_pair(1) * (kAccWarps / 2);
    auto kern = grid_acc_sliced_kernel<CPLF>;
    const int per_sm = occupancy(reinterpret_cast<const void*>(kern), kAccThreads, smem);
    if (per_sm < 0) return cudaErrorInvalidConfiguration;
    const int64_t units = static_cast<int64_t>(p.n_apps) * ((p.n_clocks + 31) / 32);
    const int blocks = grid_blocks(kAccWarps / 2, units, sm_count, per_sm);
    kern<<<blocks, kAccThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

int launch_acc_sliced_cpl(const AccParams& p, int sm_count, cudaStream_t s) {
    const int cpl = (p.n_clocks + 31) / 32;
    if (cpl <= 1) return launch_acc_sliced<1>(p, sm_count, s);
    if (cpl <= 2) return launch_acc_sliced<2>(p, sm_count, s);
    if (cpl <= 4) return launch_acc_sliced<4>(p, sm_count, s);
    if (cpl <= 7) return launch_acc_sliced<7>(p, sm_count, s);
    if (cpl <= 9) return launch_acc_sliced<9>(p, sm_count, s);
    if (cpl <= 12) return launch_acc_sliced<12>(p, sm_count, s);
    return launch_acc_sliced<16>(p, sm_count, s);
}

int launch_acc_cpl(const AccParams& p, int sm_count, cudaStream_t s) {
    const int cpl = (p.n_clocks + 31) / 32;
    if (cpl <= 1) return launch_acc<1>(p, sm_count, s);
    if (cpl <= 2) return launch_acc<2>(p, sm_count, s);
    if (cpl <= 4) return launch_acc<4>(p, sm_count, s);
    if (cpl <= 7) return launch_acc<7>(p, sm_count, s);
    if (cpl <= 9) return launch_acc<9>(p, sm_count, s);
    if (cpl <= 12) return launch_acc<12>(p, sm_count, s);
    return launch_acc<16>(p, sm_count, s);
}

// Walk-kernel geometry: warps per CTA (two per 32 apps) so the transposed
// ranks plus two stage buffers of tree windows fit the opt-in shared memory.
struct WalkGeom {
    int warps, win_nodes, stage_nodes, n_bufs, n_subs;
    int tile_apps, rb;  // apps per tile, bytes per rank (1: 1024-app tiles, two apps per lane)
    size_t smem;
};
int64_t env_i64(const char* name, int64_t dflt);
WalkGeom walk_geom(const GridParams& p, int64_t batch_apps, size_t kLimit = 227 * 1024, bool wide = false,
                   int subs = 0) {
    WalkGeom g{};
    g.n_bufs = static_cast<int>(env_i64("GDVFS_WALK_BUFS", 2));
    g.n_bufs = g.n_bufs < 2 ? 2 : (g.n_bufs > 4 ? 4 : g.n_bufs);
    const int32_t max_tree = (p.max_wint + 1) & ~1;  // the loadable prefixes are what is staged
    // 16 warps per CTA: 16 groups x 1 warp (512 apps per tile, every warp
    // walks every tree of a stage) or 8 groups x 2 warps (even / odd trees).
    g.n_subs = static_cast<int>(env_i64("GDVFS_WALK_SUBS", subs ? subs : 1)) == 2 ? 2 : 1;
    int max_groups = static_cast<int>(env_i64("GDVFS_WALK_GROUPS", 16 / g.n_subs));
    if (max_groups > 16 / g.n_subs) max_groups = 16 / g.n_subs;
    // Small batches (the configs[4] latency stream): no more app groups than
    // the batch fills, so the CTAs' work items stay short.
    while (max_groups > 1 && 32LL * (max_groups / 2) >= batch_apps) max_groups /= 2;
    if (wide) {  // 8-bit ranks: 16 warps, 1024 apps per tile
        g.n_subs = 1;
        max_groups = 16;
    }
    for (int groups = 16; groups >= 1; groups >>= 1) {
        if (groups > max_groups) continue;
        g.tile_apps = (wide ? 64 : 32) * groups;
        g.rb = wide ? 1 : 2;
        const size_t fixed = 128 + walk_rank_bytes(p.n_cols, g.tile_apps, g.rb) + walk_jobs_bytes(g.n_subs * groups) +
                             static_cast<size_t>(g.n_bufs) * kStageTrees * 16 + 16;
        if (fixed + g.n_bufs * 8 * 4 > kLimit) continue;
        int64_t stage = static_cast<int64_t>((kLimit - fixed) / (8 * g.n_bufs)) & ~1;
        if (stage > 16384) stage = 16384;
        // Tree window: whole trees when a pair fits one stage buffer, else
        // the largest top-level prefix that does (the rest is read from L2).
        int64_t win = env_i64("GDVFS_WIN_NODES", 0);
        if (win <= 0) win = max_tree < stage / 2 ? max_tree : stage / 2;
        win &= ~1LL;
        if (win < 2) win = 2;
        if (2 * win > stage || (wide && groups != 16)) continue;
        g.warps = g.n_subs * groups;
        g.win_nodes = static_cast<int>(win);
        g.stage_nodes = static_cast<int>(stage);
        g.smem = fixed + g.n_bufs * static_cast<size_t>(g.stage_nodes) * 8;
        return g;
    }
    g.warps = 0;  // too many columns
    return g;
}

int64_t env_i64(const char* name, int64_t dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoll(e) : dflt;
}

// Residue-table pool slots per app: half the trees, i.e. one table (two
// slots: a table may grow to depth 4 in place) per four (app, tree) pairs
// -- 12 % of the pairs hold a table at configs[3], 16 % with trained
// configs[1] models.  GDVFS_POOL_DIV overrides the divisor; tables that do
// not fit fall back to FULL records.
int64_t pool_per_app(const GridParams& p) {
    int64_t div = env_i64("GDVFS_POOL_DIV", 2);
    if (div < 1) div = 1;
    return (static_cast<int64_t>(p.e_trees) + p.t_trees) / div + 2;
}

// Latency mode for small batches: one warp pair per (app, 32-clock slice)
// instead of per app (GDVFS_ACC_SLICED=0/1 forces it).
bool acc_sliced(int64_t n_apps) {
    const int64_t f = env_i64("GDVFS_ACC_SLICED", -1);
    return f >= 0 ? f != 0 : n_apps <= 256;
}

// Apps per batch: the walk -> accumulate hand-off of one batch (records,
// residue tables, ranks) is bounded by a scratch budget (32 GiB of the 180 GB
// HBM; it streams through HBM -- beyond a few thousand apps it does not stay
// in L2 -- so the budget only sets how many batch boundaries, each with its
// kernels' tail waves, a large batch pays: 4 -> 8 -> 16 -> 32 GiB is -4 % /
// -1.5 % / -0.5 % at configs[3]).  Smaller calls allocate only what they use.
int64_t batch_apps(const GridParams& p) {
    const int64_t per_app = grid_scratch_per_app(p);
    const int64_t budget = env_i64("GDVFS_BATCH_BYTES", int64_t(1) << 35);
    int64_t b = per_app > 0 ? budget / per_app : p.n_apps;
    b = b < 256 ? 256 : b;
    return b < p.n_apps ? b : p.n_apps;
}

}  // namespace

int64_t grid_batch_apps(const GridParams& p) { return batch_apps(p); }

bool grid_fast_path_ok(const GridParams& p) {
    return p.rank16 && p.max_tree_nodes <= 65536 && walk_geom(p, batch_apps(p)).warps > 0;
}

int64_t grid_scratch_per_app(const GridParams& p) {
    const int64_t pairs = ((p.e_trees + 1) >> 1) + ((p.t_trees + 1) >> 1);
    const int64_t pool = pool_per_app(p);  // residue tables per app
    const int64_t ranks = (2LL * p.n_cols * 2 + 15) & ~15LL;
    int64_t bytes = pairs * 2 * static_cast<int64_t>(sizeof(TreeRec)) + pool * static_cast<int64_t>(sizeof(RTRec)) + ranks;
    if (acc_sliced(p.n_apps)) bytes += 2LL * p.n_clocks * 8 + 16;  // E/T staging + arrival counter
    return bytes;
}

size_t grid_scratch_bytes(const GridParams& p, bool general) {
    if (general || p.n_apps == 0) return 0;
    const int64_t b = batch_apps(p);
    const int64_t nb = (p.n_apps + b - 1) / b;
    // + one tile of rank padding (the rank layout is whole walk tiles)
    return static_cast<size_t>(b * grid_scratch_per_app(p)) + 4LL * kMaxTileApps * p.n_cols + 16 +
           static_cast<size_t>(nb) * 8 + 256;
}

int launch_grid_select(const GridParams& p, bool general, int sm_count, void* stream, void* scratch,
                       size_t scratch_bytes, int64_t* launches, LaunchMark mark, void* user) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (general) {
        const int cpl = (p.n_clocks + 31) / 32;
        int e;
        if (cpl <= 1) e = launch_general<1>(p, sm_count, s);
        else if (cpl <= 2) e = launch_general<2>(p, sm_count, s);
        else if (cpl <= 4) e = launch_general<4>(p, sm_count, s);
        else if (cpl <= 7) e = launch_general<7>(p, sm_count, s);
        else if (cpl <= 9) e = launch_general<9>(p, sm_count, s);
        else if (cpl <= 12) e = launch_general<12>(p, sm_count, s);
        else e = launch_general<16>(p, sm_count, s);
        if (launches) ++*launches;
        if (mark) mark(user, "general");
        return e;
    }
    if (p.n_apps == 0) return cudaSuccess;
    if (scratch_bytes < grid_scratch_bytes(p, false)) return cudaErrorInvalidValue;
    const int64_t B = batch_apps(p);
    const int64_t nb = (p.n_apps + B - 1) / B;
    const int64_t pe = (p.e_trees + 1) >> 1, pt = (p.t_trees + 1) >> 1;
    const int64_t pool_cap = B * pool_per_app(p);
    unsigned char* base = static_cast<unsigned char*>(scratch);
    TreeRec* rec_e = reinterpret_cast<TreeRec*>(base);
    TreeRec* rec_t = rec_e + B * pe * 2;
    RTRec* pool = reinterpret_cast<RTRec*>(rec_t + B * pt * 2);
    uint16_t* ranks = reinterpret_cast<uint16_t*>(pool + pool_cap);
    const bool sliced = acc_sliced(p.n_apps);
    double* et = reinterpret_cast<double*>(ranks + ((2LL * (B + kMaxTileApps) * p.n_cols + 7) & ~7LL));
    uint32_t* arrive = reinterpret_cast<uint32_t*>(et + (sliced ? 2LL * B * p.n_clocks : 0));
    uint32_t* counts = arrive + (sliced ? ((B + 3) & ~3LL) : 0);
    cudaError_t e = cudaSuccess;

    // Small batches: a quarter of the shared memory per CTA (shorter stage
    // buffers) so several CTAs share an SM and the few work items run in
    // parallel; fall back to the full budget if a tree pair does not fit.
    WalkGeom wg = walk_geom(p, B);
    if (wg.warps > 0 && wg.warps < 16) {
        // Small batches: the smallest shared-memory budget that still stages a
        // tree pair, so every work item's CTA is resident in ONE wave (the
        // configs[4] 64-app batch has 500 one-pair items: 57 KB CTAs fit 3
        // per SM, 444 slots -- a second wave).
        // Two warps per 32-app group (even / odd trees): a pair whose trees
        // put every app's walk on a clock node (a clock root) is resolved by
        // twice the lanes -- such items are the stragglers of a latency batch.
        for (size_t lim : {size_t(24) << 10, size_t(32) << 10, size_t(56) << 10}) {
            const WalkGeom small = walk_geom(p, B, lim, false, 2);
            if (small.warps > 0) {
                wg = small;
                break;
            }
        }
    }
    // 8-bit ranks (every feature of both models has <= 255 distinct
    // thresholds) and a batch that fills whole 1024-app tiles: wide tiles.
    // (GDVFS_WIDE=0 disables, =2 forces it for any batch that fills 16 warps.)
    const int64_t wide_knob = env_i64("GDVFS_WIDE", 1);
    if (p.rank8 && wg.warps == 16 && (wide_knob == 2 || (wide_knob == 1 && B >= 8 * 1024))) {
        const WalkGeom wide = walk_geom(p, B, 227 * 1024, true);
        if (wide.warps == 16 && wide.win_nodes >= wg.win_nodes) wg = wide;
    }
    // 16-bit ranks and tree-local child indices bound what the walk handles
    // (grid_fast_path_ok routes other models to the general kernel).
    if (wg.warps == 0 || !p.rank16 || p.max_tree_nodes > 65536) return cudaErrorNotSupported;
    const bool all_smem = ((p.max_wint + 1) & ~1) <= wg.win_nodes;
    // Lazy refills pay off when a stage holds many trees (>= 8 of the largest
    // window): warps then drift apart within a stage (trained ensembles'
    // residue-heavy trees: walk -20 %, configs[1] -6 %); stages of one or two
    // deep trees gain nothing and keep the blocking form (configs[3] +1 %).
    // GDVFS_LAZY: 0 never, 1 auto, 2 always.
    const int64_t lazy_knob = env_i64("GDVFS_LAZY", 1);
    const bool lazy = lazy_knob == 2 || (lazy_knob == 1 && wg.stage_nodes >= 8 * std::max(p.max_wint, 1));
    using WalkKern = void (*)(WalkParams);
    WalkKern walk_kern;
    if (wg.rb == 1)
        walk_kern = all_smem ? (lazy ? grid_walk_kernel<true, 1, true> : grid_walk_kernel<true, 1, false>)
                             : (lazy ? grid_walk_kernel<false, 1, true> : grid_walk_kernel<false, 1, false>);
    else
        walk_kern = all_smem ? (lazy ? grid_walk_kernel<true, 2, true> : grid_walk_kernel<true, 2, false>)
                             : (lazy ? grid_walk_kernel<false, 2, true> : grid_walk_kernel<false, 2, false>);
    int walk_per_sm = occupancy(reinterpret_cast<const void*>(walk_kern), wg.warps * 32, wg.smem);
    if (walk_per_sm < 0) return cudaErrorInvalidConfiguration;
    if (walk_per_sm < 1) walk_per_sm = 1;
    // Streamed inputs: batch b's slices go up on the copy stream, issued after
    // batch b - 1's kernels were enqueued (from pageable memory the copy call
    // blocks the host, so the kernels already queued keep the GPU busy).
    auto upload = [&](int64_t b) -> cudaError_t {
        cudaStream_t cs = static_cast<cudaStream_t>(p.copy_stream);
        const int64_t a0 = b * B, n = p.n_apps - a0 < B ? p.n_apps - a0 : B;
        cudaError_t r;
        if ((r = cudaMemcpyAsync(const_cast<double*>(p.rows) + a0 * p.n_cols, p.h_rows + a0 * p.n_cols,
                                 static_cast<size_t>(n * p.n_cols) * sizeof(double), cudaMemcpyHostToDevice, cs)) !=
            cudaSuccess)
            return r;
        if (p.n_cat > 0 &&
            (r = cudaMemcpyAsync(const_cast<double*>(p.cat_t) + a0 * p.n_cat, p.h_cat_t + a0 * p.n_cat,
                                 static_cast<size_t>(n * p.n_cat) * sizeof(double), cudaMemcpyHostToDevice, cs)) !=
                cudaSuccess)
            return r;
        if ((r = cudaMemcpyAsync(const_cast<double*>(p.budgets) + a0, p.h_budgets + a0,
                                 static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, cs)) != cudaSuccess)
            return r;
        return cudaEventRecord(static_cast<cudaEvent_t>(p.batch_ready[b]), cs);
    };
    if (p.h_rows && (e = upload(0)) != cudaSuccess) return e;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t a0 = b * B;
        const int32_t n = static_cast<int32_t>(p.n_apps - a0 < B ? p.n_apps - a0 : B);
        if (p.h_rows && (e = cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(p.batch_ready[b]), 0)) != cudaSuccess)
            return e;
        {
            const int ta = wg.tile_apps;
            const int64_t total = 2LL * ((n + ta - 1) / ta) * ta * p.n_cols;
            // The rank kernel also zeroes this batch's counters (the walk's
            // pool count; the sliced accumulate's arrival counters), saving
            // two memset launches on the latency path.
            // (Sliced: arrive[] and counts[] are adjacent; earlier batches
            // are done with theirs, stream order.)
            uint32_t* zero = sliced ? arrive : counts + 2 * b;
            const int32_t n_zero = sliced ? static_cast<int32_t>(counts + 2 * nb - arrive) : 2;
            auto rank_launch = [&](auto* rk) {
                if (total <= kRankWarpLimit) {
                    grid_rank_warp_kernel<<<static_cast<int>((total + 7) / 8), 256, 0, s>>>(
                        p.rows, p.cat_t, p.cat_cols, p.n_cat, a0, n, p.n_cols, ta, p.e_thr, p.e_thr_off, p.t_thr,
                        p.t_thr_off, rk, zero, n_zero);
                } else if (ta % 256 == 0 &&
                           !(std::getenv("GDVFS_RANK_SAMPLED") && std::getenv("GDVFS_RANK_SAMPLED")[0] == '0')) {
                    grid_rank_sampled_kernel<<<static_cast<int>(total / 256), 256, 0, s>>>(
                        p.rows, p.cat_t, p.cat_cols, p.n_cat, a0, n, p.n_cols, ta, p.e_thr, p.e_thr_off, p.t_thr,
                        p.t_thr_off, rk, zero, n_zero);
                } else {
                    int blocks = static_cast<int>((total + 255) / 256);
                    if (blocks > 16 * sm_count) blocks = 16 * sm_count;
                    grid_rank_kernel<<<blocks, 256, 0, s>>>(p.rows, p.cat_t, p.cat_cols, p.n_cat, a0, n, p.n_cols, ta,
                                                            p.e_thr, p.e_thr_off, p.t_thr, p.t_thr_off, rk, zero,
                                                            n_zero);
                }
            };
            if (wg.rb == 1) rank_launch(reinterpret_cast<uint8_t*>(ranks));
            else rank_launch(ranks);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
            if (mark) mark(user, "rank");
        }
        WalkParams w{};
        w.wnodes[0] = p.e_wnodes;
        w.wnodes[1] = p.t_wnodes;
        w.wroots[0] = p.e_wroots;
        w.wroots[1] = p.t_wroots;
        w.roots[0] = p.e_roots;
        w.roots[1] = p.t_roots;
        w.wint[0] = p.e_wint;
        w.wint[1] = p.t_wint;
        w.gnodes[0] = p.e_nodes;
        w.gnodes[1] = p.t_nodes;
        w.n_trees[0] = p.e_trees;
        w.n_trees[1] = p.t_trees;
        w.ranks = reinterpret_cast<const unsigned char*>(ranks);
        w.n_apps = n;
        w.n_cols = p.n_cols;
        w.tile_apps = wg.tile_apps;
        w.n_subs = wg.n_subs;
        w.win_nodes = wg.win_nodes;
        w.stage_nodes = wg.stage_nodes;
        w.n_bufs = wg.n_bufs;
        w.rec[0] = rec_e;
        w.rec[1] = rec_t;
        w.pool = pool;
        w.pool_count = counts + 2 * b;
        // Latency batches keep residue tables to 3 test levels (deeper ones
        // go FULL): a deep residue's depth-first resolution is the critical
        // path of a small batch's walk.  GDVFS_RES_LEVELS overrides.
        w.res_levels = static_cast<int32_t>(env_i64("GDVFS_RES_LEVELS", wg.warps < 16 ? 3 : 5));
        if (w.res_levels < 1) w.res_levels = 1;
        if (w.res_levels > 5) w.res_levels = 5;
        // Runs of 96 queued jobs for stages of one or two deep trees (their
        // refill loop keeps more lanes busy: configs[3] walk -1.6 %,
        // configs[2] -2.4 %); 64 with lazy refills (trained configs[1]: 96
        // costs +13 %).
        w.job_run = static_cast<int32_t>(env_i64("GDVFS_JOB_RUN", lazy ? 64 : 96));
        if (w.job_run > kJobCap - 32) w.job_run = kJobCap - 32;
        if (w.job_run < 1) w.job_run = 1;
        w.item_next = counts + 2 * b + 1;
        w.pool_cap = static_cast<uint32_t>(pool_cap);
        const int64_t tiles = (n + w.tile_apps - 1) / w.tile_apps;
        const int64_t max_pairs = pe > pt ? pe : pt;
        // Split-major items, one per fetch, ~16 per CTA (measured against
        // tile-major chunks: configs[2] walk -12 %, trained configs[1] -40 %,
        // configs[1] +7 %, the rank restaging per item).  GDVFS_WALK_SPLIT_MAJOR=0:
        // tile-major, ~8 items per CTA in chunks of a quarter of that.
        const bool split_major = env_i64("GDVFS_WALK_SPLIT_MAJOR", 1) != 0;
        // Large batches (>= 32 tiles) take ~32 items per CTA: shorter items
        // even out the CTAs' finishing times (configs[3] -1.3 %, configs[2]
        // -0.9 %); a small batch's items would get too short (configs[1]
        // +9 %: the rank restaging per item) and keep ~16.
        const int64_t items_per_cta = env_i64("GDVFS_WALK_ITEMS", split_major ? (tiles >= 32 ? 32 : 16) : 8);
        int64_t splits = (items_per_cta * sm_count + 2 * tiles - 1) / (2 * tiles);
        splits = env_i64("GDVFS_WALK_SPLITS", splits);
        if (splits > max_pairs) splits = max_pairs;
        if (splits < 1) splits = 1;
        w.splits = static_cast<int32_t>(splits);
        w.tiles = static_cast<int32_t>(tiles);
        w.n_items = static_cast<int32_t>(tiles * 2 * splits);
        w.split_major = split_major ? 1 : 0;
        const int64_t per_cta = (w.n_items + sm_count - 1) / sm_count;
        w.chunk = split_major ? 1 : static_cast<int32_t>(per_cta / 4 > 1 ? per_cta / 4 : 1);
        const int grid = w.n_items < sm_count * walk_per_sm ? w.n_items : sm_count * walk_per_sm;
        walk_kern<<<grid, wg.warps * 32, wg.smem, s>>>(w);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (mark) mark(user, "walk");

        AccParams a{};
        a.nodes[0] = p.e_nodes;
        a.nodes[1] = p.t_nodes;
        a.n_trees[0] = p.e_trees;
        a.n_trees[1] = p.t_trees;
        a.base[0] = p.e_base;
        a.base[1] = p.t_base;
        a.lr[0] = p.e_lr;
        a.lr[1] = p.t_lr;
        a.rec[0] = rec_e;
        a.rec[1] = rec_t;
        a.pool = pool;
        a.rows = p.rows;
        a.cat_t = p.cat_t;
        a.cat_cols = p.cat_cols;
        a.sm = p.sm;
        a.mem = p.mem;
        a.budgets = p.budgets;
        a.out = p.out;
        a.e_out = p.e_out;
        a.t_out = p.t_out;
        a.a0 = a0;
        a.n_apps = n;
        a.n_cols = p.n_cols;
        a.n_cat = p.n_cat;
        a.n_clocks = p.n_clocks;
        a.mode = p.mode;
        a.objective = p.objective;
        a.best_effort = p.best_effort;
        a.out_stride = p.out_stride;
        if (sliced) {
            a.et = et;
            a.arrive = arrive;
            if ((e = static_cast<cudaError_t>(launch_acc_sliced_cpl(a, sm_count, s))) != cudaSuccess) return e;
        } else if ((e = static_cast<cudaError_t>(launch_acc_cpl(a, sm_count, s))) != cudaSuccess) {
            return e;
        }
        if (mark) mark(user, "acc");
        if (launches) *launches += 3;
        if (p.h_rows && b + 1 < nb && (e = upload(b + 1)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace gd
#ifdef GD_WALK_TRACE
extern "C" int gd_debug_walk_trace(unsigned long long* out, int n) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, gd::g_wtrace, static_cast<size_t>(n) * 64));
}
#endif
