// planner.cpp -- host-side planner for the B200 permutation kernels.
//
// GPU analog of the reference's planning layer:
//   merge_dimensions   /root/reference/pkg/src/vecperm/planner.py:211-241 (verbatim semantics)
//   select_block       planner.py:277-352 (re-done at GPU scale: tiles of KBs,
//                      not w <= 16 lanes; no power-of-two padding)
//   BlockPlan.phases   planner.py:178-201 (ragged tiles are predicated in-kernel
//                      instead of separate main/tail loops)
//   format_plan        planner.py:386-419 (vpg_plan_describe)
//
// Classification:
//   merged rank 1                         -> COPY
//   sigma[0] == 0 and row >= 512 B        -> ROWS (K1, 128-bit copy-with-remap)
//   everything else                       -> TILE (K2/K3: smem-staged tile)
//   tiny tensors                          -> GATHER (K0)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <vector>

#include "plan.h"

namespace vpg {

namespace {

constexpr int kTileThreads = 256;
constexpr int64_t kGatherMaxN = 1024;
constexpr int64_t kRowsMinBytes = 512;
// cost of starting one contiguous run; with the ragged-tile factor below,
// tuned on 80 random 64-512 MiB permutations (tools/perf_sweep.py): worst
// case 0.585 -> 0.655 of copy, BASELINE choices unchanged
constexpr double kRunOverheadBytes = 128.0;
constexpr double kTileOverheadBytes = 2048.0;  // cost of one tile (decode + 2 barriers)
constexpr int64_t kTileBudgetBytes = 48 * 1024;  // staged elements per CTA
constexpr double kResidueCostFactor = 0.9;
constexpr double kSw128CostFactor = 0.85;    // 128-byte congruent rows: half the L2 sector requests of the R phase   // residue-stride shifted tiles: no W shift arithmetic
// algorithmic bytes below which tiles shrink to the 24 KiB budget (round 1,
// from cfg1-3).  Timing every tile candidate of 31 random 32-512 MiB
// permutations at 24/32/48 KiB budgets (tools/cand_data.py,
// profiles/cand_data_r2.jsonl): 24 KiB below this size is within noise of
// 48 KiB (mean 0.969 vs 0.969 of the best candidate); a 128 MiB cut measured
// 0.972 -- not enough to move it.
constexpr double kSmallProblemBytes = 512.0 * 1024 * 1024;
constexpr double kWalkWeight = 4.0;
constexpr double kSmallWordMisalignFactor = 1.5;
constexpr int kSmCount = 148;         // B200 SMs (tiny-problem tiling; launches query the device)   // walk cost (ops/element) vs relative geometry cost, per byte of element

int64_t gcd64(int64_t a, int64_t b) {
    a = a < 0 ? -a : a;
    b = b < 0 ? -b : b;
    while (b) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Expected 32-byte sectors touched by a run of `bytes` whose start is a
// multiple of `align` bytes, uniformly distributed modulo 32.
double expected_sectors(int64_t bytes, int64_t align) {
    if (align >= 32 || align <= 0) return (double)((bytes + 31) / 32);
    int64_t cnt = 0, tot = 0;
    for (int64_t o = 0; o < 32; o += align) {
        tot += (o + bytes + 31) / 32;
        ++cnt;
    }
    return (double)tot / (double)cnt;
}

struct Problem {
    int64_t budget;       // staged tile bytes per CTA buffer
    int nbuf;             // forced pipeline stages (0 = planner's choice)
    int64_t cta_smem;     // per-CTA shared-memory target (bytes)
    bool no_shift = false; // disable shifted-run reads (VPG_NO_SHIFT)
    bool no_res = false;   // disable residue row strides for shifted runs (VPG_NO_RES)
    bool no_sw128 = false; // disable the 128-byte congruent layout (VPG_NO_SW128; bulk-read plans)
    bool no_w2 = false;    // disable V x V register-transposed W blocks (VPG_NO_W2)
    bool no_wg = false;    // disable gather W blocks (VPG_WG=0)
    bool force_wg = false; // gather W blocks wherever they apply (VPG_WG=2, experiments)
    bool no_swz_addr = false; // 128-byte residue layouts without the address swizzle (VPG_NO_SWZ_ADDR)
    bool no_bulk = false;  // TMA bulk source reads off (VPG_BULK=0, pull exchanges)
    bool force_bulk = false; // TMA bulk source reads wherever they apply (VPG_BULK=1)
    bool no_swz = true;    // shifted-run chunk swizzle is opt-in (VPG_SWZ=1)
    // W as destination-linear 16-byte chunks (VPG_LIN): 0 off (default:
    // measured slower for every word size -- 4/8-byte words median -4%,
    // tools/lin_ab.py; 1/2-byte words 1.5-2.5x slower,
    // profiles/small_word_r2.txt), -1 cost model, 1 wherever it applies
    int lin_mode = 0;
    int r;
    int64_t d[kMaxRank];
    int sigma[kMaxRank];
    int pos[kMaxRank];
    int64_t in_stride[kMaxRank];
    int64_t out_stride_of_dim[kMaxRank];  // destination stride of source dim k
    int E;
    int64_t n;
    // fused sharded exchange: pin[k] = 2 for the leading input dims (they
    // index the source shard), 1 for the other leading output dims (they
    // index the destination shard), 0 otherwise.  Pinned dims never enter a
    // tile, and the input-shard digits are the slowest grid digits.
    uint8_t pin[kMaxRank] = {};
    int G = 0;          // shards (0: ordinary plan)
    int shard = 0;      // this plan's input shard (push) or output shard (pull)
    bool pull = false;  // pull exchange: pin[k] = 2 marks the leading OUTPUT dims
};

void fill_problem(Problem &P) {
    for (int j = 0; j < P.r; ++j) P.pos[P.sigma[j]] = j;
    P.in_stride[0] = 1;
    for (int k = 1; k < P.r; ++k) P.in_stride[k] = P.in_stride[k - 1] * P.d[k - 1];
    int64_t os = 1;
    for (int j = 0; j < P.r; ++j) {
        P.out_stride_of_dim[P.sigma[j]] = os;
        os *= P.d[P.sigma[j]];
    }
    P.n = os;
}

// ---------------------------------------------------------------- tile geometry
struct TileGeom {
    int64_t ext[kMaxRank];   // 0 = not in tile
    int src_dims[kMaxRank], nsrc;   // source run dims (source order)
    int n_runidx;                   // tile dims outside the source run
    int dst_dims[kMaxRank], ndst;   // destination run dims (dest order)
    int a_part, c_part;             // partial boundary dims (-1 none)
    int64_t Ls, Ld, T;
    double cost, eff_s, eff_d;
};

bool build_geom(const Problem &P, const int64_t *ext, TileGeom &g) {
    const int r = P.r;
    memcpy(g.ext, ext, sizeof(int64_t) * r);
    // source run: greedy over source order
    g.nsrc = 0;
    g.Ls = 1;
    g.a_part = -1;
    for (int k = 0; k < r && ext[k] > 0; ++k) {
        g.src_dims[g.nsrc++] = k;
        g.Ls *= ext[k];
        if (ext[k] < P.d[k]) {
            g.a_part = k;
            break;
        }
    }
    g.ndst = 0;
    g.Ld = 1;
    g.c_part = -1;
    for (int j = 0; j < r && ext[P.sigma[j]] > 0; ++j) {
        int k = P.sigma[j];
        g.dst_dims[g.ndst++] = k;
        g.Ld *= ext[k];
        if (ext[k] < P.d[k]) {
            g.c_part = k;
            break;
        }
    }
    if (g.nsrc == 0 || g.ndst == 0) return false;
    g.T = 1;
    int ntile = 0;
    for (int k = 0; k < r; ++k) {
        if (ext[k] > 0) {
            if (P.pin[k]) return false;   // shard-indexing dims stay grid digits
            g.T *= ext[k];
            ++ntile;
            // every partial dim must be a run boundary
            if (ext[k] < P.d[k] && k != g.a_part && k != g.c_part) return false;
        }
    }
    if (ntile > kMaxTileDims) return false;
    int n_s_runidx = ntile - g.nsrc, n_w_runidx = ntile - g.ndst;
    g.n_runidx = n_s_runidx;
    if (n_s_runidx > kMaxTileDims || n_w_runidx > kMaxTileDims || g.ndst > kMaxTileDims) return false;
    return true;
}

// alignment (elements) shared by all run starts on one side: gcd of the
// strides that move a run start (grid digits and run-index dims).
int64_t run_align_elems(const Problem &P, const TileGeom &g, bool src_side) {
    const int *dims = src_side ? g.src_dims : g.dst_dims;
    const int nd = src_side ? g.nsrc : g.ndst;
    int64_t gg = 0;
    for (int k = 0; k < P.r; ++k) {
        if (P.d[k] <= 1) continue;
        bool in_run = false;
        for (int i = 0; i < nd; ++i)
            if (dims[i] == k) in_run = true;
        int64_t stride = src_side ? P.in_stride[k] : P.out_stride_of_dim[k];
        if (!in_run) gg = gcd64(gg, stride);
        else if (g.ext[k] < P.d[k]) gg = gcd64(gg, stride * g.ext[k]);
    }
    return gg == 0 ? (int64_t)1 << 40 : gg;
}

void score_geom(const Problem &P, TileGeom &g) {
    const int E = P.E;
    int64_t as = run_align_elems(P, g, true) * E;
    int64_t ad = run_align_elems(P, g, false) * E;
    const double ovh_s = getenv("VPG_RUNOVH_S") ? atof(getenv("VPG_RUNOVH_S")) : kRunOverheadBytes;
    const double ovh_d = getenv("VPG_RUNOVH_D") ? atof(getenv("VPG_RUNOVH_D")) : kRunOverheadBytes;
    int64_t bs = g.Ls * E, bd = g.Ld * E;
    g.eff_s = (double)bs / (32.0 * expected_sectors(bs, gcd64(as, 32)));
    g.eff_d = (double)bd / (32.0 * expected_sectors(bd, gcd64(ad, 32)));
    // average valid elements per tile (ragged tiles carry fewer)
    double ntiles = 1.0;
    for (int k = 0; k < P.r; ++k) {
        if (g.ext[k] == 0) ntiles *= (double)P.d[k];
        else if (g.ext[k] < P.d[k]) ntiles *= std::ceil((double)P.d[k] / (double)g.ext[k]);
    }
    double t_avg = (double)P.n / ntiles;
    // ragged tiles run their full walk with idle lanes: the per-element
    // cost grows with the slots per valid element (beta measured on random
    // shapes, tools/perf_sweep.py: a 256-wide tile over a 300-long dim ran
    // at 59% of copy)
    const double beta = getenv("VPG_RAGGED_BETA") ? atof(getenv("VPG_RAGGED_BETA")) : 0.5;
    g.cost = (E / g.eff_s + E / g.eff_d + ovh_s / g.Ls + ovh_d / g.Ld) *
                 (1.0 + beta * ((double)g.T / t_avg - 1.0)) +
             kTileOverheadBytes / t_avg;
    // 1- and 2-byte words move as 16-byte vectors only when run starts keep
    // 16-byte alignment; a tile extent that breaks it (a 1024^2 byte
    // transpose tiled 171 x 128 instead of 128 x 128) falls back to
    // aligned-superset reads and scalar stores of 1-2 bytes, so such
    // geometries rank behind aligned ones
    if (E < 4 && ((as % 16) || (ad % 16))) g.cost *= kSmallWordMisalignFactor;
}

std::vector<int64_t> extent_candidates(int64_t d, int64_t cap) {
    std::vector<int64_t> v;
    if (d <= cap) v.push_back(d);
    for (int64_t p = 1; p < d && p <= cap; p <<= 1) v.push_back(p);
    for (int64_t k = 2; k <= 16; ++k) {
        int64_t e = (d + k - 1) / k;
        if (e >= 1 && e < d && e <= cap) v.push_back(e);
    }
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    return v;
}

// Candidate order: modelled cost; ties (mirror-image tiles) go to the
// smaller tile, then to the longer SOURCE run -- reads gain more from long
// runs than the write-back-cached writes (cfg5: 2 KiB reads x 1 KiB writes
// 670 us vs 1 KiB x 2 KiB 682 us; tools/pick_ab.py).
static bool better(const TileGeom &a, const TileGeom &b) {
    if (a.cost < b.cost - 1e-9) return true;
    if (a.cost > b.cost + 1e-9) return false;
    if (a.T != b.T) return a.T < b.T;
    return a.Ls > b.Ls;
}

bool select_tile(const Problem &P, TileGeom &best, int pick = -1) {
    const int r = P.r;
    const int64_t maxT = std::max<int64_t>(P.budget / P.E, 64);
    bool found = false;
    best.cost = 1e300;
    std::vector<TileGeom> all;   // every candidate, for candidate picks (autotuning, VPG_TILE_PICK)
    int64_t ext[kMaxRank];
    int64_t pre_s = 1;
    for (int a = 0; a < r && pre_s <= maxT; pre_s *= P.d[a], ++a) {
        for (int64_t ea : extent_candidates(P.d[a], maxT / pre_s)) {
            for (int b = 0; b < r; ++b) {
                for (int k = 0; k < r; ++k) ext[k] = 0;
                for (int k = 0; k < a; ++k) ext[k] = P.d[k];
                ext[a] = ea;
                for (int j = 0; j < b; ++j) ext[P.sigma[j]] = P.d[P.sigma[j]];
                int c = P.sigma[b];
                int64_t T0 = 1;
                for (int k = 0; k < r; ++k)
                    if (ext[k] > 0) T0 *= ext[k];
                if (T0 > maxT) break;
                std::vector<int64_t> ecs;
                if (ext[c] == P.d[c]) ecs.push_back(P.d[c]);
                else if (c == a) ecs.push_back(ea);
                else ecs = extent_candidates(P.d[c], maxT / T0);
                for (int64_t ec : ecs) {
                    int64_t e2[kMaxRank];
                    memcpy(e2, ext, sizeof(int64_t) * r);
                    if (e2[c] != P.d[c]) e2[c] = ec;
                    TileGeom g;
                    if (!build_geom(P, e2, g)) continue;
                    if (g.T > maxT) continue;
                    score_geom(P, g);
                    all.push_back(g);
                    if (!found || better(g, best)) {
                        best = g;
                        found = true;
                    }
                }
            }
        }
    }
    if (const char *e = getenv("VPG_TILE_PICK"))
        if (*e) pick = atoi(e);
    if (pick >= 0) {
        std::stable_sort(all.begin(), all.end(), better);
        std::vector<TileGeom> uniq;   // distinct (Ls, Ld, T)
        for (const TileGeom &g : all) {
            bool dup = false;
            for (const TileGeom &u : uniq)
                if (u.Ls == g.Ls && u.Ld == g.Ld && u.T == g.T) dup = true;
            if (!dup) uniq.push_back(g);
        }
        if ((size_t)pick >= uniq.size()) return false;       // no such candidate
        best = uniq[(size_t)pick];
    }
    return found;
}

// Shared-memory bank model: wavefronts for one warp access of 32 lanes to
// element offsets `off` (elements of E bytes).
int warp_wavefronts(const uint32_t *off, int nlanes, int E) {
    int wb = std::max(4, E);             // bytes per bank word
    int lanes_per_phase = 32 / (wb / 4);
    int nbanks = 128 / wb;
    int total = 0;
    for (int p0 = 0; p0 < nlanes; p0 += lanes_per_phase) {
        std::vector<std::vector<uint64_t>> bank(nbanks);
        int deg = 0;
        for (int l = p0; l < std::min(nlanes, p0 + lanes_per_phase); ++l) {
            uint64_t w = ((uint64_t)off[l] * E) / wb;
            auto &b = bank[w % nbanks];
            if (std::find(b.begin(), b.end(), w) == b.end()) b.push_back(w);
            deg = std::max(deg, (int)b.size());
        }
        total += std::max(deg, 1);
    }
    return total;
}

// ------------------------------------------------------------- phase walks
struct PDimH {
    int64_t e, g, s;
    int slot;
    int64_t cmul;
    int64_t hmul = 0;    // shifted-run mode, W phase: source alignment shift per step
};

// Vectorisation choice for one tile: R groups the leading source-run entry
// into 16-byte cp.async chunks; W groups V consecutive dim-0 elements into
// one 16-byte shared-memory load feeding V coalesced scalar stores.
struct VecChoice {
    int vr = 1, vw = 1;
    bool rshift = false;   // R reads 16-byte aligned supersets of misaligned runs
    bool bulk = false;     // R as one cp.async.bulk per source run (producer warp + mbarriers)
    int swz = 0;           // shifted-run mode: chunk swizzle (0 off, else 1 + row shift)
    bool rres = false;     // shifted-run mode with residue row strides (no per-element shift in W)
    bool sw128 = false;    // aligned runs: unpadded rows congruent to their source lines mod 128 B, chunk-swizzled
    bool w2 = false;       // (sw128 only) W in V x V register-transposed blocks with 16-byte stores
    bool swz_addr = true;  // (128-byte residue layouts) address swizzle; off when the bank model prefers plain
    bool res16 = false;    // residue modulus of one 16-byte chunk (TMA bulk reads of misaligned runs)
    bool lin = false;      // W as destination-linear 16-byte chunks (LinDesc)
    int wk = 0;            // W in k x V interleave blocks (k = extent of the destination-innermost dim)
    int wg = 0;            // W in gather blocks: wg destination-innermost elements -> one store (V: 16 bytes; 2, 4, 8 < V: narrow blocks)
};

// smem strides of the tile dims for a given pitch (source run dense, run
// index dims scaled by the pitch).
void tile_sstrides(const Problem &Pb, const TileGeom &g, uint32_t pitch, int64_t *sstr, bool *in_src) {
    for (int k = 0; k < Pb.r; ++k) in_src[k] = false;
    int64_t acc = 1;
    for (int i = 0; i < g.nsrc; ++i) {
        int k = g.src_dims[i];
        in_src[k] = true;
        sstr[k] = acc;
        acc *= g.ext[k];
    }
    // rows (source runs) are ordered by the destination order of their
    // run-index dims: the W phase's lanes then walk consecutive rows, which
    // an odd chunk pitch spreads over all banks (in source order a
    // run-index dim that W visits early can land on a row stride that is a
    // multiple of 8 chunks and alias banks)
    acc = pitch;
    for (int j = 0; j < Pb.r; ++j) {
        const int k = Pb.sigma[j];
        if (g.ext[k] == 0 || in_src[k]) continue;
        sstr[k] = acc;
        acc *= g.ext[k];
    }
}

// Residue row strides for misaligned source runs (shifted-run mode without
// a per-element shift).  Each run-index dim k gets an smem stride S_k with
// S_k == in_stride[k] (mod M, M = res_modulus: 128 bytes of elements), and
// the tile sits at smem offset (source tile base mod M).  Every run then
// starts at the same offset modulo M in shared and in global memory, so its
// 16-byte aligned global superset lands on a 16-byte aligned smem chunk of
// the congruent 128-byte block (R: one L2 request per sector) and the W
// phase reads element (run, e) at an affine offset.  S_1 >= NCK*V (chunks
// per run) and S_{k+1} >= e_k * S_k keep the aligned row spans disjoint.
// Returns the elements one tile buffer needs (M - 1 of base shift included).
int64_t tile_sstrides_res(const Problem &Pb, const TileGeom &g, uint32_t pitch, int V, int64_t *sstr,
                          bool *in_src, int64_t M) {
    for (int k = 0; k < Pb.r; ++k) in_src[k] = false;
    int64_t acc = 1;
    for (int i = 0; i < g.nsrc; ++i) {
        int k = g.src_dims[i];
        in_src[k] = true;
        sstr[k] = acc;
        acc *= g.ext[k];
    }
    const int64_t nck = (g.Ls + V - 1 + V - 1) / V;
    auto with_res = [&](int64_t lo, int64_t res) {
        int64_t r = ((res % M) + M) % M;
        int64_t x = lo + (((r - lo) % M) + M) % M;
        return x;
    };
    int64_t need = std::max<int64_t>((int64_t)pitch, nck * V);
    int64_t last = 0;   // offset of the last run
    for (int j = 0; j < Pb.r; ++j) {
        const int k = Pb.sigma[j];
        if (g.ext[k] == 0 || in_src[k]) continue;
        sstr[k] = with_res(need, Pb.in_stride[k]);
        last += (g.ext[k] - 1) * sstr[k];
        need = sstr[k] * g.ext[k];
    }
    return (last + (M - 1) + nck * V + V - 1) / V * V;
}

// Residue modulus (elements) of the residue row strides: 128 bytes, so each
// run also sits at its source line's offset modulo 128 B and the per-lane
// cp.async requests each L2 sector about once (cfg3: 2.49M -> 1.66M L2 read
// sectors, ncu).  Those plans use the address swizzle (kSwzAddr) and 128-byte
// aligned stage buffers: cfg3 18.4 vs 20.5 us flushed, 15.0 vs 16.7 us steady
// (VPG_RES_MOD=16 restores the chunk-only congruence; with 128 B but no
// swizzle, VPG_NO_SWZ_ADDR=1, the time does not improve).
int64_t res_modulus(int E) {
    static const int64_t bytes = getenv("VPG_RES_MOD") ? std::max(16L, atol(getenv("VPG_RES_MOD"))) : 128;
    return std::max<int64_t>(16 / E, bytes / E);
}

// Phase dims (fastest first) with adjacent dims fused when they are
// contiguous in BOTH global and shared memory (and carry no checked slot).
// R with vr > 1: the leading entry is grouped by vr.  W with vw > 1: dim 0
// is grouped by vw (its V elements are one smem vector, stored separately).
std::vector<PDimH> phase_dims(const Problem &Pb, const TileGeom &g, const int64_t *sstr,
                              const int *slot_of_dim, bool write, int vec, int64_t hmask = 0, bool w2 = false,
                              int wk = 0, int wg = 0) {
    std::vector<PDimH> L;
    bool in_run[kMaxRank] = {false};
    for (int i = 0; i < g.nsrc; ++i) in_run[g.src_dims[i]] = true;
    for (int i = 0; i < Pb.r; ++i) {
        int k = write ? Pb.sigma[i] : i;
        if (g.ext[k] == 0) continue;
        if (write && wk > 0 && i == 0) continue;    // k x V blocks: the innermost dim is inside each block
        PDimH d{g.ext[k], write ? Pb.out_stride_of_dim[k] : Pb.in_stride[k], sstr[k], slot_of_dim[k], 1};
        if (write && hmask && !in_run[k]) d.hmul = Pb.in_stride[k] & hmask;
        // W: dim 0 groups by V (one smem vector); with w2 the destination's
        // innermost dim (first in W order) groups by V too (V rows per block)
        if (write && vec > 1 && (k == 0 || (w2 && i == 0))) {
            d.e /= vec;
            d.g *= vec;
            d.s *= vec;
            d.cmul = vec;
        }
        // W gather blocks: the destination-innermost dim groups by wg (= V)
        if (write && wg > 1 && i == 0) {
            d.e /= wg;
            d.g *= wg;
            d.s *= wg;
            d.cmul = wg;
        }
        if (!L.empty()) {
            PDimH &p = L.back();
            if (p.slot < 0 && d.slot < 0 && d.g == p.g * p.e && d.s == p.s * p.e &&
                !(write && vec > 1 && k == 0) && p.hmul == 0 && d.hmul == 0) {
                p.e *= d.e;
                continue;
            }
        }
        L.push_back(d);
    }
    if (!write && vec > 1) {
        PDimH &f = L.front();
        f.e /= vec;
        f.g *= vec;
        f.s *= vec;
        f.cmul *= vec;
    }
    return L;
}

// R dims in shifted-run mode: the whole source run becomes NCK 16-byte
// chunks (one leading entry), followed by the run-index dims.
std::vector<PDimH> shift_r_dims(const Problem &Pb, const TileGeom &g, const int64_t *sstr, const int *slot_of_dim,
                                int V) {
    std::vector<PDimH> L;
    const int64_t nck = (g.Ls + V - 1 + V - 1) / V;
    L.push_back(PDimH{nck, V, V, -1, 1});
    bool in_run[kMaxRank] = {false};
    for (int i = 0; i < g.nsrc; ++i) in_run[g.src_dims[i]] = true;
    for (int k = 0; k < Pb.r; ++k) {
        if (g.ext[k] == 0 || in_run[k]) continue;
        PDimH d{g.ext[k], Pb.in_stride[k], sstr[k], slot_of_dim[k], 1};
        if (L.size() > 1) {
            PDimH &p = L.back();
            if (p.slot < 0 && d.slot < 0 && d.g == p.g * p.e && d.s == p.s * p.e) {
                p.e *= d.e;
                continue;
            }
        }
        L.push_back(d);
    }
    return L;
}

void set_pdim(PhaseDim &pd, int64_t e, int64_t g, int64_t s, int slot, int64_t cmul, int64_t hmul = 0) {
    pd.hmul = (uint16_t)hmul;
    pd.pad_ = 0;
    pd.div = make_fastdiv((uint32_t)e);
    pd.gstride = g;
    pd.sstride = (uint32_t)s;
    pd.slot = (int16_t)slot;
    pd.cmul = (uint16_t)cmul;
}

// Choose the thread part (prefix dims, split factor f) maximising lane use;
// fill the phase descriptor.  Returns the utilisation estimate.
//
// Threads beyond one thread part share the outer loop.  Two ways:
//   * separable groups: G divides the extent of one outer dim j, and the
//     group index becomes one more thread dim (coordinate g of dim j, the
//     outer dim keeps extent E_j/G at G times the stride).  Every thread
//     then walks the same outer entries (ngroups = 1), so a specialised
//     kernel unrolls the whole walk with constant offsets;
//   * interleaved groups (ngroups = G): thread group g takes outer entries
//     g, g+G, ...; each entry is decoded at run time (about a dozen
//     instructions per entry, amortised over the n_in inner steps).
// The score charges interleaved groups that decode cost.
double make_phase(const std::vector<PDimH> &L, int NT, PhaseDesc &pd, uint32_t &lim_split) {
    memset(&pd, 0, sizeof(pd));
    const int m = (int)L.size();
    double best = -1.0, best_u = 0.0;
    int bh = 0, bj = -1;
    int64_t bf = 1, bG = 1;
    int64_t P = 1;
    const bool no_sep = getenv("VPG_NO_SEPGROUPS") != nullptr;
    for (int h = 0; h < m && P <= NT; P *= L[h].e, ++h) {
        if (h + 1 > kMaxPhaseDims) break;
        for (int64_t f = 1; f <= L[h].e && P * f <= NT; ++f) {
            int64_t ntp = P * f;
            int64_t steps = (L[h].e + f - 1) / f;
            int64_t rest = 1;
            for (int i = h + 1; i < m; ++i) rest *= L[i].e;
            int64_t n_outer = steps > 1 ? rest : (h + 1 < m ? rest / L[h + 1].e : 1);
            int64_t n_in = steps > 1 ? steps : (h + 1 < m ? L[h + 1].e : 1);
            const int first_outer = steps > 1 ? h + 1 : h + 2;
            int nout_dims = m - first_outer;
            if (nout_dims > kMaxPhaseDims) continue;
            if (n_outer < 1) n_outer = 1;
            double pad = (double)L[h].e / (double)(f * steps);
            // coalescing: consecutive lanes must walk globally contiguous
            // elements; `avail` = contiguous extent of the leading dims,
            // `cover` = how much of it one thread part spans
            int64_t avail = L[0].e, cover = h == 0 ? f : L[0].e;
            bool contig = true;
            for (int i = 1; i < m; ++i) {
                if (L[i].g != L[i - 1].g * L[i - 1].e) break;
                avail *= L[i].e;
                if (i < h) cover *= L[i].e;
                else if (i == h && contig) cover *= f;
            }
            for (int i = 1; i <= h && i < m; ++i)
                if (L[i].g != L[i - 1].g * L[i - 1].e) contig = false;
            if (!contig) cover = h == 0 ? f : L[0].e;
            double coal = std::min(1.0, (double)std::min<int64_t>(cover, 32) / (double)std::min<int64_t>(32, avail));
            auto consider = [&](int64_t G, int j, bool sep) {
                double lane = (double)(G * ntp) / NT;
                double bal = sep ? 1.0 : (double)n_outer / (double)(G * ((n_outer + G - 1) / G));
                double u = lane * pad * bal * coal;
                // interleaved groups decode every outer entry at run time
                double eff = (!sep && G > 1) ? u / (1.0 + 2.0 / (double)n_in) : u;
                // ties: bigger thread parts (fewer outer-table steps), longer inner loops
                double score = eff + 1e-3 * std::log2((double)ntp) + 1e-4 * (steps * f == L[h].e) +
                               1e-6 * std::min<int64_t>(n_in, 64) + (sep ? 1e-5 : 0.0);
                if (score > best) {
                    best = score;
                    best_u = u;
                    bh = h;
                    bf = f;
                    bG = G;
                    bj = sep ? j : -1;
                }
            };
            int64_t G = NT / ntp;
            if (G > n_outer) G = n_outer;
            if (G < 1) G = 1;
            consider(G, -1, G == 1);
            if (!no_sep && pd.nthr_dims + 2 <= kMaxPhaseDims && h + 2 <= kMaxPhaseDims)
                for (int j = first_outer; j < m; ++j)
                    for (int64_t Gs = 2; Gs <= L[j].e && ntp * Gs <= NT; ++Gs)
                        if (L[j].e % Gs == 0) consider(Gs, j, true);
        }
    }
    const int h = bh;
    const int64_t f = bf;
    int64_t ntp = 1;
    pd.nthr_dims = 0;
    for (int i = 0; i < h; ++i) {
        set_pdim(pd.thr[pd.nthr_dims++], L[i].e, L[i].g, L[i].s, L[i].slot, L[i].cmul, L[i].hmul);
        ntp *= L[i].e;
    }
    int64_t steps = (L[h].e + f - 1) / f;
    int split_slot = L[h].slot;
    bool padded = steps * f != L[h].e;
    if (padded && split_slot < 0) {
        split_slot = 2;
        lim_split = (uint32_t)(L[h].e * L[h].cmul);
    }
    set_pdim(pd.thr[pd.nthr_dims++], f, L[h].g, L[h].s, split_slot, L[h].cmul, L[h].hmul);
    ntp *= f;
    // separable groups: coordinate g of outer dim bj as the last thread dim
    if (bj >= 0) {
        const PDimH &dj = L[bj];
        set_pdim(pd.thr[pd.nthr_dims++], bG, dj.g, dj.s, dj.slot, dj.cmul, dj.hmul);
        ntp *= bG;
    }
    int first_outer;
    if (steps > 1) {
        pd.n_in = (uint32_t)steps;
        pd.g_in = L[h].g * f;
        pd.s_in = (uint32_t)(L[h].s * f);
        if (split_slot >= 0) pd.c_in[split_slot] = (uint32_t)(f * L[h].cmul);
        pd.h_in = (uint32_t)(f * L[h].hmul);
        first_outer = h + 1;
    } else if (h + 1 < m) {
        pd.n_in = (uint32_t)L[h + 1].e;
        pd.g_in = L[h + 1].g;
        pd.s_in = (uint32_t)L[h + 1].s;
        if (L[h + 1].slot >= 0) pd.c_in[L[h + 1].slot] = (uint32_t)L[h + 1].cmul;
        pd.h_in = (uint32_t)L[h + 1].hmul;
        first_outer = h + 2;
    } else {
        pd.n_in = 1;
        pd.g_in = 0;
        pd.s_in = 0;
        first_outer = m;
    }
    pd.nout_dims = 0;
    int64_t n_outer = 1;
    for (int i = first_outer; i < m; ++i) {
        if (i == bj) {
            if (L[i].e / bG > 1) {
                set_pdim(pd.out[pd.nout_dims++], L[i].e / bG, L[i].g * bG, L[i].s * bG, L[i].slot,
                         L[i].cmul * bG, L[i].hmul * bG);
                n_outer *= L[i].e / bG;
            }
            continue;
        }
        set_pdim(pd.out[pd.nout_dims++], L[i].e, L[i].g, L[i].s, L[i].slot, L[i].cmul, L[i].hmul);
        n_outer *= L[i].e;
    }
    pd.n_outer = (uint32_t)n_outer;
    pd.nthr = (uint32_t)ntp;
    int64_t G = bj >= 0 ? 1 : NT / ntp;
    if (G > n_outer) G = n_outer;
    if (G < 1) G = 1;
    pd.ngroups = (uint32_t)G;
    pd.mask_full = padded ? (1u << split_slot) : 0u;
    pd.mask_ragged = pd.mask_full;
    for (const PDimH &d : L)
        if (d.slot == 0 || d.slot == 1) pd.mask_ragged |= 1u << d.slot;
    return best_u;
}

// smem element offsets seen by the lanes of one warp at inner step 0 of its
// first outer entry (simulation of the kernel's mapping, for the bank model).
uint32_t host_swizzle(const PhaseDesc &pd, uint32_t s, int V) {
    if (!pd.swz) return s;
    if (pd.swz == kSwzAddr) {
        uint32_t lv = 0;
        while ((1 << lv) < V) ++lv;
        return s ^ (((s >> (lv + 3)) & 7u) << lv);
    }
    const uint32_t P = pd.spitch.d, r = s / P, c = s - r * P, f = (r >> (pd.swz - 1)) & 7u;
    return r * P + ((((c / V) ^ f) * V) | (c % V));
}

void phase_warp_offsets(const PhaseDesc &pd, int warp, uint32_t *off, int &nl, uint32_t hmask = 0, int V = 1) {
    nl = 0;
    for (int l = 0; l < 32; ++l) {
        uint32_t t = (uint32_t)(warp * 32 + l);
        if (t >= pd.nthr * pd.ngroups) break;
        uint32_t grp = t / pd.nthr, tr = t % pd.nthr;
        uint32_t s = 0, h = 0;
        for (int i = 0; i < pd.nthr_dims; ++i) {
            uint32_t q = tr / pd.thr[i].div.d;
            s += (tr - q * pd.thr[i].div.d) * pd.thr[i].sstride;
            h += (tr - q * pd.thr[i].div.d) * pd.thr[i].hmul;
            tr = q;
        }
        uint32_t o = grp;
        for (int i = 0; i < pd.nout_dims; ++i) {
            uint32_t q = o / pd.out[i].div.d;
            s += (o - q * pd.out[i].div.d) * pd.out[i].sstride;
            h += (o - q * pd.out[i].div.d) * pd.out[i].hmul;
            o = q;
        }
        off[nl++] = host_swizzle(pd, s + (h & hmask), V);
    }
}

// Can phase R / W be vectorised by V for this geometry (pitch-independent part)?
bool r_vectorizable(const Problem &Pb, const TileGeom &g, int V) {
    if (V <= 1) return false;
    bool in_run[kMaxRank] = {false};
    for (int i = 0; i < g.nsrc; ++i) in_run[g.src_dims[i]] = true;
    // run starts move by the strides of run-index dims, grid dims and the
    // tile step along a partial run boundary: all must keep 16-byte alignment
    for (int k = 0; k < Pb.r; ++k) {
        if (Pb.d[k] <= 1) continue;
        if (!in_run[k] && Pb.in_stride[k] % V) return false;
        if (in_run[k] && g.ext[k] < Pb.d[k] && (Pb.in_stride[k] * g.ext[k]) % V) return false;
    }
    // the grouped leading R entry: whole run, dims 0..a-1, or dim 0 alone (a == 0)
    int64_t unit = g.a_part >= 0 ? g.Ls / g.ext[g.a_part] : g.Ls;
    int64_t lead = g.a_part < 0 ? g.Ls : (g.a_part == 0 ? g.ext[0] : unit);
    if (lead % V) return false;
    if (g.a_part == 0 && (Pb.d[0] % g.ext[0]) % V) return false;   // ragged run lengths
    return true;
}

// W in V x V blocks: the destination-innermost dim sigma[0] is a tile dim
// grouped by V, and every destination offset of a group start is a multiple
// of V (16-byte stores; d[sigma[0]] % V == 0 makes all other destination
// strides, the shard size included, multiples of V).
// elements of the source run before its last (partial) dim, when that dim
// is sigma[0] and they form whole 128-byte lines; 0 otherwise
int64_t w2_in_run_rows(const Problem &Pb, const TileGeom &g) {
    if (g.nsrc < 2 || g.src_dims[g.nsrc - 1] != Pb.sigma[0]) return 0;
    const int64_t lrow = g.Ls / g.ext[Pb.sigma[0]];
    return (lrow * Pb.E) % 128 == 0 ? lrow : 0;
}

bool w2_vectorizable(const Problem &Pb, const TileGeom &g, int V) {
    const int k1 = Pb.sigma[0];
    if (k1 == 0 || g.ext[k1] == 0 || g.ext[k1] % V || Pb.d[k1] % V) return false;
    // the V rows of a block are smem rows (sigma[0] a run-index dim, the
    // first in destination order: stride = pitch), so they share a swizzle
    // group.  sigma[0] may also be the partial last dim of the source run
    // when the run part before it is a whole number of 128-byte lines: the
    // contiguous run is then swizzled as rows of that length (a batched
    // transpose whose source-innermost dim is one 128-byte line, u8
    // attention K^T: tools/cand_scan.py)
    for (int i = 0; i < g.nsrc; ++i)
        if (g.src_dims[i] == k1 && (i + 1 != g.nsrc || !w2_in_run_rows(Pb, g))) return false;
    if (Pb.G >= 1 && (Pb.n / Pb.G) % V) return false;
    return true;
}

// W in k x V interleave blocks: the destination-innermost dim c = sigma[0]
// is small (k = 2..8, wholly inside the tile, its own smem rows) and the
// next destination dim is source dim 0, grouped by V.  A block = k smem
// vectors (one per c, V consecutive dim-0 elements each) = k*V consecutive
// destination elements, stored as k 16-byte chunks (image CHW -> HWC: 3 x
// 16 bytes per block).  Block starts keep 16-byte alignment when d[0] and
// the tile's dim-0 extent are multiples of V.  Returns k, or 0.
// W in gather blocks: V consecutive destination-innermost elements (scalar
// smem loads sstride apart) packed into one 16-byte store -- the
// destination-innermost dim sigma[0] has a tile extent and a full extent
// that are multiples of V, so every block starts 16-byte aligned.  Where the W phase would otherwise store one 1-, 2- or 4-byte
// word per lane (misaligned source runs, residue rows).
bool wg_vectorizable(const Problem &Pb, const TileGeom &g, int V) {
    if (V <= 1) return false;
    const int k1 = Pb.sigma[0];
    if (k1 == 0 || g.ext[k1] == 0 || g.ext[k1] % V || Pb.d[k1] % V) return false;
    // (sigma[0] may also be the partial last dim of the source run -- NCHW ->
    // NHWC with 7x7 maps stages one contiguous 49 x 256 block: the V
    // elements of a block are then 49 apart in smem; scalar loads take any
    // stride)
    if (Pb.G >= 1 && (Pb.n / Pb.G) % V) return false;
    return true;
}

int wk_extent(const Problem &Pb, const TileGeom &g, int V) {
    if (V <= 1 || Pb.r < 2) return 0;
    const int c = Pb.sigma[0];
    if (c == 0 || Pb.sigma[1] != 0) return 0;
    const int64_t k = Pb.d[c];
    if (k < 2 || k > 8 || g.ext[c] != k) return 0;
    for (int i = 0; i < g.nsrc; ++i)
        if (g.src_dims[i] == c) return 0;
    if (g.ext[0] == 0 || g.ext[0] % V || Pb.d[0] % V) return 0;
    if (Pb.G >= 1 && (Pb.n / Pb.G) % V) return 0;
    return (int)k;
}

bool w_vectorizable(const Problem &Pb, const TileGeom &g, int V) {
    if (V <= 1) return false;
    if (g.ext[0] == 0 || g.ext[0] % V) return false;
    if (g.ext[0] < Pb.d[0] && (Pb.d[0] % g.ext[0]) % V) return false;  // ragged dim-0 extents
    // dim 0 is also the destination's stride-1 dim: each smem vector is one
    // 16-byte destination chunk (one store), aligned when d[0] is a multiple
    // of V (short rows below the rows kernel's 512 bytes: attention head
    // splits of 64-128 fp16/u8 elements)
    if (Pb.sigma[0] == 0) return Pb.d[0] % V == 0 && !(Pb.G >= 1 && (Pb.n / Pb.G) % V);
    return true;
}

// 128-byte congruent layout for 16-byte source reads: the run is a whole
// number of 128-byte lines and a power of two (cheap swizzle divide), and
// every stride that moves a run start (run-index dims, grid digits, the
// partial source dim's tile step, the shard bias) keeps 128-byte alignment.
// Swizzled unpadded rows need only runs of a power of two of whole 128-byte
// lines (sw128_layout_ok); the congruence with the source lines (the L2
// request saving) needs the strides too (sw128_possible).
bool sw128_layout_ok(const Problem &Pb, const TileGeom &g) {
    return (g.Ls * Pb.E) % 128 == 0 && (g.Ls & (g.Ls - 1)) == 0;
}

bool sw128_possible(const Problem &Pb, const TileGeom &g) {
    const int64_t E = Pb.E;
    if (!sw128_layout_ok(Pb, g)) return false;
    if (Pb.G >= 1 && ((Pb.n / Pb.G) * E) % 128) return false;   // shard bases keep the congruence
    bool in_run[kMaxRank] = {false};
    for (int i = 0; i < g.nsrc; ++i) in_run[g.src_dims[i]] = true;
    for (int k = 0; k < Pb.r; ++k) {
        if (Pb.d[k] <= 1) continue;
        if (!in_run[k] && (Pb.in_stride[k] * E) % 128) return false;
        if (in_run[k] && g.ext[k] < Pb.d[k] && (Pb.in_stride[k] * g.ext[k] * E) % 128) return false;
    }
    return true;
}

// W as destination-linear 16-byte chunks (LinDesc, tile_write_lin): for 4-
// and 8-byte words whose W phase would otherwise store one word per lane
// (no vector grouping, no per-element shift), with destination runs of at
// least 2 chunks and an offset table of at most 16 KiB.
constexpr uint64_t kLinTableMax = 16384;
uint64_t lin_table_bytes(int64_t Ld, int V) {
    const uint64_t cpr = (uint64_t)((Ld + V - 2) / V + 1);
    return (uint64_t)V * cpr * (uint64_t)V * 2;
}

bool lin_applicable(const Problem &Pb, const TileGeom &g, const VecChoice &vc) {
    if (Pb.lin_mode == 0 || Pb.E >= 16) return false;
    if (vc.vw > 1 || vc.w2 || vc.wk || vc.wg || vc.bulk || (vc.rshift && !vc.rres)) return false;
    const int V = 16 / Pb.E;
    if (g.Ld < 2 * V || g.ndst > kMaxLinDims || g.T / g.Ld > 0xffffffffLL) return false;
    int nx = 0;
    for (int k = 0; k < Pb.r; ++k)
        if (g.ext[k] > 0) ++nx;
    if (nx - g.ndst > kMaxPhaseDims) return false;
    return lin_table_bytes(g.Ld, V) <= kLinTableMax;
}

// Run dims = the destination run (only its last dim may be partial, so the
// valid positions of a ragged run are a prefix); run-index dims in
// destination order.
void fill_lin(const Problem &Pb, const TileGeom &g, const int64_t *sstr, const int *slot_of_dim, int NT,
              TileParams &tp) {
    LinDesc &L = tp.lin;
    const int V = 16 / Pb.E;
    L.on = 1;
    L.nt = (uint32_t)NT;
    L.run_len = (uint32_t)g.Ld;
    L.cpr = (uint32_t)((g.Ld + V - 2) / V + 1);
    L.cprd = make_fastdiv(L.cpr);
    L.nchunks = (uint32_t)(g.T / g.Ld) * L.cpr;
    bool in_run[kMaxRank] = {false};
    L.nrd = g.ndst;
    for (int i = 0; i < g.ndst; ++i) {
        const int k = g.dst_dims[i];
        in_run[k] = true;
        set_pdim(L.rd[i], g.ext[k], Pb.out_stride_of_dim[k], sstr[k], i + 1 == g.ndst ? slot_of_dim[k] : -1, 1);
    }
    const int kl = g.dst_dims[g.ndst - 1];
    L.last_slot = slot_of_dim[kl];
    L.last_unit = (uint32_t)(g.Ld / g.ext[kl]);
    L.nxd = 0;
    for (int j = 0; j < Pb.r; ++j) {
        const int k = Pb.sigma[j];
        if (g.ext[k] == 0 || in_run[k]) continue;
        set_pdim(L.xd[L.nxd++], g.ext[k], Pb.out_stride_of_dim[k], sstr[k], slot_of_dim[k], 1);
    }
}

// smem element offset of destination-run position j (host mirror of the
// kernel's table entries)
uint32_t lin_offset(const LinDesc &L, uint32_t j) {
    uint32_t off = 0;
    for (int k = 0; k < L.nrd; ++k) {
        const uint32_t e = L.rd[k].div.d, q = j / e;
        off += (j - q * e) * L.rd[k].sstride;
        j = q;
    }
    return off;
}

// smem wavefronts of one warp's V loads of a chunk step (lanes on chunk
// slots 0..31 of a run, averaged over the run's start offsets m) with the
// bank-spreading rotation `rs` (32 = none)
double lin_waves(const Problem &Pb, const PhaseDesc &d, const LinDesc &L, uint32_t rs) {
    const int V = 16 / Pb.E;
    uint32_t off[32];
    double waves = 0.0;
    for (int m = 0; m < V; ++m)
        for (int k = 0; k < V; ++k) {
            int nl = 0;
            for (int l = 0; l < 32; ++l) {
                const int e = (k + (rs < 32 ? (l >> rs) : 0)) & (V - 1);
                const int j = l * V + e - m;
                if (j < 0 || j >= (int)L.run_len) continue;
                off[nl++] = host_swizzle(d, lin_offset(L, (uint32_t)j), V);
            }
            if (nl) waves += warp_wavefronts(off, nl, Pb.E);
        }
    return waves / V;
}

// Fill TileParams for geometry g, smem pitch (elements) and vector choice.
double fill_tile_params(const Problem &Pb, const TileGeom &g, uint32_t pitch, int NT, VecChoice vc,
                        TileParams &tp) {
    memset(&tp, 0, sizeof(tp));
    const int r = Pb.r;
    tp.Ls = (uint32_t)g.Ls;
    tp.Ld = (uint32_t)g.Ld;
    tp.T = (uint32_t)g.T;
    tp.pitch = pitch;
    const uint32_t Ns = (uint32_t)(g.T / g.Ls);
    tp.tile_elems_alloc = Ns * pitch;
    int64_t sstr[kMaxRank];
    bool in_src[kMaxRank];
    const int V = 16 / Pb.E;
    const int64_t M = vc.res16 ? V : res_modulus(Pb.E);
    if (vc.rres) tp.tile_elems_alloc = (uint32_t)tile_sstrides_res(Pb, g, pitch, V, sstr, in_src, M);
    else tile_sstrides(Pb, g, pitch, sstr, in_src);
    int slot_of_dim[kMaxRank];
    for (int k = 0; k < r; ++k) slot_of_dim[k] = -1;
    if (g.a_part >= 0) slot_of_dim[g.a_part] = 0;
    if (g.c_part >= 0 && g.c_part != g.a_part) slot_of_dim[g.c_part] = 1;
    const int64_t hmask = vc.rshift && !vc.rres ? V - 1 : 0;
    double u0 = make_phase(vc.rshift ? shift_r_dims(Pb, g, sstr, slot_of_dim, V)
                                     : phase_dims(Pb, g, sstr, slot_of_dim, false, vc.vr),
                           NT, tp.ph[0], tp.lim_split[0]);
    double u1 = make_phase(phase_dims(Pb, g, sstr, slot_of_dim, true, vc.vw, hmask, vc.w2, vc.wk,
                                      vc.wg), NT, tp.ph[1], tp.lim_split[1]);
    if (vc.w2) {
        tp.ph[1].w2 = 1;
        tp.ph[1].vrow = (uint32_t)sstr[Pb.sigma[0]];    // == pitch (w2_vectorizable)
    } else if (vc.wk) {
        tp.ph[1].w2 = (uint32_t)vc.wk;                  // >= 2: k x V interleave blocks
        tp.ph[1].vrow = (uint32_t)sstr[Pb.sigma[0]];    // smem stride of the innermost destination dim
    } else if (vc.wg) {
        tp.ph[1].w2 = kW2Gather + (vc.wg == V ? 0u : (uint32_t)vc.wg);
        tp.ph[1].vrow = (uint32_t)sstr[Pb.sigma[0]];
    }
    if (vc.lin) fill_lin(Pb, g, sstr, slot_of_dim, NT, tp);
    tp.ph[0].rshift = vc.rshift ? (vc.rres ? 2u : 1u) : 0u;
    tp.hmask = (uint32_t)hmask;
    tp.rres = vc.rres ? (uint32_t)(M - 1) : 0u;
    if (vc.rres && M * Pb.E >= 128 && !Pb.no_swz_addr && vc.swz_addr)
        for (int ph = 0; ph < 2; ++ph) tp.ph[ph].swz = kSwzAddr;
    if ((vc.swz && vc.rshift && vc.vw == 1 && !vc.bulk) || (vc.sw128 && !vc.bulk)) {
        // congruent layout: XOR by row (W lanes walk rows), or by row group
        // of V rows with w2 (W lanes walk V-row groups)
        uint32_t lv = 0;
        while ((1 << lv) < V) ++lv;
        for (int ph = 0; ph < 2; ++ph) {
            tp.ph[ph].swz = vc.sw128 ? (vc.w2 ? 1u + lv : 1u) : (uint32_t)vc.swz;
            // (V x V blocks over sigma[0] inside the source run: rows of the
            // run part before it, w2_in_run_rows)
            const int64_t lrow = vc.w2 ? w2_in_run_rows(Pb, g) : 0;
            tp.ph[ph].spitch = make_fastdiv(lrow ? (uint32_t)lrow : pitch);
        }
    }
    if (tp.lin.on) {
        uint32_t best_rs = 32;
        double best_w = lin_waves(Pb, tp.ph[1], tp.lin, 32);
        static const bool no_rot = getenv("VPG_LIN_ROT") && atoi(getenv("VPG_LIN_ROT")) == 0;   // experiments
        for (uint32_t rs = 0; rs < 3 && !no_rot; ++rs) {
            const double w = lin_waves(Pb, tp.ph[1], tp.lin, rs);
            if (w < best_w - 1e-9) {
                best_w = w;
                best_rs = rs;
            }
        }
        tp.lin.rot_shift = best_rs;
    }
    if (vc.bulk) {
        tp.bulk = 1;
        tp.nruns = (uint32_t)(g.T / g.Ls);
        tp.run_bytes = (uint32_t)(g.Ls * Pb.E);
        tp.run_unit_bytes = (uint32_t)((g.a_part >= 0 ? g.Ls / g.ext[g.a_part] : g.Ls) * Pb.E);
        tp.nrdims = 0;
        for (int k = 0; k < r; ++k) {
            if (g.ext[k] == 0 || in_src[k]) continue;
            set_pdim(tp.rdims[tp.nrdims++], g.ext[k], Pb.in_stride[k], sstr[k], slot_of_dim[k], 1);
        }
    }
    tp.n_elems = Pb.n;
    tp.ph[0].vec = (uint32_t)vc.vr;
    tp.ph[1].vec = (uint32_t)vc.vw;
    tp.ph[1].vstride = vc.vw > 1 ? Pb.out_stride_of_dim[0] : 0;
    // grid digits
    struct Dg {
        int64_t ext, ss, ds;
        int dim;     // partial tile dim (-1: whole grid dim)
        int src;     // input-shard dim index (-1: other)
    };
    std::vector<Dg> dg;
    for (int k = 0; k < r; ++k) {
        if (g.ext[k] == 0)
            dg.push_back({Pb.d[k], Pb.in_stride[k], Pb.out_stride_of_dim[k], -1, Pb.pin[k] == 2 ? k : -1});
        else if (g.ext[k] < Pb.d[k])
            dg.push_back({(Pb.d[k] + g.ext[k] - 1) / g.ext[k], Pb.in_stride[k] * g.ext[k],
                          Pb.out_stride_of_dim[k] * g.ext[k], k, -1});
    }
    // destination-stride order (the reference's counter digits,
    // planner.py:324-342); input-shard digits last, inner to outer, so a
    // shard's tiles form one contiguous range of the tile index
    // (pull exchange: the pinned digits index the OUTPUT shard, so they rank
    // by output position)
    std::stable_sort(dg.begin(), dg.end(), [&Pb](const Dg &x, const Dg &y) {
        if ((x.src >= 0) != (y.src >= 0)) return y.src >= 0;
        if (x.src >= 0) return Pb.pull ? Pb.pos[x.src] < Pb.pos[y.src] : x.src < y.src;
        static const bool by_src = getenv("VPG_ORDER_SRC") != nullptr;   // experiments
        return by_src ? x.ss < y.ss : x.ds < y.ds;
    });
    tp.ngrid = (int32_t)dg.size();
    tp.grid_a = tp.grid_c = -1;
    uint64_t cum = 1;
    for (size_t i = 0; i < dg.size(); ++i) {
        tp.grid[i].cum = make_fastdiv((uint32_t)std::min<uint64_t>(cum, 0xffffffffull));
        tp.grid[i].ext = make_fastdiv((uint32_t)dg[i].ext);
        tp.grid[i].src_stride = dg[i].ss;
        tp.grid[i].dst_stride = dg[i].ds;
        if (dg[i].dim >= 0 && dg[i].dim == g.a_part) tp.grid_a = (int32_t)i;
        if (dg[i].dim >= 0 && dg[i].dim == g.c_part && g.c_part != g.a_part) tp.grid_c = (int32_t)i;
        cum *= (uint64_t)dg[i].ext;
    }
    tp.num_tiles = (uint32_t)std::min<uint64_t>(cum, 0xffffffffull);
    if (Pb.G >= 1) {
        const uint64_t per = cum / (uint64_t)Pb.G;
        tp.nshards = (uint32_t)Pb.G;
        tp.num_tiles = (uint32_t)std::min<uint64_t>(per, 0xffffffffull);
        tp.tile_begin = (uint32_t)std::min<uint64_t>(per * (uint64_t)Pb.shard, 0xffffffffull);
        tp.shard_elems = Pb.n / Pb.G;
        if (Pb.pull) {
            tp.pull = 1;
            tp.src_bias = 0;
            tp.dst_bias = tp.shard_elems * Pb.shard;
            tp.n_elems = Pb.n;            // source offsets are global
            const uint64_t S = (uint64_t)tp.shard_elems;
            tp.shard_shift = 0;
            if (S > 1 && (S & (S - 1)) == 0)
                while ((1ull << tp.shard_shift) < S) ++tp.shard_shift;
            tp.shard_div = make_fastdiv((uint32_t)std::min<uint64_t>(S, 0xffffffffull));
        } else {
            tp.src_bias = tp.shard_elems * Pb.shard;
            tp.n_elems = tp.shard_elems;  // source bounds: the local shard
        }
    }
    tp.src_span = 1;
    for (int k = 0; k < r; ++k)
        if (g.ext[k] > 0) tp.src_span += (g.ext[k] - 1) * Pb.in_stride[k];
    tp.e_a = g.a_part >= 0 ? (uint32_t)g.ext[g.a_part] : 1u;
    tp.d_a = g.a_part >= 0 ? (uint32_t)Pb.d[g.a_part] : 1u;
    bool c_slot = g.c_part >= 0 && g.c_part != g.a_part;
    tp.e_c = c_slot ? (uint32_t)g.ext[g.c_part] : 1u;
    tp.d_c = c_slot ? (uint32_t)Pb.d[g.c_part] : 1u;
    // dynamic smem layout
    uint32_t o = 0;
    auto take = [&](uint64_t bytes, uint32_t al) {
        o = (o + al - 1) / al * al;
        uint32_t at = o;
        o += (uint32_t)bytes;
        return at;
    };
    tp.ph[0].off_tab = take(kOuterEntryBytes * tp.ph[0].n_outer, 16);
    tp.ph[1].off_tab = take(kOuterEntryBytes * tp.ph[1].n_outer, 16);
    uint64_t buf_bytes = ((uint64_t)tp.tile_elems_alloc * Pb.E + 15) / 16 * 16;
    if (vc.rres && M * Pb.E >= 128) {
        // every stage buffer 128-byte aligned (the residue congruence is mod 128 B)
        buf_bytes = (buf_bytes + 127) / 128 * 128;
        tp.tile_elems_alloc = (uint32_t)(buf_bytes / Pb.E);
    }
    // lin mode: u16 table entries hold smem element offsets inside one buffer
    if (tp.lin.on && tp.tile_elems_alloc >= 65536u) memset(&tp.lin, 0, sizeof(tp.lin));
    if (tp.lin.on) tp.lin.tab_off = take(lin_table_bytes(g.Ld, V), 16);
    // pipeline depth: as many stages as fit the per-CTA smem target (two
    // CTAs per SM), at least 2, at most 8 (1- and 2-byte words too: their
    // vectorised reads are 16-byte cp.async, their scalar reads synchronous)
    uint32_t stages = 1;
    {
        uint64_t room = (uint64_t)Pb.cta_smem > o + 1024 ? (uint64_t)Pb.cta_smem - o - 1024 : 0;
        stages = (uint32_t)std::min<uint64_t>(8, std::max<uint64_t>(2, room / buf_bytes));
        if (Pb.nbuf > 0) stages = (uint32_t)Pb.nbuf;
    }
    tp.nbuf = stages;
    tp.off_buf = take(buf_bytes * tp.nbuf, 128);
    tp.smem_bytes = (o + 15) / 16 * 16 + 128;     // + slack: the kernel aligns its base to 128 bytes
    return u0 * u1;
}

// Modelled per-tile cost of a (pitch, vector) choice: smem wavefronts of
// both phases (simulated warp by warp) plus issued memory instructions.
double tile_cost(const Problem &Pb, const TileParams &tp) {
    double cost = 0.0;
    uint32_t off[32];
    int nl;
    for (int ph = 0; ph < 2; ++ph) {
        const PhaseDesc &d = tp.ph[ph];
        if (ph == 1 && tp.lin.on) {
            // lin W: per warp chunk step one table load, V scalar smem loads
            // (lanes on consecutive chunk slots of one run) and one 16-byte
            // store, plus the slot decode
            const LinDesc &L = tp.lin;
            const double waves = lin_waves(Pb, d, L, L.rot_shift);
            const double ops = std::ceil((double)L.nchunks / 32.0);
            cost += ops * (1.0 + waves + 1.0 + 2.0);
            continue;
        }
        const int V = (int)d.vec;
        const int abytes = Pb.E * V;
        int64_t waves = 0, warps = 0;
        for (int w = 0; w < 8; ++w) {
            phase_warp_offsets(d, w, off, nl, ph == 1 ? tp.hmask : 0, 16 / Pb.E > 0 ? 16 / Pb.E : 1);
            if (!nl) continue;
            for (int l = 0; l < nl; ++l) off[l] /= (uint32_t)V;     // in access units
            waves += warp_wavefronts(off, nl, abytes);
            ++warps;
        }
        if (!warps) continue;
        // warp-level memory ops actually issued by the walk (idle lanes included)
        const double nwarps = std::ceil((double)d.nthr * d.ngroups / 32.0);
        const double ops = nwarps * d.n_in * std::ceil((double)d.n_outer / d.ngroups);
        const double avg_w = (double)waves / (double)warps;
        const bool checked = d.mask_full != 0;
        // LDGSTS: issue + global request + smem; 8 (was 4) lets 16-byte
        // aligned-superset reads win over 4-byte ones on misaligned runs
        // (odd 2-D transposes 0.70 -> 0.78 of copy; random-shape p10 +1-3%)
        const double kr = getenv("VPG_R_OP_COST") ? atof(getenv("VPG_R_OP_COST")) : 8.0;
        if (ph == 0) cost += ops * (kr + avg_w + (checked ? 2.0 : 0.0));
        else if (d.w2 == 1) cost += ops * (V * avg_w + V + 1.0 + (checked ? 2.0 : 0.0));    // V LDS.128 + V STG.128
        else if (d.w2 >= kW2Gather) {
            // Vg scalar LDS + one store (+ packing)
            const int Vg = d.w2 == kW2Gather ? 16 / Pb.E : (int)(d.w2 - kW2Gather);
            cost += ops * (Vg * avg_w + 1.0 + 0.25 * Vg + (checked ? 2.0 : 0.0));
        }
        else if (d.w2 >= 2) cost += ops * (d.w2 * avg_w + d.w2 + 1.0 + (checked ? 2.0 : 0.0)); // k LDS.128 + k STG.128
        else cost += ops * (avg_w + (V > 1 ? V : 1) + 1.0 + (checked ? 2.0 : 0.0)); // LDS + STGs
    }
    return cost;
}

// Every source run of the tile starts at a multiple of V elements: the
// strides that move a run start (run-index dims, grid dims, the tile step
// along a partial run dim, the shard bias) are multiples of V.
bool src_starts_aligned(const Problem &Pb, const TileGeom &g, int V) {
    bool in_run[kMaxRank] = {false};
    for (int i = 0; i < g.nsrc; ++i) in_run[g.src_dims[i]] = true;
    for (int k = 0; k < Pb.r; ++k) {
        if (Pb.d[k] <= 1) continue;
        if (!in_run[k] && Pb.in_stride[k] % V) return false;
        if (in_run[k] && g.ext[k] < Pb.d[k] && (Pb.in_stride[k] * g.ext[k]) % V) return false;
    }
    if (Pb.G >= 1 && (Pb.n / Pb.G) % V) return false;
    return true;
}

// Choose pitch and vectorisation that minimise the modelled tile cost.
void choose_pitch_vec(const Problem &Pb, const TileGeom &g, int NT, uint32_t &pitch_out, VecChoice &vc_out) {
    // 16-byte vectors for every word size below 16 bytes (1- and 2-byte
    // words too: fp16/bf16 and byte tensors, including aligned-superset
    // reads of misaligned runs); TMA bulk modes exist for 4- and 8-byte words
    const int V = Pb.E < 16 ? 16 / Pb.E : 1;
    const bool rv = r_vectorizable(Pb, g, V);
    const bool wv = w_vectorizable(Pb, g, V);
    // shifted-run reads: misaligned source runs long enough to amortise the
    // superset (up to V-1 extra elements at each end)
    const bool rs = V > 1 && !rv && g.Ls >= 2 * V && !Pb.no_shift;
    double best = -1.0;
    pitch_out = (uint32_t)g.Ls;
    struct Opt {
        int vr, vw;
        bool rshift;
    };
    std::vector<Opt> opts;
    for (int vr : {1, V})
        for (int vw : {1, V}) {
            if ((vr > 1 && !rv) || (vw > 1 && !wv)) continue;
            opts.push_back({vr, vw, false});
        }
    if (rs) opts.push_back({V, 1, true});
    // swizzled unpadded rows: wherever the layout fits; the L2 saving (cost
    // factor) only where the rows are congruent to their source lines
    const bool s128 = rv && !Pb.no_sw128 && sw128_layout_ok(Pb, g);
    const double s128_factor = sw128_possible(Pb, g) ? kSw128CostFactor : 1.0;
    // the same layout with the W phase in gather blocks (16-byte stores)
    auto wg_try = [&](VecChoice vc, uint32_t pitch, double factor) {
        if (vc.vw > 1 || vc.w2 || vc.wk || vc.bulk || vc.lin || (vc.rshift && !vc.rres) || Pb.no_wg) return;
        // the widest block the destination-innermost extent allows: V (16-byte
        // stores), or for 1- and 2-byte words V/2, V/4 ... >= 2 (8- and 4-byte
        // stores; VPG_WG_NARROW=0 keeps the full width only)
        static const bool narrow = !(getenv("VPG_WG_NARROW") && atoi(getenv("VPG_WG_NARROW")) == 0);
        int wgw = 0;
        for (int w = V; w >= 2; w /= 2) {
            static const int narrow_maxE = getenv("VPG_WG_NARROW_E") ? atoi(getenv("VPG_WG_NARROW_E")) : 2;
            if (w < V && (Pb.E > narrow_maxE || !narrow)) break;
            if (wg_vectorizable(Pb, g, w)) {
                wgw = w;
                break;
            }
        }
        if (!wgw) return;
        vc.wg = wgw;
        TileParams tp;
        fill_tile_params(Pb, g, pitch, NT, vc, tp);
        const double c = tile_cost(Pb, tp) * factor * (Pb.force_wg ? 1e-6 : 1.0);
        if (getenv("VPG_DEBUG_PLAN"))
            fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u vr %d rshift %d rres %d gather cost %.1f per-elem %.3f\n",
                    (long long)g.Ls, (long long)g.Ld, pitch, vc.vr, (int)vc.rshift, (int)vc.rres, c, c / (double)g.T);
        if (best < 0 || c < best - 1e-9) {
            best = c;
            pitch_out = pitch;
            vc_out = vc;
        }
    };
    // the same layout with the W phase as destination-linear 16-byte chunks
    auto lin_try = [&](VecChoice vc, uint32_t pitch, double factor) {
        if (!lin_applicable(Pb, g, vc)) return;
        vc.lin = true;
        TileParams tp;
        fill_tile_params(Pb, g, pitch, NT, vc, tp);
        if (!tp.lin.on) return;
        double c = tile_cost(Pb, tp) * factor;
        if (Pb.lin_mode == 1) c *= 1e-6;    // forced wherever it applies
        if (getenv("VPG_DEBUG_PLAN"))
            fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u vr %d rshift %d rres %d swz %d lin cost %.1f per-elem %.3f\n",
                    (long long)g.Ls, (long long)g.Ld, pitch, vc.vr, (int)vc.rshift, (int)vc.rres, (int)vc.swz_addr,
                    c, c / (double)g.T);
        if (best < 0 || c < best - 1e-9) {
            best = c;
            pitch_out = pitch;
            vc_out = vc;
        }
    };
    for (const Opt &op : opts) {
        if (s128 && op.vr > 1 && !op.rshift && (int64_t)(g.T / g.Ls) * g.Ls * Pb.E <= Pb.budget + 8192) {
            // congruent rows (pitch = run, no padding), chunk swizzle against
            // the W bank conflicts; per-lane cp.async then requests each L2
            // sector once instead of ~twice
            for (int w2 = 0; w2 < 3; ++w2) {
                if (w2 == 1 && !(op.vw > 1 && !Pb.no_w2 && w2_vectorizable(Pb, g, V))) continue;
                if (w2 == 2 && !(op.vw > 1 && !Pb.no_w2 && wk_extent(Pb, g, V))) continue;
                TileParams tp;
                VecChoice vc;
                vc.vr = op.vr;
                vc.vw = op.vw;
                vc.sw128 = true;
                vc.w2 = w2 == 1;
                vc.wk = w2 == 2 ? wk_extent(Pb, g, V) : 0;
                fill_tile_params(Pb, g, (uint32_t)g.Ls, NT, vc, tp);
                double c = tile_cost(Pb, tp) * s128_factor;
                if (getenv("VPG_DEBUG_PLAN"))
                    fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %lld vr %d vw %d sw128 w2 %d cost %.1f per-elem %.3f\n",
                            (long long)g.Ls, (long long)g.Ld, (long long)g.Ls, vc.vr, vc.vw, w2, c, c / (double)g.T);
                if (best < 0 || c < best - 1e-9) {
                    best = c;
                    pitch_out = (uint32_t)g.Ls;
                    vc_out = vc;
                }
                lin_try(vc, (uint32_t)g.Ls, s128_factor);
                wg_try(vc, (uint32_t)g.Ls, s128_factor);
            }
        }
        if (op.rshift && !Pb.no_swz && op.vw == 1) {
            // swizzled rows: pitch a multiple of 8 chunks, row shift 0..3
            const int64_t base = (g.Ls + V - 1 + V - 1) / V * V;
            const int64_t p8 = (base + 8 * V - 1) / (8 * V) * (8 * V);
            for (int sw = 1; sw <= 4; ++sw) {
                const uint32_t pitch = (uint32_t)p8;
                if ((int64_t)(g.T / g.Ls) * pitch * Pb.E > Pb.budget + 16384) break;
                TileParams tp;
                VecChoice vc;
                vc.vr = op.vr;
                vc.vw = op.vw;
                vc.rshift = true;
                vc.swz = sw;
                fill_tile_params(Pb, g, pitch, NT, vc, tp);
                double c = tile_cost(Pb, tp);
                if (getenv("VPG_DEBUG_PLAN"))
                    fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u shift-swizzle %d cost %.1f per-elem %.3f\n",
                            (long long)g.Ls, (long long)g.Ld, pitch, sw, c, c / (double)g.T);
                if (best < 0 || c < best - 1e-9) {
                    best = c;
                    pitch_out = pitch;
                    vc_out = vc;
                }
            }
        }
        if (op.rshift && !Pb.no_res) {
            // residue row strides: pitch candidates NCK*V + pad (rounded up to
            // the first run-index dim's residue inside tile_sstrides_res)
            const int64_t base = (g.Ls + V - 1 + V - 1) / V * V;
            for (int pad = 0; pad <= 32 * 2 + 1; ++pad) {
                // odd/even pad index: address swizzle on/off (the bank model
                // decides; with 128-byte residues the W lanes' banks are set
                // by the source strides and the swizzle can add conflicts)
                const uint32_t pitch = (uint32_t)(base + pad / 2);
                if ((int64_t)(g.T / g.Ls) * pitch * Pb.E > Pb.budget + 8192) break;
                TileParams tp;
                VecChoice vc;
                vc.vr = op.vr;
                vc.vw = op.vw;
                vc.rshift = true;
                vc.rres = true;
                vc.swz_addr = (pad & 1) == 0;
                fill_tile_params(Pb, g, pitch, NT, vc, tp);
                // no per-element shift arithmetic in W: cheaper per element
                double c = tile_cost(Pb, tp) * kResidueCostFactor *
                           (res_modulus(Pb.E) * Pb.E >= 128 ? kSw128CostFactor : 1.0);   // 128-byte congruence
                if (getenv("VPG_DEBUG_PLAN"))
                    fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u residue swz %d cost %.1f per-elem %.3f\n",
                            (long long)g.Ls, (long long)g.Ld, pitch, (int)vc.swz_addr, c, c / (double)g.T);
                if (best < 0 || c < best - 1e-9) {
                    best = c;
                    pitch_out = pitch;
                    vc_out = vc;
                }
                lin_try(vc, pitch, kResidueCostFactor * (res_modulus(Pb.E) * Pb.E >= 128 ? kSw128CostFactor : 1.0));
                wg_try(vc, pitch, kResidueCostFactor * (res_modulus(Pb.E) * Pb.E >= 128 ? kSw128CostFactor : 1.0));
            }
        }
        if (op.rshift && Pb.force_bulk && !Pb.no_bulk && (Pb.E == 4 || Pb.E == 8) && g.n_runidx <= kMaxPhaseDims) {
            // TMA bulk reads of misaligned runs: one cp.async.bulk per run's
            // 16-byte aligned superset (producer warp, tile_body_bulk) into
            // rows with 16-byte residue strides.  The bulk engine keeps L2
            // requests at one per sector whatever the smem offset (per-lane
            // cp.async into rows not congruent mod 128 B requests them ~2x),
            // so the strides are free modulo 128 B: the pitch is chosen for
            // the W lanes' banks.  Experimental (VPG_BULK=1).
            const int64_t base = (g.Ls + V - 1 + V - 1) / V * V;
            double bb = -1.0;
            for (int pad = 0; pad <= 32; ++pad) {
                const uint32_t pitch = (uint32_t)(base + pad);
                if ((int64_t)(g.T / g.Ls) * pitch * Pb.E > Pb.budget + 8192) break;
                TileParams tp;
                VecChoice vc;
                vc.vr = op.vr;
                vc.vw = op.vw;
                vc.rshift = true;
                vc.rres = true;
                vc.res16 = true;
                vc.swz_addr = false;
                vc.bulk = true;
                fill_tile_params(Pb, g, pitch, NT, vc, tp);
                const double c = tile_cost(Pb, tp);
                if (getenv("VPG_DEBUG_PLAN"))
                    fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u bulk-residue cost %.1f per-elem %.3f\n",
                            (long long)g.Ls, (long long)g.Ld, pitch, c, c / (double)g.T);
                if (bb < 0 || c < bb - 1e-9) {
                    bb = c;
                    pitch_out = pitch;
                    vc_out = vc;
                    best = 0.0;     // forced: wins over every per-lane option
                }
            }
            return;
        }
        if (op.rshift && op.vw > 1) continue;     // narrow W vectors: residue rows only
        const int step = (op.vr > 1 || op.vw > 1) ? V : 1;
        const int64_t base = op.rshift ? (g.Ls + V - 1 + V - 1) / V * V : g.Ls;
        static const int pad_max = getenv("VPG_PAD_MAX") ? atoi(getenv("VPG_PAD_MAX")) : 32;   // experiments
        for (int pad = 0; pad <= pad_max; pad += step) {
            uint32_t pitch = (uint32_t)(base + pad);
            if ((int64_t)(g.T / g.Ls) * pitch * Pb.E > Pb.budget + 8192) break;
            TileParams tp;
            VecChoice vc;
            vc.vr = op.vr;
            vc.vw = op.vw;
            vc.rshift = op.rshift;
            fill_tile_params(Pb, g, pitch, NT, vc, tp);
            double c = tile_cost(Pb, tp);
            if (getenv("VPG_DEBUG_PLAN"))
                fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u vr %d vw %d shift %d cost %.1f per-elem %.3f\n",
                        (long long)g.Ls, (long long)g.Ld, pitch, vc.vr, vc.vw, (int)vc.rshift, c, c / (double)g.T);
            if (best < 0 || c < best - 1e-9) {
                best = c;
                pitch_out = pitch;
                vc_out = vc;
            }
            lin_try(vc, pitch, 1.0);
            wg_try(vc, pitch, 1.0);
            // k x V interleave blocks on the same layout (16-byte aligned rows)
            if (op.vw > 1 && !op.rshift && !Pb.no_w2 && (pitch * Pb.E) % 16 == 0 && wk_extent(Pb, g, V)) {
                VecChoice vk = vc;
                vk.wk = wk_extent(Pb, g, V);
                fill_tile_params(Pb, g, pitch, NT, vk, tp);
                const double ck = tile_cost(Pb, tp);
                if (getenv("VPG_DEBUG_PLAN"))
                    fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u wk %d cost %.1f per-elem %.3f\n",
                            (long long)g.Ls, (long long)g.Ld, pitch, vk.wk, ck, ck / (double)g.T);
                if (best < 0 || ck < best - 1e-9) {
                    best = ck;
                    pitch_out = pitch;
                    vc_out = vk;
                }
            }
        }
    }
    // Narrow W vectors on residue rows (1- and 2-byte words), where the choice
    // so far is the plain scalar W walk: source runs misaligned to 16 bytes but
    // aligned to 8 or 4 keep that alignment in shared memory (rows sit at
    // their global offset modulo 16 bytes), so the W phase loads 8 or 4 bytes
    // along source dim 0 at once and stores the elements one by one.  Gather
    // blocks keep priority: they widen the stores, which measured better (u8
    // (72,1917,1944) reversed 0.75 of copy_ with gather blocks, 0.54 with
    // 4-byte W vectors).  VPG_WV_NARROW=0: off.
    static const bool wv_narrow = !(getenv("VPG_WV_NARROW") && atoi(getenv("VPG_WV_NARROW")) == 0);
    // Only where source dim 0 lies outside the tile's destination run: inside
    // it, a lane's vector elements would take the places of its neighbours'
    // and each store instruction would scatter over short segments (u8
    // (7,26,11,7,23,23,72) -> (0,3,1,4,5,6,2), dim 0 second in the destination:
    // 0.73 -> 0.33 of copy_).
    if (best > 0 && Pb.E <= 2 && wv_narrow && Pb.sigma[0] != 0 && Pb.out_stride_of_dim[0] >= g.Ld &&
        vc_out.rshift && vc_out.rres && vc_out.vw == 1 &&
        !vc_out.wg && !vc_out.lin && !vc_out.w2 && !vc_out.wk && !vc_out.bulk && !vc_out.res16) {
        for (int vn = V / 2; vn * Pb.E >= 4; vn /= 2) {
            if (!w_vectorizable(Pb, g, vn) || !src_starts_aligned(Pb, g, vn)) continue;
            VecChoice v2 = vc_out;
            v2.vw = vn;
            TileParams tp;
            fill_tile_params(Pb, g, pitch_out, NT, v2, tp);
            const double c = tile_cost(Pb, tp) * kResidueCostFactor *
                             (res_modulus(Pb.E) * Pb.E >= 128 ? kSw128CostFactor : 1.0);
            if (getenv("VPG_DEBUG_PLAN"))
                fprintf(stderr, "[plan] Ls %lld Ld %lld pitch %u residue narrow W vector %d cost %.1f per-elem %.3f\n",
                        (long long)g.Ls, (long long)g.Ld, pitch_out, vn, c, c / (double)g.T);
            if (c < best - 1e-9) {
                best = c;
                vc_out = v2;
            }
            break;
        }
    }
}

}  // namespace

// ----------------------------------------------------------------- merge
// planner.py:211-241
// `pin` (optional): pinned dims (sharded plans) never fuse with a neighbour;
// `opin` receives the pin of every merged dim.
int merge_dims(int rank, const int64_t *dims, const int32_t *sigma, int64_t *od, int32_t *os, const uint8_t *pin,
               uint8_t *opin) {
    std::vector<int> keep;
    for (int k = 0; k < rank; ++k)
        if (dims[k] > 1) keep.push_back(k);
    if (keep.empty()) {
        od[0] = 1;
        os[0] = 0;
        if (opin) opin[0] = 0;
        return 1;
    }
    std::vector<int> renum(rank, -1);
    for (size_t i = 0; i < keep.size(); ++i) renum[keep[i]] = (int)i;
    int m = (int)keep.size();
    std::vector<int64_t> d(m);
    for (int i = 0; i < m; ++i) d[i] = dims[keep[i]];
    std::vector<int> sg;
    for (int j = 0; j < rank; ++j)
        if (renum[sigma[j]] >= 0) sg.push_back(renum[sigma[j]]);
    std::vector<int> pos(m);
    for (int j = 0; j < m; ++j) pos[sg[j]] = j;
    auto pinned = [&](int k) { return pin && pin[keep[k]]; };
    std::vector<std::vector<int>> groups{{0}};
    for (int k = 1; k < m; ++k) {
        if (pos[k] == pos[k - 1] + 1 && !pinned(k) && !pinned(k - 1)) groups.back().push_back(k);
        else groups.push_back({k});
    }
    int ng = (int)groups.size();
    for (int gi = 0; gi < ng; ++gi) {
        int64_t p = 1;
        for (int k : groups[gi]) p *= d[k];
        od[gi] = p;
        if (opin) opin[gi] = pin ? pin[keep[groups[gi][0]]] : 0;
    }
    std::vector<int> order(ng);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return pos[groups[x][0]] < pos[groups[y][0]]; });
    for (int j = 0; j < ng; ++j) os[j] = order[j];
    return ng;
}

// ----------------------------------------------------------------- shards
// Leading factors: walk dims outermost first taking whole dims, or the
// outer factor of the dim that completes the product, until it equals G
// (sharded.py _lead_split).  cuts[k] = outer factor taken from dim k.
static bool lead_cuts(const std::vector<int> &outer_first, const int64_t *dims, int64_t G,
                      std::map<int, int64_t> &cuts, std::string *err) {
    int64_t rem = G;
    for (int k : outer_first) {
        if (rem == 1) break;
        const int64_t d = dims[k];
        if (d <= rem && rem % d == 0) {
            cuts[k] = d;
            rem /= d;
        } else if (d % rem == 0) {
            cuts[k] = rem;
            rem = 1;
        } else {
            *err = "cannot shard: dim of size " + std::to_string(d) + " vs remaining factor " + std::to_string(rem);
            return false;
        }
    }
    if (rem != 1) {
        *err = "tensor has fewer than " + std::to_string(G) + " leading elements";
        return false;
    }
    return true;
}

// Split dims so that the leading input dims and the leading output dims each
// multiply to exactly G; pin those (2 = input shard digits, 1 = output).
// Inner-first in and out.
static bool refine_for_shards(int rank, const int64_t *dims, const int32_t *sigma, int G,
                              std::vector<int64_t> &rd, std::vector<int32_t> &rs, std::vector<uint8_t> &pin,
                              std::string *err, bool pull = false) {
    std::vector<int> in_of, out_of;
    for (int k = rank - 1; k >= 0; --k) in_of.push_back(k);
    for (int j = rank - 1; j >= 0; --j) out_of.push_back(sigma[j]);
    std::map<int, int64_t> cin, cout;
    if (!lead_cuts(in_of, dims, G, cin, err) || !lead_cuts(out_of, dims, G, cout, err)) return false;
    std::vector<std::vector<int64_t>> pieces(rank);   // inner-first factors of each dim
    for (int k = 0; k < rank; ++k) {
        std::vector<int64_t> cuts;
        for (auto *m : {&cin, &cout}) {
            auto it = m->find(k);
            if (it != m->end() && it->second > 1 && it->second < dims[k]) cuts.push_back(it->second);
        }
        std::sort(cuts.begin(), cuts.end());
        cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
        if (cuts.size() == 2 && cuts[1] % cuts[0]) {
            *err = "cannot shard: dim " + std::to_string(k) + " needs incompatible splits";
            return false;
        }
        std::vector<int64_t> outer_first;
        int64_t prev = 1;
        for (int64_t c : cuts) {
            outer_first.push_back(c / prev);
            prev = c;
        }
        outer_first.push_back(dims[k] / prev);
        pieces[k].assign(outer_first.rbegin(), outer_first.rend());
    }
    std::vector<int> first(rank);
    rd.clear();
    for (int k = 0; k < rank; ++k) {
        first[k] = (int)rd.size();
        for (int64_t f : pieces[k]) rd.push_back(f);
    }
    const int rr = (int)rd.size();
    if (rr > VPG_MAX_RANK) {
        *err = "refined rank exceeds " + std::to_string(VPG_MAX_RANK);
        return false;
    }
    rs.clear();
    for (int j = 0; j < rank; ++j)
        for (size_t i = 0; i < pieces[sigma[j]].size(); ++i) rs.push_back(first[sigma[j]] + (int)i);
    pin.assign(rr, 0);
    if (G > 1 && pull) {
        // pull: the leading OUTPUT dims index the plan's output shard -- the
        // slowest grid digits; the input-shard dims stay free (every source
        // chunk finds its shard at run time)
        int64_t prod = 1;
        for (int j = rr - 1; j >= 0 && prod < G; --j) {
            pin[rs[j]] = 2;
            prod *= rd[rs[j]];
        }
    } else if (G > 1) {
        int64_t prod = 1;
        for (int k = rr - 1; k >= 0 && prod < G; --k) {
            pin[k] = 2;
            prod *= rd[k];
        }
        prod = 1;
        for (int j = rr - 1; j >= 0 && prod < G; --j) {
            if (!pin[rs[j]]) pin[rs[j]] = 1;
            prod *= rd[rs[j]];
        }
    }
    return true;
}

// Stride-1-preserving permutations go to the ROWS kernel when its rows are
// long enough and 16-byte vectorisable; rows of odd length fall back to
// narrow accesses there, and the tile kernel (aligned-superset reads) moves
// them faster unless they are long 8-byte rows (tools/shape_ab.py: 69 x 8 B
// rows 0.56 vs 0.98 of copy through the tile kernel; 1001 x 4 B 0.58 vs 0.79;
// 1025 x 8 B 0.85 both).
// Rows whose length is not a multiple of 16 bytes go to the tile kernel,
// which stages them through residue-strided smem rows and keeps 16-byte
// accesses: 8-byte words with odd row lengths of 65-16385 elements ran at
// 1.06-1.15 of a same-size copy_ there against 0.75-1.02 in the rows kernel
// (word-width vectors; tools/rows_vs_tile.py, profiles/rows_vs_tile_r2.txt).
static bool rows_suitable(int64_t Lr, int E) {
    const int64_t V = std::max(1, 16 / E);
    if (Lr * E < kRowsMinBytes) return false;
    return Lr % V == 0;
}

// ----------------------------------------------------------------- plan
static void describe(vpg_plan *p) {
    char buf[4096];
    int o = 0;
    auto put = [&](const char *fmt, auto... args) {
        if (o < (int)sizeof(buf)) o += snprintf(buf + o, sizeof(buf) - o, fmt, args...);
    };
    static const char *names[] = {"copy", "rows(K1)", "tile(K2/K3)", "gather(K0)"};
    put("kernel class: %s\n", names[p->kernel_class]);
    put("elem bytes: %d\n", p->elem_bytes);
    put("merged dims (inner-first): (");
    for (int k = 0; k < p->rank; ++k) put(k ? ",%lld" : "%lld", (long long)p->dims[k]);
    put(")\nmerged sigma (inner-first): (");
    for (int k = 0; k < p->rank; ++k) put(k ? ",%d" : "%d", p->sigma[k]);
    put(")\nelements: %lld\n", (long long)p->n);
    if (p->kernel_class == VPG_KERNEL_TILE) {
        const TileParams &t = p->tile;
        put("tile elements: %u (src run %u x %u runs, dst run %u x %u runs)\n", t.T, t.Ls, t.T / t.Ls,
            t.Ld, t.T / t.Ld);
        put("smem pitch: %u, smem bytes: %u, buffers: %u\n", t.pitch, t.smem_bytes, t.nbuf);
        put("ragged boundary dims: a(extent %u of %u) c(extent %u of %u)\n", t.e_a, t.d_a, t.e_c,
            t.d_c);
        for (int ph = 0; ph < 2; ++ph) {
            const PhaseDesc &d = t.ph[ph];
            put("phase %s: %u threads x %u groups, thread dims %d, inner %u steps, outer %u (dims %d), "
                "check mask full=%u ragged=%u\n",
                ph ? "W" : "R", d.nthr, d.ngroups, d.nthr_dims, d.n_in, d.n_outer, d.nout_dims,
                d.mask_full, d.mask_ragged);
        }
        if (t.ph[0].swz == kSwzAddr) put("smem address swizzle: 16-byte chunk ^= 128-byte block index\n");
        else if (t.ph[0].swz) put("smem chunk swizzle: row >> %u\n", t.ph[0].swz - 1);
        put("vector elems: R %u%s, W %u%s\n", t.ph[0].vec,
            t.bulk ? (t.ph[0].rshift == 2
                          ? " (TMA bulk copy per source run: aligned supersets of misaligned runs, 16-byte residue "
                            "row strides, producer warp)"
                          : " (TMA bulk copy per source run, producer warp)")
                   : (t.ph[0].rshift == 2 ? " (aligned supersets of misaligned runs, residue row strides)"
                                       : t.ph[0].rshift ? " (aligned supersets of misaligned runs)" : ""),
            t.ph[1].vec, t.ph[1].w2 == 1 ? " (VxV register-transposed blocks, 16-byte stores)"
                         : t.ph[1].w2 == kW2Gather ? " (gather blocks: 16-byte stores of destination-innermost runs)"
                         : t.ph[1].w2 == kW2Gather + 2 ? " (gather blocks of 2: narrow stores of destination-innermost runs)"
                         : t.ph[1].w2 == kW2Gather + 4 ? " (gather blocks of 4: narrow stores of destination-innermost runs)"
                         : t.ph[1].w2 == kW2Gather + 8 ? " (gather blocks of 8: narrow stores of destination-innermost runs)"
                         : t.ph[1].w2 >= 2 ? " (k x V interleave blocks, 16-byte stores)" : "");
        if (t.ph[1].w2 >= 2 && t.ph[1].w2 < kW2Gather)
            put("W interleave: k = %u destination-innermost elements per dim-0 element\n", t.ph[1].w2);
        if (t.lin.on)
            put("W lin: destination-linear %u-byte chunks, one store each (runs of %u elements, %u chunk slots x %u "
                "runs, offset table %u bytes, bank rotation %s)\n",
                16u, t.lin.run_len, t.lin.cpr, t.lin.nchunks / t.lin.cpr,
                (unsigned)lin_table_bytes(t.lin.run_len, 16 / p->elem_bytes),
                t.lin.rot_shift < 32 ? ("lane >> " + std::to_string(t.lin.rot_shift)).c_str() : "none");
        put("lane utilisation (R*W): %.3f\n", p->tile_util);
        put("cost model: geometry %.4f (sector efficiency src %.3f, dst %.3f), walk %.4f per element\n",
            p->geom_cost, p->eff_s, p->eff_d, p->walk_cost);
        put("specialised (NVRTC) kernel: %s\n", p->jit ? "yes" : "no");
        put("tiles: %u, grid digits: %d\n", t.num_tiles, t.ngrid);
        if (p->shards > 0 && t.pull)
            put("sharded exchange (pull): output shard %d of %d, tiles [%u, %u), reads from %d input shards\n",
                p->shard_index, p->shards, t.tile_begin, t.tile_begin + t.num_tiles, p->shards);
        else if (p->shards > 0)
            put("sharded exchange: shard %d of %d, tiles [%u, %u), stores into %d output shards\n",
                p->shard_index, p->shards, t.tile_begin, t.tile_begin + t.num_tiles, p->shards);
    } else if (p->kernel_class == VPG_KERNEL_ROWS) {
        put("rows: %u x %lld elements, vector %u elements, %u threads/row\n", p->rows.nrows,
            (long long)p->rows.row_len, p->rows.vec, 1u << p->rows.tpr_log2);
        if (p->rows.row_len * p->elem_bytes >= 2560 && (p->rows.row_len * p->elem_bytes) % 16 == 0)
            put("rows vector elems: TMA bulk pipeline (global -> smem -> global) when the buffers are 16-byte aligned\n");
    }
    put("predicted sector efficiency: %.3f\n", p->predicted_eff);
    p->text.assign(buf, std::min<int>(o, sizeof(buf) - 1));
}

// Inputs of rank > VPG_MAX_RANK are accepted when their size-1 dims, which
// merge_dimensions drops anyway (planner.py:222-227), bring the rank within
// the limit: validate over the full rank, then squeeze (sigma renumbered).
// The reference has no rank cap (core.py:58-88).
bool squeeze_unit_dims(int &rank, const int64_t *&dims, const int32_t *&sigma, std::vector<int64_t> &sd,
                       std::vector<int32_t> &ss, std::string *err) {
    if (rank <= VPG_MAX_RANK) return true;
    if (rank > (1 << 20)) {
        *err = "rank " + std::to_string(rank) + " is out of range";
        return false;
    }
    std::vector<int> seen(rank, 0), renum(rank, -1);
    for (int k = 0; k < rank; ++k) {
        if (dims[k] < 1) {
            *err = "dimension " + std::to_string(dims[k]) + " is not positive";
            return false;
        }
        if (sigma[k] < 0 || sigma[k] >= rank || seen[sigma[k]]) {
            *err = "map is not a bijection on 0.." + std::to_string(rank - 1);
            return false;
        }
        seen[sigma[k]] = 1;
    }
    sd.clear();
    ss.clear();
    for (int k = 0; k < rank; ++k)
        if (dims[k] > 1) {
            renum[k] = (int)sd.size();
            sd.push_back(dims[k]);
        }
    for (int j = 0; j < rank; ++j)
        if (renum[sigma[j]] >= 0) ss.push_back(renum[sigma[j]]);
    if (sd.empty()) {
        sd.push_back(1);
        ss.push_back(0);
    }
    if ((int)sd.size() > VPG_MAX_RANK) {
        *err = "rank after dropping size-1 dims (" + std::to_string(sd.size()) + ") exceeds " +
               std::to_string(VPG_MAX_RANK);
        return false;
    }
    rank = (int)sd.size();
    dims = sd.data();
    sigma = ss.data();
    return true;
}

vpg_status make_plan(int rank, const int64_t *dims, const int32_t *sigma, int E, unsigned flags,
                     vpg_plan **out, std::string *err, int shards, int shard_index) {
    std::vector<int64_t> sq_d;
    std::vector<int32_t> sq_s;
    if (!squeeze_unit_dims(rank, dims, sigma, sq_d, sq_s, err)) return VPG_EINVAL;
    if (rank < 1 || rank > VPG_MAX_RANK) {
        *err = "rank must be in 1.." + std::to_string(VPG_MAX_RANK);
        return VPG_EINVAL;
    }
    if (!(E == 1 || E == 2 || E == 4 || E == 8 || E == 16)) {
        *err = "element width must be one of 1, 2, 4, 8, 16 bytes";
        return VPG_EINVAL;
    }
    std::vector<int> seen(rank, 0);
    for (int k = 0; k < rank; ++k) {
        if (dims[k] < 1) {
            *err = "dimension " + std::to_string(dims[k]) + " is not positive";
            return VPG_EINVAL;
        }
        if (sigma[k] < 0 || sigma[k] >= rank || seen[sigma[k]]) {
            *err = "map is not a bijection on 0.." + std::to_string(rank - 1);
            return VPG_EINVAL;
        }
        seen[sigma[k]] = 1;
    }
    Problem P;
    P.E = E;
    bool small_problem = false;
    // development knobs (documented in DESIGN.md): override the tiling policy
    P.budget = kTileBudgetBytes;
    P.nbuf = 0;
    P.cta_smem = 110 * 1024;
    {
        // small problems (a few tiles per CTA): half-size tiles and a smaller
        // per-CTA staging target, so twice as many CTAs per SM run
        // independent pipelines (steady-state, tools/sweep.py SWEEP_MODE=
        // steady: cfg2 10.6 -> 10.1 us, cfg3 18.3 -> 17.0 us, cfg1 25.8 ->
        // 24.7 us; cfg5's 4 GiB keeps the large tiles: 664 vs 686 us)
        int64_t nel = 1;
        for (int k = 0; k < rank; ++k) nel *= dims[k];
        const char *sm = getenv("VPG_SMALL");      // 0: no small-problem tiling (experiments)
        const char *sb = getenv("VPG_SMALL_BYTES");   // algorithmic-bytes threshold (experiments)
        const double small_bytes = sb ? atof(sb) : kSmallProblemBytes;
        if ((double)nel * E * 2.0 < small_bytes && !(sm && atoi(sm) == 0)) {
            P.budget = 24 * 1024;
            P.cta_smem = 75 * 1024;
            small_problem = true;
            // tiny problems: tiles small enough for ~4 per SM, so the grid
            // fills the GPU (a 1 MiB byte transpose is 64 tiles of 16 KiB)
            // (opt-in, VPG_TINY=1: a wash once such plans run specialised
            // kernels, tools/tiny_probe.py)
            const char *tb = getenv("VPG_TINY");
            const int64_t tiny = (int64_t)((double)nel * E / (4.0 * kSmCount));
            if (tb && atoi(tb) == 1 && tiny < P.budget) P.budget = std::max<int64_t>(4096, tiny);
        }
    }
    int persist_mode = -1;  // -1 auto, 0 one tile per CTA, 1 persistent
    int force_threads = 0;
    if (const char *e = getenv("VPG_TILE_BUDGET")) P.budget = std::max(1024L, atol(e));
    if (const char *e = getenv("VPG_NBUF")) P.nbuf = std::max(1, std::min(8, atoi(e)));
    if (const char *e = getenv("VPG_CTA_SMEM")) P.cta_smem = std::min(220L * 1024, std::max(16L * 1024, atol(e)));
    if (const char *e = getenv("VPG_PERSIST")) persist_mode = atoi(e);
    if (const char *e = getenv("VPG_THREADS")) force_threads = atoi(e);
    if (getenv("VPG_NO_SHIFT")) P.no_shift = true;
    if (getenv("VPG_NO_RES")) P.no_res = true;
    if (getenv("VPG_NO_SW128")) P.no_sw128 = true;
    if (getenv("VPG_NO_W2")) P.no_w2 = true;
    if (const char *e = getenv("VPG_WG")) {
        P.no_wg = atoi(e) == 0;
        P.force_wg = atoi(e) == 2;
    }
    if (const char *e = getenv("VPG_LIN")) P.lin_mode = *e ? atoi(e) : 0;
    // (a blanket "no address swizzle unless 4-byte words" rule measured neutral
    // over 200 random shapes: +10..18% on some plans, -13..15% on others,
    // profiles/swz_addr_ab_r2.txt -- the bank model keeps the choice)
    if (const char *e = getenv("VPG_NO_SWZ_ADDR")) P.no_swz_addr = !*e || atoi(e) != 0;
    // the chunk swizzle removes the W bank conflicts of shifted runs but costs
    // a divide and a few integer ops per element: measured 28.4 vs 20.5 us on
    // cfg3, 216 vs 247 us on an odd 8-byte 2-D transpose -- opt-in
    if (const char *e = getenv("VPG_SWZ")) P.no_swz = atoi(e) == 0;
    // TMA bulk copies of the source runs: chosen per plan (see make_plan);
    // VPG_BULK=0 never, VPG_BULK=1 wherever the runs allow it
    if (const char *e = getenv("VPG_BULK")) {
        P.no_bulk = atoi(e) == 0;
        P.force_bulk = atoi(e) != 0;
    }
    // sharded exchange plans: refine and pin the shard-indexing dims first
    std::vector<int64_t> rdims(dims, dims + rank);
    std::vector<int32_t> rsig(sigma, sigma + rank);
    std::vector<uint8_t> rpin(rank, 0);
    if (shards > 0) {
        if (shards > kMaxShards || shard_index < 0 || shard_index >= shards) {
            *err = "shards must be in 1.." + std::to_string(kMaxShards) + " and shard_index in 0..shards-1";
            return VPG_EINVAL;
        }
        const bool pull = (flags & VPG_SHARD_PULL) != 0;
        if (!refine_for_shards(rank, dims, sigma, shards, rdims, rsig, rpin, err, pull)) return VPG_EUNSUPPORTED;
        P.G = shards;
        P.shard = shard_index;
        P.pull = pull;
        if (pull) P.no_swz = true;   // the chunk swizzle assumes one source buffer
        // TMA bulk reads assume one source buffer (pull), and the bulk
        // kernel's producer/consumer split carries no device-side exchange
        // barrier (tile_body.cuh shard_barrier_*): exchanges stay per-lane
        P.no_bulk = true;
    }
    const int rrank = (int)rdims.size();
    if (flags & VPG_NO_MERGE) {
        P.r = 0;
        for (int k = 0; k < rrank && k < kMaxRank; ++k) {
            P.d[k] = rdims[k];
            P.sigma[k] = rsig[k];
            P.pin[k] = rpin[k];
        }
        P.r = rrank;
    } else {
        int64_t md[VPG_MAX_RANK];
        int32_t ms[VPG_MAX_RANK];
        uint8_t mp[VPG_MAX_RANK];
        P.r = merge_dims(rrank, rdims.data(), rsig.data(), md, ms, rpin.data(), mp);
        if (P.r > kMaxRank) {
            *err = "merged rank exceeds " + std::to_string(kMaxRank);
            return VPG_EUNSUPPORTED;
        }
        for (int k = 0; k < P.r; ++k) {
            P.d[k] = md[k];
            P.sigma[k] = ms[k];
            P.pin[k] = mp[k];
        }
    }
    if (P.r > kMaxRank) {
        *err = "rank exceeds " + std::to_string(kMaxRank);
        return VPG_EUNSUPPORTED;
    }
    fill_problem(P);
    vpg_plan *p = new vpg_plan();
    p->elem_bytes = E;
    p->rank = P.r;
    for (int k = 0; k < P.r; ++k) {
        p->dims[k] = P.d[k];
        p->sigma[k] = P.sigma[k];
    }
    p->n = P.n;
    p->shards = shards;
    p->shard_index = shard_index;
    p->predicted_eff = 1.0;
    // a sharded exchange is always a tile plan (per-tile destination shard)
    if (shards > 0) {
        flags |= VPG_FORCE_TILE;
        flags &= ~(unsigned)VPG_FORCE_GATHER;
    }
    bool identity = true;
    for (int k = 0; k < P.r; ++k)
        if (P.sigma[k] != k) identity = false;

    if ((flags & VPG_FORCE_GATHER) || (P.n <= kGatherMaxN && !(flags & VPG_FORCE_TILE))) {
        if (P.n >= (int64_t)1 << 32) {
            delete p;
            *err = "gather kernel limited to 2^32 elements";
            return VPG_EUNSUPPORTED;
        }
        p->kernel_class = VPG_KERNEL_GATHER;
        GatherParams &gp = p->gather;
        gp.n = (uint32_t)P.n;
        gp.rank = P.r;
        for (int j = 0; j < P.r; ++j) {
            gp.ext[j] = make_fastdiv((uint32_t)P.d[P.sigma[j]]);
            gp.src_stride[j] = P.in_stride[P.sigma[j]];
        }
        p->threads = 256;
        p->grid_hint = (P.n + 255) / 256;
        p->predicted_eff = 0.25;
    } else if (identity && !(flags & VPG_FORCE_TILE)) {
        p->kernel_class = VPG_KERNEL_COPY;
        p->copy.n = P.n;
        p->threads = 256;
        p->grid_hint = 148 * 8;
    } else if (P.sigma[0] == 0 && rows_suitable(P.d[0], E) && !(flags & VPG_FORCE_TILE)) {
        p->kernel_class = VPG_KERNEL_ROWS;
        RowsParams &rp = p->rows;
        int64_t Lr = P.d[0];
        int64_t nrows = P.n / Lr;
        if (nrows >= ((int64_t)1 << 32)) {
            delete p;
            *err = "rows kernel limited to 2^32 rows";
            return VPG_EUNSUPPORTED;
        }
        uint32_t V = std::max(1, 16 / E);
        while (V > 1 && Lr % V) V >>= 1;
        rp.vec = V;
        rp.row_len = Lr;
        rp.nrows = (uint32_t)nrows;
        rp.row_vecs = (uint32_t)(Lr / V);
        uint32_t tpr = 32;
        while (tpr > 1 && tpr / 2 >= rp.row_vecs) tpr >>= 1;
        rp.tpr_log2 = 0;
        while ((1u << rp.tpr_log2) < tpr) ++rp.tpr_log2;
        rp.ndig = P.r - 1;
        for (int j = 1; j < P.r; ++j) {
            rp.dig[j - 1].ext = make_fastdiv((uint32_t)P.d[P.sigma[j]]);
            rp.dig[j - 1].src_stride = P.in_stride[P.sigma[j]];
        }
        p->threads = 256;
        p->grid_hint = 148 * 8;
        int64_t bytes = Lr * E;
        p->predicted_eff = (double)bytes / (32.0 * expected_sectors(bytes, gcd64(bytes, 32)));
    } else {
        TileGeom g;
        // flags bits 8..15: pick the n-th best tile candidate (autotuning)
        const int pick = (int)((flags >> 8) & 0xff) - 1;
        if (!select_tile(P, g, pick)) {
            delete p;
            *err = pick >= 0 ? "no such tile candidate" : "no tile fits the shared-memory budget";
            return VPG_EUNSUPPORTED;
        }
        p->kernel_class = VPG_KERNEL_TILE;
        int threads = g.T >= 1024 ? kTileThreads : (g.T >= 256 ? 128 : 64);
        if (force_threads >= 32 && force_threads <= 1024) threads = force_threads / 32 * 32;
        uint32_t pitch;
        VecChoice vc;
        choose_pitch_vec(P, g, threads, pitch, vc);
        // V x V register-transposed W blocks (16-byte stores on both sides)
        // are the fastest W mode; when the model's first tile cannot use them
        // and a later candidate within 30% of its geometry cost can, take that
        // one (batched 2048 x 128 transposes, attention K^T: a contiguous
        // 8192-element source block with scalar-width stores ran 0.81 / 0.71
        // of copy_ in f32 / bf16, the 64 x 128 V x V tile 1.04 / 1.00,
        // tools/cand_scan.py; on the 31 random shapes of
        // profiles/cand_data_r2.jsonl the rule changes 1-2 plans, none worse)
        const char *vxv = getenv("VPG_PREFER_VXV");    // 0: off (experiments)
        if (pick < 0 && !vc.w2 && !P.force_bulk && !(vxv && atoi(vxv) == 0)) {
            for (int k = 1; k < 10; ++k) {
                TileGeom gk;
                if (!select_tile(P, gk, k)) break;
                if (gk.cost > 1.3 * g.cost) continue;
                const int tk = gk.T >= 1024 ? kTileThreads : (gk.T >= 256 ? 128 : 64);
                const int thk = force_threads >= 32 && force_threads <= 1024 ? force_threads / 32 * 32 : tk;
                uint32_t pk;
                VecChoice vk;
                choose_pitch_vec(P, gk, thk, pk, vk);
                if (vk.w2) {
                    g = gk;
                    threads = thk;
                    pitch = pk;
                    vc = vk;
                    break;
                }
            }
        }
        // Small problems with misaligned source runs also consider the 32 KiB
        // budget (their residue rows pad a tile by up to a third) and keep it
        // when the geometry cost plus the walk cost (issued smem/memory ops
        // per element, weight 4 per byte of element; 4 and 8 select alike on
        // the calibration shapes except cfg3, whose 32 KiB tile runs 3%
        // faster in the steady protocol) is lower.  Round 2 kept
        // the 32 KiB tile unconditionally (from cfg3: 18.65 -> 18.03 us
        // flushed); timing every candidate of 31 random permutations
        // (tools/cand_data.py, profiles/cand_data_r2.jsonl) showed that as the
        // worst budget policy -- 0.77 and 0.73 of the best candidate on two
        // shapes whose 32 KiB tiles walk with idle lanes -- and this rule the
        // best simple one (0.975 mean of the best candidate).  VPG_SMALL_MIS:
        // 1 = always take the 32 KiB tile, 0 = never.
        const char *smis = getenv("VPG_SMALL_MIS");
        const int small_mis = smis ? atoi(smis) : -1;
        if (vc.rshift && small_problem && pick < 0 && !getenv("VPG_TILE_BUDGET") && small_mis != 0) {
            Problem P2 = P;
            P2.budget = 32 * 1024;
            TileGeom g2;
            if (select_tile(P2, g2, -1)) {
                const int t2 = g2.T >= 1024 ? kTileThreads : (g2.T >= 256 ? 128 : 64);
                const int thr2 = force_threads >= 32 && force_threads <= 1024 ? force_threads / 32 * 32 : t2;
                uint32_t pitch2;
                VecChoice vc2;
                choose_pitch_vec(P2, g2, thr2, pitch2, vc2);
                bool take = vc2.rshift;
                if (take && small_mis < 0) {
                    TileParams a, b;
                    fill_tile_params(P, g, pitch, threads, vc, a);
                    fill_tile_params(P2, g2, pitch2, thr2, vc2, b);
                    const double gmin = std::min(g.cost, g2.cost);
                    const double ca = g.cost / gmin + kWalkWeight * tile_cost(P, a) / (double)g.T / E;
                    const double cb = g2.cost / gmin + kWalkWeight * tile_cost(P2, b) / (double)g2.T / E;
                    take = cb < ca;
                }
                if (take) {
                    P = P2;
                    g = g2;
                    threads = thr2;
                    pitch = pitch2;
                    vc = vc2;
                }
            }
        }
        // optionally the vectorised R phase runs as TMA bulk copies, one per
        // source run (16-byte aligned runs of whole 16-byte chunks; VPG_BULK=1)
        // TMA bulk copies (one cp.async.bulk per source run, producer warp +
        // mbarriers) instead of per-lane 16-byte cp.async: the per-lane form
        // requests every 32-byte sector from L2 about twice (ncu
        // lts__t_sectors_srcunit_tex_op_read = 1.96x the data, bulk 1.00x),
        // which costs 2-15% once runs are long; below ~2 KiB the TMA issue
        // cost per run wins (tools/perf_sweep.py, VPG_BULK=0 vs 1: 2-6 KiB
        // source runs with >= 512-byte destination runs +3..15%, 256-byte
        // runs -10..-25%; cfg5 729 -> 713 us)
        const bool long_runs = g.Ls * E >= 2048 && g.Ld * E >= 512;
        auto bulk_for = [&](const VecChoice &v) {
            return (E == 4 || E == 8) && v.vr > 1 && !v.rshift && !P.no_bulk && (long_runs || P.force_bulk) &&
                   (g.Ls * E) % 16 == 0 &&
                   (g.a_part < 0 ||
                    ((g.Ls / g.ext[g.a_part]) * (P.d[g.a_part] % g.ext[g.a_part]) * E) % 16 == 0) &&
                   g.n_runidx <= kMaxPhaseDims;
        };
        // the congruent layout (1x L2 sectors with per-lane cp.async, V x V W
        // blocks) beats bulk reads into padded rows where it applies (cfg5:
        // 690 vs 708 us flushed, 703 vs 729 us steady); bulk covers the long
        // runs it cannot take (not a power of two, or not 128-byte aligned)
        vc.bulk = (vc.bulk && vc.rshift) || (!vc.sw128 && bulk_for(vc));
        p->tile_util = fill_tile_params(P, g, pitch, threads, vc, p->tile);
        p->geom_cost = g.cost;
        p->walk_cost = tile_cost(P, p->tile) / (double)g.T;
        p->eff_s = g.eff_s;
        p->eff_d = g.eff_d;
        // variant without 16-byte source reads, for misaligned base pointers
        VecChoice vs = vc;
        vs.vr = 1;
        vs.rshift = false;
        vs.bulk = false;
        vs.w2 = false;      // 16-byte destination stores need an aligned dst too
        vs.wk = 0;
        vs.wg = 0;
        if (P.sigma[0] == 0) vs.vw = 1;   // (its vector W would be 16-byte stores)
        if (vs.vw > 1 && vs.vw * P.E < 16) vs.vw = 1;   // narrow W vectors need the residue rows
        vs.lin = false;
        fill_tile_params(P, g, pitch, threads, vs, p->tile_unaligned);
        // the tile count must fit the 32-bit tile index
        double nt = 1.0;
        for (int i = 0; i < p->tile.ngrid; ++i) nt *= p->tile.grid[i].ext.d;
        if (nt >= 4294967296.0) {
            delete p;
            *err = "more than 2^32 tiles";
            return VPG_EUNSUPPORTED;
        }
        p->threads = threads;
        p->tile.persistent = persist_mode < 0 ? 1u : (uint32_t)persist_mode;
        p->tile_unaligned.persistent = p->tile.persistent;
        // per-case specialisation pays off once the tensor is large enough to
        // amortise a one-off NVRTC compile (cached in-process and on disk)
        const char *je = getenv("VPG_JIT");
        // (1 MiB: the ahead-of-time kernel runs 2-2.5x slower than the
        // specialised one on 1-6 MiB permutations -- 3.6x the instructions,
        // tools/tiny_probe.py jit -- and a compile takes 0.3-0.7 s once per
        // plan, cached in-process and on disk)
        // Below it the specialised kernel still runs 2-3x faster (7-8 us vs
        // 13-24 us flushed on 150 KiB - 1 MiB problems, profiles/tiny_jit_r2.txt)
        // but the compile dominates one-off calls: build_program(jit=True),
        // VPG_JIT=1 or VPG_JIT_MIN_BYTES opt in.
        static const int64_t jit_min = getenv("VPG_JIT_MIN_BYTES") ? atoll(getenv("VPG_JIT_MIN_BYTES")) : ((int64_t)1 << 20);
        bool big = P.n / std::max(1, P.G) * E >= jit_min;
        p->jit = (flags & VPG_FORCE_JIT) ? 1 : (flags & VPG_NO_JIT) ? 0 : je ? (atoi(je) != 0) : big;
        p->grid_hint = std::min<int64_t>(p->tile.num_tiles, 148 * 4);
        p->predicted_eff = 2.0 / (1.0 / g.eff_s + 1.0 / g.eff_d);
    }
    describe(p);
    *out = p;
    return VPG_OK;
}

}  // namespace vpg
