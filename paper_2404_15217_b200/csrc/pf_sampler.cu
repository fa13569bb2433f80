// Batched overlap_fraction and the epoch_stream sampler.
//
// epoch_stream (pkg/sampler.py:196-227) is sequential: a slide draw, then up
// to max_attempts candidates of sample_patch (140-184), each consuming one
// mpp draw and - when the footprint fits - two coordinate draws, until one is
// accepted by overlap_fraction >= min_foreground.  All draws come from
// counter-based SplitMix64 streams (pkg/rng.py), so when every (slide, mpp)
// footprint fits and no randrange rejection occurs, candidate number m of the
// stream on slide s is a pure function of (s, m):
//     mpp draw m+1, coords draws 2m+1, 2m+2.
// The sampler therefore (1) evaluates the acceptance bit A(s, m) of every
// slide for a window of attempts in parallel — one warp per candidate, FP64
// overlap test bit-exact with the reference — and (2) walks the slide draws in
// stream order with a single warp, taking for each draw the first accepted
// attempt within its max_attempts budget (an ordered compaction of the accept
// bitmaps via find-first-set).  Exhausted draws consume max_attempts attempts
// and no sequence number, exactly like the reference.  Whenever the
// assumptions do not hold (a footprint that does not fit, a rejected draw,
// a window that ran out) the walk continues on the sequential exact path.
#include <algorithm>


#include "pf_common.cuh"
#include "pf_poly.cuh"

namespace pf {

// ---------------------------------------------------------------------------
// pf_overlap_fraction: one warp per rect.
// ---------------------------------------------------------------------------
__global__ void overlap_kernel(const void* blob, const double* rects, int n, int grid, double* out) {
    extern __shared__ __align__(16) uint32_t s_masks[];
    const int warp_in_block = threadIdx.x >> 5;
    const int q = blockIdx.x * (blockDim.x >> 5) + warp_in_block;
    if (q >= n) return;
    const PolyView P = poly_view(blob);
    uint32_t* sm = s_masks + warp_in_block * (overlap_smem_bytes(grid) / 4);
    const double x = rects[4 * q], y = rects[4 * q + 1], w = rects[4 * q + 2], h = rects[4 * q + 3];
    const int c = warp_overlap_count(P, x, y, w, h, grid, sm);
    if ((threadIdx.x & 31) == 0) out[q] = c < 0 ? 0.0 : __ddiv_rn((double)c, (double)grid * (double)grid);
}

// ---------------------------------------------------------------------------
// Sampler helpers (pkg/rng.py, pkg/sampler.py)
// ---------------------------------------------------------------------------
constexpr int kFastDraws = 8192;  // slide draws precomputed per fast walk (int32)

struct SamplerWs {
    uint32_t* bitmaps;  // [n_slides][window/32]
    int4* cands;        // [n_slides][window]: x, y, mpp_idx, -
    int32_t* reject_at; // first window offset whose coords draws were rejected
    int32_t* n_queue;   // kCountBase + candidates queued for the overlap test this round
    int32_t* queue;     // [n_slides * window]: candidates the raster left undecided
    int2* acc;          // [n_slides * window]: per queued candidate (covered cells, parts done)
    uint16_t* na;       // [n_slides * window]: next-accept table (sample_table_kernel)
    int32_t* fdraw;     // [kFastDraws]: the call's slide draws (sample_table_kernel)
    int32_t* draws_ok;  // kCountBase unless a precomputed slide draw was rejected
    int2* emits;        // [window]: (slide, window offset) of specs emitted by the walk
};

__host__ __device__ inline SamplerWs carve_ws(void* ws, int n_slides, int window) {
    SamplerWs w;
    uint8_t* p = reinterpret_cast<uint8_t*>(ws);
    w.reject_at = reinterpret_cast<int32_t*>(p);
    w.n_queue = reinterpret_cast<int32_t*>(p + 4);
    w.draws_ok = reinterpret_cast<int32_t*>(p + 8);  // PF_WALK_TIMING stamps start at byte 32
    p += 256;
    w.bitmaps = reinterpret_cast<uint32_t*>(p);
    p += (((size_t)n_slides * (window / 32) * 4) + 255) / 256 * 256;
    w.cands = reinterpret_cast<int4*>(p);
    p += (size_t)n_slides * window * 16;
    w.queue = reinterpret_cast<int32_t*>(p);
    p += (size_t)n_slides * window * 4;
    w.acc = reinterpret_cast<int2*>(p);
    p += (size_t)n_slides * window * 8;
    w.fdraw = reinterpret_cast<int32_t*>(p);
    p += (size_t)kFastDraws * 4;
    w.na = reinterpret_cast<uint16_t*>(p);
    p += ((size_t)n_slides * window * 2 + 15) / 16 * 16;
    w.emits = reinterpret_cast<int2*>(p);
    return w;
}

__host__ __device__ inline int64_t ws_bytes(int n_slides, int window) {
    return 256 + ((int64_t)n_slides * (window / 32) * 4 + 255) / 256 * 256 +
           (int64_t)n_slides * window * 28 + (int64_t)kFastDraws * 4 + ((int64_t)n_slides * window * 2 + 15) / 16 * 16 +
           (int64_t)(window + 1) * 8;
}

// RandomStream.weighted_index (rng.py:88-103) given the stream draw u.
__device__ __forceinline__ int weighted_pick(uint64_t u, const double* w, int n, double total) {
    const double v = __dadd_rn(0.0, __dmul_rn(u64_to_unit(u), __dsub_rn(total, 0.0)));
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        acc = __dadd_rn(acc, w[i]);
        if (v < acc) return i;
    }
    return n - 1;
}

// The reference sums the weights on every call (rng.py:95); the sum is the same each time,
// so per-candidate callers take it precomputed (host sum in the same order, IEEE binary64).
__host__ __device__ inline double weight_total(const double* w, int n) {
    double total = 0.0;
    for (int i = 0; i < n; ++i) total = total + w[i];
    return total;
}

__device__ __forceinline__ int weighted_pick(uint64_t u, const double* w, int n) {
    return weighted_pick(u, w, n, weight_total(w, n));
}

// Per-launch constants of the speculative evaluation, computed once on the host.
struct EvalConsts {
    double weight_total;  // sum of cfg.mpp_weight
    int32_t need;         // accept_cells(cfg.grid, cfg.min_foreground)
};

__device__ __forceinline__ void emit_spec(const pf_sampler_config& cfg, const pf_sampler_slide& sl,
                                          const pf_slide_desc& sd, int s, int x, int y, int mi,
                                          int64_t seq, pf_patch_spec* out) {
    pf_patch_spec sp;
    sp.seq = seq;
    sp.target_mpp = cfg.mpp[mi];
    sp.slide = s;
    sp.x = x;
    sp.y = y;
    sp.width = sl.fp[mi];
    sp.height = sl.fp[mi];
    sp.out_size = cfg.patch_size;
    sp.mpp_idx = mi;
    sp.level = sl.level[mi];
    sp.side = sl.side[mi];
    const double ds = (double)sd.downsample[sp.level];
    sp.sx = (int32_t)floor(__dadd_rn(__ddiv_rn((double)x, ds), 0.5));
    sp.sy = (int32_t)floor(__dadd_rn(__ddiv_rn((double)y, ds), 0.5));
    sp.flags = 0;
    *out = sp;
}

// ---------------------------------------------------------------------------
// Speculative evaluation of every (slide, window offset) candidate, in two passes.
//
// sample_classify_kernel, a thread per candidate: the mpp and coordinate draws, then bounds
// on the window's covered-cell count from the slide's classification raster (pf_raster.cu):
// lattice cells inside clean-inside raster cells are covered, inside clean-outside ones not.
// When the bounds settle "count >= need" the candidate is decided on the spot (its bitmap bit
// set or not); the rest are queued.
//
// sample_eval_kernel, kEvalParts warps per queued candidate, each counting a quarter of its
// lattice cell rows (pf_poly.cuh warp_overlap_count_rows); the last part to finish compares
// the total with the threshold.  One resident grid (few large blocks: the block launch ramp of
// ~2000 small ones cost ~10 us) strides the parts over its warps.  Only windows near the
// tissue border reach this pass (~2 % of the candidates), so it is short, and splitting them
// keeps its length at a fraction of one window's latency.
// ---------------------------------------------------------------------------
constexpr int kEvalWarps = 8;
#ifndef PF_EVAL_MIN_BLOCKS
#define PF_EVAL_MIN_BLOCKS 4
#endif
constexpr int32_t kCountBase = 0x7f7f7f7f;  // the round's memset value of reject_at / n_queue
constexpr int kEvalParts = 4;  // a queued window's cell rows are counted by this many warps

constexpr int kClassifyThreads = 64;  // ~45 k candidates: small blocks spread evenly over the SMs

__global__ void __launch_bounds__(kClassifyThreads) sample_classify_kernel(pf_sampler_config cfg, const pf_sampler_slide* slides,
                                                              const pf_sampler_state* state, SamplerWs ws, int window,
                                                              int n, EvalConsts k) {
    if (state->status != PF_OK || state->emitted >= n) return;
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (uint32_t)cfg.n_slides * (uint32_t)window) return;
    const int s = (int)(q / (uint32_t)window), a = (int)(q % (uint32_t)window);
    const pf_sampler_slide& sl = slides[s];
    const uint64_t m0 = state->c_mpp, c0 = state->c_coords;
    const int mi = weighted_pick(stream_u64(cfg.key_mpp, m0 + (uint64_t)a + 1), cfg.mpp_weight, cfg.n_mpps,
                                 k.weight_total);
    const uint64_t nx = (uint64_t)(sl.x_hi[mi] - sl.x_lo[mi] + 1);
    const uint64_t ny = (uint64_t)(sl.y_hi[mi] - sl.y_lo[mi] + 1);
    const uint64_t vx = stream_u64(cfg.key_coords, c0 + 2ull * (uint64_t)a + 1);
    const uint64_t vy = stream_u64(cfg.key_coords, c0 + 2ull * (uint64_t)a + 2);
    if (!randrange_accepts_n(vx, nx) || !randrange_accepts_n(vy, ny)) {
        atomicMin(ws.reject_at, a);
        return;
    }
    const int x = sl.x_lo[mi] + (int)mod_u64(vx, nx);
    const int y = sl.y_lo[mi] + (int)mod_u64(vy, ny);
    const int fp = sl.fp[mi];
    ws.cands[q] = make_int4(x, y, mi, 0);
    int lo = 0, hi = cfg.grid * cfg.grid;
    if (sl.raster)
        raster_bounds_thread(reinterpret_cast<const RasterHeader*>(sl.raster), (double)x, (double)y, (double)fp,
                             cfg.grid, lo, hi);
    if (lo >= k.need || hi < k.need) {  // decided by the bounds on the covered-cell count
        if (lo >= k.need) atomicOr(ws.bitmaps + (size_t)s * (window / 32) + (a >> 5), 1u << (a & 31));
    } else {
        const uint32_t at = atomicAdd(reinterpret_cast<unsigned*>(ws.n_queue), 1u) - (uint32_t)kCountBase;
        PF_CHECK(at < (uint32_t)cfg.n_slides * (uint32_t)window);
        ws.queue[at] = (int)q;
        ws.acc[at] = make_int2(0, 0);
    }
}

// One part of a queued candidate: the covered cells of cell rows [part, part + 1) * grid /
// kEvalParts, added to the candidate's total; the part that completes it sets the bit.
__device__ __forceinline__ void eval_part(const pf_sampler_config& cfg, const pf_sampler_slide* slides,
                                          const SamplerWs& ws, int window, const EvalConsts& k, uint32_t item,
                                          uint32_t* sm) {
    const int lane = threadIdx.x & 31;
#ifdef PF_EVAL_TIMING
    uint64_t t_0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_0));
#endif
    const uint32_t at = item / kEvalParts;
    const int part = (int)(item % kEvalParts);
    const uint32_t q = (uint32_t)__ldg(ws.queue + at);
    PF_CHECK(q < (uint32_t)cfg.n_slides * (uint32_t)window);
    const int s = (int)(q / (uint32_t)window), a = (int)(q % (uint32_t)window);
    const pf_sampler_slide& sl = slides[s];
    const int4 cd = ws.cands[q];
    const int fp = sl.fp[cd.z];
    const PolyView P = poly_view(reinterpret_cast<const void*>(sl.poly_blob));
    const int r_lo = part * cfg.grid / kEvalParts, r_hi = (part + 1) * cfg.grid / kEvalParts;
    const int c = warp_overlap_count_rows(P, (double)cd.x, (double)cd.y, (double)fp, cfg.grid, sm, r_lo, r_hi);
    if (lane == 0) {
        atomicAdd(&ws.acc[at].x, c);
        __threadfence();
        if (atomicAdd(&ws.acc[at].y, 1) == kEvalParts - 1) {
            const int total = atomicAdd(&ws.acc[at].x, 0);
            if (total >= k.need) atomicOr(ws.bitmaps + (size_t)s * (window / 32) + (a >> 5), 1u << (a & 31));
        }
#ifdef PF_EVAL_TIMING
        uint64_t t_1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_1));
        atomicMax(reinterpret_cast<unsigned long long*>(ws.reject_at) + 21, (unsigned long long)t_1);
        // part latency (ns) and start offset into the unused tail of the queue array
        if (item < 8192) {
            ws.queue[16384 + 2 * item] = (int)(t_1 - t_0);
            ws.queue[16384 + 2 * item + 1] = (int)(t_0 & 0x7fffffff);
        }
#endif
    }
}

__global__ void __launch_bounds__(kEvalWarps * 32, PF_EVAL_MIN_BLOCKS) sample_eval_kernel(pf_sampler_config cfg,
                                   const pf_sampler_slide* slides, const pf_sampler_state* state, SamplerWs ws,
                                   int window, int n, EvalConsts k) {
    extern __shared__ __align__(16) uint32_t s_masks[];
    if (state->status != PF_OK || state->emitted >= n) return;
    const int lane = threadIdx.x & 31;
#ifdef PF_EVAL_TIMING  // warp-pass span (tools/eval_timing.py)
    if (lane == 0) {
        uint64_t t_0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_0));
        atomicMin(reinterpret_cast<unsigned long long*>(ws.reject_at) + 20, (unsigned long long)t_0);
    }
#endif
    // queue complete (stream order); every queued candidate is kEvalParts work items of about
    // equal cost, strided over the resident warps (no claim counter to contend on)
    const uint32_t total = ((uint32_t)*ws.n_queue - (uint32_t)kCountBase) * kEvalParts;
    uint32_t* sm = s_masks + (threadIdx.x >> 5) * (overlap_smem_bytes_chunked(cfg.grid) / 4);
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < total; i += nwarps)
        eval_part(cfg, slides, ws, window, k, i, sm);
}

// ---------------------------------------------------------------------------
// Next-accept table and slide draws for the walk, on many CTAs (the walk is one CTA: built
// there, the table alone took ~8 us of it).  Blocks [0, n_slides): one slide's table; the
// rest: the call's slide draws.
//
// entry (slide, a) = where a fresh draw starting at offset a leaves the walk:
//   f + 1            its first accepted attempt f (a spec); | 0x4000 when f + 1 reaches the
//                    window end (the walk's fast loop leaves on any flag bit),
//   0x8000 | a + M   no accept within M = max_attempts (ExhaustedAttemptsError),
//   0xffff           the window (or a rejected coords draw) ends inside the draw
// ---------------------------------------------------------------------------
constexpr int kTableThreads = 512;

__global__ void __launch_bounds__(kTableThreads) sample_table_kernel(pf_sampler_config cfg,
                                                                     const pf_sampler_slide* slides,
                                                                     const pf_sampler_state* state, SamplerWs ws,
                                                                     int window, int n) {
    __shared__ uint32_t s_bm[2048];   // window <= 65536
    __shared__ uint16_t s_next[2048];  // first non-zero word at or after w
    if (state->status != PF_OK || state->emitted >= n) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const int words = window / 32;
    if ((int)blockIdx.x >= cfg.n_slides) {  // slide draws (sample_slide, sampler.py:130-137)
        const int n_fd = min(kFastDraws, 2 * (n - state->emitted) + 256);
        const int i = ((int)blockIdx.x - cfg.n_slides) * kTableThreads + tid;
        if (i >= n_fd) return;
        const uint64_t v = stream_u64(cfg.key_slide, state->c_slide + 1 + (uint64_t)i);
        int sidx;
        if (cfg.strategy == 0) {
            const uint64_t nn = (uint64_t)cfg.n_slides;
            sidx = randrange_accepts(v, randrange_limit(nn)) ? (int)(v % nn) : -1;
        } else {
            double total = 0.0;
            for (int k = 0; k < cfg.n_slides; ++k) total = __dadd_rn(total, slides[k].weight);
            const double u = __dadd_rn(0.0, __dmul_rn(u64_to_unit(v), __dsub_rn(total, 0.0)));
            double acc = 0.0;
            sidx = cfg.n_slides - 1;
            for (int k = 0; k < cfg.n_slides; ++k) {
                acc = __dadd_rn(acc, slides[k].weight);
                if (u < acc) {
                    sidx = k;
                    break;
                }
            }
        }
        if (sidx < 0) *ws.draws_ok = 0;  // a rejected draw (p ~ n / 2^64): the general walk handles it
        ws.fdraw[i] = sidx;
        return;
    }
    const int sl = blockIdx.x;
    PF_CHECK(words <= 2048);
    const uint32_t* bm = ws.bitmaps + (size_t)sl * words;
    for (int i = tid; i < words; i += kTableThreads) s_bm[i] = bm[i];
    __syncthreads();
    if (tid < 32) {  // suffix min of the non-zero word indices, 32 words per step from the end
        int carry = words;
        for (int base = ((words - 1) >> 5) << 5; base >= 0; base -= 32) {
            const int wi = base + lane;
            int v = (wi < words && s_bm[wi] != 0u) ? wi : words;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_down_sync(0xffffffffu, v, o);
                if (lane + o < 32) v = min(v, u);
            }
            v = min(v, carry);
            if (wi < words) s_next[wi] = (uint16_t)v;
            carry = __shfl_sync(0xffffffffu, v, 0);
        }
    }
    __syncthreads();
    const int max_att = cfg.max_attempts;
    const int wlim_t = min(window, *ws.reject_at);
    uint16_t* na = ws.na + (size_t)sl * window;
    for (int a = tid; a < window; a += kTableThreads) {  // consecutive threads, consecutive entries
        const int wd = a >> 5;
        const uint32_t m = s_bm[wd] & (0xffffffffu << (a & 31));
        int f;
        if (m) {
            f = wd * 32 + __ffs(m) - 1;
        } else {
            f = 0x7fffffff;  // first accept after this word
            if (wd + 1 < words) {
                const int w2 = s_next[wd + 1];
                if (w2 < words) f = w2 * 32 + __ffs(s_bm[w2]) - 1;
            }
        }
        uint32_t e;
        if (f < min(a + max_att, wlim_t)) e = (uint32_t)(f + 1) | (f + 1 >= wlim_t ? 0x4000u : 0u);
        else if (a + max_att <= wlim_t) e = 0x8000u | (uint32_t)(a + max_att);
        else e = 0xffffu;
        na[a] = (uint16_t)e;
    }
}

// ---------------------------------------------------------------------------
// Ordered walk (single warp).  Lane 0 drives; lanes help with slide draws.
// ---------------------------------------------------------------------------
struct WalkState {
    uint64_t c_slide, c_coords, c_mpp;
    int64_t seq, failures, attempts, slow;
    int32_t emitted, cur_slide, cur_used, status;
};

__device__ inline void load_ws(const pf_sampler_state* st, WalkState& w) {
    w.c_slide = st->c_slide;
    w.c_coords = st->c_coords;
    w.c_mpp = st->c_mpp;
    w.seq = st->seq;
    w.failures = st->consecutive_failures;
    w.attempts = st->attempts;
    w.slow = st->slow_evals;
    w.emitted = st->emitted;
    w.cur_slide = st->cur_slide;
    w.cur_used = st->cur_used;
    w.status = st->status;
}

__device__ inline void store_ws(pf_sampler_state* st, const WalkState& w) {
    st->c_slide = w.c_slide;
    st->c_coords = w.c_coords;
    st->c_mpp = w.c_mpp;
    st->seq = w.seq;
    st->consecutive_failures = w.failures;
    st->attempts = w.attempts;
    st->slow_evals = w.slow;
    st->emitted = w.emitted;
    st->cur_slide = w.cur_slide;
    st->cur_used = w.cur_used;
    st->status = w.status;
}

// sample_slide (sampler.py:130-137): one call = one randrange / weighted_index.
__device__ inline int draw_slide(const pf_sampler_config& cfg, const pf_sampler_slide* slides,
                                 uint64_t& c_slide) {
    if (cfg.strategy == 0) {
        const uint64_t n = (uint64_t)cfg.n_slides;
        const uint64_t lim = randrange_limit(n);
        while (true) {
            const uint64_t v = stream_u64(cfg.key_slide, ++c_slide);
            if (randrange_accepts(v, lim)) return (int)(v % n);
        }
    }
    const uint64_t u = stream_u64(cfg.key_slide, ++c_slide);
    double total = 0.0;
    for (int i = 0; i < cfg.n_slides; ++i) total = __dadd_rn(total, slides[i].weight);
    const double v = __dadd_rn(0.0, __dmul_rn(u64_to_unit(u), __dsub_rn(total, 0.0)));
    double acc = 0.0;
    for (int i = 0; i < cfg.n_slides; ++i) {
        acc = __dadd_rn(acc, slides[i].weight);
        if (v < acc) return i;
    }
    return cfg.n_slides - 1;
}

__device__ inline int64_t failure_limit(const pf_sampler_config& cfg) {
    return max((int64_t)100, (int64_t)10 * cfg.n_slides);
}

// One exact attempt of sample_patch on the current slide (warp-wide).
// Returns 1 if a spec was emitted.
__device__ inline int slow_attempt(const pf_sampler_config& cfg, const pf_sampler_slide* slides,
                                   const pf_slide_desc* descs, WalkState& w, pf_patch_spec* out,
                                   uint32_t* sm) {
    const int s = w.cur_slide;
    const pf_sampler_slide& sl = slides[s];
    const int mi = weighted_pick(stream_u64(cfg.key_mpp, ++w.c_mpp), cfg.mpp_weight, cfg.n_mpps);
    w.cur_used += 1;
    w.attempts += 1;
    if (sl.x_hi[mi] < sl.x_lo[mi] || sl.y_hi[mi] < sl.y_lo[mi]) return 0;  // no coords draw
    const uint64_t nx = (uint64_t)(sl.x_hi[mi] - sl.x_lo[mi] + 1);
    const uint64_t ny = (uint64_t)(sl.y_hi[mi] - sl.y_lo[mi] + 1);
    uint64_t v;
    do { v = stream_u64(cfg.key_coords, ++w.c_coords); } while (!randrange_accepts(v, randrange_limit(nx)));
    const int x = sl.x_lo[mi] + (int)(v % nx);
    do { v = stream_u64(cfg.key_coords, ++w.c_coords); } while (!randrange_accepts(v, randrange_limit(ny)));
    const int y = sl.y_lo[mi] + (int)(v % ny);
    const PolyView P = poly_view(reinterpret_cast<const void*>(sl.poly_blob));
    const int fp = sl.fp[mi];
    const bool accept = warp_overlap_accept(P, (double)x, (double)y, (double)fp, (double)fp, cfg.grid, sm,
                                            cfg.min_foreground);
    w.slow += 1;
    if (accept) {
        if ((threadIdx.x & 31) == 0) emit_spec(cfg, sl, descs[s], s, x, y, mi, w.seq, out + w.emitted);
        w.seq += 1;
        w.emitted += 1;
        w.failures = 0;
        w.cur_slide = -1;
        return 1;
    }
    return 0;
}

// Walk with the speculation table: warp 0 consumes slide draws in stream order
// against the accept bitmaps staged in shared memory; each emitted spec is
// recorded as (slide, window offset) and materialised afterwards by the whole
// block.  The exact sequential path finishes whatever the table cannot decide.
constexpr int kWalkThreads = 512;
constexpr int kDrawCache = 256;

__device__ inline double k_total_weight(const pf_sampler_config& cfg, const pf_sampler_slide* slides) {
    double total = 0.0;
    for (int k = 0; k < cfg.n_slides; ++k) total = __dadd_rn(total, slides[k].weight);
    return total;
}

__global__ void __launch_bounds__(kWalkThreads) sample_walk_kernel(
    pf_sampler_config cfg, const pf_sampler_slide* slides, const pf_slide_desc* descs, pf_sampler_state* state,
    SamplerWs ws, int window, int n, int use_table, int finish, int bitmaps_in_smem, int next_table, int2* emit_list,
    pf_patch_spec* out) {
    extern __shared__ __align__(16) uint32_t s_dyn[];
    __shared__ int16_t s_draw[kDrawCache];
    __shared__ int s_first, s_last;
    __shared__ int64_t s_seq0;  // stream seq at entry: warp 0 rewrites *state at exit
    WalkState w;
#ifdef PF_WALK_TIMING  // phase timestamps into the workspace's reserved header (tools/walk_timing.py)
#define PF_WT(i) do { if (threadIdx.x == 0) { uint64_t t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); reinterpret_cast<uint64_t*>(ws.reject_at)[4 + (i) + (finish ? 8 : 0)] = t_; } } while (0)
#else
#define PF_WT(i) ((void)0)
#endif
    PF_WT(0);
    load_ws(state, w);
    if (w.status != PF_OK || w.emitted >= n) return;
    const uint64_t m0_round = w.c_mpp;  // window offset 0 of this round's bitmaps
    const int tid = threadIdx.x, lane = tid & 31;
    const int max_att = cfg.max_attempts;
    const int64_t flimit = failure_limit(cfg);
    const int words = window / 32;
    if (tid == 0) {
        s_first = w.emitted;
        s_last = w.emitted;
        s_seq0 = state->seq;
    }
    if (use_table) {
        const uint32_t* bm_all = ws.bitmaps;
        // Shared layout: bitmaps [n_slides * words] (padded to 16 B), next-accept table
        // na[n_slides][window] (uint16), the call's slide draws fdraw[kFastDraws] (int32: 16-bit
        // ones get packed in pairs by the compiler, which then waits on the prefetch load at
        // once), the fast walk's emits semit[] ((slide << 16) | window offset: a global store
        // per draw on the one-thread chain costs more than the chain itself)
        const int bm_bytes = cfg.n_slides * words * 4;
        uint16_t* na = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(s_dyn) + ((bm_bytes + 15) & ~15));
        int32_t* fdraw = reinterpret_cast<int32_t*>(na + (size_t)cfg.n_slides * window);  // window % 32 == 0
        int32_t* semit = fdraw + kFastDraws;
        __shared__ int s_fast;
        __shared__ __align__(8) uint64_t s_bar;
        int n_fd = 0;
        if (next_table) {
            // bitmaps, table and draws in three bulk copies (TMA) on one mbarrier, issued by one
            // thread: the per-thread copy loop of 98 KB was ~3 us of the walk
            n_fd = min(kFastDraws, 2 * (n - w.emitted) + 256);
            PF_CHECK(((bm_bytes + 15) & ~15) + cfg.n_slides * window * 2 + kFastDraws * 4 + window * 4 <=
                     (int)dynamic_smem_size());
            const uint32_t na_bytes = (uint32_t)cfg.n_slides * (uint32_t)window * 2u;
            const uint32_t fd_bytes = ((uint32_t)n_fd * 4u + 15u) & ~15u;
            const bool bm_bulk = (bm_bytes & 15) == 0;
            const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
            if (tid == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                const uint32_t total = na_bytes + fd_bytes + (bm_bulk ? (uint32_t)bm_bytes : 0u);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(total) : "memory");
                auto bulk = [bar](void* dst, const void* src, uint32_t bytes) {
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            (uint32_t)__cvta_generic_to_shared(dst)),
                        "l"(src), "r"(bytes), "r"(bar)
                        : "memory");
                };
                if (bm_bulk) bulk(s_dyn, ws.bitmaps, (uint32_t)bm_bytes);
                bulk(na, ws.na, na_bytes);
                bulk(fdraw, ws.fdraw, fd_bytes);
                s_fast = *ws.draws_ok == kCountBase;
            }
            if (!bm_bulk)
                for (int i = tid; i < cfg.n_slides * words; i += kWalkThreads) s_dyn[i] = ws.bitmaps[i];
            __syncthreads();  // barrier initialised (and the fallback bitmap copy done)
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                    : "=r"(done)
                    : "r"(bar)
                    : "memory");
            bm_all = s_dyn;
        } else if (bitmaps_in_smem) {
            for (int i = tid; i < cfg.n_slides * words; i += kWalkThreads) s_dyn[i] = ws.bitmaps[i];
            bm_all = s_dyn;
            __syncthreads();
        } else {
            __syncthreads();
        }
        PF_WT(1);
        PF_WT(2);
        PF_WT(3);
        if (next_table && s_fast) {
            if (tid == 0) {  // one thread: no divergence bookkeeping inside the chain
                const uint64_t m0 = w.c_mpp;
                const int wlim = min(window, *ws.reject_at);
                int a = 0, j = 0, emitted = w.emitted, used = 0;
                int64_t failures = w.failures;
                int status = w.status;
                bool mid_draw = false;
                int s = w.cur_slide;
                if (s >= 0) {  // a draw resumed from the previous call: its budget is max_att - cur_used
                    used = w.cur_used;
                    const int budget = max_att - used;
                    const int span = min(budget, wlim);
                    const uint32_t* bm = bm_all + (size_t)s * words;
                    int f = 0x7fffffff;
                    for (int x = 0; x < span && f == 0x7fffffff; ++x)
                        if ((bm[x >> 5] >> (x & 31)) & 1u) f = x;
                    if (f != 0x7fffffff) {
                        semit[emitted - s_first] = (s << 16) | f;
                        ++emitted;
                        a = f + 1;
                        failures = 0;
                        s = -1;
                    } else if (span == budget) {
                        a = budget;
                        if (++failures >= flimit) status = PF_ERR_NO_SAMPLABLE;
                        s = -1;
                    } else {
                        a = span;
                        used += span;
                        mid_draw = true;
                    }
                }
                // The chain a <- entry(slide_j, a).  Fast loop for the common case (an accept below the
                // window end, flag bits clear): table load, emit, next offset -- a handful of
                // instructions per draw on one warp's dependent path; anything flagged (exhaustion,
                // window end) or the last spec / last precomputed draw leaves to the general step.
                if (!mid_draw && emitted < n && status == PF_OK && n_fd > 0) {
                    // draws j+1 .. j+4 held in registers: each shared load has iterations to land
                    // before the register rotation moves it (a move waits for its load)
                    int sj = fdraw[0];
                    int s_nxt = fdraw[min(1, n_fd - 1)], s_n2 = fdraw[min(2, n_fd - 1)];
                    int s_n3 = fdraw[min(3, n_fd - 1)], s_n4 = fdraw[min(4, n_fd - 1)];
                    const uint16_t* row = na + (size_t)sj * window;
                    j = 1;
                    if (a >= wlim) {  // the window ends at this draw's first attempt
                        s = sj, used = 0, mid_draw = true;
                    } else {
                        int n_left = n - emitted;  // specs still wanted when a fast segment starts
                        int32_t* el = semit + (emitted - s_first);
                        int k = 0;  // specs emitted by the fast loop
                        while (true) {
                            uint32_t e;
                            // plain accepts while the stream goes on, eight per back edge (a taken
                            // branch per draw costs as much as the draw on one warp)
#define PF_FAST_DRAW                                                                            \
    e = row[a];                                                                                 \
    if (!(e < 0x4000u && k + 1 < n_left && j < n_fd)) break;                                    \
    el[k] = (sj << 16) | ((int)e - 1);                                                          \
    ++k;                                                                                        \
    a = (int)e;                                                                                 \
    sj = s_nxt;                                                                                 \
    row = na + (size_t)sj * window;                                                             \
    ++j;                                                                                        \
    s_nxt = s_n2, s_n2 = s_n3, s_n3 = s_n4;                                                     \
    s_n4 = fdraw[min(j + 3, n_fd - 1)];
                            for (;;) {
                                PF_FAST_DRAW PF_FAST_DRAW PF_FAST_DRAW PF_FAST_DRAW
                                PF_FAST_DRAW PF_FAST_DRAW PF_FAST_DRAW PF_FAST_DRAW
                            }
#undef PF_FAST_DRAW
                            if (k > 0) failures = 0;
                            // general step for this draw
                            emitted += k;
                            el += k;
                            k = 0;
                            e &= (e == 0xffffu || (e & 0x8000u)) ? 0xffffu : 0x3fffu;  // drop the 0x4000 mark
                            const bool acc = e < 0x8000u, win = e == 0xffffu;
                            if (acc) {
                                PF_CHECK(emitted - s_first < window);
                                semit[emitted - s_first] = (sj << 16) | ((int)e - 1);
                                ++emitted;
                                failures = 0;
                                a = (int)e;
                            } else if (!win) {
                                a = (int)(e & 0x7fffu);
                                if (++failures >= flimit) status = PF_ERR_NO_SAMPLABLE;
                            } else {  // the window ends inside this draw
                                used = wlim - a;
                                a = wlim;
                                s = sj, mid_draw = true;
                                break;
                            }
                            if (emitted >= n || status != PF_OK || j == n_fd) break;
                            if (a >= wlim) {  // the next draw starts at the window end
                                s = s_nxt, used = 0, mid_draw = true;
                                ++j;
                                break;
                            }
                            el = semit + (emitted - s_first);
                            n_left = n - emitted;
                            sj = s_nxt;
                            row = na + (size_t)sj * window;
                            ++j;
                            s_nxt = s_n2, s_n2 = s_n3, s_n3 = s_n4;
                            s_n4 = fdraw[min(j + 3, n_fd - 1)];
                        }
                    }
                }
                if (!mid_draw) used = 0;
                w.c_slide += (uint64_t)j;
                w.c_mpp = m0 + (uint64_t)a;
                w.c_coords += 2ull * (uint64_t)a;
                w.attempts += a;
                w.seq += emitted - w.emitted;
                w.emitted = emitted;
                w.failures = failures;
                w.status = status;
                // a draw taken from the table but not finished stays current (cur_slide); a draw
                // taken and finished is consumed; j counts the table entries taken
                w.cur_slide = mid_draw ? s : -1;
                w.cur_used = mid_draw ? used : 0;
                s_last = emitted;
                store_ws(state, w);
            }
            __syncthreads();
            if (tid < 32) load_ws(state, w);
        }
        // general walk over the bitmaps: the whole round without a table, else whatever the fast
        // walk's precomputed draws did not cover (its emits then continue in shared memory)
        const bool fast_emits = next_table && s_fast;
        if (tid < 32 && w.emitted < n && w.status == PF_OK) {
            const uint64_t m0 = m0_round;
            const int wlim = min(window, *ws.reject_at);
            int draw_pos = kDrawCache, draw_cnt = kDrawCache;
            uint64_t draw_base = w.c_slide;  // counter of s_draw[0] is draw_base + 1
            while (w.emitted < n && w.status == PF_OK) {
                if (w.cur_slide < 0) {
                    if (draw_pos == draw_cnt) {  // refill: 32 lanes draw the next kDrawCache counters
                        draw_base = w.c_slide;
                        __syncwarp();  // every lane has read its last s_draw entry
                        for (int i = lane; i < kDrawCache; i += 32) {
                            const uint64_t v = stream_u64(cfg.key_slide, draw_base + 1 + (uint64_t)i);
                            int sidx;
                            if (cfg.strategy == 0) {
                                const uint64_t nn = (uint64_t)cfg.n_slides;
                                sidx = randrange_accepts(v, randrange_limit(nn)) ? (int)(v % nn) : -1;
                            } else {
                                double total = 0.0;
                                for (int k = 0; k < cfg.n_slides; ++k) total = __dadd_rn(total, slides[k].weight);
                                const double u = __dadd_rn(0.0, __dmul_rn(u64_to_unit(v), __dsub_rn(total, 0.0)));
                                double acc = 0.0;
                                sidx = cfg.n_slides - 1;
                                for (int k = 0; k < cfg.n_slides; ++k) {
                                    acc = __dadd_rn(acc, slides[k].weight);
                                    if (u < acc) {
                                        sidx = k;
                                        break;
                                    }
                                }
                            }
                            s_draw[i] = (int16_t)sidx;
                        }
                        __syncwarp();
                        draw_pos = 0;
                    }
                    const int sidx = s_draw[draw_pos++];
                    w.c_slide += 1;
                    if (sidx < 0) continue;  // rejected draw: randrange retries with the next counter
                    w.cur_slide = sidx;
                    w.cur_used = 0;
                }
                const int a0 = (int)(w.c_mpp - m0);
                const int budget = max_att - w.cur_used;
                const int span = min(budget, wlim - a0);
                int found = -1;
                if (span > 0) {
                    const uint32_t* bm = bm_all + (size_t)w.cur_slide * words;
                    const int wfirst = a0 >> 5, wlast = (a0 + span - 1) >> 5;
                    // common case first (acceptance ~0.5): the next accepted offset lies in a0's word
                    uint32_t b0 = bm[wfirst] & (0xffffffffu << (a0 & 31));
                    if (wfirst == wlast) {
                        const int e = (a0 + span - 1) & 31;
                        b0 &= (e == 31) ? 0xffffffffu : ((1u << (e + 1)) - 1u);
                    }
                    if (b0) found = wfirst * 32 + __ffs(b0) - 1;
                    for (int base = wfirst + 1; base <= wlast && found < 0; base += 32) {
                        const int wi = base + lane;
                        uint32_t bits = 0;
                        if (wi <= wlast) {
                            bits = bm[wi];
                            if (wi == wlast) {
                                const int e = (a0 + span - 1) & 31;
                                bits &= (e == 31) ? 0xffffffffu : ((1u << (e + 1)) - 1u);
                            }
                        }
                        const uint32_t ball = __ballot_sync(0xffffffffu, bits != 0);
                        if (ball) {
                            const int src = __ffs(ball) - 1;
                            const uint32_t b = __shfl_sync(0xffffffffu, bits, src);
                            found = (base + src) * 32 + __ffs(b) - 1;
                        }
                    }
                }
                if (found >= 0) {
                    const int consumed = found - a0 + 1;
                    w.c_mpp += consumed;
                    w.c_coords += 2ull * consumed;
                    w.attempts += consumed;
                    if (lane == 0) {  // < window per round
                        PF_CHECK(w.emitted - s_first < window);
                        if (fast_emits) semit[w.emitted - s_first] = (w.cur_slide << 16) | found;
                        else emit_list[w.emitted - s_first] = make_int2(w.cur_slide, found);
                    }
                    w.seq += 1;
                    w.emitted += 1;
                    w.failures = 0;
                    w.cur_slide = -1;
                } else if (span == budget) {
                    w.c_mpp += span;  // ExhaustedAttemptsError: redraw, no seq consumed
                    w.c_coords += 2ull * span;
                    w.attempts += span;
                    w.cur_slide = -1;
                    w.failures += 1;
                    if (w.failures >= flimit) w.status = PF_ERR_NO_SAMPLABLE;
                } else {
                    w.c_mpp += span;  // window (or a rejected draw) reached
                    w.c_coords += 2ull * span;
                    w.attempts += span;
                    w.cur_used += span;
                    break;
                }
            }
            // unused precomputed draws were never consumed: c_slide already counts only consumed ones
            if (lane == 0) s_last = w.emitted;
        }
        __syncthreads();
        PF_WT(4);
        // materialise the emitted specs in parallel
        const int first = s_first, last = s_last;
        const int64_t seq0 = s_seq0;
        for (int i = first + tid; i < last; i += kWalkThreads) {
            int2 e;
            if (fast_emits) {
                const int v = semit[i - first];
                e = make_int2(v >> 16, v & 0xffff);
            } else {
                e = emit_list[i - first];
            }
            const int4 cd = ws.cands[(size_t)e.x * window + e.y];
            emit_spec(cfg, slides[e.x], descs[e.x], e.x, cd.x, cd.y, cd.z, seq0 + (i - first), out + i);
        }
    }
    PF_WT(5);
    if (tid >= 32) return;
    if (finish) {
        uint32_t* sm = s_dyn;
        while (w.emitted < n && w.status == PF_OK) {
            if (w.cur_slide < 0) {
                w.cur_slide = draw_slide(cfg, slides, w.c_slide);
                w.cur_used = 0;
            }
            if (w.cur_used >= max_att) {
                w.cur_slide = -1;
                w.failures += 1;
                if (w.failures >= flimit) w.status = PF_ERR_NO_SAMPLABLE;
                continue;
            }
            slow_attempt(cfg, slides, descs, w, out, sm);
        }
    }
    __syncwarp();
    if (lane == 0) store_ws(state, w);
}

__global__ void sample_begin_kernel(pf_sampler_state* state) {
    state->emitted = 0;
    state->status = PF_OK;
}

// ---------------------------------------------------------------------------
// Capped replay (pkg/sampler.py:230-281): output i = stored[randrange(n_stored)] from
// the "cache" stream, draws consumed in order.  One block: every thread draws for its
// outputs at counters c0 + 1 + i; a rejected draw (v >= floor(2^64/n)*n, probability
// n/2^64) shifts all later counters, so then one thread redoes the batch serially.
// ---------------------------------------------------------------------------
__global__ void capped_draw_kernel(uint64_t key, uint64_t* counter, const pf_patch_spec* stored, int n_stored,
                                   int n, pf_patch_spec* out) {
    __shared__ int any_reject;
    const uint64_t c0 = *counter;
    const uint64_t lim = randrange_limit((uint64_t)n_stored);
    if (threadIdx.x == 0) any_reject = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (!randrange_accepts(stream_u64(key, c0 + 1 + (uint64_t)i), lim)) any_reject = 1;
    __syncthreads();
    if (!any_reject) {
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            out[i] = stored[stream_u64(key, c0 + 1 + (uint64_t)i) % (uint64_t)n_stored];
        if (threadIdx.x == 0) *counter = c0 + (uint64_t)n;
        return;
    }
    if (threadIdx.x == 0) {
        uint64_t c = c0;
        for (int i = 0; i < n; ++i) {
            uint64_t v;
            do v = stream_u64(key, ++c);
            while (!randrange_accepts(v, lim));
            out[i] = stored[v % (uint64_t)n_stored];
        }
        *counter = c;
    }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_overlap_fraction(const void* poly_blob_dev, const double* rects_dev, int32_t n,
                                   int32_t grid, double* out_dev, void* stream) {
    if (n < 0 || grid < 32 || grid > kMaxGrid || (n > 0 && (!poly_blob_dev || !rects_dev || !out_dev)))
        return fail(PF_ERR_INVALID_ARG, "pf_overlap_fraction: bad arguments (32 <= grid <= 256)");
    if (n == 0) return PF_OK;
    const int warps = 4;
    const size_t smem = (size_t)warps * overlap_smem_bytes(grid);
    int rc = check_cuda(cudaFuncSetAttribute(overlap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "cudaFuncSetAttribute");
    if (rc) return rc;
    overlap_kernel<<<(n + warps - 1) / warps, warps * 32, smem, as_stream(stream)>>>(poly_blob_dev, rects_dev, n,
                                                                                 grid, out_dev);
    return after_launch("overlap_kernel");
}

extern "C" int pf_sample_workspace_bytes(const pf_sampler_config* cfg, int32_t window, int64_t* bytes) {
    if (!cfg || !bytes || window < 32 || window % 32 != 0)
        return fail(PF_ERR_INVALID_ARG, "pf_sample_workspace_bytes: window must be a positive multiple of 32");
    *bytes = ws_bytes(cfg->n_slides, window);
    return PF_OK;
}

extern "C" int pf_sample(const pf_sampler_config* cfg, const pf_sampler_slide* slides_dev,
                         const pf_slide_desc* slide_descs_dev, pf_sampler_state* state_dev, int32_t n,
                         pf_patch_spec* out_dev, void* workspace, int64_t workspace_bytes, int32_t window,
                         int32_t rounds, int32_t all_fit, void* stream) {
    if (!cfg || !slides_dev || !slide_descs_dev || !state_dev || n < 0 || (n > 0 && !out_dev))
        return fail(PF_ERR_INVALID_ARG, "pf_sample: bad arguments");
    if (cfg->n_slides < 1) return fail(PF_ERR_NO_SAMPLABLE, "no slides provided");
    if (cfg->n_mpps < 1 || cfg->n_mpps > PF_MAX_MPPS || cfg->grid < 32 || cfg->grid > kMaxGrid ||
        cfg->max_attempts < 1)
        return fail(PF_ERR_INVALID_ARG, "pf_sample: bad config");
    if (n == 0) return PF_OK;
    if (window < 32 || window % 32 != 0 || (int64_t)cfg->n_slides * window >= (int64_t)1 << 31) rounds = 0;
    if (rounds > 0 && (!workspace || workspace_bytes < ws_bytes(cfg->n_slides, window)))
        return fail(PF_ERR_INVALID_ARG, "pf_sample: workspace too small");
    if (!all_fit) rounds = 0;
    cudaStream_t st = as_stream(stream);
    sample_begin_kernel<<<1, 1, 0, st>>>(state_dev);
    int rc = after_launch("sample_begin_kernel");
    if (rc) return rc;
    const int warps = kEvalWarps;
    // per warp: slab/edge cache + chunked row masks (3.7 KB at grid 128)
    const size_t eval_smem = (size_t)warps * overlap_smem_bytes_chunked(cfg->grid);
    const size_t bm_bytes_all = (size_t)cfg->n_slides * (window / 32) * 4;
    const int bm_in_smem = rounds > 0 && bm_bytes_all <= 160 * 1024;
    // next-accepted-offset table beside the bitmaps (uint16 offsets: window < 0xffff)
    const size_t nt_bytes = (bm_bytes_all + 15) / 16 * 16 + (size_t)cfg->n_slides * window * 2 + (size_t)kFastDraws * 4 +
                            (size_t)window * 4;
    // entries: f + 1 below the 0x4000 window-end mark (window <= 0x3fff), 0x8000 | a + M
    const int next_table = bm_in_smem && window < 0x4000 && window + cfg->max_attempts < 0x7fff &&
                           nt_bytes <= 200 * 1024;
    const size_t walk_smem = std::max((size_t)overlap_smem_bytes(cfg->grid),
                                      next_table ? nt_bytes : (bm_in_smem ? bm_bytes_all : (size_t)0));
    rc = check_cuda(cudaFuncSetAttribute(sample_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)walk_smem),
                    "cudaFuncSetAttribute");
    if (rc) return rc;
    rc = check_cuda(cudaFuncSetAttribute(sample_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)eval_smem), "cudaFuncSetAttribute");
    if (rc) return rc;
    static thread_local int eval_grid = 0, eval_grid_dev = -1;  // resident evaluation blocks, whole GPU
    static thread_local size_t eval_grid_smem = 0;
    int cur_dev = 0;
    if ((rc = check_cuda(cudaGetDevice(&cur_dev), "cudaGetDevice"))) return rc;
    if (eval_grid == 0 || eval_grid_dev != cur_dev || eval_grid_smem != eval_smem) {
        int dev = cur_dev, sms = 0, per_sm = 0;
        if ((rc = check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute")))
            return rc;
        if ((rc = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sample_eval_kernel, warps * 32,
                                                                           eval_smem), "cudaOccupancy")))
            return rc;
        eval_grid = std::max(1, sms * std::max(1, per_sm));
        eval_grid_dev = cur_dev;
        eval_grid_smem = eval_smem;
    }
    SamplerWs ws{};
    if (rounds > 0) ws = carve_ws(workspace, cfg->n_slides, window);
    EvalConsts consts{};
    consts.weight_total = weight_total(cfg->mpp_weight, cfg->n_mpps);
    consts.need = accept_cells(cfg->grid, cfg->min_foreground);
    for (int r = 0; r < rounds; ++r) {
        const size_t bm_bytes = (size_t)cfg->n_slides * (window / 32) * 4;
        rc = check_cuda(cudaMemsetAsync(ws.bitmaps, 0, bm_bytes, st), "cudaMemsetAsync");
        if (rc) return rc;
        // reject_at, n_queue and draws_ok all start at kCountBase (0x7f bytes)
        rc = check_cuda(cudaMemsetAsync(ws.reject_at, 0x7f, 12, st), "cudaMemsetAsync");
        if (rc) return rc;
        const int64_t cands = (int64_t)cfg->n_slides * window;
        sample_classify_kernel<<<(unsigned)((cands + kClassifyThreads - 1) / kClassifyThreads), kClassifyThreads, 0,
                                 st>>>(*cfg, slides_dev, state_dev, ws, window,
                                                                                n, consts);
        if ((rc = after_launch("sample_classify_kernel"))) return rc;
        const int64_t blocks = std::min<int64_t>((cands + warps - 1) / warps, eval_grid);
        sample_eval_kernel<<<(unsigned)blocks, warps * 32, eval_smem, st>>>(*cfg, slides_dev, state_dev, ws, window, n,
                                                                             consts);
        if ((rc = after_launch("sample_eval_kernel"))) return rc;
        if (next_table) {
            const int draw_blocks = (std::min(kFastDraws, 2 * n + 256) + kTableThreads - 1) / kTableThreads;
            sample_table_kernel<<<cfg->n_slides + draw_blocks, kTableThreads, 0, st>>>(*cfg, slides_dev, state_dev, ws,
                                                                                      window, n);
            if ((rc = after_launch("sample_table_kernel"))) return rc;
        }
        sample_walk_kernel<<<1, kWalkThreads, walk_smem, st>>>(*cfg, slides_dev, slide_descs_dev, state_dev, ws,
                                                                window, n, 1, r == rounds - 1, bm_in_smem,
                                                                next_table, ws.emits, out_dev);
        if ((rc = after_launch("sample_walk_kernel"))) return rc;
    }
    if (rounds == 0) {
        sample_walk_kernel<<<1, kWalkThreads, walk_smem, st>>>(*cfg, slides_dev, slide_descs_dev, state_dev, ws,
                                                                window, n, 0, 1, 0, 0, nullptr, out_dev);
        if ((rc = after_launch("sample_walk_kernel"))) return rc;
    }
    return PF_OK;
}

extern "C" int pf_capped_draw(uint64_t key, uint64_t* counter_dev, const pf_patch_spec* stored_dev,
                              int32_t n_stored, int32_t n, pf_patch_spec* out_dev, void* stream) {
    if (!counter_dev || n < 0 || (n > 0 && (!out_dev || !stored_dev)))
        return fail(PF_ERR_INVALID_ARG, "pf_capped_draw: bad arguments");
    if (n_stored < 1) return fail(PF_ERR_INVALID_ARG, "pf_capped_draw: cannot draw from an empty cache");
    if (n == 0) return PF_OK;
    capped_draw_kernel<<<1, 1024, 0, as_stream(stream)>>>(key, counter_dev, stored_dev, n_stored, n, out_dev);
    return after_launch("capped_draw_kernel");
}
