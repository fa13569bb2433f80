// Host-backed tile tier: a compacted level whose HBM slot pool is smaller
// than its reachable tile set, backed by a pinned, device-mapped host copy of every reachable
// tile.  Replaces the reference's on-demand TileCache + fetch_chunk (pkg/store.py:270-319,
// 611-649) -- LRU of decoded tiles, fetched on a miss -- with a batch-granular device-side cache:
//
//   the sampler runs one batch ahead, so before batch b's crops are cut its specs are known:
//   1. mark:   every tile a spec's window touches is stamped "used by b"; a non-resident tile is
//              put on the miss list once (a per-tile request flag);
//   2. assign: each miss takes a victim slot -- one no batch >= b - 1 uses (batch b - 1 may still
//              be in flight; batches <= b - 2 have finished: the loader orders the prefetch of b
//              after the crops of b - 2) -- found by a clock hand over the pool; the evicted
//              tile's map entry returns to the zero hole, the new tile's points at the slot;
//   3. fill:   one CTA per miss copies the tile from the mapped host store (zero-copy reads over
//              PCIe, 16-byte vectors) into its slot.
//
// All three run on the caller's stream with no host round trip; running out of victim slots
// (a batch needing more tiles than the pool holds) sets the slide's fault word.
#include <cuda_runtime.h>

#include "pf_common.cuh"

namespace pf {
namespace {

__device__ __forceinline__ void tier_fault(const pf_slide_desc& sd, int code) {
    if (sd.status_word) atomicCAS(reinterpret_cast<int*>(sd.status_word), 0, code);  // the first fault sticks
}

// 1. one thread per (spec, tile of its window); windows at levels without a tier are skipped
__global__ void tier_mark_kernel(const pf_slide_desc* slides, const pf_tile_tier* tiers, const pf_patch_spec* specs,
                                 int n, int32_t batch, int max_tiles_per_spec) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int spec = i / max_tiles_per_spec, k = i - spec * max_tiles_per_spec;
    if (spec >= n) return;
    const pf_patch_spec sp = specs[spec];
    const pf_tile_tier& tr = tiers[sp.slide];
    if (!tr.slot_owner || tr.level != sp.level) return;
    const pf_slide_desc& sd = slides[sp.slide];
    const int L = sp.level, T = sd.tile_size;
    const int x0 = max(sp.sx, 0), y0 = max(sp.sy, 0);
    const int x1 = min(sp.sx + sp.side - 1, sd.width[L] - 1), y1 = min(sp.sy + sp.side - 1, sd.height[L] - 1);
    const int tx0 = x0 / T, ty0 = y0 / T, ntx = x1 / T - tx0 + 1, nty = y1 / T - ty0 + 1;
    if (k >= ntx * nty) return;
    const int tx = tx0 + k % ntx, ty = ty0 + k / ntx;
    const int t = ty * sd.tiles_x[L] + tx;
    int32_t* map = reinterpret_cast<int32_t*>(sd.tile_map[L]);
    int32_t* last = reinterpret_cast<int32_t*>(tr.slot_last_use);
    int32_t* req = reinterpret_cast<int32_t*>(tr.requested);
    int32_t* cnt = reinterpret_cast<int32_t*>(tr.counters);
    const int slot = map[t];
    if (slot > 0) {
        last[slot] = batch;  // benign race: every writer stores the same value
        return;
    }
    if (reinterpret_cast<const int64_t*>(tr.host_index)[t] < 0) {
        tier_fault(sd, PF_ERR_OUT_OF_BOUNDS);  // not in the host store either: the plan missed it
        return;
    }
    if (atomicCAS(req + t, 0, 1) == 0) {
        const int m = atomicAdd(cnt + 0, 1);
        if (m < tr.max_miss) reinterpret_cast<int32_t*>(tr.miss_list)[m] = t;
        else tier_fault(sd, PF_ERR_CAPACITY);
    }
}

// 2. one block per tier: victims by a clock hand over slots 1..n_slots, claimed in block-wide
//    rounds of blockDim candidates (ballot + prefix) until every miss has a slot
__global__ void tier_assign_kernel(const pf_slide_desc* slides, const pf_tile_tier* tiers, int32_t batch) {
    const pf_tile_tier& tr = tiers[blockIdx.x];
    if (!tr.slot_owner) return;
    const pf_slide_desc& sd = slides[blockIdx.x];
    int32_t* cnt = reinterpret_cast<int32_t*>(tr.counters);
    const int n_miss = min(cnt[0], tr.max_miss);
    if (n_miss == 0) return;
    int32_t* map = reinterpret_cast<int32_t*>(sd.tile_map[tr.level]);
    int32_t* owner = reinterpret_cast<int32_t*>(tr.slot_owner);
    int32_t* last = reinterpret_cast<int32_t*>(tr.slot_last_use);
    const int32_t* miss = reinterpret_cast<const int32_t*>(tr.miss_list);
    int32_t* vict = reinterpret_cast<int32_t*>(tr.victims);
    __shared__ int s_taken, s_scanned, s_lastq;
    __shared__ int s_warp[32];
    if (threadIdx.x == 0) s_taken = 0, s_scanned = 0, s_lastq = -1;
    __syncthreads();
    const int hand0 = cnt[2];
    const int ns = tr.n_slots;
    while (true) {
        const int taken = s_taken, scanned = s_scanned;
        if (taken >= n_miss || scanned >= ns) break;
        const int q = scanned + threadIdx.x;
        const int slot = 1 + (hand0 + q) % ns;
        const bool ok = q < ns && last[slot] < batch - 1;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        int before = 0;
        for (int w = 0; w < warp; ++w) before += s_warp[w];
        const int rank = taken + before + __popc(bal & ((1u << lane) - 1u));
        if (ok && rank < n_miss) vict[rank] = slot;
        if (ok && rank == n_miss - 1) s_lastq = q;
        int total = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += s_warp[w];
        __syncthreads();
        if (threadIdx.x == 0) {
            s_taken = taken + total;
            s_scanned = scanned + (int)blockDim.x;
        }
        __syncthreads();
    }
    const int got = min(s_taken, n_miss);
    if (threadIdx.x == 0) {
        if (got < n_miss) tier_fault(sd, PF_ERR_CAPACITY);  // pool smaller than one batch's tiles
        // the hand moves past the last slot taken (or the whole scan when the pool ran out)
        const int adv = s_lastq >= 0 ? s_lastq + 1 : min(s_scanned, ns);
        cnt[2] = (hand0 + adv) % ns;
        cnt[1] = got;
    }
    __syncthreads();
    for (int m = threadIdx.x; m < got; m += blockDim.x) {
        const int slot = vict[m], t = miss[m];
        PF_CHECK(slot >= 1 && slot <= ns);
        const int old = owner[slot];
        if (old >= 0) map[old] = 0;  // evicted: back to the zero hole
        owner[slot] = t;
        last[slot] = batch;
        map[t] = slot;
    }
}

// 3. persistent fill: one CTA per SM walks the (tier, miss) pairs; every thread keeps four 16-byte
//    zero-copy loads in flight (PCIe latency hiding with one CTA of SM footprint, so the crops of
//    the batch in flight keep the rest of the SM)
__global__ void __launch_bounds__(512) tier_fill_kernel(const pf_slide_desc* slides, const pf_tile_tier* tiers,
                                                        int n_tiers) {
    for (int ti = 0; ti < n_tiers; ++ti) {
        const pf_tile_tier& tr = tiers[ti];
        if (!tr.slot_owner) continue;
        const int32_t* cnt = reinterpret_cast<const int32_t*>(tr.counters);
        const int n = cnt[1];
        const pf_slide_desc& sd = slides[ti];
        const int T = sd.tile_size;
        const size_t tb = (size_t)T * T * 3;
        const size_t nv = tb / 16;
        for (int m = blockIdx.x; m < n; m += gridDim.x) {
            const int t = reinterpret_cast<const int32_t*>(tr.miss_list)[m];
            const int slot = reinterpret_cast<const int32_t*>(tr.victims)[m];
            const int64_t h = reinterpret_cast<const int64_t*>(tr.host_index)[t];
            const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(tr.host_tiles) + (size_t)h * tb);
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sd.level_ptr[tr.level]) + (size_t)slot * tb);
            size_t i = threadIdx.x;
            for (; i + 3 * blockDim.x < nv; i += 4 * blockDim.x) {
                const uint4 a = src[i], b = src[i + blockDim.x], c = src[i + 2 * blockDim.x], d = src[i + 3 * blockDim.x];
                dst[i] = a;
                dst[i + blockDim.x] = b;
                dst[i + 2 * blockDim.x] = c;
                dst[i + 3 * blockDim.x] = d;
            }
            for (; i < nv; i += blockDim.x) dst[i] = src[i];
        }
    }
}

// 4. clear the request flags of this batch's misses and the miss counter (stats accumulate)
__global__ void tier_reset_kernel(const pf_tile_tier* tiers) {
    const pf_tile_tier& tr = tiers[blockIdx.x];
    if (!tr.slot_owner) return;
    int32_t* cnt = reinterpret_cast<int32_t*>(tr.counters);
    const int n_miss = min(cnt[0], tr.max_miss);
    int32_t* req = reinterpret_cast<int32_t*>(tr.requested);
    const int32_t* miss = reinterpret_cast<const int32_t*>(tr.miss_list);
    for (int m = threadIdx.x; m < n_miss; m += blockDim.x) req[miss[m]] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        reinterpret_cast<unsigned long long*>(cnt + 4)[0] += (unsigned long long)cnt[1];  // tiles filled, total
        cnt[0] = 0;
        cnt[1] = 0;
    }
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" int pf_host_alloc_mapped(int64_t bytes, void** host_ptr, void** dev_ptr) {
    if (bytes < 1 || !host_ptr || !dev_ptr) return fail(PF_ERR_INVALID_ARG, "pf_host_alloc_mapped: bad arguments");
    int rc = check_cuda(cudaHostAlloc(host_ptr, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable),
                        "pf_host_alloc_mapped: cudaHostAlloc");
    if (rc) return rc;
    return check_cuda(cudaHostGetDevicePointer(dev_ptr, *host_ptr, 0), "pf_host_alloc_mapped: cudaHostGetDevicePointer");
}

extern "C" int pf_host_free(void* host_ptr) {
    if (!host_ptr) return PF_OK;
    return check_cuda(cudaFreeHost(host_ptr), "pf_host_free");
}

extern "C" int pf_tier_prefetch(const pf_slide_desc* slides_dev, const pf_tile_tier* tiers_dev, int32_t n_slides,
                                const pf_patch_spec* specs_dev, int32_t n, int32_t batch, int32_t max_fill,
                                int32_t max_tiles_per_spec, void* stream) {
    if (!slides_dev || !tiers_dev || n_slides < 1 || n < 0 || (n > 0 && !specs_dev) || batch < 2 || max_fill < 1 ||
        max_tiles_per_spec < 1)
        return fail(PF_ERR_INVALID_ARG, "pf_tier_prefetch: bad arguments (batch ids start at 2)");
    if (n == 0) return PF_OK;
    cudaStream_t st = as_stream(stream);
    const long long threads = (long long)n * max_tiles_per_spec;
    tier_mark_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(slides_dev, tiers_dev, specs_dev, n, batch,
                                                                     max_tiles_per_spec);
    int rc = after_launch("tier_mark_kernel");
    if (rc) return rc;
    tier_assign_kernel<<<n_slides, 1024, 0, st>>>(slides_dev, tiers_dev, batch);
    if ((rc = after_launch("tier_assign_kernel"))) return rc;
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    tier_fill_kernel<<<sms, 512, 0, st>>>(slides_dev, tiers_dev, n_slides);
    if ((rc = after_launch("tier_fill_kernel"))) return rc;
    tier_reset_kernel<<<n_slides, 256, 0, st>>>(tiers_dev);
    return after_launch("tier_reset_kernel");
}
