// scan.cuh — single-pass device-wide exclusive scan (decoupled look-back) used for
// the order-preserving compactions of the cull query and of the tree build.
//
// A persistent grid takes tiles from an atomic ticket in launch order; each
// tile publishes its aggregate, looks back over its predecessors (flag 1 =
// aggregate, 2 = inclusive prefix) and publishes its inclusive prefix.  Tiles
// are acquired in increasing order by running CTAs, so the look-back never
// waits on an unscheduled tile.  The item count may live in device memory
// (so the launch needs no host round trip).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

struct V1 {
    int x;
};
__device__ __forceinline__ V1 vadd(V1 a, V1 b) { return V1{a.x + b.x}; }
__device__ __forceinline__ int4 vadd(int4 a, int4 b)
{
    return make_int4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ V1 vzero(V1) { return V1{0}; }
__device__ __forceinline__ int4 vzero(int4) { return make_int4(0, 0, 0, 0); }
__device__ __forceinline__ V1 vshfl_up(V1 a, int d) { return V1{__shfl_up_sync(0xffffffffu, a.x, d)}; }
__device__ __forceinline__ int4 vshfl_up(int4 a, int d)
{
    return make_int4(__shfl_up_sync(0xffffffffu, a.x, d), __shfl_up_sync(0xffffffffu, a.y, d),
                     __shfl_up_sync(0xffffffffu, a.z, d), __shfl_up_sync(0xffffffffu, a.w, d));
}
__device__ __forceinline__ void vstore_volatile(V1 *p, V1 v) { *(volatile int *)&p->x = v.x; }
__device__ __forceinline__ void vstore_volatile(int4 *p, int4 v)
{
    volatile int *q = (volatile int *)p;
    q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
}
__device__ __forceinline__ V1 vload_volatile(const V1 *p) { return V1{*(const volatile int *)&p->x}; }
__device__ __forceinline__ int4 vload_volatile(const int4 *p)
{
    const volatile int *q = (const volatile int *)p;
    return make_int4(q[0], q[1], q[2], q[3]);
}

template <typename T>
struct ScanTiles {
    int32_t *flag;   // [ntiles], zeroed before the launch
    T *agg;          // [ntiles]
    T *pre;          // [ntiles]
    int32_t *ticket; // zeroed before the launch
};

// Block-wide exclusive scan of one value per thread; returns the thread's
// exclusive prefix and writes the block total to *total (all threads).
// Warp-inclusive shuffle scan, then warp 0 scans the THREADS/32 warp totals in
// place (inclusive over warps), so a thread reads two entries instead of looping
// over all warps: integer sums, so the result does not depend on the grouping.
template <typename T, int THREADS>
__device__ __forceinline__ T block_excl_scan(T v, T *total, T *smem_warp /*[THREADS/32]*/)
{
    constexpr int NW = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = vshfl_up(inc, d);
        if (lane >= d) inc = vadd(inc, o);
    }
    if (lane == 31) smem_warp[warp] = inc;
    __syncthreads();
    if (NW > 1 && warp == 0) {
        T s = lane < NW ? smem_warp[lane] : vzero(v);
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            T o = vshfl_up(s, d);
            if (lane >= d) s = vadd(s, o);
        }
        if (lane < NW) smem_warp[lane] = s;
    }
    __syncthreads();
    const T wpre = warp > 0 ? smem_warp[warp - 1] : vzero(v);
    *total = smem_warp[NW - 1];
    __syncthreads();   // smem_warp may be reused by the next call
    // exclusive = wpre + inclusive-of-previous-lanes
    T ex = vshfl_up(inc, 1);
    if (lane == 0) ex = vzero(v);
    return vadd(wpre, ex);
}

__device__ __forceinline__ V1 vshfl_xor(V1 a, int d) { return V1{__shfl_xor_sync(0xffffffffu, a.x, d)}; }
__device__ __forceinline__ int4 vshfl_xor(int4 a, int d)
{
    return make_int4(__shfl_xor_sync(0xffffffffu, a.x, d), __shfl_xor_sync(0xffffffffu, a.y, d),
                     __shfl_xor_sync(0xffffffffu, a.z, d), __shfl_xor_sync(0xffffffffu, a.w, d));
}

// Warp-parallel look-back: called by all 32 lanes of ONE warp; returns (in every
// lane) the exclusive prefix of `tile`.  Each round inspects the 32 nearest
// unresolved predecessors with one round trip: it waits until all of them have
// published at least their aggregate, sums the aggregates down to the nearest
// inclusive prefix (flag 2) and stops there, else moves the window back.
template <typename T>
__device__ __forceinline__ T tile_lookback(ScanTiles<T> st, int tile, T agg)
{
    const int lane = threadIdx.x & 31;
    T excl = vzero(agg);
    if (tile == 0) {
        if (lane == 0) {
            vstore_volatile(&st.pre[0], agg);
            __threadfence();
            *(volatile int32_t *)&st.flag[0] = 2;
        }
        return excl;
    }
    if (lane == 0) {
        vstore_volatile(&st.agg[tile], agg);
        __threadfence();
        *(volatile int32_t *)&st.flag[tile] = 1;
    }
    int j = tile - 1 - lane;
    while (true) {
        int f = j >= 0 ? *(volatile int32_t *)&st.flag[j] : 2;
        if (__any_sync(0xffffffffu, f == 0)) continue;
        __threadfence();
        T v = vzero(agg);
        if (j >= 0) v = (f == 2) ? vload_volatile(&st.pre[j]) : vload_volatile(&st.agg[j]);
        const unsigned m2 = __ballot_sync(0xffffffffu, f == 2);
        const int stop = m2 ? __ffs(m2) - 1 : 31;
        if (lane > stop) v = vzero(agg);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v = vadd(v, vshfl_xor(v, d));
        excl = vadd(excl, v);
        if (m2) break;
        j -= 32;
    }
    if (lane == 0) {
        vstore_volatile(&st.pre[tile], vadd(excl, agg));
        __threadfence();
        *(volatile int32_t *)&st.flag[tile] = 2;
    }
    return excl;
}

// Get the next tile index for this CTA (all threads); returns -1 when done.
__device__ __forceinline__ int next_tile(int32_t *ticket, int64_t n, int tile_items, int *s_tile)
{
    if (threadIdx.x == 0) *s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    int t = *s_tile;
    __syncthreads();
    return ((int64_t)t * tile_items < n) ? t : -1;
}
