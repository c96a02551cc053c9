// args.hpp -- kernel argument blocks of the 2D and 3D N.5D sweeps (shared by the host and the
// kernel instances; plain data, no device code).
#pragma once
#include <cstdint>
#include <cuda.h>   // CUtensorMap (type only; the map is encoded on the host)

namespace an5d {

struct Sweep2DArgs {
    const void* src;      // sweep input  (level 0)
    void* dst;            // sweep output (level degree)
    int64_t pitch;        // row stride in elements
    int64_t Ey;           // local rows (streaming extent of the local array, ring/ghosts included)
    int64_t g_off;        // global row index of local row 0 (slab mode; 0 on one GPU)
    int64_t gEy;          // global streaming extent
    int64_t out_lo;       // local output rows [out_lo, out_hi) (interior only)
    int64_t out_hi;
    int64_t h;            // stream-block length h_SN
    int64_t n_units;      // (tile, stream block) units of this sweep
    unsigned long long* ctr;  // dynamic unit counter pair {next, finished blocks}; zero on entry
    unsigned long long* scratch;  // 1024 x 32 zero slots: the other lanes' no-op atomics (kernel2d.cuh)
    int64_t n_sb;         // stream blocks
    int32_t* wc;          // debug: per-cell store counts (local Ey x Ex, dense), or nullptr
    long long* unit_ns;   // debug: per-unit (start, end, smid) globaltimer stamps, or nullptr
    const int4* runs;     // unit -> {tile_x, first stream block, end stream block}, or nullptr
                          // (then unit = one stream block in the fixed edge-first order)
    // fused halo exchange (NEXT N1): output rows [out_lo, send_lo_end) are also stored into
    // peer_lo at element offset (local offset + peer_lo_shift), rows [send_hi_begin, out_hi) into
    // peer_hi -- the neighbours' ghost rows, peer-mapped (NVLink P2P / CUDA IPC); nullptr = none
    void* peer_lo;
    void* peer_hi;
    int64_t peer_lo_shift, peer_hi_shift;
    int64_t send_lo_end, send_hi_begin;
    int64_t fstride;      // multi-field systems: element distance between consecutive fields (0: one field)
    int Ex;               // x extent (ring included)
    int C;                // compute width per tile (aligned to 16 bytes)
    int H;                // loaded halo per side (>= degree*rad, multiple of the vector width)
    int n_tiles_x;
};

struct Sweep3DArgs {
    const void* src;
    void* dst;
    int64_t pz, py;          // plane and row strides (elements)
    int64_t Ez;              // local planes
    int64_t g_off, gEz;      // global index of local plane 0, global z extent (slab mode)
    int64_t out_lo, out_hi;  // local output planes [out_lo, out_hi)
    int64_t h;               // stream-block length
    int64_t n_units;         // units of this sweep (= blocks)
    int64_t n_sb;            // stream blocks
    int32_t* wc;             // debug store counts (dense Ez x Ey x Ex) or nullptr
    const int4* runs;        // unit -> {tile y, tile x, first stream block, end stream block}, or
                             // nullptr (then unit = one stream block in the fixed frame-first order)
    void* peer_lo;           // fused halo exchange: as Sweep2DArgs (planes instead of rows)
    void* peer_hi;
    int64_t peer_lo_shift, peer_hi_shift;
    int64_t send_lo_end, send_hi_begin;
    int Ey, Ex;
    int Cy, Cx;              // compute region per tile
    int Hy, Hx;              // loaded halo per side (Hy = degree*rad; Hx rounded to 16 bytes)
    int nty, ntx;            // tiles along y, x
    int x_off;               // TMA x coordinate of array x = 0 (the map starts 16-byte aligned before it)
};

}  // namespace an5d
