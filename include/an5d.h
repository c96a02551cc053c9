/*
 * an5d.h -- C ABI of the B200-native N.5D temporally blocked stencil library (libAN5D).
 *
 * Method: AN5D, Matsumura et al., arXiv 2001.01473 ("PAPER.md" below, cited P:<line>).
 *   - Problem: a double-buffered grid A[2] with a constant (Dirichlet) boundary ring, updated by a
 *     star or box stencil of radius rad with constant coefficients for I_T time steps
 *     (fig:jacobi2d P:400-418, Table 2).
 *   - Method: N.5D blocking = overlapped-tile temporal blocking (halo b_T*rad per side, recomputed
 *     redundantly) on top of (N-1)-D spatial blocking that streams along the outermost
 *     dimension, with the streaming dimension divided into stream blocks
 *      and box stencils computed by associative partial sums.
 *   - Host loop of sweeps, each advancing up to b_T steps, with a final-block adjustment.
 *
 * Conventions (all functions):
 *   - Layout: row-major, innermost dimension x contiguous.  The STREAMING dimension is the
 *     OUTERMOST array dimension (y in 2D, z in 3D): "the loop after the time loop represents the
 *     streaming dimension".  `extents` are given outermost first and INCLUDE the rad-wide
 *     boundary ring on every face: extent_i = I_S_i + 2*rad.
 *   - `pitches` (may be NULL = dense): element strides of the ndim-1 outer dimensions, outermost
 *     first (2D: {row stride}; 3D: {plane stride, row stride}).
 *   - Alignment (B200 128-bit vector path): the address of element x = rad of every row must be
 *     16-byte aligned, i.e. (base + rad*elem_size) % 16 == 0 and every pitch*elem_size % 16 == 0.
 *     Violations return AN5D_ERR_UNSUPPORTED before any launch (the Python binding allocates
 *     compliant views: paper_2001_01473_b200.empty_grid).
 *   - Pointers named grid_* are DEVICE pointers owned by the caller; the library retains none of
 *     them after a call returns and never allocates grid-sized memory.  A plan owns small device
 *     scheduling state: the dynamic-unit counters and the run tables of the geometries it has
 *     swept (16 bytes per unit, at most 64 tables cached; uploaded synchronously on first use of a
 *     geometry, so do not capture a geometry's first sweep in a CUDA graph); an5d_destroy frees it.
 *   - Environment (tuning / test knobs, read per call): AN5D_RUN_FRAC (fraction of the y/z-
 *     interior stream blocks scheduled as long runs, default 0.85, 0 = one stream block per unit),
 *     AN5D_RUN_WARPS (resident blocks the run table is shaped for; tests), AN5D_FORCE_CFG
 *     ("bT,vec,h" overrides the planner), AN5D_HBM_GBS (planner bandwidth), AN5D_UNIT_PROFILE
 *     (debug per-unit timing dump; synchronises).
 *   - Streams: every launch goes to `cuda_stream` (a cudaStream_t; NULL = legacy default stream)
 *     and is asynchronous.  Argument/feasibility errors are detected before any launch, so an
 *     error return means nothing was written.  CUDA launch errors surface as AN5D_ERR_CUDA.
 *   - No C++ exception crosses this ABI.  an5d_last_error() returns a thread-local message.
 *   - Threading: a plan may be used from one thread at a time; distinct plans are independent.
 */
#ifndef AN5D_H
#define AN5D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AN5D_OK = 0,
    AN5D_ERR_INVALID_ARGUMENT = 1,   /* null pointer, bad ndim/radius/shape/dtype, T < 0, ...   */
    AN5D_ERR_INFEASIBLE_CONFIG = 2,  /* empty compute region b_S - 2*b_T*rad < 1         */
    AN5D_ERR_BLOCK_TOO_LARGE = 3,    /* tile does not fit the kernel instance / thread limits    */
    AN5D_ERR_SHAPE_MISMATCH = 4,     /* extents smaller than 2*rad+1, coefficient count wrong,   */
                                     /* STAR table with a non-zero off-axis entry               */
    AN5D_ERR_UNSUPPORTED = 5,        /* no kernel instance for (ndim,rad,shape,dtype,b_T,vec),   */
                                     /* or misaligned base/pitch for the vector path            */
    AN5D_ERR_CUDA = 6,               /* a CUDA runtime error (message in an5d_last_error)       */
    AN5D_ERR_OUT_OF_MEMORY = 7,
    AN5D_ERR_NCCL = 8                /* NCCL missing or failed (an5d_set_comm slab mode)         */
} an5d_status;

/* STAR / BOX: P:127-142.  GRADIENT: the non-linear gradient2d row of Table 2, 2D,
 * radius 1 only: f' = c f + 1/sqrt(c_0 + sum_{i=-1,+1} ((f - f(x+i,y))^2 + (f - f(x,y+i))^2)),
 * c = the table's centre entry (every other entry must be 0), c_0 = an5d_create's `divisor`
 * argument (not folded); runs on the direct-gather (non-associative) 2D kernel. */
typedef enum { AN5D_STAR = 0, AN5D_BOX = 1, AN5D_GRADIENT = 2 } an5d_shape;
typedef enum { AN5D_F32 = 0, AN5D_F64 = 1 } an5d_dtype;   /* single and double */

typedef struct an5d_plan an5d_plan; /* opaque */

/* Blocking configuration (P:516-519 compile-time parameters of the paper; run-time here).
 * Any field set to 0 is chosen by the host planner (an5d_plan_config).                        */
typedef struct {
    int bT;          /* temporal blocking degree b_T of a full sweep                      */
    int bS[2];       /* logical spatial tile b_S_i INCLUDING the 2*b_T*rad halo, blocked dims     */
                     /* only: 2D {b_S_x, 0}; 3D {b_S_y, b_S_x}.  The kernel loads   */
                     /* b_S_x rounded up so that halos are whole 16-byte vectors.    */
    int64_t h;       /* stream-block length h_SN along the streaming dimension       */
    int vec;         /* cells per thread along y (3D) or x (2D): register tiling factor V        */
    int direct;      /* 0: associative partial sums (the default for both   */
                     /*    shapes).  1: the non-associative "Otherwise" variant of Table 1       */
                     /*    (P:262-270): each level gathers an output from its 2*rad+1 input rows */
                     /*    at once -- kept for the partial-sum on/off comparison (BASELINE       */
                     /*    config 4).  2D only (else AN5D_ERR_UNSUPPORTED); the planner never    */
                     /*    picks 1 by itself.  Values other than 0/1: AN5D_ERR_INVALID_ARGUMENT. */
    int n_thr;       /* threads per thread block of the kernel layout (P:316 n_thr); with bS it    */
                     /* selects the layout: 2D 32 (one warp per tile); 3D 256 (16 x 16 threads, */
                     /* 64-wide tiles) or 512 (32 x 16 threads: 64-wide fp64 tiles at half the  */
                     /* registers per thread, or 128-wide fp32 tiles).  0 = planner / default.  */
                     /* 3D bS[0] (the loaded tile height) also names the thread-block-cluster   */
                     /* layouts (2 / 4 blocks stacked along y sharing y halos through DSMEM: 64 / */
                     /* 128 rows) and, at b_T = 1, the output-stationary tiles (threads on the  */
                     /* 64 x 32 compute region only: bS = {32 + 2 rad, 64 + 2 rad}).            */
} an5d_config;

/* Bookkeeping of one sweep of degree bT under `cfg` (bit-exact).        */
typedef struct {
    int ndim, rad, bT;
    int64_t interior[3];        /* I_S_i, outermost first (streaming dim first)                 */
    int bS[2];                  /* logical tile b_S_i (blocked dims, outer..x)                   */
    int bS_loaded[2];           /* cells actually loaded per tile (x rounded to 16-byte halos)  */
    int compute[2];             /* compute region b_S_i - 2*b_T*rad                      */
    int halo_loaded[2];         /* loaded halo per side (>= b_T*rad)                  */
    int64_t n_tiles[2];         /* ceil(I_S_i / compute_i)                               */
    int64_t n_tb;               /* prod n_tiles                                          */
    int64_t h;                  /* stream-block length h_SN                                      */
    int64_t n_stream_blocks;    /* ceil(I_S_N / h_SN)                                    */
    int64_t n_tb_prime;         /* n_stream_blocks * n_tb                                */
    int64_t stream_overlap;     /* 2*sum_{T=0}^{bT-1} rad*(bT-T) = rad*bT*(bT+1)     */
    int n_thr;                  /* threads per thread block of the kernel instance               */
    int units_per_block;        /* independent tiles handled by one thread block                 */
    int64_t grid_blocks;        /* thread blocks launched per sweep                              */
    size_t smem_bytes;          /* dynamic shared memory per thread block                        */
    int regs_per_thread;        /* from cudaFuncGetAttributes of the instance (0 if unknown)     */
    int vec;                    /* register tiling factor V                                      */
    int64_t n_units;            /* units one launch schedules = entries of the host run table     */
                                /* (consecutive stream blocks of one tile streamed in one pass,   */
                                /* each paying stream_overlap once); n_tb_prime    */
                                /* when AN5D_RUN_FRAC=0                                           */
} an5d_geometry;

/* Create a plan (Table 2).
 *   ndim 2|3; radius 1..4 ("1st to 4th-order"); shape STAR|BOX.
 *   coeffs: dense table of (2r+1)^ndim doubles, index order (d_outer, ..., d_x), each d in
 *     [-r, r]; entry (d) multiplies the neighbour at offset +d: new[x] = sum_d c_d * old[x+d].
 *     STAR tables must have 0 on every entry with more than one non-zero offset component.
 *   divisor: 1.0 = none; j-stencils (j2d5pt, j2d9pt, j3d27pt) divide the sum by c_0 (Table 2).
 *     GRADIENT: c_0, the constant under the square root, not folded; it must be finite and
 *     >= the dtype's smallest normal number (FLT_MIN / DBL_MIN), else AN5D_ERR_UNSUPPORTED.
 *     Applied as in the paper's fast-math build: 1/c_0 is folded into
 *     the coefficients.  Each folded tap is one of the two dtype neighbours of c_d / c_0, chosen
 *     so that the taps' sum is as close as possible to sum_d c_d / c_0 (compensated rounding,
 *     DESIGN.md reading R-8b: plain rounding biases the sum and a T-step run amplifies the bias
 *     T-fold).  divisor == 1: coefficients are rounded once (to nearest) to dtype.
 *   Copies the table; caller keeps ownership of `coeffs`.  On success *out owns the plan until
 *   an5d_destroy.                                                                               */
an5d_status an5d_create(int ndim, int radius, an5d_shape shape, const double* coeffs,
                        size_t n_coeffs, double divisor, an5d_dtype dtype, an5d_plan** out);

/* A multi-field SYSTEM (NEXT N4: "multi-output temporal blocking to optimize multi-statement
 * stencils"): n_fields arrays advance together, one statement per array, and statement i
 * reads the PREVIOUS step of every array through its own Table-2-shaped table:
 *     A_i'(x) = sum_j sum_d coeffs[i][j][d] * A_j(x + d)
 * One sweep streams all arrays and carries every statement through b_T steps (2D kernels).
 *   coeffs: n_fields * n_fields dense (2r+1)^ndim tables, block (i, j) at (i n_fields + j)(2r+1)^ndim,
 *     each rounded once to dtype; STAR blocks must be 0 off-axis.  No divisor.
 *   n_fields 1..8 (kernels are instantiated for 1 and 2; others: AN5D_ERR_UNSUPPORTED at run);
 *   ndim 2 (3D with n_fields > 1: AN5D_ERR_UNSUPPORTED).
 *   With n_fields > 1 every call taking `pitches` (an5d_run, an5d_sweep, an5d_copy_ring,
 *   an5d_tune, an5d_plan_config, an5d_describe) reads pitches[0] = the element distance from one
 *   field's array to the next (grids are n_fields arrays of identical layout, field-major; a
 *   multiple of 16 bytes) followed by the ndim-1 usual pitches (NULL: dense fields and rows).
 *   Slab runs (an5d_run_slab, an5d_sweep_peer with peers) take single-field plans only.        */
an5d_status an5d_create_system(int ndim, int radius, an5d_shape shape, int n_fields, const double* coeffs,
                               size_t n_coeffs, an5d_dtype dtype, an5d_plan** out);

/* Advance the grid by T time steps (host loop of sweeps).
 *   grid_in / grid_out: device arrays with identical extents/pitches (the paper's A[2]).
 *   On return grid_out holds step T (interior) and the input ring; grid_in's interior is used as
 *   scratch and is clobbered when T >= 2 (reading R-7: the sweep count is made odd by
 *   splitting one sweep, generalising the paper's final-block adjustment).  T == 0 copies.
 *   cfg: NULL or fields 0 -> host planner.  cuda_stream: cudaStream_t.                          */
an5d_status an5d_run(an5d_plan* plan, void* grid_in, void* grid_out, const int64_t* extents,
                     const int64_t* pitches, int64_t T, const an5d_config* cfg, void* cuda_stream);

/* One sweep of degree `degree` (1 <= degree <= cfg->bT) reading src, writing dst, for the slab
 * mode of multi-GPU runs: the local array holds planes
 * [outer_offset, outer_offset + extents[0]) of a global array whose outermost extent is
 * global_outer_extent; only global planes within rad of the global faces are ring planes.
 * Output planes written: local [out_lo, out_hi) (clipped to the global interior).  Ring cells of
 * dst must already equal src's (an5d_copy_ring).  Single-GPU: outer_offset = 0,
 * global_outer_extent = extents[0], out_lo = rad, out_hi = extents[0] - rad.                   */
an5d_status an5d_sweep(an5d_plan* plan, const void* src, void* dst, const int64_t* extents,
                       const int64_t* pitches, int degree, const an5d_config* cfg,
                       int64_t outer_offset, int64_t global_outer_extent, int64_t out_lo,
                       int64_t out_hi, int32_t* debug_write_count, void* cuda_stream);

/* ---- Fused halo exchange (slab mode on several GPUs) --------------
 * A sweep of a slab can store its outermost output planes -- the planes the neighbouring slabs
 * hold as ghost planes -- straight into the NEIGHBOURS' destination buffers, from the same
 * kernel that computes them (the thread that stores a plane also stores it to the peer), so no
 * separate exchange step exists.  The buffers are peer-mapped: another GPU's memory opened with
 * an5d_ipc_open (NVLink P2P through NVSwitch), or another buffer on the same GPU.  Ordering
 * between the slabs is stream-ordered with 32-bit flags (an5d_stream_signal / an5d_stream_wait):
 * before sweep i every rank waits until its neighbours have finished sweep i-1 (their ghost
 * stores into its src are complete, and they no longer read the buffer this sweep writes into). */
typedef struct {
    void* peer_dst[2];            /* [0] lower / [1] upper neighbour's buffer of the same parity as */
                                  /* dst (device pointers valid on this device), or NULL           */
    int64_t peer_plane_shift[2];  /* plane index in the neighbour's local array minus the plane    */
                                  /* index here (= my outer_offset - the neighbour's outer_offset) */
    int64_t send_planes[2];       /* the lowest [0] / highest [1] send_planes output planes of this */
                                  /* sweep are also stored there (0 = none)                         */
} an5d_peer_store;

/* an5d_sweep with peer stores.  The neighbours' arrays must have this array's extents beyond the
 * outermost dimension, the same pitches and the same alignment (checked: AN5D_ERR_UNSUPPORTED).
 * peers == NULL is an5d_sweep.                                                                 */
an5d_status an5d_sweep_peer(an5d_plan* plan, const void* src, void* dst, const int64_t* extents,
                            const int64_t* pitches, int degree, const an5d_config* cfg,
                            int64_t outer_offset, int64_t global_outer_extent, int64_t out_lo,
                            int64_t out_hi, const an5d_peer_store* peers, int32_t* debug_write_count,
                            void* cuda_stream);

/* Stream-ordered flag write (after all prior work on the stream, with a memory barrier: the
 * stream's earlier stores -- peer stores included -- are visible before the flag) and wait
 * (the stream blocks until *flag >= value).  flag: a device pointer (own or peer-mapped).      */
an5d_status an5d_stream_signal(uint32_t* flag, uint32_t value, void* cuda_stream);
an5d_status an5d_stream_wait(const uint32_t* flag, uint32_t value, void* cuda_stream);

/* CUDA IPC of a device allocation (one process per GPU): an5d_ipc_export writes the 64-byte
 * handle of the allocation containing ptr and ptr's byte offset in it; an5d_ipc_open maps a
 * handle from another process (peer access enabled lazily) and returns the allocation's base
 * (add the offset); an5d_ipc_close unmaps it.                                                 */
an5d_status an5d_ipc_export(const void* ptr, void* handle64, int64_t* offset);
an5d_status an5d_ipc_open(const void* handle64, void** base);
an5d_status an5d_ipc_close(void* base);

/* The whole T-step run of one slab with the fused exchange, stream-ordered on cuda_stream (the
 * library-owned multi-GPU data plane; no NCCL):  ring copy of the GLOBAL ring planes/cells, then
 * per sweep i: wait until each neighbour's flag >= epoch + i, an5d_sweep_peer over the owned planes
 * [own_lo, own_hi) (local indices) storing d_next*rad boundary planes into the neighbours'
 * buffers of dst's parity, write own flag = epoch + i + 1.  On return links->epoch has advanced by
 * the number of sweeps (every rank must run the same T and b_T); grid_out's owned planes hold step
 * T once the stream reaches that point.  CUDA-graph capturable (flags, kernels and copies only).
 * Errors as an5d_sweep_peer; AN5D_ERR_INVALID_ARGUMENT if a side gives buffers without a flag.   */
typedef struct {
    void* peer_bufs[2][2];        /* [0 lower / 1 upper][the neighbour's buffer paired with grid_in, */
                                  /* with grid_out]: device pointers valid here, or NULL            */
    int64_t peer_plane_shift[2];  /* my outer_offset - the neighbour's outer_offset                */
    uint32_t* peer_flag[2];       /* the neighbours' progress flags (peer-mapped), or NULL          */
    uint32_t* flag;               /* this slab's progress flag (device memory)                      */
    uint32_t epoch;               /* sweeps every slab completed before this run (in / out)         */
} an5d_slab_links;

an5d_status an5d_run_slab(an5d_plan* plan, void* grid_in, void* grid_out, const int64_t* extents,
                          const int64_t* pitches, int64_t T, const an5d_config* cfg, int64_t outer_offset,
                          int64_t global_outer_extent, int64_t own_lo, int64_t own_hi,
                          an5d_slab_links* links, void* cuda_stream);

/* ---- Library-owned NCCL slab mode (BASELINE north_star (d):
 * "slab decomposition of the outermost dimension ... exchanging bT*rad-deep halos every bT steps
 * (NCCL send/recv), overlapped with interior compute") ------------------------------------------
 * an5d_comm_unique_id: ncclGetUniqueId into out128 (128 bytes).  Rank 0 calls it and hands the
 *   bytes to the other ranks out of band (e.g. torch.distributed.broadcast_object_list).
 * an5d_set_comm: the plan joins an NCCL communicator of nranks ranks (ncclCommInitRank; one
 *   process per GPU, the current device; collective: every rank calls it).  From then on an5d_run
 *   treats its grids as this rank's slab of the streaming (outermost) dimension: local plane 0 is
 *   global plane outer_offset of a global array of global_outer_extent planes; on each side that
 *   has a neighbour (rank > 0 below, rank < nranks-1 above) the outermost ghost_planes local
 *   planes are the neighbour's (ghost_planes >= b_T*rad of the run, else AN5D_ERR_UNSUPPORTED
 *   before any launch).  grid_in must hold the input on every local plane, ghosts included; on
 *   return (stream-ordered) grid_out's owned planes hold step T.  Per sweep of degree d: the
 *   boundary output planes first, then the d_next*rad outermost owned planes of the output are
 *   ncclSend/ncclRecv-exchanged with the neighbours in one group on a library-owned comm stream
 *   while the interior planes are computed on cuda_stream; the next sweep waits for both.
 *   Every rank must run the same T and configuration.  nranks == 1: a plain run.
 *   nccl_unique_id == NULL: detach (destroys the communicator).  NCCL is loaded at run time
 *   ("libnccl.so.2" -- the one the process already has, e.g. torch's; AN5D_NCCL_LIB overrides);
 *   a missing library or an NCCL failure -> AN5D_ERR_NCCL.  Single-field plans only.
 *   The fused exchange (an5d_run_slab) is the alternative without NCCL on the data path.       */
an5d_status an5d_comm_unique_id(void* out128);
an5d_status an5d_set_comm(an5d_plan* plan, const void* nccl_unique_id, int rank, int nranks,
                          int64_t global_outer_extent, int64_t outer_offset, int ghost_planes);

/* Copy the rad-wide ring cells of src into dst (O(surface) kernel).  With outer_offset /
 * global_outer_extent as in an5d_sweep, only global ring planes/rows/columns are copied.       */
an5d_status an5d_copy_ring(an5d_plan* plan, const void* src, void* dst, const int64_t* extents,
                           const int64_t* pitches, int64_t outer_offset,
                           int64_t global_outer_extent, void* cuda_stream);

/* The configuration the host planner picks for (extents, T) on the current device (B200 model,
 * DESIGN.md "Planner"); fields of `hint` that are non-zero are kept.                            */
an5d_status an5d_plan_config(an5d_plan* plan, const int64_t* extents, int64_t T,
                             const an5d_config* hint, an5d_config* out);

/* Tuned configuration (the paper's procedure): rank every configuration with the
 * model of an5d_plan_config, run the best stream-block length of each of the top_k distinct
 * (bT, vec, layout) configurations -- plus the best one of every kernel layout the top_k missed --
 * on the device and return the fastest (measured over two sweeps after a warm-up
 * sweep).  Non-zero fields of `hint` are kept, as in an5d_plan_config.
 *   grid_in: read only.  grid_out: overwritten (interior) -- pass the buffers of the following
 *   an5d_run, which rewrites grid_out entirely.  Same extents/pitches/alignment rules as an5d_run.
 *   best_seconds_per_cell_step: optional (NULL); the winner's measured time per cell and step.
 *   Synchronises cuda_stream (a blocking host call; do it once, outside any timed region).
 *   Errors: as an5d_run; AN5D_ERR_CUDA if no candidate could run.                              */
an5d_status an5d_tune(an5d_plan* plan, const void* grid_in, void* grid_out, const int64_t* extents,
                      const int64_t* pitches, int64_t T, const an5d_config* hint, int top_k,
                      an5d_config* out, double* best_seconds_per_cell_step, void* cuda_stream);

/* Bookkeeping introspection for one sweep of degree cfg->bT (bit-exact tests).                 */
an5d_status an5d_describe(an5d_plan* plan, const int64_t* extents, const an5d_config* cfg,
                          an5d_geometry* out);

/* Sweep schedule of T steps at degree bT (P:432-441 with reading R-7): writes up to `cap`
 * degrees to `degrees`, the count to *n_sweeps and whether a trailing interior copy is needed
 * (bT == 1 with an even T) to *trailing_copy.  Pure host function.                             */
an5d_status an5d_schedule(int64_t T, int bT, int* degrees, int64_t cap, int64_t* n_sweeps,
                          int* trailing_copy);

/* ---- The paper's performance model (section 5), pure host arithmetic ------------
 * Thread census of one sweep of degree bT over the whole grid for the PAPER's execution model
 * (one cell per thread, n_thr = prod b_S threads per block), with the readings of
 * DESIGN.md "Planner" (SURVEY C-12, C-13): level T = 1..bT computes and reads shared memory on
 * its valid region prod (b_S_i - 2 T rad) over h + 2 rad (bT - T) planes;
 * every thread writes shared memory at levels 0..bT-1; global reads n_thr (h + 2 bT rad), global
 * writes prod C_i * h per (tile, stream block); Table 3 "practical" shared-memory
 * reads; FLOPs per cell from Table 2 with eff_ALU for k-1 FMA + 1 MUL (+1 MUL for
 * /c_0); eff_SM with n_SM in the wave count (reading C-12).
 * time_model = max(time_comp, time_sm, time_gm) / eff_SM.                        */
typedef struct {
    int n_sm;                    /* SM count (Table 4: V100 80, P100 56; B200 148)              */
    int max_threads_per_sm;      /* 2048                                             */
    double peak_comp_gflops;     /* FP peak of the dtype, GFLOP/s (Table 4)                      */
    double peak_gm_gbs;          /* measured external-memory throughput, GB/s (Table 4)          */
    double peak_sm_gbs;          /* measured shared-memory throughput, GB/s (Table 4)            */
} an5d_device_params;

typedef struct {
    double th_comp, th_sm_read, th_sm_write, th_gm_read, th_gm_write;  /* per sweep, whole grid  */
    int64_t n_tb, n_tb_prime;    /* thread blocks per stream block / per sweep    */
    int n_thr;                   /* threads per block                                            */
    double flops_per_cell;       /* Table 2                                                      */
    double eff_alu, eff_sm;
    double time_comp, time_sm, time_gm, time_model;  /* seconds per sweep of degree bT            */
    double gflops;               /* useful GFLOP/s: prod I * bT * F / time_model (Table 5 Model) */
    int bottleneck;              /* 0 compute, 1 shared memory, 2 global memory                  */
} an5d_model_result;

/* Evaluate the model for one configuration.  interior: I_S_i, outermost (streaming) first.
 * bS: 2D {b_S_x}, 3D {b_S_y, b_S_x} (tile incl. halo).  Errors: AN5D_ERR_INVALID_ARGUMENT (bad
 * argument), AN5D_ERR_INFEASIBLE_CONFIG (b_S - 2 bT rad < 1 or n_thr > max_threads_per_sm).   */
an5d_status an5d_model_paper(int ndim, int radius, an5d_shape shape, int has_divisor, an5d_dtype dtype,
                             const int64_t* interior, int bT, const int* bS, int64_t h,
                             const an5d_device_params* dev, an5d_model_result* out);

/* The paper's "Tuned" search: every (bT, bS, h) of the paper's space -- 2D bT 1..16,
 * bS in {128, 256, 512}, h in {256, 512, 1024}; 3D bT 1..8, bS (y x x) in {16x16, 16x32, 32x32,
 * 16x64}, h in {128, 256} -- minus the configurations the register rule prunes (P:778-784:
 * at least bT (2 rad + 1) + bT + 20 registers per thread in single, 2 bT (2 rad + 1) + bT + 30 in
 * double precision; more than 255 per thread or 65,536 per block is pruned), ranked by the
 * model's GFLOP/s.  Writes the best min(cap, count) configurations (bT, bS, h filled) and their
 * predicted GFLOP/s to out_cfg / out_gflops (either may be NULL) and the number of feasible
 * configurations to *n_feasible.                                                              */
an5d_status an5d_model_paper_search(int ndim, int radius, an5d_shape shape, int has_divisor,
                                    an5d_dtype dtype, const int64_t* interior,
                                    const an5d_device_params* dev, int cap, an5d_config* out_cfg,
                                    double* out_gflops, int* n_feasible);

/* Number of kernel launches the last an5d_run on this plan issued (for bench gpu_launches).    */
int64_t an5d_last_launch_count(const an5d_plan* plan);

an5d_status an5d_destroy(an5d_plan* plan);
const char* an5d_last_error(void);
const char* an5d_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AN5D_H */
