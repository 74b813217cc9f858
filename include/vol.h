/*
 * vol.h — C ABI of the B200 hashed-voxel-grid primal-dual TV regulariser (arXiv 1604.03734 §III).
 *
 * Citations: P:n = PAPER.md line n (the paper's LaTeX), S:n = SPEC.md line n.  Readings of ambiguous
 * passages are listed in DESIGN.md ("Readings", SURVEY.md §8(c) c-1 … c-20).
 *
 * Data model ("8 voxels in each dimension (512 total)", S:37 x-fastest):
 *   - a volume is n allocated 8³ blocks with integer block coordinates (x, y, z) (int32);
 *   - every per-voxel array is [n][512] float32 in the caller's block order, voxel index
 *     x + 8y + 64z inside a block, global voxel coordinate 8·B + (x, y, z);
 *   - f is the fused TSDF, W the fusion weight; Ω = {allocated voxels with W > 0}
 *     (reading c-13); unallocated blocks are Ω̄.
 *
 * Pointers: every input/output pointer may be host (pageable or pinned) or device memory; the
 * library detects which with cudaPointerGetAttributes.  Host outputs are written synchronously
 * (the call returns after the copy); device outputs are written asynchronously on the handle's
 * stream.  The library copies every input: the caller may free inputs when the call returns.
 *
 * Ownership: the caller owns the optional device workspace passed to vol_create and keeps it
 * alive until vol_destroy; with workspace == NULL the library allocates (and frees) its own.
 * A handle is not thread-safe: one host thread and one CUDA stream per handle.
 *
 * Errors: every call returns a vol_status; vol_last_error() gives a thread-local message for the
 * last failing call of the calling thread.  No call ever falls back to a CPU implementation.
 */
#ifndef HVG_VOL_H
#define HVG_VOL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vol_s *vol_t;

typedef enum {
    VOL_OK = 0,
    VOL_EINVAL = 1,  /* usage: bad sizes, bad parameters, NULL handle (S:542 class "usage")          */
    VOL_EDATA = 2,   /* data: duplicate block coordinates, NaN/Inf in f or W, W < 0, empty Ω */
    VOL_ENOMEM = 3,  /* workspace too small or device allocation failed (S:542 class "resource")     */
    VOL_ECUDA = 4,   /* CUDA runtime error (message in vol_last_error)                                */
    VOL_ENCCL = 5,   /* NCCL error in the sharded path                                                */
    VOL_ENOTSUP = 6  /* feature not built into this library                                          */
} vol_status;

/* Solver options.  vol_default_opts() fills the defaults marked (d).                              */
typedef struct {
    float theta;     /* over-relaxation θ of Eq. 9 (reading c-3); (d) 1.0 (Table I) */
    int data_term;   /* 0 (d): W-weighted L1 shrinkage toward f (north_star, TV-L1);
                        1: W-weighted L2 prox, paper Eq. 8                               */
    int init;        /* 0 (d): warm start u = ū = f, p = 0; 1: u = ū = 0 on Ω, p = 0 */
    int resume;      /* 0 (d): initialise before iterating; 1: continue from the current state        */
    int kernel;      /* 0 (d): the product path = 2;
                        1: two-kernel baseline (dual kernel, then primal+relax kernel; single GPU only);
                        2: skewed fused schedule (one HBM sweep per iteration: primal k + dual k+1 per
                           launch, ū never stored inside the loop; sharded: a (u, p) halo before
                           every launch);
                        3: one-pass fused kernel (dual k + primal k per launch; sharded: (ū, p) halo).
                        All four give bit-identical results                        */
    int freeze;      /* 1 (d): with the L1 data term, voxels whose primal step is provably the identity
                        for the whole call (τλW >= τ(3+√3) plus rounding margin, and u = ū = f in both
                        buffers at the start of the call) are not recomputed nor rewritten — the result
                        is bit-identical; 0: every Ω voxel is updated every iteration               */
    int exchange;    /* 1 (d): a sharded volume exchanges its halo every iteration;
                        0: the exchange chain (pack, NCCL send/recv, unpack) is replaced by a no-op with
                        the same partition and the same launches — the result is WRONG; for timing only
                        (exposed halo µs/iteration = T(1) − T(0)).  Ignored when unsharded */
} vol_opts;

/* Multi-GPU description (route-axis spatial sharding).  NULL = single GPU.          */
typedef struct {
    int rank;               /* this process's rank in [0, world)                                   */
    int world;              /* number of ranks (one GPU each)                                      */
    const int32_t *part;    /* [n_global] owner rank of each block (host pointer)                  */
    const void *nccl_id;    /* 128-byte ncclUniqueId created by rank 0 and broadcast by the caller
                               (NCCL transport; with world == 1 the sharded runtime runs with no
                               peers); NULL: loopback transport (world > 1) or plain single GPU      */
} vol_dist;

/* Defaults for vol_opts (see field comments). */
void vol_default_opts(vol_opts *opts);

/* Device bytes vol_create needs for a volume of n_global blocks (exact for dist == NULL; for a
 * sharded volume pass the same dist as to vol_create, the value then covers local + ghost blocks).
 * block_xyz may be NULL when dist == NULL.  Device coordinates of a sharded volume are read on the
 * legacy default stream (the call takes no stream): writes to them on another stream must be
 * complete.  Returns 0 on invalid arguments.                                                      */
size_t vol_workspace_bytes(const int32_t *block_xyz, int64_t n_global, const vol_dist *dist);

/* Build a volume:
 *   block_xyz [n_global][3] int32 block coordinates (host or device), all distinct, each in
 *             (−2^30, 2^30);
 *   f, W      [n_local][512] float32 (host or device): the blocks this rank owns, in global order
 *             (n_local = n_global when dist == NULL); f finite, W finite and >= 0;
 *   dist      NULL (single GPU) or the sharding description;
 *   workspace device buffer of >= vol_workspace_bytes(...) bytes, or NULL (library allocates);
 *   stream    cudaStream_t for every later call on this handle (NULL = legacy default stream).
 * Builds on the device: the spatial hash h(x,y,z) = ((u32)x·73856093 ⊕ (u32)y·19349669 ⊕
 * (u32)z·83492791) mod T with T = next power of two >= 2n, a CSR bucket table ordered by caller
 * index (reading c-14), and the 6-neighbour block table (−x,+x,−y,+y,−z,+z; −1 = unallocated).
 * Errors: VOL_EINVAL (n_global < 1, NULL pointers, 2^23 or more local + ghost blocks on one GPU —
 * the iteration kernels index voxels with 32 bits), VOL_EDATA (duplicate coordinates — the first
 * repeated pair is named in vol_last_error —, coordinates out of range, non-finite f/W, W < 0),
 * VOL_ENOMEM, VOL_ECUDA.                                                                          */
vol_status vol_create(const int32_t *block_xyz, int64_t n_global, const float *f, const float *W,
                      const vol_dist *dist, void *workspace, size_t workspace_bytes, void *stream,
                      vol_t *out);

/* vol_create with the weights given as exact 8-bit observation counts (W is a count, Eq. 1: w_k = w_{k-1}
 * + 1 capped at w_max): W8 [n_local][512] uint8 (host or device), otherwise as vol_create.
 * Equivalent to vol_create with W = (float)W8 — bit for bit — with a quarter of the weight bytes to copy
 * (the end-to-end bench passes host weights this way).  Errors as vol_create; VOL_EINVAL if W8 is NULL. */
vol_status vol_create_w8(const int32_t *block_xyz, int64_t n_global, const float *f, const uint8_t *W8,
                         const vol_dist *dist, void *workspace, size_t workspace_bytes, void *stream, vol_t *out);

/* Run `iters` Chambolle–Pock iterations (SURVEY §8(a) rows a-2 … a-6):
 *   dual ascent with Huber damping + projection  q = (p + σ∇_Ω ū)/(1 + σε),  p = q / max(1, ‖q‖₂)
 *   primal step                                  ũ = u + τ·div_Ω p  (sign: reading c-2)
 *   data prox (opts->data_term)                  L1: shrink ũ toward f by τλW;  L2: (ũ+τλWf)/(1+τλW)
 *   over-relaxation                              ū = u' + θ(u' − u),  u = u'
 * with the Ω-masked forward gradient (Eq. 3) and backward divergence (Eq. 4,
 * P:252-263) across block faces.  Constraints: λ > 0, ε >= 0, τ > 0, σ > 0, 12·τσ <= 1 + 1e-6
 * (‖∇_Ω‖² <= 12), iters >= 0 (0 = initialise only unless resuming).  Asynchronous on the handle's
 * stream.  Errors: VOL_EINVAL (parameters), VOL_EDATA (global Ω empty), VOL_ECUDA/ENCCL.   */
vol_status vol_regularise(vol_t v, float lambda, float eps, float tau, float sigma, int32_t iters,
                          const vol_opts *opts);

/* Copy u [n_local][512] float32 in the caller's block order into u_out (host or device);
 * Ω̄ voxels hold f (they are never written).                                                */
vol_status vol_read_u(vol_t v, float *u_out);

/* Energy of the current state (Eq. 2, Huber TV, W-weighted data
 * term, reading c-1), fp64 deterministic reduction over all ranks:
 *   primal = Σ_Ω H_ε(‖∇_Ω u‖₂) + λ Σ_Ω W|u−f|   (data_term 0)  or  + (λ/2) Σ_Ω W(u−f)²  (1);
 *   dual   = SURVEY §8(c) dual value at the current p (L1: rescaled to |div p| <= λW); may be NULL.
 * Synchronous.                                                                                    */
vol_status vol_energy(vol_t v, float lambda, float eps, int data_term, double *primal, double *dual);

/* State checkpoint: u, ū (current relaxed primal), p = [3][n_local][512] (component-
 * major).  Any pointer may be NULL to skip it.  vol_load_state sets p = 0 on Ω̄ and ū = u = f there. */
vol_status vol_read_state(vol_t v, float *u, float *ubar, float *p);
vol_status vol_load_state(vol_t v, const float *u, const float *ubar, const float *p);

/* Store tables for bit-exact checks (caller indices; single-GPU volumes only):
 *   *T; bucket_start [T+1] uint32; bucket_entry [n] int32; nbr [n][6] int32.  Pointers may be NULL. */
vol_status vol_read_tables(vol_t v, uint32_t *T, uint32_t *bucket_start, int32_t *bucket_entry,
                           int32_t *nbr);

/* Sizes: allocated blocks on this rank, ghost blocks held, total Ω voxels on this rank.           */
vol_status vol_info(vol_t v, int64_t *n_local, int64_t *n_ghost, int64_t *n_omega);

/* Per-stream durations of the LAST iteration of the last vol_regularise call on an NCCL-sharded volume
 * (SURVEY §8(d) "boundary-chain vs interior-kernel durations from per-stream events"), in ms, from CUDA
 * events: interior_ms = launch A (blocks without a remote neighbour, compute stream); exchange_ms = the
 * halo chain pack → NCCL send/recv → unpack (communication stream, overlapping launch A); boundary_ms =
 * launch B (blocks with a remote neighbour, after the halo).  Waits for those events.  Any output pointer
 * may be NULL.  VOL_EINVAL if the volume is not NCCL-sharded or has not iterated yet.                  */
vol_status vol_shard_timing(vol_t v, float *interior_ms, float *exchange_ms, float *boundary_ms);

/* Number of kernel launches the last vol_regularise issued (counted on the host; graph nodes count). */
int64_t vol_last_launches(vol_t v);

/* Kernels launched by this library in this process so far (graph replays count every node). */
int64_t vol_total_launches(void);

/* Block until all work on the handle's stream is done. */
vol_status vol_sync(vol_t v);

void vol_destroy(vol_t v);

/* Thread-local message of the last error ("" if none). */
const char *vol_last_error(void);

/* Sharded volumes ----------------------------------------------------------------
 * NCCL transport: rank 0 calls vol_nccl_unique_id, the caller broadcasts the 128 bytes (e.g. with
 * torch.distributed), every rank passes them in dist->nccl_id to vol_create (collective: all ranks
 * call vol_create, vol_regularise and vol_energy together).  Per iteration each rank exchanges one
 * message per neighbouring rank (ū, p of the ghost blocks) with ncclSend/ncclRecv, overlapped with
 * the interior blocks.
 * Loopback transport (tests on one GPU): `world` handles created in one process with
 * dist->nccl_id == NULL; vol_group_connect exchanges the static ghost data once, then
 * vol_regularise_group / vol_group_energy run the same plan, pack/unpack and two-launch schedule
 * with device-to-device copies, on handles[0]'s stream.  The result equals the single-GPU result
 * bit for bit.                                                                                   */
vol_status vol_nccl_unique_id(void *out128);
vol_status vol_group_connect(vol_t *handles, int world);
vol_status vol_regularise_group(vol_t *handles, int world, float lambda, float eps, float tau, float sigma,
                                int32_t iters, const vol_opts *opts);
vol_status vol_group_energy(vol_t *handles, int world, float lambda, float eps, int data_term, double *primal,
                            double *dual);

/* Direct-store halo transport (the paper's "boundary conditions" of a block taken from its
 * neighbours, fetched across GPUs).  A sharded volume whose peers are all connected writes,
 * in its boundary launch, the (u, p) of every block a peer reads straight into that peer's ghost rows
 * (peer memory over NVLink; in one process, another volume's workspace) and signals a per-source counter
 * in the peer's memory; the peer waits for it before its own boundary launch.  No pack, no NCCL, no
 * unpack inside the loop; results are bit-identical to the other transports.  Collective: every rank
 * connects every peer it exchanges with, and all ranks use the transport for the same calls.
 *   vol_peer_info(v, info, cap, &n)  this rank's descriptor for its peers (n int64: ranks, sizes,
 *                                    receive offsets, byte offsets of the field buffers and counters
 *                                    inside the workspace); info = NULL queries n.
 *   vol_connect_peer(v, q, ws, info, n)   register peer q whose workspace is mapped at device address
 *                                    `ws` in this process (its vol_peer_info in `info`); peers this rank
 *                                    has no halo with are ignored.  After the last needed peer the
 *                                    volume switches to direct stores (vol_transport = 3).
 *   vol_ipc_handle(v, handle64, &off) the CUDA IPC handle (64 bytes) of the allocation holding this
 *                                    volume's workspace and the workspace's offset inside it;
 *   vol_connect_peer_ipc(v, q, handle64, off, info, n)  opens it (cudaIpcOpenMemHandle, NVLink peer
 *                                    access) and connects peer q; the mapping is closed by vol_destroy.
 *   vol_transport(v)                 0 unsharded, 1 NCCL, 2 loopback copies, 3 direct stores.        */
vol_status vol_peer_info(vol_t v, int64_t *info, int64_t cap, int64_t *n);
vol_status vol_connect_peer(vol_t v, int peer, void *peer_workspace, const int64_t *info, int64_t n);
vol_status vol_ipc_handle(vol_t v, void *handle64, int64_t *offset);
vol_status vol_connect_peer_ipc(vol_t v, int peer, const void *handle64, int64_t offset, const int64_t *info,
                                int64_t n);
int vol_transport(vol_t v);

/* Host-only helpers (no GPU needed), used by the sharding planner tests -------------------------- */

/* The block hash of vol_create (no device work). */
uint32_t vol_block_hash(int32_t x, int32_t y, int32_t z, uint32_t T);

/* Shard plan of `rank`: counts of local blocks, ghost blocks, and per-peer send /
 * receive block counts.  Fills ghost_global [n_ghost] (global indices of ghost blocks, receive
 * order), send_global [n_send] (global indices of local blocks sent, grouped by peer in rank order)
 * and peer_send / peer_recv [world] (blocks sent to / received from each peer) when non-NULL.
 * Call with NULL arrays first to get the sizes.  Returns VOL_OK or VOL_EINVAL/VOL_EDATA.          */
vol_status vol_plan_shard(const int32_t *block_xyz, int64_t n_global, const int32_t *part, int world,
                          int rank, int64_t *n_local, int64_t *n_ghost, int64_t *n_send,
                          int64_t *ghost_global, int64_t *send_global, int64_t *peer_send,
                          int64_t *peer_recv);

/* Route-axis partition (the regulariser is block-local with boundary
 * conditions from the neighbour blocks, so the cut surface between ranks is the halo).  Host only.
 *   block_xyz   [n_global][3] int32 block coordinates (host memory);
 *   route       [n_route][3] float64 polyline vertices in metres (the camera path), n_route >= 1;
 *   block_edge  block edge length in metres (8 x voxel size); a block's centre is (b + 0.5)*block_edge;
 *   world       number of ranks; part [n_global] (out): owner rank of every block;
 *   arc         [n_global] (out, nullable): arc length (metres) of the route point nearest to each
 *               block centre (the first segment wins a tie in distance).
 * Blocks are ordered by (arc, x, y, z) and cut into `world` contiguous ranges of equal block count:
 * rank r owns positions [r*n/world, (r+1)*n/world).  The result is a pure function of the arguments
 * (every rank computes the same map).  Returns VOL_OK or VOL_EINVAL.                               */
vol_status vol_partition_route(const int32_t *block_xyz, int64_t n_global, const double *route, int32_t n_route,
                               double block_edge, int world, int32_t *part, double *arc);

/* Destroy every cached NCCL communicator of this process (teardown; volumes still using one must be
 * destroyed first).  Communicators are cached per (unique id, world, rank, device) so that volumes
 * created over one process group share one; a communicator that reports an asynchronous error is
 * aborted and evicted automatically.                                                              */
vol_status vol_release_comms(void);

/* Isosurface extraction ("extract the surface", P:132-133 zero-crossing
 * level set).  Readings X-1 … X-7: marching tetrahedra over the cells spanned by every
 * voxel g and g + {0,1}^3 (voxel centres (g + ½)·voxel metres) whose 8 corners are allocated with
 * W > 0 and W >= w_min (no geometry next to Ω̄); each cell split into the 6 Freudenthal tetrahedra;
 * inside ⇔ value < 0; vertex on an edge with ends lo < hi (global coordinates, lexicographic)
 * p = P_lo + t(P_hi − P_lo), t = v_lo/(v_lo − v_hi) in fp32; triangles oriented toward value > 0;
 * triangles with two identical vertices dropped.  Output: triangle soup [m][3][3] float32 (x, y, z
 * of 3 vertices), ordered by caller block, cell (voxel order), tetrahedron, triangle.
 *   field   0: the current u (u = f from vol_create until the first vol_regularise), 1: the fused f;
 *   tris    host or device buffer of max_tris triangles, or NULL to count only; *n_tris receives m.
 * A device buffer is filled in one ordered pass (count, look-back, emit); a host buffer is sized by a
 * counting pass first.  Synchronous.  Errors: VOL_EINVAL, VOL_ENOMEM (m > max_tris; *n_tris = m; a
 * device buffer then holds the first max_tris triangles, a host buffer is untouched), VOL_ENOTSUP
 * (sharded volume), VOL_ECUDA.                                                                      */
vol_status vol_extract(vol_t v, int field, float voxel, float w_min, float *tris, int64_t max_tris, int64_t *n_tris);

/* Depth-map estimation from rectified stereo (paper §IV) ----------
 * Readings S-1 … S-12.  Batched: images are [F][H][W] float32 intensities in [0, 1].
 *   census   window 3 or 5, bit k (row-major, centre skipped) = neighbour < centre,
 *            clamp-to-edge borders;
 *   cost     ρ(x, y, d) = Hamming(sig_R(x, y), sig_L(x + d, y)) (bits), d = 0 … n_disp−1, the right
 *            image is the reference; x + d outside the image → win² − 1;
 *   tensor   T = exp(−γ|∇I_R|^β) n nᵀ + n⊥ n⊥ᵀ, central differences, identity where |∇I| < 1e-6,
 *            evaluated in fp64 and rounded to fp32;
 *   solver   E = α₁Σ|T∇d − w|₂ + α₂Σ|∇w|_F + 1/(2θ)Σ(d − a)² + λΣρ(a) (P:526 + quadratic relaxation):
 *            init a = d = winner-take-all; `outer` rounds of `inner` Chambolle–Pock iterations on (d, w)
 *            (steps τ, σ with 12τσ <= 1), then a ← argmin over integer d of the coupling + data term
 *            with a parabola sub-pixel step; θ from theta0 to theta_end geometrically.              */
typedef struct {
    int32_t width, height;   /* W, H of every image                                                */
    int32_t n_disp;          /* D: candidate disparities 0 … D−1 (pixels)                          */
    int32_t window;          /* census window: 3 or 5                                              */
    int32_t outer, inner;    /* data-step rounds; Chambolle–Pock iterations per round               */
    float lambda;            /* λ_2D (Table I: 0.5)                                                */
    float alpha1, alpha2;    /* α₁, α₂ (Table I: 1.0, 5.0)                                         */
    float beta, gamma;       /* β, γ (Table I: 1.0, 4.0)                                           */
    float theta0, theta_end; /* coupling schedule (default 1.0 → 0.01)                             */
    float tau, sigma;        /* primal / dual steps (default 1/√12 each)                           */
} vol_stereo_params;

void vol_stereo_default_params(vol_stereo_params *params);

/* Device bytes vol_stereo needs for n_frames pairs (inputs on the host included). */
size_t vol_stereo_workspace_bytes(int32_t n_frames, const vol_stereo_params *params);

/* Solve n_frames rectified pairs.  left, right [F][H][W] (both host or both device); outputs (all host
 * or all device): disparity d [F][H][W], w [F][2][H][W] per frame-major plane order [2][F][H][W]
 * (may be NULL), a [F][H][W] (last data step, may be NULL).  workspace >= vol_stereo_workspace_bytes
 * or NULL (library allocates).  Synchronous for host pointers, else asynchronous on `stream`.
 * Errors: VOL_EINVAL (parameters: sizes, window, 12τσ > 1 …), VOL_ENOMEM, VOL_ECUDA.              */
vol_status vol_stereo(const float *left, const float *right, int32_t n_frames, const vol_stereo_params *params,
                      void *workspace, size_t workspace_bytes, void *stream, float *disparity, float *w, float *a);

/* Census signatures [F][H][W] uint32 of img [F][H][W] (device pointers; for checks).               */
vol_status vol_stereo_census(const float *img, int32_t n_frames, int32_t height, int32_t width, int32_t window,
                             void *stream, uint32_t *sig);
/* Tensor fields T [3][F][H][W] = (T11, T12, T22) of img (device pointers; for checks).              */
vol_status vol_stereo_tensor(const float *img, int32_t n_frames, int32_t height, int32_t width, float beta,
                             float gamma, void *stream, float *T);
/* depth = fx_baseline / d for d > d_min, else 0 (invalid); device pointers.                 */
vol_status vol_disparity_to_depth(const float *disparity, int64_t n, float fx_baseline, float d_min, void *stream,
                                  float *depth);

/* TSDF fusion of posed depth maps (paper §III-A, Eq. 1) ----------
 * Readings F-1 … F-10.  For every depth map k = 0 … K−1 in sequence the paper
 * allocates the blocks where frame k observes a surface and then updates every voxel of
 * every allocated block:
 *   allocation  every valid pixel (i, j) (depth d finite, 0 < d <= max_range) allocates the blocks met
 *               by its viewing ray between camera depths max(d − μ, 0) and d + μ (F-5), visited by a
 *               6-connected walk over the block lattice (F-7);
 *   update      p_c = R^T (p_g − t) (F-2) for the voxel centre p_g = (8B + i + ½)·v; nearest
 *               pixel (floor(fx·x_c/z_c + cx + ½), floor(fy·y_c/z_c + cy + ½)) (F-1); if z_c > 0,
 *               the pixel is inside and its depth valid: u_SDF = d − z_c; Eq. 1: if
 *               u_SDF >= −μ then u_TSDF = clamp(u_SDF, −μ, μ)/μ (F-3), f = (u_TSDF + w·f)/(w + 1),
 *               w = min(w + 1, w_max) (F-4).  Unobserved voxels keep f = 0, W = 0.
 * All arithmetic is IEEE fp32 in that written order (F-10).                                         */
typedef struct {
    float fx, fy;       /* focal lengths in pixels (> 0)                                            */
    float cx, cy;       /* principal point in pixels; pixel (i, j) is the unit square centred at (i, j) */
    int32_t width;      /* W: columns of every depth map                                            */
    int32_t height;     /* H: rows                                                                  */
} vol_camera;

typedef struct {
    float voxel;        /* voxel edge v in metres (blocks are 8v)                                   */
    float mu;           /* truncation distance μ in metres (Eq. 1)                                  */
    float max_range;    /* depths > max_range are invalid (F-9)                                     */
    float w_max;        /* weight cap (F-4); >= 1, a huge value gives the paper's uncapped w         */
} vol_fusion_params;

/* Counters of one vol_fuse call ("Returns counts").                                   */
typedef struct {
    int64_t pixels_valid;   /* valid depth pixels over all frames (each allocates its band)          */
    int64_t blocks;         /* allocated blocks                                                      */
    int64_t block_frames;   /* (block, frame) pairs evaluated by the update pass after the
                               conservative frustum/range cull (frames since the block's allocation) */
    int64_t voxel_updates;  /* Eq. 1 updates applied (u_SDF >= −μ on a valid in-image pixel)          */
    float ms_alloc;         /* CUDA-event duration of the allocation kernel on the stream (ms)        */
    float ms_integrate;     /* CUDA-event duration of the update kernel on the stream (ms)            */
} vol_fusion_stats;

/* Device bytes vol_fuse needs for up to max_blocks allocated blocks (worst case: host inputs and
 * host outputs).  Returns 0 on invalid arguments.                                                 */
size_t vol_fuse_workspace_bytes(int64_t max_blocks, int32_t n_frames, const vol_camera *cam);

/* Fuse K = n_frames depth maps into a new set of blocks:
 *   depth     [K][H][W] float32 metres (host or device); non-finite, <= 0 or > max_range = invalid;
 *   poses     [K][12] float32 row-major T_gc = [R | t] (camera-to-global, p_g = R p_c + t), host or
 *             device;
 *   max_blocks capacity of the outputs; workspace device buffer of >= vol_fuse_workspace_bytes(...)
 *             or NULL (the library allocates and frees its own); stream cudaStream_t or NULL;
 *   outputs   (all host or all device) block_xyz [max_blocks][3] int32, first_frame [max_blocks]
 *             int32 (frame that allocated the block; may be NULL), f, W [max_blocks][512] float32;
 *             rows 0 … n−1 hold the n allocated blocks sorted by (x, y, z) (F-9); *n_blocks (host)
 *             receives n; stats (host, may be NULL) receives the counters above (reading them
 *             synchronises the stream).
 * Synchronous with respect to the host for *n_blocks (the count is read back); device outputs are
 * complete when the stream reaches that point.  Errors: VOL_EINVAL (arguments), VOL_EDATA (a block
 * walk leaves the coordinate range (−2^20, 2^20) or is longer than 4096 blocks), VOL_ENOMEM (more
 * than max_blocks blocks: *n_blocks then holds the count reached, retry with a larger capacity; or
 * workspace too small), VOL_ECUDA.                                                                  */
vol_status vol_fuse(const float *depth, int32_t n_frames, const vol_camera *cam, const float *poses,
                    const vol_fusion_params *params, int64_t max_blocks, void *workspace, size_t workspace_bytes,
                    void *stream, int32_t *block_xyz, int32_t *first_frame, float *f, float *W,
                    int64_t *n_blocks, vol_fusion_stats *stats);

/* Continue a fusion (reading F-11; "New incoming data can be added at any time"): the n_prev
 * blocks prev_xyz [n_prev][3] with their prev_f, prev_W [n_prev][512] (host or device; e.g. the
 * outputs of an earlier call) are in the set before the first new frame (allocating frame −1) and are
 * updated by the new depth maps exactly as if all frames had been fused in one call — the output is
 * bit-identical to fusing the old and new frames together.  Other arguments as vol_fuse; max_blocks
 * counts the previous blocks too.  Errors as vol_fuse, plus VOL_EDATA when prev_xyz repeats a block. */
vol_status vol_fuse_incremental(const int32_t *prev_xyz, const float *prev_f, const float *prev_W, int64_t n_prev,
                                const float *depth, int32_t n_frames, const vol_camera *cam, const float *poses,
                                const vol_fusion_params *params, int64_t max_blocks, void *workspace,
                                size_t workspace_bytes, void *stream, int32_t *block_xyz, int32_t *first_frame,
                                float *f, float *W, int64_t *n_blocks, vol_fusion_stats *stats);

#ifdef __cplusplus
}
#endif
#endif /* HVG_VOL_H */
