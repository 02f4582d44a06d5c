/*
 * rdcnn_cuda.h -- C-ABI of the B200-native FitzHugh-Nagumo RD-CNN stepper.
 *
 * Drop-in boundary for the reference's time-stepping path.  Every entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj/include/rdcnn/):
 *
 *   rdcnn_params_from_gene   make_params<float>(Gene)          model.hpp:24-32
 *   rdcnn_sim_create         StepBuffers<float>(GridState)     kernels.hpp:22-38
 *   rdcnn_sim_upload         GridState<float> u/v planes        grid.hpp:31-53
 *   rdcnn_sim_init           init_center_square / full_random  init.hpp:20-48
 *   rdcnn_sim_init_image     init_from_image (typ=3)           init.hpp:51-64
 *   rdcnn_sim_advance        step() x n / run_timed()          kernels.hpp:233-259,
 *                                                               engine.hpp:98-106
 *   rdcnn_sim_download       bufs.front readback               engine.hpp:83-92
 *   rdcnn_checksum_f32/_f64  checksum(GridState<T>)            grid.hpp:101-116
 *   rdcnn_sim_create_f64     StepBuffers<double>               kernels.hpp:22-38
 *   rdcnn_init_*_host        init_* on host buffers            init.hpp:20-48
 *
 * Conventions: plain pointers and sizes only; status codes mirror the CLI
 * exit codes (rdcnn_cli.cpp:28-31): 0 ok, 1 invalid argument, 2 blow-up,
 * 3 CUDA/device failure.  Every non-zero status leaves a message in the
 * calling thread's rdcnn_last_error().  A handle owns its device buffers and
 * its CUDA stream; it may be used by one host thread at a time, distinct
 * handles are independent (reference SPEC.md:212).  No global mutable state.
 *
 * Host layout: row-major planes, index = i*cols + j, batch-major for batched
 * handles (grid g occupies [g*rows*cols, (g+1)*rows*cols)).
 */
#ifndef RDCNN_CUDA_H
#define RDCNN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RDCNN_ABI_VERSION 1

enum rdcnn_status {
  RDCNN_OK = 0,
  RDCNN_EINVAL = 1,
  RDCNN_EBLOWUP = 2,
  RDCNN_ECUDA = 3
};

enum rdcnn_mode {
  RDCNN_STRICT = 0, /* default: the reference's results bit for bit (every finite
                       value, the blow-up iteration).  fp32 launches use the
                       exactly-equal substitutions the genes allow (fused -4*c
                       tails, gated 2-op x/3, Dv == 1 product skipped; DESIGN.md
                       section 4); RDCNN_DIV3=3|2|u pins simpler instances. */
  RDCNN_FAST = 1    /* opt-in: FMA-contracted, not bit-exact; checked at the
                       reference tolerance after 10 steps (test_kernels.cpp:159-172)
                       and statistically to 10^4 steps (regime labels of the full
                       cfg4 sweep identical, cfg2 growth curve within 6.4e-5:
                       profiles/fast_mode_r02.json, tests/test_fast_mode_gpu.py) */
};

/* Gene narrowed to fp32 in kernel order (gene_to_vector, gene.hpp:39-41). */
typedef struct rdcnn_params_f32 {
  float dt, a, b, eps, c, du, dv;
} rdcnn_params_f32;

/* fp64 gene (make_params<double>, model.hpp:24-32: no narrowing). */
typedef struct rdcnn_params_f64 {
  double dt, a, b, eps, c, du, dv;
} rdcnn_params_f64;

typedef struct rdcnn_sim* rdcnn_sim_t;

int rdcnn_abi_version(void);
const char* rdcnn_last_error(void);
int rdcnn_device_count(int* n);

/* gene7 = {dt, a, b, eps, c, Du, Dv} as doubles; narrows each with T(x). */
void rdcnn_params_from_gene(const double gene7[7], rdcnn_params_f32* out);

/* rows, cols >= 3 (grid.hpp:49-52); batch >= 1 independent grids of the same
 * shape; device = CUDA ordinal; mode = rdcnn_mode. */
int rdcnn_sim_create(int rows, int cols, int batch, int device, int mode,
                     rdcnn_sim_t* out);
/* fp64 lattice (GridState<double>; the reference templates instantiate both
 * precisions, grid.hpp:13-28).  Strict mode only.  Use the *_f64 entry
 * points for its state and genes; the fp32 ones reject it. */
int rdcnn_sim_create_f64(int rows, int cols, int batch, int device,
                         rdcnn_sim_t* out);
/* 4 (fp32) or 8 (fp64). */
int rdcnn_sim_precision(rdcnn_sim_t sim, int* bytes);
void rdcnn_sim_destroy(rdcnn_sim_t sim);

/* n = 1 (shared gene) or n = batch (one gene per grid, sweep.hpp:296-309). */
int rdcnn_sim_set_params(rdcnn_sim_t sim, const rdcnn_params_f32* p, int n);
int rdcnn_sim_set_params_f64(rdcnn_sim_t sim, const rdcnn_params_f64* p, int n);

/* Synchronous host<->device copies of the current state (front buffer).
 * Pinned host memory gets full link bandwidth; pageable memory also works. */
int rdcnn_sim_upload(rdcnn_sim_t sim, const float* u, const float* v);
int rdcnn_sim_download(rdcnn_sim_t sim, float* u, float* v);
int rdcnn_sim_upload_f64(rdcnn_sim_t sim, const double* u, const double* v);
int rdcnn_sim_download_f64(rdcnn_sim_t sim, double* u, double* v);

/* Device-side initial states, bit-identical to the reference initialisers:
 * typ 1 = init_center_square, typ 2 = init_full_random (every grid of a
 * batch from the same seed, sweep.hpp:307 default).  */
int rdcnn_sim_init(rdcnn_sim_t sim, int typ, uint64_t seed);
/* typ 3: u = v = float(ka) * float(px/255.0) from an 8-bit rows x cols image
 * (image.hpp:283, init.hpp:51-64); one image for every grid of a batch. */
int rdcnn_sim_init_image(rdcnn_sim_t sim, const uint8_t* px, double ka);

/* Advance every grid by `steps` iterations (steps >= 0).  Returns
 * RDCNN_EBLOWUP if any grid produced a non-finite value; then
 * first_bad_iter[g] (array of batch entries, may be NULL) holds the 1-based
 * iteration within this call at which grid g first went non-finite, 0 for
 * grids that stayed finite.  A blown-up grid stops at that iteration: its
 * state is the state right after it (reference run_timed leaves bufs.front
 * there, engine.hpp:103-104); the other grids complete all steps. */
int rdcnn_sim_advance(rdcnn_sim_t sim, long steps, long* first_bad_iter);

/* Device time of the last advance (CUDA events on the handle's stream). */
int rdcnn_sim_elapsed_ms(rdcnn_sim_t sim, double* ms);
/* Kernel launches issued by the last advance (including blow-up replays). */
int rdcnn_sim_launch_count(rdcnn_sim_t sim, long* n);
/* Tuning: maximum time levels per launch (1, 2, 4 or 8; default 4) and the
 * rows per warp segment (0 = automatic). */
int rdcnn_sim_set_tuning(rdcnn_sim_t sim, int max_levels, int seg_rows);
/* Small single lattices (batch 1, fp32, cols 128 or 256, rows = C*R with
 * C, R <= 16 -- e.g. the reference's 256x256 default) advance in ONE launch
 * of a persistent 16-CTA thread-block cluster: state in registers, row
 * halos through shared memory and DSMEM, one cluster barrier per step,
 * exact per-step blow-up stop.  mode 0: automatic (default), 1: required
 * (advance fails with RDCNN_EINVAL when the shape does not fit), -1: off. */
int rdcnn_sim_set_persistent(rdcnn_sim_t sim, int mode);
/* Profiling: one K-level launch over the whole state with per-warp tracing;
 * host_trace receives {start ns, end ns, smid} per warp (globaltimer), cap
 * entries at most; *n_warps = warps launched.  Advances the state by
 * `levels` iterations. */
int rdcnn_sim_trace_launch(rdcnn_sim_t sim, int levels, unsigned long long* host_trace,
                           long long cap, long long* n_warps);
/* The handle's CUDA stream (cudaStream_t) for interop with other libraries. */
int rdcnn_sim_stream(rdcnn_sim_t sim, void** stream);
/* Device pointers of the current front planes (plane u, plane v; float or
 * double per rdcnn_sim_precision), for zero-copy interop; valid until the
 * next advance/destroy. */
int rdcnn_sim_device_state(rdcnn_sim_t sim, void** u, void** v);

/* ---- slab mode: one row slab of a larger torus, for multi-GPU runs -------
 * The slab owns rows [0, rows) of its shard and `ghost` halo rows above and
 * below.  Device layout per buffer: (rows + 2*ghost) rows, each row = u cols
 * then v cols (interleaved, so `ghost` rows of both planes are one
 * contiguous message).  The caller exchanges halos with its ring neighbours
 * between phases (NCCL send/recv, see paper_2102_10340_b200/slab.py):
 *   rdcnn_slab_step_boundary(k)   rows [0,ghost) and [rows-ghost,rows) -> back
 *   ... send back rows [0,ghost) up / [rows-ghost,rows) down, receive ghosts ...
 *   rdcnn_slab_step_interior(k)   rows [ghost, rows-ghost) -> back
 *   rdcnn_slab_swap()
 * k <= ghost levels per block.  `stream` is the cudaStream_t to launch on,
 * taken literally (0 = the legacy default stream; pass rdcnn_sim_stream()'s
 * value for the handle's own stream). */
int rdcnn_slab_create(int rows, int cols, int ghost, int device, int mode,
                      rdcnn_sim_t* out);
/* Initialise the slab as rows [row_offset, row_offset+rows) of a
 * global_rows x cols lattice built by init typ (1 or 2) from seed. */
int rdcnn_slab_init(rdcnn_sim_t sim, int typ, uint64_t seed, int global_rows,
                    int row_offset);
int rdcnn_slab_step_boundary(rdcnn_sim_t sim, int k, void* stream);
int rdcnn_slab_step_interior(rdcnn_sim_t sim, int k, void* stream);
int rdcnn_slab_swap(rdcnn_sim_t sim);
/* Device pointers (in floats) into the front (which=0) or back (which=1)
 * buffer: the first owned row and the first top-ghost row; row pitch is
 * 2*cols floats. */
int rdcnn_slab_rows_ptr(rdcnn_sim_t sim, int which, float** first_row,
                        float** first_ghost_row);
/* Any non-finite value stored so far (1) or not (0); *tag = launch tag. */
int rdcnn_slab_poll_blowup(rdcnn_sim_t sim, int* bad, unsigned* tag);

/* Native ring (no host work per block).  Rank 0 calls rdcnn_nccl_unique_id
 * and shares the 128 bytes with every rank (e.g. a torch.distributed
 * broadcast); each rank then attaches its slab.  world == 1 closes the ring
 * on itself (the torus row wrap as two device copies, no NCCL).  NCCL is
 * resolved at run time from the libnccl.so.2 already in the process. */
int rdcnn_nccl_unique_id(uint8_t id[128]);
int rdcnn_slab_attach_ring(rdcnn_sim_t sim, const uint8_t id[128], int rank,
                           int world);
/* NCCL ring: exchange the front buffer's edge rows into the ring's ghosts
 * (once, after initialising the slabs).  Peer ring: only completes the
 * state (the neighbours read it in place); barrier the ranks afterwards. */
int rdcnn_slab_fill_ghosts(rdcnn_sim_t sim);
/* Advance by `steps`.  Peer ring: one fused launch per block of k <= ghost
 * levels.  NCCL ring: per block, boundary kernel -> NCCL ring exchange on a
 * comm stream overlapped with the interior kernel.
 * On a non-finite value returns RDCNN_EBLOWUP with *first_bad = the first
 * iteration of the first bad block (block granularity). */
int rdcnn_slab_advance(rdcnn_sim_t sim, long steps, long* first_bad);

/* Fused peer ring (the default multi-GPU transport): the halo exchange runs
 * INSIDE the step kernel.  Per block, one launch computes every owned row;
 * the warps producing the first/last `ghost` rows stage the level-0 rows
 * beyond the slab straight from the ring neighbours' input buffers (peer
 * memory: CUDA IPC mappings over NVLink, or plain pointers when the
 * neighbour lives in the same process) and, when done, publish a
 * per-direction word with a release store ("my edge rows are written, and I
 * have finished reading yours"); the neighbours' edge warps acquire it.  No
 * NCCL, no exchange copies, no host work per block.
 *
 * Protocol: every rank exports its descriptor, the descriptors are shared
 * (e.g. torch.distributed all_gather_object), every rank attaches with its
 * ring neighbours' descriptors (prev = rank-1, next = rank+1 mod world; world
 * 1 passes its own), calls rdcnn_slab_fill_ghosts, and the ranks barrier once
 * before the first block.  All ranks must then run the same blocks.  Destroy
 * only after a barrier (neighbours read this slab's rows in place). */
typedef struct {
  uint8_t ipc[3][64];   /* cudaIpcMemHandle_t: buffer 0, buffer 1, sync words */
  uint64_t ptr[3];      /* the same allocations as device pointers (exporter's process) */
  int64_t pid;          /* exporting process */
  int32_t device, rows, cols, ghost;
  int32_t ipc_ok;       /* 0: IPC export failed (in-process rings only) */
} rdcnn_slab_peer_desc;
int rdcnn_slab_peer_export(rdcnn_sim_t sim, rdcnn_slab_peer_desc* out);
int rdcnn_slab_attach_peers(rdcnn_sim_t sim, int rank, int world,
                            const rdcnn_slab_peer_desc* prev,
                            const rdcnn_slab_peer_desc* next);
/* One fused block of k levels on `stream` (NULL: the handle's stream); for
 * drivers that interleave several in-process ranks on one stream.  The ring
 * must have been made ready (rdcnn_slab_fill_ghosts + a barrier). */
int rdcnn_slab_step_fused(rdcnn_sim_t sim, int k, void* stream);

/* Exact blow-up iteration for slab runs (engine.hpp:79 BlowUpError(iter+1)).
 * With the checkpoint on, the first rdcnn_slab_advance after the state was
 * set (upload/init), and then one advance every 2048 iterations
 * (RDCNN_CKPT_INTERVAL), keeps its input aside: the fused peer ring tees it
 * from the first block's own level-0 reads, the NCCL ring copies it.
 * rdcnn_slab_checkpoint_age gives the iterations from the checkpoint to the
 * start of the last advance; rdcnn_slab_restore makes the checkpoint the
 * front buffer again.  The ranks then agree on the first bad block (min over
 * ranks), restore, synchronise (no rank may start the re-advance while a
 * neighbour's buffer still holds the post-blow-up rows its peer reads would
 * pull), re-advance age + that block's first iteration - 1 steps and step
 * one level at a time until any rank flags -- see slab.py
 * SlabStepper.advance.  (Freezing every rank at the first flag instead
 * cannot work: a rank's neighbours learn of it one block later, ranks at
 * distance d only d blocks later, by when they have overwritten the state
 * the replay needs.) */
int rdcnn_slab_checkpoint_enable(rdcnn_sim_t sim, int on);
int rdcnn_slab_restore(rdcnn_sim_t sim);
int rdcnn_slab_checkpoint_age(rdcnn_sim_t sim, long* age);

/* ---- in-process multi-device ring ------------------------------------------
 * One global_rows x cols torus split into n row slabs in ONE process, slab r
 * on CUDA device devices[r] (entries may repeat: slabs sharing a GPU run
 * their blocks interleaved on one stream).  Slab r owns rows
 * [offset_r, offset_r + rows_r), rows_r = global_rows/n (+1 for the first
 * global_rows % n slabs), each >= 2*ghost.  The halo exchange is the fused
 * peer ring above (edge warps read the neighbours' rows in place over NVLink
 * peer access); one host thread per device drives its slabs; no NCCL, no
 * torch.distributed.  Replaces the row-band parallelism of
 * kern::step_parallel (kernels.hpp:153-174) across GPUs (the
 * devices[]/n_devices create of §8b).
 *
 * rdcnn_ring_advance reports the reference's exact iteration
 * (engine.hpp:79, BlowUpError(iter+1)) and leaves the post-blow-up state
 * (engine.hpp:103-104): the first block of each advance tees its input into
 * a per-slab checkpoint; on a flag every slab restores it, re-advances to
 * the first bad block and steps one level at a time.  With
 * rdcnn_ring_set_exact(ring, 0) it reports the first iteration of the first
 * bad block instead. */
typedef struct rdcnn_ring* rdcnn_ring_t;
int rdcnn_ring_create(int global_rows, int cols, const int* devices, int n_devices,
                      int ghost, int mode, rdcnn_ring_t* out);
void rdcnn_ring_destroy(rdcnn_ring_t ring);
/* Slab r's handle (owned by the ring; slab-mode entry points only), its
 * first global row, its row count and device.  Any output may be NULL. */
int rdcnn_ring_slab(rdcnn_ring_t ring, int r, rdcnn_sim_t* slab, int* row_offset,
                    int* rows, int* device);
int rdcnn_ring_set_params(rdcnn_ring_t ring, const rdcnn_params_f32* p);
/* Time levels per block: 1, 2, 4 or 8, at most ghost (default ghost). */
int rdcnn_ring_set_levels(rdcnn_ring_t ring, int max_levels);
int rdcnn_ring_set_exact(rdcnn_ring_t ring, int on);
/* typ 1 or 2 over the global lattice (init_center_square / init_full_random). */
int rdcnn_ring_init(rdcnn_ring_t ring, int typ, uint64_t seed);
/* Global row-major planes (global_rows*cols each), split by slab. */
int rdcnn_ring_upload(rdcnn_ring_t ring, const float* u, const float* v);
int rdcnn_ring_download(rdcnn_ring_t ring, float* u, float* v);
int rdcnn_ring_advance(rdcnn_ring_t ring, long steps, long* first_bad_iter);
/* Device time of the last advance: max over devices (CUDA events). */
int rdcnn_ring_elapsed_ms(rdcnn_ring_t ring, double* ms);
int rdcnn_ring_launch_count(rdcnn_ring_t ring, long* n);
/* Profiling: one block of `levels` on every slab with per-warp tracing;
 * out receives n entries of 6 words {slab, start ns, end ns, smid, ns the
 * warp waited for its neighbours' ready words, bytes it staged from peer
 * memory} (cap entries at most).  Advances the state by `levels`. */
int rdcnn_ring_trace_block(rdcnn_ring_t ring, int levels, unsigned long long* out,
                           long long cap, long long* n);

/* ---- snapshot store and analysis (batched sweeps, frames) ----------------
 * Replaces the host-side post-processing of sweep.hpp:48-112 and
 * frame.hpp:28-66 for device-resident runs.  A handle reserves `nframes`
 * slots of its u planes (all grids); rdcnn_sim_frame_capture copies the
 * current u planes into a slot (device to device).  Statistics are per grid
 * of the batch and exact: min/max, and the median as std::nth_element picks
 * it (rank floor(n/2)); counts of |double(x) - median| > threshold. */
int rdcnn_sim_frames_reserve(rdcnn_sim_t sim, int nframes);
int rdcnn_sim_frame_capture(rdcnn_sim_t sim, int slot);
/* u planes of all grids of one slot (float or double per precision). */
int rdcnn_sim_frame_download(rdcnn_sim_t sim, int slot, void* u);
int rdcnn_sim_frame_stats(rdcnn_sim_t sim, int slot, double* mins, double* maxs,
                          double* medians);
int rdcnn_sim_frame_active(rdcnn_sim_t sim, int slot, const double* medians,
                           const double* thresholds, long long* counts);
/* normalize_frame(_fixed): 8-bit rows*cols image of grid `grid`'s u plane in
 * `slot` (slot < 0: the current state), mapping [lo, hi] to 0..255 with
 * lround and clamping; 128 everywhere when hi <= lo. */
int rdcnn_sim_frame_normalize(rdcnn_sim_t sim, int slot, int grid, double lo,
                              double hi, uint8_t* out);
/* normalize_frame (frame.hpp:28-44): the same map with [lo, hi] = the
 * plane's own min/max, found by a whole-device reduction (finite planes);
 * *lo / *hi receive them (either may be NULL).  One call per processed image
 * (edge detection: init_image -> advance -> this). */
int rdcnn_sim_frame_normalize_auto(rdcnn_sim_t sim, int slot, int grid,
                                   uint8_t* out, double* lo, double* hi);

/* checksum (grid.hpp:100-126) of every grid of the current state, computed
 * on the device (one thread per grid: FNV-1a 64 over u's bytes then v's);
 * out[batch].  Equal to rdcnn_checksum_f32/_f64 of the downloaded planes. */
int rdcnn_sim_checksums(rdcnn_sim_t sim, uint64_t* out);

/* ---- host helpers (reference-identical, no device needed) --------------- */
int rdcnn_init_center_square_host(int rows, int cols, uint64_t seed, float* u,
                                  float* v);
int rdcnn_init_full_random_host(int rows, int cols, uint64_t seed, float* u,
                                float* v);
uint64_t rdcnn_checksum_f32(const float* u, const float* v, size_t cells);
int rdcnn_init_center_square_host_f64(int rows, int cols, uint64_t seed,
                                      double* u, double* v);
int rdcnn_init_full_random_host_f64(int rows, int cols, uint64_t seed, double* u,
                                    double* v);
uint64_t rdcnn_checksum_f64(const double* u, const double* v, size_t cells);

/* ---- self-test of the device arithmetic -------------------------------------
 * Sweeps all 2^32 fp32 bit patterns x on the device and counts those where
 * div3_rn(x) differs from IEEE x/3 (finite x) or is finite (non-finite x);
 * domain 0: every x, domain 1: x = u*u for every u; domain 2: the gated
 * two-op quotient of strict fp32 launches (fhn_stencil.cuh div3_rn2) inside
 * RN(c - x/3) at c = +-2^-90 and c = 1, every x >= +0 (0 mismatches).  */
int rdcnn_selftest_div3(int device, int domain, uint64_t* mismatches,
                        uint32_t* first_bad);
/* fp64: `samples` inputs spanning every exponent (and their squares) against
 * IEEE division; mismatches and the smallest failing bit pattern. */
int rdcnn_selftest_div3_f64(int device, uint64_t samples, uint64_t* mismatches,
                            uint64_t* first_bad);

#ifdef __cplusplus
}
#endif

#endif /* RDCNN_CUDA_H */
