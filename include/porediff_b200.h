/*
 * porediff_b200.h — C ABI of the B200-native FTCS reaction-diffusion step on
 * the 8^Dims sparse block grid (arXiv 2304.11165; reference `porediff`).
 *
 * The reference has no C ABI: its surface is the header-only C++ templates in
 * /root/reference/proj/include/porediff (SparseBlockGrid, FtcsStepper,
 * ftcs_step, run_simulation, total_mass, max_diffusivity). Every entry point
 * below replaces one of those members, cited as file:line. The C++ drop-in
 * headers in include/porediff/ (and the Python mirror in
 * paper_2304_11165_b200/porediff.py) are thin layers over exactly these calls.
 *
 * Conventions
 *  - All functions return an int status (PD_OK or one PD_E_* code); on error
 *    the message is retrievable with pd_last_error() (thread-local).
 *  - Codes 1..6 map one-to-one onto the reference exception taxonomy
 *    (errors.hpp:9-41); PD_E_CUDA signals a device/driver failure.
 *  - Chunk arrays are in ascending chunk linear index (the reference's
 *    traversal order, sparse_block_grid.hpp:283-293); a chunk's ordinal is its
 *    position in that order. Keys are int32[Dims] per chunk (x fastest).
 *    Masks are uint64[V/64] per chunk, bit (offset&63) of word (offset>>6)
 *    (sparse_block_grid.hpp:45-50). Offsets are x-fastest inside the chunk
 *    (sparse_block_grid.hpp:99-103). Slabs are V scalars per chunk,
 *    chunk-ordinal-major (sparse_block_grid.hpp:43,180-187).
 *  - scalar_bytes is 8 (double, the parity mode) or 4 (float).
 *  - Calls are synchronous at return (stream-ordered internally).
 */
#ifndef POREDIFF_B200_H
#define POREDIFF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PD_OK = 0,
    PD_E_INPUT = 1,     /* porediff::input_error     (errors.hpp:14) */
    PD_E_BOUNDS = 2,    /* porediff::bounds_error    (errors.hpp:19) */
    PD_E_PROPERTY = 3,  /* porediff::property_error  (errors.hpp:24) */
    PD_E_IO = 4,        /* porediff::io_error        (errors.hpp:29) */
    PD_E_STABILITY = 5, /* porediff::stability_error (errors.hpp:34) */
    PD_E_NUMERIC = 6,   /* porediff::numeric_error   (errors.hpp:39) */
    PD_E_CUDA = 7       /* device / driver failure (no reference analogue) */
};

enum { PD_REACTION_NONE = 0, PD_REACTION_SURFACE_SINK = 1, PD_REACTION_VOLUMETRIC = 2 };
enum { PD_BC_NO_FLUX = 0, PD_BC_DIRICHLET = 1 };

/* porediff::SimulationConfig + ReactionSpec + FaceBc (solver.hpp:38-97).
 * The volumetric time factor std::function is replaced by per-step factors
 * passed to pd_stepper_run (the host evaluates T(time_factor(s*dt)) as
 * solver.hpp:230-234 does). */
typedef struct pd_sim_config {
    double dt;
    int64_t n_steps;
    double b_low, b_up;            /* PhaseBand (geometry.hpp:43-46) */
    double boundary_epsilon;
    int32_t reaction_kind;         /* PD_REACTION_* */
    int32_t source_prop;           /* volumetric: property index of f(x) */
    double rate;                   /* surface sink k >= 0 */
    double band_half_width;        /* surface sink w > 0 */
    int32_t bc_type[6];            /* [axis*2+side], PD_BC_* */
    double bc_value[6];
    int64_t record_every;
    int32_t enforce_stability;
    int32_t has_time_factor;       /* volumetric: factors array supplied */
} pd_sim_config;

/* porediff::StepDiagnostics (solver.hpp:99-106) minus wall_seconds. */
typedef struct pd_diag {
    int64_t step;
    double time;
    double total_mass;
    double min_u;
    double max_u;
} pd_diag;

typedef struct pd_grid pd_grid;
typedef struct pd_stepper pd_stepper;

/* Last error message of the calling thread ("" if none). */
const char* pd_last_error(void);
/* Number of CUDA devices visible (0 on a CPU-only host; never errors). */
int pd_device_count(void);
/* Library build string (arch, precision modes). */
const char* pd_version(void);

/* ---- device sparse block grid (replaces SparseBlockGrid storage,
 *      sparse_block_grid.hpp:30-304) ---------------------------------------- */

/* Creates a device grid: geometry (grid_geometry.hpp:23-112), chunk keys and
 * masks in ascending linear order, n_props zero-initialised columns
 * (sparse_block_grid.hpp:58-73,268-281). `device` selects the CUDA device. */
int pd_grid_create(int dims, int scalar_bytes, const int64_t* size, const double* spacing,
                   int64_t n_chunks, const int32_t* keys, const uint64_t* masks,
                   int n_props, int device, pd_grid** out);
int pd_grid_destroy(pd_grid* g);
/* Host<->device copy of one logical property's slabs (n_chunks*V scalars).
 * Resolves the double-buffer column mapping like channel_data
 * (sparse_block_grid.hpp:180-187). */
int pd_grid_upload(pd_grid* g, int prop, const void* host_slabs);
int pd_grid_download(pd_grid* g, int prop, void* host_slabs);
/* Same, device pointer to device pointer (no host staging). */
int pd_grid_upload_device(pd_grid* g, int prop, const void* dev_slabs);
/* Runs all further work of this grid (and its steppers) on an external CUDA
 * stream (cudaStream_t, e.g. torch.cuda.current_stream()); NULL restores the
 * grid's own stream. Used to order the step with NCCL halo exchanges. */
int pd_grid_set_stream(pd_grid* g, void* stream);
/* Packs / unpacks the one-node face plane `face` (axis*2+side: side 0 = the
 * chunk's coordinate-0 plane, 1 = coordinate-7 plane) of n chunks (device
 * ordinal list) of one logical property to / from a contiguous device
 * buffer of n*V/8 scalars (halo exchange for z-slab sharding). */
int pd_grid_pack_face(pd_grid* g, int prop, const int32_t* dev_ordinals, int64_t n, int face,
                      void* dev_out);
int pd_grid_unpack_face(pd_grid* g, int prop, const int32_t* dev_ordinals, int64_t n, int face,
                        const void* dev_in);
/* O(1) column swap (sparse_block_grid.hpp:88-91). */
int pd_grid_swap(pd_grid* g, int prop_a, int prop_b);
/* Current physical column of a logical property (for host mirrors). */
int pd_grid_column_of(const pd_grid* g, int prop, int* column);
/* Raw device pointer of a logical property's slabs (stream-ordered use). */
int pd_grid_device_ptr(pd_grid* g, int prop, void** ptr);
int pd_grid_info(const pd_grid* g, int64_t* n_chunks, int64_t* active_nodes);
/* Chunk arrays back to the host (keys int32[n*dims], masks uint64[n*words]). */
int pd_grid_download_layout(const pd_grid* g, int32_t* keys, uint64_t* masks);

/* total_mass (solver.hpp:158-171): per-chunk sequential sum of active values,
 * pairwise_sum over ordinals (parallel.hpp:68-84), times cell volume. */
int pd_grid_total_mass(pd_grid* g, int prop, double* out);
/* max_diffusivity (solver.hpp:139-154): max over active nodes, 0 if none. */
int pd_grid_max_active(pd_grid* g, int prop, double* out);
/* min/max over active nodes with the reference's fold semantics
 * (snapshot_diagnostics, solver.hpp:282-301). */
int pd_grid_minmax_active(pd_grid* g, int prop, double* mn, double* mx);

/* ---- FTCS stepper (replaces FtcsStepper, solver.hpp:183-467) ------------- */

/* Validates the config (solver.hpp:304-331; messages identical) and builds the
 * per-run constants, neighbour table (solver.hpp:333-351) and the static
 * fluid / sink bitmasks derived from phi. prop_* are logical property
 * indices of phi, u, D, u_next (and the volumetric source, or -1). */
int pd_stepper_create(pd_grid* g, const pd_sim_config* cfg, int prop_phi, int prop_u,
                      int prop_d, int prop_next, pd_stepper** out);
int pd_stepper_destroy(pd_stepper* s);
/* Restricts the step (and its diagnostics partials) to the chunk ordinals
 * [begin, end) — the chunks a rank owns under z-slab sharding; the other
 * chunks of the grid are read-only ghost halos. Default: all chunks. */
int pd_stepper_set_range(pd_stepper* s, int64_t begin, int64_t end);
/* Asynchronous stepping for overlapped multi-GPU runs. Enqueues the step
 * kernel for the owned sub-range [begin, end) on the grid's stream (see
 * pd_grid_set_stream): reads logical u, writes logical u_next, no swap, no
 * diagnostics, no host synchronisation. Steps are stream-ordered; a
 * non-finite node is recorded on the device and reported by
 * pd_stepper_status. pd_stepper_swap then swaps u / u_next
 * (solver.hpp:262) once every sub-range of the step has been enqueued. */
int pd_stepper_enqueue(pd_stepper* s, int64_t step_index, int64_t begin, int64_t end, double factor);
int pd_stepper_swap(pd_stepper* s);
/* Synchronises and reports (then clears) a non-finite node of the enqueued
 * steps as numeric_error "non-finite value at step <step_number>, node (...)". */
int pd_stepper_status(pd_stepper* s, int64_t step_number);
/* Exact diagnostics across ranks: per-chunk sequential mass and
 * min / max of the current u over the owned range, into caller device arrays
 * of end-begin doubles (stream-ordered). Ranks own ascending ordinal ranges,
 * so their arrays concatenated in rank order are the global per-chunk
 * partials; pd_reduce_partials folds them exactly like total_mass /
 * snapshot_diagnostics (pairwise_sum over global ordinals, parallel.hpp:68-84;
 * left-preference min/max) into row = {mass*cell_volume, min, max}. */
int pd_stepper_partials(pd_stepper* s, double* dev_mass, double* dev_min, double* dev_max);
int pd_reduce_partials(pd_grid* g, const double* dev_mass, const double* dev_min, const double* dev_max, int64_t n,
                       double* row);
/* Strict stability bound for the grid's current D (solver.hpp:220-224). */
int pd_stepper_stability_bound(pd_stepper* s, double* out);
/* Step-0 row (snapshot_diagnostics, solver.hpp:282-301). */
int pd_stepper_snapshot_diag(pd_stepper* s, pd_diag* out);
/* Advances n_steps steps starting at global step index step0 (the state
 * entering is u at step0*dt), exactly as n calls of FtcsStepper::step
 * (solver.hpp:228-279): after each step u and u_next are swapped. A row is
 * produced for every step s (global, 0-based) with (s+1) % record_every == 0
 * or s+1 == final_step, where final_step is the caller's run length
 * (run_simulation's record rule, solver.hpp:512-517); rows receives at most
 * n_steps rows and *n_rows the count. factors: per-step source factor T(g(t))
 * (volumetric with time factor) or NULL (=1). On a non-finite node the
 * numeric_error message of solver.hpp:250-260 is returned and the grid is left
 * exactly as the reference leaves it (u = pre-step state, u_next written). */
int pd_stepper_run(pd_stepper* s, int64_t step0, int64_t n_steps, int64_t final_step,
                   const double* factors, pd_diag* rows, int64_t* n_rows);
/* One step from global step index step_index with a diagnostics row: exactly
 * FtcsStepper::step (solver.hpp:228-279) -- a non-finite node raises the
 * numeric_error, a non-finite total mass does NOT (that check belongs to
 * run_simulation, solver.hpp:514-515) and is returned in the row. factor:
 * the step's source factor T(g(t)) (1 without a time factor). */
int pd_stepper_step(pd_stepper* s, int64_t step_index, double factor, pd_diag* row);
/* ---- steady-state observers (north_star (3); no reference counterpart:
 * checked against a NumPy restatement, tests/test_observe.py) ------------- */
/* With on != 0, every row pd_stepper_run records also yields the convergence
 * norm max over active nodes of |u(step) - u(step-1)| (exact, order-free). */
int pd_stepper_set_convergence(pd_stepper* s, int on);
/* Convergence norms of the rows of the last pd_stepper_run (row order). */
int pd_stepper_convergence(const pd_stepper* s, double* out, int64_t cap, int64_t* n);
/* Diffusive flux of the current u through the plane between node layers
 * `layer` and `layer`+1 of `axis`: face_sum = sum over faces with both nodes
 * fluid of dh * (u_{L+1} - u_L), dh = (d_a + d_b) * T(0.5) (the reference's
 * face coefficient, solver.hpp:430-433), chunk sums folded pairwise in
 * ordinal order; flux = -face_sum / h_axis * (face area). */
int pd_stepper_plane_flux(pd_stepper* s, int axis, int64_t layer, double* face_sum, double* flux,
                          int64_t* faces);
/* Device time (ms, CUDA events) of the last pd_stepper_run's step kernels. */
int pd_stepper_last_ms(const pd_stepper* s, double* ms);
/* Launches of the step kernel so far (benchmark accounting). */
int pd_stepper_launch_count(const pd_stepper* s, int64_t* launches);

/* ---- geometry build on the device (north_star subsystem 1; reference
 *      build_sparse_grid geometry.hpp:148-176 on synthetic::SpherePacking
 *      synthetic.hpp:25-56 and the hash initial condition config.hpp:558) ---- */

/* Evaluates the sphere-pack fluid SDF (synthetic.hpp:32-40) at every node of
 * a cell-centred geometry, activates b_low+eps < phi < b_up-eps
 * (geometry.hpp:163-170), allocates chunks in ascending linear order and
 * fills phi. n_props columns; phi goes to prop_phi. The resulting grid is
 * bit-identical (keys, masks, phi) to build_sparse_grid on field_from(sdf). */
int pd_build_sphere_pack_grid(int scalar_bytes, const int64_t* size, const double* spacing,
                              const double* origin, int64_t n_spheres,
                              const double* centers /* n*3 */, const double* radii,
                              double b_low, double b_up, int n_props, int prop_phi,
                              int device, pd_grid** out);
/* Same, but only the chunks whose key lies in [chunk_lo, chunk_hi) per axis
 * are built (keys stay global): one shard of a decomposed domain, including
 * its ghost chunk layers. An empty region yields a grid with 0 chunks. */
int pd_build_sphere_pack_region(int scalar_bytes, const int64_t* size, const double* spacing,
                                const double* origin, int64_t n_spheres, const double* centers,
                                const double* radii, double b_low, double b_up,
                                const int64_t* chunk_lo, const int64_t* chunk_hi, int n_props,
                                int prop_phi, int device, pd_grid** out);
/* D = d_min + d_max/(1+exp(-(g1+g2*phi))) on active nodes
 * (populate_diffusion_channel, geometry.hpp:182-206). exp is the reference
 * libm's, restated bit for bit (csrc/pd_libm_exp.h), so D is the reference's
 * bits. */
int pd_grid_populate_diffusion(pd_grid* g, int prop_phi, int prop_d, double d_min,
                               double d_max, double gamma1, double gamma2);
/* smooth_diffusion_coefficient (geometry.hpp:182-187) for n host values of
 * phi, evaluated on `device` (same bits as the reference); validation as the
 * reference (input_error on d_min < 0 or d_max <= 0). */
int pd_smooth_diffusion_coefficients(const double* phi, int64_t n, double d_min, double d_max,
                                     double gamma1, double gamma2, double* out, int device);
/* u = hash_unit_value(seed, flat_index) on active nodes (config.hpp:558-564). */
int pd_grid_fill_hash(pd_grid* g, int prop, uint64_t seed);
/* Fills a property with a constant on active nodes. */
int pd_grid_fill_const(pd_grid* g, int prop, double value);

/* ---- FRAP / effective diffusivity support (reference analysis.hpp:147-225)
 * ------------------------------------------------------------------------ */

/* build_free_box_grid (analysis.hpp:147-153): every node of the box active,
 * chunks in ascending linear index; prop_phi (>= 0) is set to phi_value on
 * every node, all other properties zero. */
int pd_grid_create_full(int dims, int scalar_bytes, const int64_t* size, const double* spacing, int n_props,
                        int prop_phi, double phi_value, int device, pd_grid** out);
/* run_frap initial condition (analysis.hpp:179-186): u = (node in [lo, hi)) ?
 * 0 : 1 and D = T(d_molecular) on every active node; returns the active
 * counts inside the box (region) and overall (phase). */
int pd_grid_frap_init(pd_grid* g, int prop_u, int prop_d, const int64_t* lo, const int64_t* hi,
                      double d_molecular, int64_t* region, int64_t* phase);
/* The run_frap observer's region mass before the cell-volume factor
 * (analysis.hpp:211-216): sum of double(value) over the active nodes of
 * [lo, hi) in lexicographic order (axis 0 fastest), sequential, bit-exact. */
int pd_grid_box_sum(pd_grid* g, int prop, const int64_t* lo, const int64_t* hi, double* out);
/* Attaches that observer to a stepper: pd_stepper_run then also evaluates the
 * box sum of the post-step u at every recorded step; NULL detaches. */
int pd_stepper_set_region(pd_stepper* s, const int64_t* lo, const int64_t* hi);
/* Box sums of the rows produced by the last pd_stepper_run (row order). */
int pd_stepper_region_sums(const pd_stepper* s, double* out, int64_t cap, int64_t* n);

/* ---- level-set geometry stage (north_star subsystem 2; reference
 *      levelset.hpp:13-191, geometry.hpp:67-176, dense_field.hpp:12-82) ----- */

/* A dense field on the device: one T array over the box, axis 0 fastest
 * (DenseField<T,Dims>, dense_field.hpp:12-82; grid_geometry.hpp:73-77). */
typedef struct pd_field pd_field;

/* porediff::LevelSetOptions (levelset.hpp:13-20). */
typedef struct pd_levelset_options {
    int32_t max_iterations;       /* 1000 */
    double tolerance;             /* 1e-3: stop when max band update < tolerance*h */
    double pseudo_time_step;      /* 0.5 (units of h) */
    double band_width_for_error;  /* 4.0 (unused by the sweep) */
    double residual_band_width;   /* 6.0: |phi| <= width*h nodes monitored */
    int32_t rescale_initial;      /* 1: start from sign(phi)*h */
} pd_levelset_options;

/* porediff::RedistanceDiagnostics (levelset.hpp:22-26). */
typedef struct pd_redistance_diag {
    int32_t iterations;
    double final_residual;  /* last max band update, in units of h */
    int32_t converged;
} pd_redistance_diag;

int pd_field_create(int dims, int scalar_bytes, const int64_t* size, const double* spacing, const double* origin,
                    int device, pd_field** out);
int pd_field_destroy(pd_field* f);
int pd_field_upload(pd_field* f, const void* host_values);
/* Same from device memory (e.g. a level set computed by another library). */
int pd_field_upload_device(pd_field* f, const void* dev_values);
int pd_field_download(pd_field* f, void* host_values);
int pd_field_device_ptr(pd_field* f, void** ptr);
/* mask_to_indicator (geometry.hpp:67-77): bits (one byte per voxel, axis 0
 * fastest) -> +1 / -1. */
int pd_field_from_mask(pd_field* f, const uint8_t* host_bits, int64_t n_bits);
/* filter_thin_features (geometry.hpp:121-142): opening of the positive phase
 * by a cubic window of min_thickness_cells nodes per axis, in place. */
int pd_field_filter_thin(pd_field* f, int min_thickness_cells);
/* sussman_redistance (levelset.hpp:115-191), in place; bit-exact sweeps and
 * stopping rule. */
int pd_field_redistance(pd_field* f, const pd_levelset_options* opts, pd_redistance_diag* out);
/* build_sparse_grid (geometry.hpp:148-176) from a device level set: a node is
 * active iff T(b_low)+eps < phi < T(b_up)-eps; chunks in ascending linear
 * index; phi copied into prop_phi, other properties zero. */
int pd_build_grid_from_field(const pd_field* f, double b_low, double b_up, int n_props, int prop_phi,
                             pd_grid** out);

/* ---- snapshots (reference snapshot.hpp:195-348) --------
 * Byte-identical "SBGR" (sparse grid) and "SBGD" (dense field) containers,
 * streamed from / to the device in batches through pinned staging buffers.
 * I/O failures are PD_E_IO with the reference's messages. */

/* SnapshotInfo (snapshot.hpp:41-50); property names come back as
 * consecutive NUL-terminated strings in names_buf. */
typedef struct pd_snapshot_info {
    char magic[5];  /* "SBGD" or "SBGR" */
    uint32_t version, scalar_bits, dims;
    uint64_t size[3];
    double spacing[3], origin[3];
    uint32_t n_properties;
} pd_snapshot_info;

/* write_sparse_snapshot: names in registration order (one per property),
 * origin[dims] (the device grid keeps no origin). Payloads are written in
 * registration order regardless of u/u_next swaps. */
int pd_grid_write_snapshot(pd_grid* g, const char* path, const char* const* names, int n_names,
                           const double* origin);
/* read_sparse_snapshot for the given rank and scalar width: creates the
 * device grid; origin[dims] and the names are returned. */
int pd_grid_read_snapshot(const char* path, int dims, int scalar_bytes, int device, pd_grid** out, double* origin,
                          char* names_buf, size_t names_cap, int* n_names);
int pd_field_write_snapshot(pd_field* f, const char* path);
int pd_field_read_snapshot(const char* path, int dims, int scalar_bytes, int device, pd_field** out);
/* peek_snapshot: header only. */
int pd_peek_snapshot(const char* path, pd_snapshot_info* info, char* names_buf, size_t names_cap);

/* Work per z chunk layer of a sphere-pack domain without building it
 * (allocated chunks and active nodes per layer, cc[2] entries each; either
 * output may be NULL): for work-balanced z-slab cuts. */
int pd_sphere_pack_layer_work(int scalar_bytes, const int64_t* size, const double* spacing, const double* origin,
                              int64_t n_spheres, const double* centers, const double* radii, double b_low,
                              double b_up, int device, int64_t* chunks_per_layer, int64_t* active_per_layer);
/* Same, plus the fully active chunks per layer (the candidates for the march
 * kernels' cheaper uniform path): the per-layer step cost model of the
 * cost-weighted slab cuts (shard.py). */
int pd_sphere_pack_layer_cost(int scalar_bytes, const int64_t* size, const double* spacing, const double* origin,
                              int64_t n_spheres, const double* centers, const double* radii, double b_low,
                              double b_up, int device, int64_t* chunks_per_layer, int64_t* active_per_layer,
                              int64_t* full_per_layer);

/* ---- fused multi-GPU halo exchange over peer memory (
 * pd_peer.cu) ---------------------------------------------------------------
 * Replaces the pack -> NCCL send/recv -> unpack exchange (pd_grid_pack_face /
 * pd_grid_unpack_face) for 3-D FP64 z-slab shards: the step kernel stores
 * each boundary chunk's new z=0 (side 0, lower neighbour) or z=7 (side 1,
 * upper neighbour) plane straight into the neighbour's ghost chunk, and
 * per-neighbour step counters in peer memory order the steps (wait before a
 * step, signal after it). Across processes the neighbour's columns and
 * counters are mapped with CUDA IPC (pd_grid_make_shareable,
 * pd_grid_ipc_handles, pd_stepper_sync_ipc_handle, pd_ipc_open); within one
 * process the raw pointers are passed. */
int pd_grid_make_shareable(pd_grid* g);            /* columns -> cudaMalloc (IPC-exportable) */
int pd_grid_ipc_handles(pd_grid* g, void* out);    /* n_props handles of pd_ipc_handle_size() bytes */
int pd_grid_column_ptrs(pd_grid* g, void** out);   /* n_props physical column pointers */
int pd_ipc_handle_size(void);
int pd_ipc_open(const void* handle, int device, void** ptr);
int pd_ipc_close(void* ptr, int device);
/* the stepper's two step-counter words ([0] raised by the lower neighbour,
 * [1] by the upper one), created on first use */
int pd_stepper_sync_words(pd_stepper* s, void** ptr);
int pd_stepper_sync_ipc_handle(pd_stepper* s, void* out);
/* side 0 = lower, 1 = upper neighbour: its physical column pointers (n_cols =
 * n_props, same property order), its counter words, and the n pairs (own
 * boundary chunk ordinal -> neighbour's ghost chunk ordinal). From then on
 * every step of pd_stepper_run / pd_stepper_enqueue (whole owned range) waits,
 * pushes and signals. peer_sync NULL removes the side. */
int pd_stepper_set_peer(pd_stepper* s, int side, void* const* peer_cols, int n_cols, void* peer_sync,
                        const int32_t* src_ords, const int32_t* dst_ords, int64_t n);
/* zero the own counters and the step epoch (all ranks, then a host barrier,
 * before the first exchanged step) */
/* Time the fused exchange's per-step wait spent blocked on the neighbours'
 * step counters (total ns and number of waits since the last reset): the
 * load imbalance between slabs (bench.py reports it per rank). */
int pd_stepper_peer_stats(pd_stepper* s, uint64_t* wait_ns, int64_t* waits);
int pd_stepper_peer_reset(pd_stepper* s);

/* ---- VTK export (reference vtk.hpp:57-143, scalar_text.hpp:20-28; SURVEY
 * §8f row 4) ---------------------------------------------------------------
 * Legacy ASCII STRUCTURED_POINTS files, byte-identical to the reference's
 * write_vtk: the text of every node is produced on the device by an exact
 * "%.17g" / "%.9g" formatter and streamed to the file in batches. */

/* format_scalar (scalar_text.hpp:20-28): the text the device formatter
 * produces for v ("%.17g" when scalar_bytes is 8, "%.9g" of the float value
 * when 4, "nan" for any NaN), NUL-terminated; cap >= 26 always suffices. */
int pd_format_scalar(double v, int scalar_bytes, char* buf, size_t cap, int* len);
/* write_vtk (vtk.hpp:57-111) of a dense dataset: n_arrays scalar arrays of
 * node_count values (scalar_bytes each; host or device pointers) and an
 * optional int32 mask array (same residency), lattice size/spacing/origin of
 * `dims` entries (2-D lattices get a third extent of 1). Names are checked
 * like the reference (empty, whitespace, duplicates; PD_E_INPUT). */
int pd_write_vtk(const char* path, const char* title, int dims, const int64_t* size, const double* spacing,
                 const double* origin, int scalar_bytes, int n_arrays, const char* const* names,
                 const void* const* values, int values_on_device, const int32_t* mask, int device);
/* write_vtk(vtk_from_sparse(grid, channels, blank)) (vtk.hpp:115-143) fused on
 * the device: logical properties props[0..n_sel) written under `names`,
 * inactive nodes print `blank` (cast to the grid scalar), then the mask array
 * (1 = active). */
int pd_grid_write_vtk(pd_grid* g, const char* path, const char* title, const int* props, const char* const* names,
                      int n_sel, double blank, const double* origin);
/* vtk_from_sparse (vtk.hpp:115-143) arrays: property `prop` densified onto
 * the full lattice (x fastest; inactive = blank) and/or the int32 mask, into
 * host buffers (either may be NULL). */
int pd_grid_densify(pd_grid* g, int prop, double blank, void* host_values, int32_t* host_mask);

#ifdef __cplusplus
}
#endif
#endif /* POREDIFF_B200_H */
