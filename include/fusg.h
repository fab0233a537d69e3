/* fusg.h — C-ABI of the B200-native volume-potential harmonic solver (arXiv 2011.03009).
 *
 * Drop-in boundary for the reference's hot path (the public headers under
 * /root/reference/proj/include/fus/).
 * Plain C types only: fields are interleaved complex128 (re, im) arrays, x fastest,
 * index = ix + Nx*(iy + Ny*iz) (include/fus/grid.hpp:41-43).  Functions whose pointer
 * arguments are named *_dev take device pointers (CUDA global memory); *_host take host
 * pointers.  Every function returns fusg_status; exceptions never cross this boundary and
 * fusg_last_error() returns the thread-local message of the last failure.  Error classes
 * mirror the reference's exception types (std::invalid_argument, std::out_of_range,
 * std::runtime_error).
 *
 * Each entry cites the reference interface it replaces.
 */
#ifndef FUSG_H_
#define FUSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fusg_status {
  FUSG_OK = 0,
  FUSG_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  FUSG_OUT_OF_RANGE = 2,     /* std::out_of_range     */
  FUSG_RUNTIME = 3,          /* std::runtime_error    */
  FUSG_CUDA = 4,             /* CUDA runtime failure  */
  FUSG_NCCL = 5,             /* NCCL failure          */
  FUSG_OOM = 6,              /* device allocation     */
  FUSG_NOT_CONVERGED = 7     /* fus::ConvergenceError (GMRES; a std::runtime_error) */
} fusg_status;

/* VoxelGrid (include/fus/grid.hpp:30-50): covered box, spacing, voxel counts, harmonic. */
typedef struct fusg_grid {
  double lo[3];
  double hi[3];
  double dx;
  int32_t dims[3];
  int32_t harmonic;
} fusg_grid;

/* Wavenumber (include/fus/medium.hpp:26-30). */
typedef struct fusg_wavenumber {
  double k_re, k_im;
  int32_t harmonic;
  double omega;
} fusg_wavenumber;

/* Medium (include/fus/medium.hpp:12-23), name omitted. */
typedef struct fusg_medium {
  double rho0, c0, beta, alpha0, eta;
} fusg_medium;

/* BowlTransducer (include/fus/transducer.hpp:15-28); points_host is n_points x 3. */
typedef struct fusg_bowl {
  double f0, focal_length, outer_radius, power;
  int32_t n_points;
  const double* points_host;
} fusg_bowl;

/* StageTiming (include/fus/cascade.hpp:25-32) plus the stages the reference leaves
 * untimed (p1 evaluation, rhs assembly); seconds, measured with CUDA events. */
typedef struct fusg_stage_timing {
  int32_t harmonic;
  uint64_t voxels;
  double meshing_s, interpolation_s, kernel_s, potential_s;
  double p1_s, rhs_s;
} fusg_stage_timing;

typedef struct fusg_ctx fusg_ctx;       /* one CUDA device + stream + workspace */
typedef struct fusg_kernel fusg_kernel; /* GreenKernel: cached octant spectrum */

const char* fusg_last_error(void);
const char* fusg_version(void);

/* ---------------------------------------------------------------- host arithmetic
 * Bit-exact restatements (compiled without FMA contraction, like the reference). */

/* make_grid (src/grid.cpp:12-34); anchor_or_null may be NULL. */
fusg_status fusg_make_grid(const double req_lo[3], const double req_hi[3], double dx,
                           int32_t harmonic, const double* anchor_or_null, fusg_grid* out);
/* complex_wavenumber (src/medium.cpp:31-45). */
fusg_status fusg_complex_wavenumber(const fusg_medium* m, double f0, int32_t n,
                                    fusg_wavenumber* out);
/* self_weight / equivalent_sphere_radius (src/potential.cpp:55-70). */
fusg_status fusg_self_weight(const fusg_wavenumber* k, double dx, double out[2]);
double fusg_equivalent_sphere_radius(double dx);
/* next_fast_size (src/potential.cpp:36-43) and the padded box the device path uses. */
int32_t fusg_next_fast_size(int32_t n);
fusg_status fusg_padded_dims(const fusg_grid* g, int32_t pad_small_primes, int32_t out[3]);
/* Padded lengths with compile-time-planned kernels (conv = 0: x / y passes, 1: z pass C),
 * ascending; writes up to cap of them to out and returns how many exist. */
int32_t fusg_static_lengths(int32_t conv, int32_t* out, int32_t cap);
/* distribute_points (src/transducer.cpp:22-70): out_host is n_points x 3. */
fusg_status fusg_distribute_points(double focal_length, double outer_radius, int32_t n_points,
                                   double* out_host);
/* plan_nested_meshes (src/grid.cpp:81-112) / plan_single_mesh (src/cascade.cpp:109-118).
 * out_grids[i] is the grid of harmonic i+2 (n_harmonics-1 entries); domains_lo/hi are the
 * planned domains D_i (3 doubles each); reference receives the fine reference mesh. */
fusg_status fusg_plan_nested_meshes(const fusg_bowl* t, const fusg_medium* m, double d,
                                    int32_t n_w, int32_t n_harmonics, double width_scale,
                                    int32_t single_mesh, fusg_grid* out_grids,
                                    double* domains_lo, double* domains_hi,
                                    fusg_grid* reference, double* w_out);
/* rhs coefficient beta omega^2 n^2 / (2 rho0 c0^4) (src/cascade.cpp:32-34). */
double fusg_rhs_coefficient(const fusg_medium* m, double omega, int32_t n);
/* Seeded test input (tests/acceptance.cpp:30-36): std::mt19937 + U(-1,1), re then im. */
fusg_status fusg_random_vector(int64_t n, uint32_t seed, double* out_host);

/* ---------------------------------------------------------------- device context */
fusg_status fusg_ctx_create(int32_t device, fusg_ctx** out);
fusg_status fusg_ctx_destroy(fusg_ctx* ctx);
/* The context's CUDA stream (cudaStream_t); NULL stream arguments below mean this one. */
void* fusg_ctx_stream(fusg_ctx* ctx);
fusg_status fusg_ctx_synchronize(fusg_ctx* ctx);
/* Number of kernels of this library launched on the context so far. */
uint64_t fusg_ctx_launch_count(fusg_ctx* ctx);

/* ---------------------------------------------------------------- volume potential
 * GreenKernel (include/fus/potential.hpp:28-48, src/potential.cpp:72-159). */

/* GreenKernel::GreenKernel (src/potential.cpp:72-118): builds the octant spectrum on the
 * device. The padded box is the smallest {2,3,5,7}-smooth size >= 2N-1 per axis (or
 * next_fast_size(2N) with pad_small_primes): the same discrete operator (offset_of,
 * src/potential.cpp:88-94) as the reference's 2N box. */
fusg_status fusg_kernel_create(fusg_ctx* ctx, const fusg_grid* grid, const fusg_wavenumber* k,
                               int32_t pad_small_primes, fusg_kernel** out);
fusg_status fusg_kernel_destroy(fusg_kernel* kernel);
fusg_status fusg_kernel_padded(const fusg_kernel* kernel, int32_t out[3]);
/* Device bytes held by the kernel (spectrum + apply workspace). */
uint64_t fusg_kernel_device_bytes(const fusg_kernel* kernel);
/* GreenKernel::apply (src/potential.cpp:120-151) times `scale` (1 for apply, -1 for the
 * cascade's p_n = -apply(f_n), src/cascade.cpp:100). f_dev/u_dev: N complex128 on device;
 * u_dev must not alias f_dev. stream may be NULL (context stream). Asynchronous. */
fusg_status fusg_kernel_apply(fusg_kernel* kernel, const double* f_dev, double* u_dev,
                              double scale, void* stream);
/* Measurement hook: `reps` back-to-back applies on the context stream with CUDA events
 * between the five passes (A: fwd x, B: fwd y, C: fwd z * K^ inv z, D: inv y, E: inv x);
 * pass_ms receives the mean duration of each pass. */
fusg_status fusg_kernel_apply_timed(fusg_kernel* kernel, const double* f_dev, double* u_dev,
                                    double scale, int32_t reps, double pass_ms[5]);
/* Host-vector drop-in for GreenKernel::apply(const VectorXcd&): host->device copy, apply,
 * device->host copy, synchronous. */
fusg_status fusg_kernel_apply_host(fusg_kernel* kernel, const double* f_host, double* u_host,
                                   double scale);

/* ---------------------------------------------------------------- incident field
 * Equal-area monopole (Rayleigh-type) sum amp * sum_i e^{ikd}/(4 pi d)
 * (src/transducer.cpp:107-132,179-196). Fails with FUSG_INVALID_ARGUMENT when an
 * evaluation point coincides with a source (d < 1e-12, :112-113). */
fusg_status fusg_monopole_grid(fusg_ctx* ctx, const double* src_host, int32_t n_src,
                               const fusg_grid* grid, double k_re, double k_im, double amp,
                               double* out_dev, void* stream);
/* The z-slab [z0, z0 + nz) of fusg_monopole_grid's field (Nx * Ny * nz values, bitwise the
 * same planes): the multi-GPU p1 shards the incident field by z-planes with no collective
 * (SURVEY.md 8(e)); each rank evaluates its own slab. */
fusg_status fusg_monopole_grid_zslab(fusg_ctx* ctx, const double* src_host, int32_t n_src,
                                     const fusg_grid* grid, int32_t z0, int32_t nz, double k_re,
                                     double k_im, double amp, double* out_dev, void* stream);
fusg_status fusg_monopole_points(fusg_ctx* ctx, const double* src_host, int32_t n_src,
                                 const double* pts_dev, int64_t n_pts, double k_re, double k_im,
                                 double amp, double* out_dev, void* stream);
/* evaluate_potential_at (src/potential.cpp:161-201): the volume potential of the device field
 * f_dev on `grid` at n_pts arbitrary host points (n_pts x 3), O(N M): sum over voxels with
 * f != 0 of vol G(r) f, self_weight f when r < 1e-9 dx. Deterministic (fixed-order partial
 * sums); out_host receives n_pts complex128 values. */
fusg_status fusg_evaluate_potential_at(fusg_ctx* ctx, const fusg_grid* grid, const fusg_wavenumber* k,
                                       const double* f_dev, const double* pts_host, int64_t n_pts,
                                       double* out_host);
/* shrink_domain_by_threshold (src/grid.cpp:114-139): index box [lo, hi] of the voxels with
 * |f| >= max|f| 10^q0 (q0 >= 0: the maximum only); the DomainBox is lo + idx dx,
 * lo + (hi + 1) dx. FUSG_INVALID_ARGUMENT for an identically zero field. */
fusg_status fusg_field_threshold_box(fusg_ctx* ctx, const fusg_grid* grid, const double* f_dev, double q0,
                                     int32_t lo_idx[3], int32_t hi_idx[3], double* max_abs_out);
/* localisedness_map (src/analysis.cpp:80-90): q_dev[i] = log10(|f_i| / max|f|), -inf where f_i = 0. */
fusg_status fusg_localisedness_map(fusg_ctx* ctx, const double* f_dev, int64_t count, double* q_dev);
/* radiated_power (src/transducer.cpp:134-155): deterministic fixed-order reduction. */
fusg_status fusg_radiated_power(fusg_ctx* ctx, const double* src_host, int32_t n_src,
                                double x_disc, double R, double k_re, double k_im, double amp,
                                double rho0, double c0, int32_t n_r, int32_t n_theta,
                                double* out_host);

/* ---------------------------------------------------------------- source / transfer */
/* rhs_source (src/cascade.cpp:21-40): out = coeff * sum_{m=1}^{n-1} p_m p_{n-m};
 * lower_dev holds n-1 device pointers (p_1 .. p_{n-1}), each `count` complex128. */
fusg_status fusg_rhs_source(fusg_ctx* ctx, int32_t n, const double* const* lower_dev,
                            int64_t count, const fusg_medium* m, double omega, double* out_dev,
                            void* stream);
/* The paper's full quadratic source (Eq. cascade_1) truncated at M harmonics:
 * out = coeff * [sum_{m=1}^{n-1} p_m p_{n-m} + 2 sum_{m=n+1}^{M} p_m conj(p_{m-n})], coeff as
 * fusg_rhs_source. fields_dev holds M device pointers p_1 .. p_M (p_n, entry n-1, is read only
 * through p_{2n} conj(p_n), so it may be null when 2n > M). M = n-1 is bitwise fusg_rhs_source. The reference keeps only the first
 * sum (src/cascade.cpp:36-39); this entry serves iterated sweeps. Parity: numpy restatement. */
fusg_status fusg_rhs_source_full(fusg_ctx* ctx, int32_t n, const double* const* fields_dev, int32_t M,
                                 int64_t count, const fusg_medium* m, double omega, double* out_dev,
                                 void* stream);
/* interpolate (src/grid.cpp:141-195): trilinear transfer onto target voxel centres. */
fusg_status fusg_interpolate(fusg_ctx* ctx, const fusg_grid* src, const double* f_dev,
                             const fusg_grid* target, double* out_dev, void* stream);
/* z-slab transfer for the multi-GPU cascade: target planes [tz0, tz0 + tnz)
 * from source planes [sz0, sz0 + snz) held in f_slab_dev (a source z-slab with its halo);
 * bitwise the same values as fusg_interpolate.  fusg_interpolate_source_planes gives the
 * source plane range [z_lo, z_hi] a target slab reads (nested grids: its own planes plus a
 * one-plane halo).  FUSG_INVALID_ARGUMENT when the slab lacks a needed plane. */
fusg_status fusg_interpolate_source_planes(const fusg_grid* src, const fusg_grid* target, int32_t tz0,
                                           int32_t tnz, int32_t* z_lo, int32_t* z_hi);
fusg_status fusg_interpolate_zslab(fusg_ctx* ctx, const fusg_grid* src, int32_t sz0, int32_t snz,
                                   const double* f_slab_dev, const fusg_grid* target, int32_t tz0, int32_t tnz,
                                   double* out_dev, void* stream);

/* ---------------------------------------------------------------- recursion
 * run_cascade (src/cascade.cpp:42-107), device resident. grids[i] is the planned grid of
 * harmonic i+2; out_dev[n] receives p_{n+1} (p_1 lives on grids[0]) and must hold
 * grids[max(n-1,0)].count complex128. timings has n_harmonics-1 rows (harmonics 2..n). */
typedef struct fusg_cascade_desc {
  fusg_medium medium;
  fusg_bowl transducer;
  const fusg_grid* grids;
  int32_t n_harmonics;
  int32_t recompute_p1_each_grid;
  int32_t pad_small_primes;
} fusg_cascade_desc;
fusg_status fusg_run_cascade(fusg_ctx* ctx, const fusg_cascade_desc* desc, double* const* out_dev,
                             fusg_stage_timing* timings, double* source_normalization);

/* ---------------------------------------------------------------- VIE mode
 * SURVEY.md 8(f) rank 2 (src/vie.cpp). Fields are N complex128 device vectors on the kernel's
 * grid; a medium map is N interleaved (c, beta) doubles (the raster order, x fastest). */
/* MediumMap::wavenumber_contrast (src/vie.cpp:11-23): out = k_n(x)^2 - kbar_n^2 with
 * k_n(x) = (n omega / c(x), Im kbar_n) where c != background c0, else 0. map_dev: device map. */
fusg_status fusg_vie_contrast(fusg_ctx* ctx, const double* map_dev, int64_t count, const fusg_medium* background,
                              double f0, int32_t n, double* out_dev, void* stream);
/* vie_operator_apply (src/vie.cpp:133-139): out = p - V[contrast .* p]. */
fusg_status fusg_vie_operator_apply(fusg_kernel* kernel, const double* contrast_dev, const double* p_dev,
                                    double* out_dev, void* stream);
/* gmres (src/vie.cpp:141-236) on device vectors with a caller operator: op(user, in, out)
 * computes out = A in (device pointers, N complex128) and returns a status. x_dev receives the
 * solution; the relative-residual history goes to history_host (up to history_capacity
 * entries; history_len = full length). FUSG_NOT_CONVERGED past max_iter (history filled). */
typedef fusg_status (*fusg_operator_fn)(void* user, const double* in_dev, double* out_dev);
fusg_status fusg_gmres(fusg_ctx* ctx, fusg_operator_fn op, void* user, const double* rhs_dev, int64_t count,
                       double tol, int32_t max_iter, int32_t restart, double* x_dev, double* history_host,
                       int32_t history_capacity, int32_t* history_len, int32_t* iterations);
/* solve_vie (src/vie.cpp:238-242): (I - V[contrast .]) x = rhs by restarted GMRES. */
fusg_status fusg_solve_vie(fusg_kernel* kernel, const double* rhs_dev, const double* contrast_dev, double tol,
                           int32_t max_iter, int32_t restart, double* x_dev, double* history_host,
                           int32_t history_capacity, int32_t* history_len, int32_t* iterations);
/* VieConfig (include/fus/vie.hpp:75-79). */
typedef struct fusg_vie_config {
  double tol;
  int32_t max_iter, restart;
} fusg_vie_config;
/* run_cascade_inhomogeneous (src/vie.cpp:244-323): the master map (map_grid, map_host) is
 * resampled onto every harmonic's grid; background supplies the wavenumbers and the source
 * field. out_dev[n-1] receives p_n; timings[i-2] carries harmonic and voxels. */
fusg_status fusg_run_cascade_inhomogeneous(fusg_ctx* ctx, const fusg_cascade_desc* desc, const fusg_grid* map_grid,
                                           const double* map_host, const fusg_medium* background,
                                           const fusg_vie_config* vie, double* const* out_dev,
                                           fusg_stage_timing* timings, double* source_normalization);
/* Device-to-device copy on the context stream, synchronous (for caller-supplied operators). */
fusg_status fusg_device_copy(fusg_ctx* ctx, void* dst_dev, const void* src_dev, uint64_t bytes);

/* ---------------------------------------------------------------- slab sharding
 * rank r of G owns z-planes [z0, z0+nz) of f and u (ragged split: the first
 * N mod G ranks take one extra plane) and spectral kx columns [x0, x0+nx) of the padded box.
 * The apply transposes z-slab -> x-slab after the forward x pass and back before the inverse
 * x pass (one all-to-all each way). The kernel spectrum is held per x-slab: a rank keeps only
 * the folded octant rows its kx columns need (fusg_kernel_octant_rows). */
fusg_status fusg_slab_range(int32_t n, int32_t nranks, int32_t rank, int32_t* begin, int32_t* count);
/* Exchange plan of rank `rank` (arrays of nranks, complex128 element offsets/counts):
 * a_off/a_cnt[q]: block of A_r [Px][nz_r][Ny] holding rank q's kx columns (sent to q in the
 * forward transpose, received from q in the inverse one); r_off/r_cnt[p]: block of the staging
 * buffer [p][nx_r][nz_p][Ny] received from p (forward) / sent to p (inverse). Host only. */
fusg_status fusg_slab_exchange_plan(const fusg_grid* global_grid, int32_t nranks, int32_t rank,
                                    int64_t* a_off, int64_t* a_cnt, int64_t* r_off, int64_t* r_cnt);
/* NCCL transport: one process per GPU. Rank 0 creates the id; every rank attaches with it. */
fusg_status fusg_nccl_unique_id(uint8_t id[128]);
fusg_status fusg_ctx_attach_nccl(fusg_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[128]);
/* GreenKernel for rank `rank` of an nranks-way decomposition of the GLOBAL grid. */
fusg_status fusg_kernel_create_slab(fusg_ctx* ctx, const fusg_grid* global_grid,
                                    const fusg_wavenumber* k, int32_t pad_small_primes,
                                    int32_t nranks, int32_t rank, fusg_kernel** out);
/* Folded kx rows [kf0, kf0 + knf) of the octant spectrum this kernel holds (unsharded: 0 and
 * Px/2 + 1; x-slab kernels: the fold of their kx columns). */
fusg_status fusg_kernel_octant_rows(const fusg_kernel* kernel, int32_t* kf0, int32_t* knf);
fusg_status fusg_kernel_slab(const fusg_kernel* kernel, int32_t* z0, int32_t* nz, int32_t* x0,
                             int32_t* nx);
/* This rank's apply: f_dev/u_dev are its z-slab [nz][Ny][Nx]; collective over the context's
 * NCCL communicator (all ranks call it). */
fusg_status fusg_kernel_apply_slab(fusg_kernel* kernel, const double* f_dev, double* u_dev,
                                   double scale, void* stream);
/* Loopback transport: all ranks of one decomposition in this process on one device (same
 * context), exchanging by device copies; same blocks and kernels as the NCCL path. */
fusg_status fusg_kernel_apply_slab_loopback(fusg_kernel* const* ranks, int32_t nranks,
                                            const double* const* f_dev, double* const* u_dev,
                                            double scale);
/* Fused peer-memory transposes (<= 8 ranks; padded x and y lengths 256, 512 or 768): the
 * forward x pass stores every kx segment straight into the x-slab of the rank owning kx and the
 * inverse y pass stores every z-row straight into the A slab of the rank owning z, over NVLink
 * (CUDA IPC mappings). No exchange buffers or pack/unpack copies.
 *  - ipc_handles: this rank's two 64-byte CUDA IPC handles (x-slab, A slab);
 *  - attach_peers: `handles` = every rank's 128 bytes in rank order (gathered by the caller);
 *  - apply_slab_p2p: this rank's apply; all ranks call it (two 1-int NCCL barriers per apply);
 *  - apply_slab_loopback_p2p: the fused path for all ranks in this process on one device. */
/* Peer-store plan of rank `rank` (arrays of nranks <= 8; host only), with owner(key) = the last
 * q with begin[q] <= key:
 *  pass A element (y, z_local, kx) of rank r goes to rank q = owner_a(kx), x-slab flat index
 *    a_off[q] + y + z_local * a_sk[q] + kx * Nz * Ny;
 *  pass D element (z, kx_local, y) goes to rank q = owner_d(z), A-slab flat index
 *    d_off[q] + z * Ny + kx_local * d_sk[q] + y. */
fusg_status fusg_slab_peer_plan(const fusg_grid* global_grid, int32_t nranks, int32_t rank, int64_t* a_begin,
                                int64_t* a_off, int64_t* a_sk, int64_t* d_begin, int64_t* d_off,
                                int64_t* d_sk);
fusg_status fusg_kernel_slab_ipc_handles(const fusg_kernel* kernel, uint8_t out[128]);
fusg_status fusg_kernel_slab_attach_peers(fusg_kernel* kernel, const uint8_t* handles);
fusg_status fusg_kernel_apply_slab_p2p(fusg_kernel* kernel, const double* f_dev, double* u_dev,
                                       double scale, void* stream);
fusg_status fusg_kernel_apply_slab_loopback_p2p(fusg_kernel* const* ranks, int32_t nranks,
                                                const double* const* f_dev, double* const* u_dev,
                                                double scale);

#ifdef __cplusplus
}
#endif
#endif /* FUSG_H_ */
