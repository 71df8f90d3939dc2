/*
 * springsim_b200.h — C ABI of the B200-native mass-spring relaxation loop.
 *
 * The reference (`/root/reference/pkg/src/springsim`) has no FFI: its two
 * "operator" seams are the numba kernels in `_kernels.py:44-155` and the
 * Python `Engine` class in `engine.py:173-466`.  Every entry point below
 * replaces one of those seams; the reference symbol it stands in for is
 * cited beside it.  The Python host layer (`paper_2207_09334_b200/engine.py`)
 * binds these with ctypes; INTEGRATION.md shows the binding a maintainer of
 * the reference would add.
 *
 * Conventions
 *  - plain C types only; arrays are C-contiguous, row-major, caller-owned;
 *    (N,3) arrays are `double[3*N]`.  Nothing retains a host pointer after
 *    the call returns.
 *  - every function returns an `int` status (SS_OK == 0) unless stated;
 *    on failure `ss_last_error()` returns a thread-local message.
 *  - mass and spring ids are the caller's (reference) ids everywhere.
 *  - one engine must not be stepped from two threads at once
 *    (engine.py:179); distinct engines are independent.
 */
#ifndef SPRINGSIM_B200_H
#define SPRINGSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 2

/* status codes */
#define SS_OK             0
#define SS_EINVAL         1   /* bad argument (Python maps to ValueError, engine.py:184-189) */
#define SS_ECUDA          2   /* CUDA runtime error (no device, OOM, launch failure)        */
#define SS_EDIVERGED      3   /* DivergenceError (engine.py:44-52,375-381)                   */
#define SS_ENOMEM         4   /* host allocation failure                                     */
#define SS_EFALLBACK      5   /* scene document outside the native fast path: use the host parser */

/* integrators (engine.py:34-37) */
#define SS_EULER   0
#define SS_VERLET  1
#define SS_RK4     2

/* arithmetic of the device state */
#define SS_F64     0   /* validation mode: bitwise equal to reference serial mode */
#define SS_F32     1   /* production mode: displacement form, 1e-4 relative        */

/* device layouts of the incidence structure */
#define SS_LAYOUT_AUTO 0
#define SS_LAYOUT_CSR  1   /* generic per-mass CSR, any degree                      */
#define SS_LAYOUT_ELL  2   /* sliced-ELL owner records + reverse refs (16 B/spring) */
#define SS_LAYOUT_TILE 3   /* 256-mass brick tiles, TMA-staged records + smem halo   */

/* actuation modes (model.py:21-23) */
#define SS_SINUSOID            0
#define SS_CONSTANT_EXPANSION  1

/*
 * Scene description: the arrays `Engine.__init__` freezes a Scene into
 * (engine.py:192-220).  Field-for-field:
 *   x, v, f_ext  <- masses[*].x / .v / .f_ext    (double[3*n_masses])
 *   m            <- masses[*].m                   (double[n_masses])
 *   fixed        <- masses[*].fixed               (uint8[n_masses], may be NULL)
 *   si, sj       <- springs[*].i / .j             (int64[n_springs])
 *   k, l0        <- springs[*].k / .l0            (double[n_springs])
 *   group        <- index of springs[*].group in the groups table, -1 passive
 *                   (int32[n_springs], may be NULL)
 *   planes       <- scene.planes as n_planes x {nx,ny,nz,offset,penalty,friction}
 */
typedef struct ss_scene_desc {
    int64_t n_masses;
    int64_t n_springs;
    const double  *x;
    const double  *v;
    const double  *m;
    const double  *f_ext;     /* may be NULL (all zero) */
    const uint8_t *fixed;     /* may be NULL (none fixed) */
    const int64_t *si;
    const int64_t *sj;
    const double  *k;
    const double  *l0;
    const int32_t *group;     /* may be NULL */
    int32_t n_groups;
    const int32_t *group_mode;      /* SS_SINUSOID / SS_CONSTANT_EXPANSION, [n_groups] */
    const double  *group_amplitude; /* [n_groups] */
    const double  *group_frequency; /* [n_groups] */
    const double  *group_phase;     /* [n_groups] */
    int32_t n_planes;
    const double  *planes;    /* [6*n_planes] */
    double gravity[3];
    double dt;
    double damping;
    int32_t integrator;       /* SS_EULER / SS_VERLET / SS_RK4 */
    int32_t precision;        /* SS_F64 / SS_F32 */
    int32_t layout;           /* SS_LAYOUT_* */
    int32_t device;           /* CUDA ordinal */
} ss_scene_desc;

typedef struct ss_engine ss_engine;

/* Result of a batch of steps. */
typedef struct ss_step_result {
    int64_t steps_done;       /* steps committed by this call (incl. the diverging one) */
    int64_t n;                /* engine step counter after the call        (engine.py:371) */
    double  t;                /* engine time after the call, == n*dt       (engine.py:372) */
    int64_t diverged_mass;    /* lowest non-finite mass id, -1 if none     (engine.py:381) */
    int64_t diverged_step;    /* step number at which it was detected, -1  */
} ss_step_result;

int         ss_abi_version(void);
const char *ss_last_error(void);
int         ss_device_count(int *count);

/* Page-locked host buffers (cudaHostAlloc).  State arrays passed to
 * ss_set_state / ss_get_state that live in page-locked memory (these, or
 * torch pin_memory tensors) cross the bus in one DMA, without the pageable
 * staging copy.  No reference counterpart: the reference keeps its state in
 * numpy arrays (engine.py:196-208); this is the transfer path behind them. */
int ss_pinned_alloc(size_t bytes, void **out);
int ss_pinned_free(void *p);

/* Engine.__init__ (engine.py:182-246). */
int ss_create(const ss_scene_desc *desc, ss_engine **out);
int ss_destroy(ss_engine *h);

/* Engine.step(count) (engine.py:366-373): `count` steps of the configured
 * integrator, actuation tables built from the current group parameters, the
 * finiteness check after every step.  Returns SS_EDIVERGED (and fills `res`)
 * when a step produced a non-finite position or velocity; the state is then
 * the diverged state, as in the reference. */
int ss_step(ss_engine *h, int64_t count, ss_step_result *res);

/* Asynchronous variant for benchmarking: enqueues `count` steps on the
 * engine's stream and returns immediately.  Divergence is recorded on the
 * device and reported by the next ss_step / ss_sync. */
int ss_step_async(ss_engine *h, int64_t count);
int ss_sync(ss_engine *h, ss_step_result *res);
/* Block until at most `max_ahead` asynchronously enqueued steps are still
 * unfinished on the device.  Engine.step drains the command queue between
 * chunks of a long batch (engine.py:366-370 drains before every step):
 * keeping the host one chunk ahead of the device bounds how late a command
 * posted mid-batch lands, without idling the device. */
int ss_pending_wait(ss_engine *h, int64_t max_ahead);
/* cudaStream_t of the engine, as an opaque pointer (for CUDA-event timing). */
void *ss_stream(ss_engine *h);

/* Engine.forces(x, v, t) (engine.py:261-289): total force at a trial state.
 * Adds the degenerate-spring count to the engine counter like the reference. */
int ss_forces(ss_engine *h, const double *x, const double *v, double t,
              double *acc_out, int64_t *degenerate_out);

/* Engine.state / direct attribute access (engine.py:383-388, 196-202).
 * Any pointer may be NULL (that array is skipped / left unchanged);
 * *has_prev reports whether the Verlet history x_prev exists.  Setting x_prev
 * creates the history (the `engine.x_prev = ...` assignment of
 * tests/test_engine.py:170); ss_clear_prev drops it (x_prev = None). */
int ss_get_state(ss_engine *h, double *x, double *v, double *x_prev, int *has_prev);
int ss_set_state(ss_engine *h, const double *x, const double *v, const double *x_prev);
int ss_clear_prev(ss_engine *h);
int ss_get_positions(ss_engine *h, double *x);
int ss_get_time(ss_engine *h, double *t, int64_t *n);
int ss_set_time(ss_engine *h, double t, int64_t n);

/* setters (engine.py:402-424); range validation is done by the caller like
 * Engine.set_damping (engine.py:405-408), direct attribute writes are not
 * validated by the reference either. */
int ss_set_f_ext(ss_engine *h, const double *f_ext);
int ss_set_damping(ss_engine *h, double damping);
int ss_set_gravity(ss_engine *h, const double g[3]);
int ss_set_group(ss_engine *h, int32_t group, int32_t mode, double amplitude,
                 double frequency, double phase);

/* Engine.degenerate_springs (engine.py:224,271) */
int ss_degenerate_count(ss_engine *h, int64_t *count);

/* introspection: bytes of device memory, layout chosen, algorithmic bytes
 * per step as defined in SURVEY §8d / DESIGN.md §4 */
typedef struct ss_info {
    int64_t n_masses, n_springs;
    int32_t precision, layout, integrator, device;
    int64_t device_bytes;
    double  algorithmic_bytes_per_step;
    int32_t ell_width_own, ell_width_ref;
    int32_t canonical_order;   /* 1 if the ELL split order == spring-id order */
    int32_t smem_per_block;    /* TILE: dynamic shared memory per CTA */
    int64_t tile_count;        /* TILE: number of 256-mass tiles */
    int64_t tile_blob_bytes;   /* TILE: bytes of records streamed per step */
    double  tile_halo_ratio;   /* TILE: mean (tile + halo masses) / tile masses */
    double  tile_foreign_frac; /* TILE: fraction of references whose owner is in another tile */
    int32_t tile_kernel;       /* dominant kernel / record format: fp32 1 explicit, 2 compact (tile_lean_kernel; 0: step_kernel);
                                  fp64 0 explicit, 3 compact (step_kernel), 4 compact (tile_f64_kernel),
                                  5 inline (tile_f64_kernel, (k, l0) per incidence: general graphs);
                                  fp32 6 inline (tile_lean_kernel, records per incidence: general graphs),
                                  7 compact with a (k, k*l0, group) dictionary and rest vectors formed
                                  from X0 (tile_lean_kernel: positions off a lattice, e.g. jittered
                                  robot populations) */
    int32_t kernel_smem;       /* its dynamic shared memory per CTA */
} ss_info;
int ss_get_info(ss_engine *h, ss_info *info);

/* Host-only: build the tiled layout of a scene description (no device
 * needed) and report its statistics in `info`. */
int ss_plan(const ss_scene_desc *desc, ss_info *info);

/* On-device sampling for simulate()/RunResult (engine.py:476-565) and the
 * energy breakdown (engine.py:148-170, Engine.energies engine.py:390-398).
 * ss_energy_setup hands the engine the caller-order spring list (k, l0,
 * actuation group, -1 passive) and the GPE datum once.  ss_step_sampled runs
 * `count` steps; after every step whose index d (Verlet: n-1, sampled at
 * x_prev with the lagged central-difference v, exactly like the reference's
 * simulate; Euler/RK4: n) is a multiple of sample_every it records t = d*dt,
 * the positions of the n_ids traced masses (caller ids) and (epe, gpe, ke,
 * total) in device buffers, and copies the rows out once at the end (one
 * host synchronisation per call).  *rows_out = rows written (<= max_rows);
 * divergence: SS_EDIVERGED with `res` filled and no rows. */
int ss_energy_setup(ss_engine *h, int64_t n_springs, const int64_t *si, const int64_t *sj,
                    const double *k, const double *l0, const int32_t *group, double gpe_datum);
int ss_step_sampled(ss_engine *h, int64_t count, int64_t sample_every,
                    const int64_t *ids, int64_t n_ids, int64_t max_rows,
                    double *times_out, double *pos_out, double *energy_out,
                    int64_t *rows_out, ss_step_result *res);
/* Steering snapshot (service.py:378-389 SteerServer._snapshot_bytes): the
 * positions of the n_ids masses `ids` (caller ids) and (epe, gpe, ke, total)
 * at the current state (x, v, actuation at t; Engine.energies()), gathered
 * and reduced on the device.  pos_out: n_ids x 3; energy_out: 4 (may be
 * null).  Needs ss_energy_setup. */
int ss_snapshot(ss_engine *h, const int64_t *ids, int64_t n_ids, double gpe_datum, double *pos_out,
                double *energy_out);

/* Kernel launches issued so far (for the bench's gpu_launches claim). */
int64_t ss_launch_count(ss_engine *h);

/*
 * Array-native voxel lattice over an axis-aligned box, bit-identical to
 * `build_voxel_lattice(box_mesh(lo, hi), LatticeSpec(dim))` with
 * `Material(k0, l_ref=dim)` (lattice.py:89-136, model.py:87-97):
 * nodes lo + idx*dim in (i,j,k) lexicographic order, springs sorted by
 * (i, j), l0 = sqrt(fma(dz,dz,fma(dy,dy,dx*dx))) (the OpenBLAS ddot that
 * np.linalg.norm uses, lattice.py:84), k = (k0*l_ref)/l0.
 * Call once with NULL outputs to get the counts, then with buffers.
 * Only masses with plane index in [i_lo, i_hi) are emitted when i_hi > i_lo
 * (spatial slab for multi-GPU sharding); springs with at least one endpoint
 * in the slab are emitted, ids stay global.
 */
int ss_lattice_box(const double lo[3], const double hi[3], double dim,
                   double k0, double l_ref,
                   int64_t i_lo, int64_t i_hi,
                   int64_t counts_out[3], int64_t *n_masses_out, int64_t *n_springs_out,
                   double *x_out, int64_t *si_out, int64_t *sj_out,
                   double *k_out, double *l0_out, int64_t *spring_id_out);

/*
 * x-slab sharding.  A shard's scene holds its
 * owned masses plus one halo plane per neighbour, marked fixed; springs keep
 * their global ids, so results are bitwise identical to one device.
 * ss_halo_setup: caller ids of the boundary planes to send and of the halo
 * planes to receive (side lo = lower-x neighbour, hi = upper), plane order
 * identical on both sides.  Transport:
 *   - ss_nccl_unique_id + ss_halo_nccl: one process per GPU; after every
 *     substep (RK4: every stage) ss_step packs, exchanges (ncclSend/ncclRecv
 *     on the engine stream) and unpacks the planes;
 *   - ss_halo_p2p_export + ss_halo_recv_slots + ss_halo_p2p_attach: one
 *     process per GPU on one node; the step kernel itself stores its
 *     boundary planes into the neighbours' position buffers over peer
 *     memory (CUDA IPC, NVLink stores) and synchronises through device-side
 *     step flags -- no extra kernel, no host round trip, no NCCL.  export
 *     returns a 256-byte blob (IPC handles of this engine's flag mailbox and
 *     position buffers, plane sizes, step); recv_slots gives this engine's
 *     device slots of its halo plane on `side`; attach maps a neighbour's
 *     blob as side 0 (lower) or 1 (upper) together with the neighbour's
 *     recv_slots for the facing plane.  The reference has no multi-GPU path
 *     (SURVEY §8e).
 *   - ss_halo_p2p_link: the same transport between engines of one process
 *     (same device or peer-accessible devices), without IPC;
 *   - ss_step_group: several shards on one device stepped in lockstep, the
 *     planes copied device-to-device (RK4: stage by stage) or, when
 *     peer-linked, exchanged by the step kernels (virtual shards, for
 *     testing).  RK4 exchanges after every stage on every transport.
 *     The shards share one divergence step: all stop after the first
 *     non-finite step anywhere; *diverged_shard (may be null) names the
 *     lowest shard that flagged it and res->diverged_mass its local id.
 */
int ss_halo_setup(ss_engine *h, int64_t n_send_lo, const int64_t *send_lo, int64_t n_send_hi,
                  const int64_t *send_hi, int64_t n_recv_lo, const int64_t *recv_lo,
                  int64_t n_recv_hi, const int64_t *recv_hi);
int ss_nccl_unique_id(unsigned char id[128]);
int ss_halo_nccl(ss_engine *h, const unsigned char id[128], int nranks, int rank, int rank_lo, int rank_hi);
int ss_halo_p2p_export(ss_engine *h, unsigned char blob[256]);
int ss_halo_recv_slots(ss_engine *h, int side, int32_t *out);
int ss_halo_p2p_attach(ss_engine *h, int side, const unsigned char blob[256], const int32_t *peer_slots,
                       int64_t n_slots);
int ss_halo_p2p_link(ss_engine *h, int side, ss_engine *peer);
int ss_step_group(ss_engine **engines, int n, int64_t count, ss_step_result *res, int32_t *diverged_shard);

/* Engine.gpe_datum (engine.py:240-242): the height GPE is measured from,
 * read by every later on-device energy sample (service.py:462 and
 * analysis.py:755 move it after construction). */
int ss_set_gpe_datum(ss_engine *h, double datum);

/* Diagnostics: the fp64 kernel's branch-free IEEE fast paths against the
 * library operators on `n` operand pairs (device `device`).  out[4i..4i+3] =
 * (fast sqrt(a), sqrt(a), fast b/a, b/a); ok[i] bit 0 / bit 1: the sqrt /
 * division operands are inside the fast-path range (then the fast result
 * must equal the library's bit for bit; tests/test_gpu_f64_kernel.py). */
int ss_check_f64_fastpath(int32_t device, const double *a, const double *b, int64_t n,
                          double *out, int32_t *ok);

/* Scene documents (sceneio.py:57-239): native codec for the bulk "masses"
 * and "springs" arrays (paper_2207_09334_b200/csrc/sceneio.cpp).
 * ss_doc_render_*: the exact text json.dumps(doc, indent=2) writes for that
 * array (entries joined by ",\n", without the brackets), malloc'd, freed by
 * ss_doc_free_text; SS_EFALLBACK for non-finite values (the host raises the
 * reference's error).  ss_doc_parse: strict fast path over a whole ASCII
 * document; SS_EFALLBACK sends the document to the reference-exact host
 * parser (any error, unusual field, escape or literal). */
typedef struct ss_doc ss_doc;
int  ss_doc_render_masses(int64_t n, const double *m, const double *x, const double *v, const double *f,
                          const uint8_t *fixed, char **out, int64_t *len);
int  ss_doc_render_springs(int64_t n, const int64_t *si, const int64_t *sj, const double *k, const double *l0,
                           const int32_t *group, const char *const *labels, int32_t n_labels, char **out,
                           int64_t *len);
int  ss_doc_render(int64_t n_masses, const double *m, const double *x, const double *v, const double *f,
                   const uint8_t *fixed, int64_t n_springs, const int64_t *si, const int64_t *sj, const double *k,
                   const double *l0, const int32_t *group, const char *const *labels, int32_t n_labels,
                   const char *pre, const char *mid, const char *post, char **out, int64_t *len);
void ss_doc_free_text(char *p);
int  ss_doc_repr(int64_t n, const double *v, char **out, int64_t *len);
int  ss_doc_parse(const char *text, int64_t len, ss_doc **out);
int  ss_doc_info(const ss_doc *d, int64_t *n_masses, int64_t *n_springs, int32_t *n_keys, int32_t *n_labels);
int  ss_doc_key(const ss_doc *d, int32_t i, const char **name, int64_t *off, int64_t *len);
const char *ss_doc_label(const ss_doc *d, int32_t i);
int  ss_doc_masses(const ss_doc *d, double *m, double *x, double *v, double *f, uint8_t *fixed);
int  ss_doc_springs(const ss_doc *d, int64_t *si, int64_t *sj, double *k, double *l0, int32_t *group);
void ss_doc_free(ss_doc *d);

#ifdef __cplusplus
}
#endif
#endif /* SPRINGSIM_B200_H */
