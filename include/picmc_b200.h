/*
 * picmc_b200.h -- C ABI of the B200-native particle mover + charge deposition.
 *
 * The reference's operator boundary for this hot path is the Python module
 * `picmc.backends` (/root/reference/pkg/src/picmc/backends/__init__.py:45-50),
 * whose compiled twin is pkg/src/picmc/backends/_kernels.pyx.  Every entry
 * point below is plain C: device pointers, sizes, a cudaStream_t passed as
 * `void*`, and an int status.  Nothing is thrown across the ABI; the detail of
 * the last failure on the calling thread is in pb_last_error().
 *
 * Status codes map onto the reference exception hierarchy
 * (pkg/src/picmc/errors.py:4-25) in the Python wrapper:
 *   PB_ERR_INVALID  -> ValueError      (Cython buffer / argument checks)
 *   PB_ERR_CFL      -> CflViolation    (pkg/src/picmc/mover.py:142-148)
 *   PB_ERR_CONTRACT -> ContractViolation (pkg/src/picmc/core.py:256-264)
 *   PB_ERR_OVERFLOW -> EngineError     (fixed-point deposit bin overflow)
 *   PB_ERR_CUDA     -> RuntimeError    (CUDA runtime failure)
 *
 * All arrays are device memory unless stated otherwise.  Particle state is
 * fp64 and cell-relative ([0,1) in units of dx) exactly as in the reference
 * store (pkg/src/picmc/core.py:108-109); the engine layout is a flat
 * structure of arrays with an int32 cell index per particle instead of the
 * reference's per-cell slack segments.
 */
#ifndef PICMC_B200_H
#define PICMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB_ABI_VERSION 3

#define PB_OK 0
#define PB_ERR_INVALID 1
#define PB_ERR_CUDA 2
#define PB_ERR_CFL 3
#define PB_ERR_CONTRACT 4
#define PB_ERR_OVERFLOW 5
#define PB_ERR_PEER 6 /* a peer GPU did not reach a density barrier */

/* Species kinds: which arithmetic the mover applies (SpeciesDef flags,
 * pkg/src/picmc/core.py:53-81, and accel_nodes_for_species,
 * pkg/src/picmc/mover.py:211-224). */
#define PB_KIND_INACTIVE 0 /* active_mover == False: not pushed            */
#define PB_KIND_DRIFT 1    /* uncharged: x += nstep*vx, no kick (keeps -0.0) */
#define PB_KIND_KICK 2     /* charged: one-sided gather, vx += a, drift      */
#define PB_KIND_BORIS 3    /* charged + B: Boris rotation (config 4)         */

/* Particle boundary: the reference always wraps (mover.py:156); absorbing
 * walls are the config-3 extension restated in oracle/ and DESIGN.md. */
#define PB_BC_PERIODIC 0
#define PB_BC_ABSORBING 1

/* Field boundary for the density stitch (fields.py:81-92, :115-117). */
#define PB_FIELD_PERIODIC 0
#define PB_FIELD_DIRICHLET 1

#define PB_MAX_SPECIES 8

/* Fixed-point deposit: each particle adds round(x * 2^48) to R and 1 to the
 * cell count C; L = C*2^48 - R.  Integer sums are exact and associative, so
 * the density is bitwise independent of thread order and GPU count. */
#define PB_DEPOSIT_FRAC_BITS 48

typedef struct pb_species {
  double *x, *vx, *vy, *vz; /* SoA particle state, n_cap slots           */
  double *yp;               /* transverse position or NULL (sn2d)         */
  int32_t *cell;            /* owning cell of every live slot             */
  int64_t *n_dev;           /* device live count (absorbing) or NULL      */
  int64_t n;                /* host live count / upper bound of n_dev     */
  int64_t *holes;           /* absorbing: scratch list of removed slots   */
  int32_t kind;             /* PB_KIND_*                                  */
  int32_t deposit;          /* deposit bin slot, -1 for neutral species   */
  double fnstep;            /* float(nstep) (mover.py:248)                */
  double kick_coef;         /* q dt^2/(m dx), velocity_kick_coef (mover.py:38-40) */
  double boris_t[3];        /* q B dt / (2 m)                             */
  double boris_s[3];        /* t * (2 / (1 + |t|^2))                      */
  /* Optional compressed cell index read by the production mover instead of
   * `cell` (1 byte instead of 4 per charged particle): cell8[i] =
   * cell[i] - chunk_base[i / PB_CELL8_CHUNK], or PB_CELL8_ESCAPE when that
   * does not fit (then cell[i] is read).  `cell` stays authoritative and is
   * written for every mover; NULL = not used.  Rebuild with pb_cell8_build
   * after anything reorders a species. */
  int8_t *cell8;
  int32_t *chunk_base;
  /* Spatially varying B (SURVEY.md 8(b) `b_nodes_or_null`, carried per
   * species so every mover entry point -- pb_push_deposit, the canonical
   * resort / keys and the shims -- sees it without another argument):
   * b_nodes[4*j + k] = B_k at node j in tesla (k = x, y, z; slot 3 is
   * padding so one node is one 32-byte load), nc+1 nodes.  NULL = the
   * uniform boris_t / boris_s above.  Otherwise, per Boris particle in cell
   * j at cell-relative x (pre-push), with f = boris_f = q dt / (2 m):
   *   t_k = f*B_k[j] + x*(f*B_k[j+1] - f*B_k[j])   (the one-sided gather
   *                                                  of accel_nodes, mover.py:221)
   *   s_k = t_k * (2 / (1 + ((t_x*t_x + t_y*t_y) + t_z*t_z)))
   * each operation rounded separately (no FMA), restated in
   * oracle/picmc_oracle.c:boris_t_gather. */
  const double *b_nodes;
  double boris_f;
} pb_species;

#define PB_CELL8_CHUNK 2048
#define PB_CELL8_ESCAPE (-128)
#define PB_CELL8_MARGIN 32 /* chunk_base = first cell of the chunk - margin */

/* Device-resident step status, read by the host at the step's sync point. */
typedef struct pb_status {
  int32_t code;             /* PB_OK or first error code                 */
  int32_t cfl_species;      /* species of the CFL offender               */
  uint64_t cfl_index;       /* smallest offending slot (atomicMin)       */
  int64_t moved[PB_MAX_SPECIES];        /* cell transfers this step     */
  int64_t absorbed[PB_MAX_SPECIES][2];  /* [left wall, right wall]      */
  int64_t n_holes[PB_MAX_SPECIES];      /* absorbed slots to compact    */
  int64_t overflow;                     /* deposit bins over capacity   */
  uint64_t tile_next;                   /* mover work counter (chunks claimed) */
  uint64_t tile_done;                   /* claimers finished; the last one
                                           resets the counters, so they are
                                           zero again after every launch */
  uint64_t tile_next2;                  /* second work list (split mover)   */
  /* In-kernel clock of the persistent movers (k_push_split / ring / quad):
   * every block records its start (%globaltimer, min), the last warp to
   * finish adds (end - first start) to mover_ns and counts the launch, so
   * the movers' own duration is measured inside graph replays. */
  uint64_t mover_t0;                    /* UINT64_MAX between launches      */
  uint64_t mover_ns;
  uint64_t mover_launches;
} pb_status;
/* The caller resets *status before each pb_push_deposit: all zero except
 * cfl_index = mover_t0 = UINT64_MAX (the engine copies a template). */

/* ---- library ------------------------------------------------------------ */
int pb_abi_version(void);
size_t pb_status_bytes(void); /* sizeof(pb_status) as compiled */
const char *pb_last_error(void);
int pb_device_sm_count(int *out);

/* ---- parity shims with the reference kernel signatures (packed layout) --
 * offs/counts address per-cell segments of packed arrays exactly as
 * CellSortedStore does (pkg/src/picmc/core.py:100-132). */

/* fused_move (pkg/src/picmc/backends/_kernels.pyx:60-102): in place.
 * accel_or_null has nc+1 entries; NULL skips the kick entirely. */
int pb_fused_move(const double *accel_or_null, double *x, double *vx,
                  const double *vy, double *yp_or_null, const int64_t *offs,
                  const int64_t *counts, int64_t nc, double fnstep,
                  void *stream);

/* deposit_partials (_kernels.pyx:14-34): L[j]=sum(1-x), R[j]=sum(x) in slot
 * order -- sequential per cell, bitwise equal to the reference. */
int pb_deposit_partials(const double *x, const int64_t *offs,
                        const int64_t *counts, int64_t nc, double *left,
                        double *right, void *stream);

/* gather (_kernels.pyx:37-57): out[k] = a[j] + x*(a[j+1]-a[j]) in live
 * (cell-major) order; out has sum(counts) entries. */
int pb_gather(const double *nodes, const double *x, const int64_t *offs,
              const int64_t *counts, int64_t nc, double *out, void *stream);

/* fused_move_aos / fused_move_table (_kernels.pyx:105-152): the same
 * arithmetic on a row-major table (ncols >= 4, columns x, vx, vy, vz[, yp]);
 * per cell j rows [starts[j], starts[j]+counts[j]).  A single cell's table
 * (fused_move_table) is nc = 1 with accel = {aj, aj1}. */
int pb_fused_move_aos(double *tab, int64_t ncols, const int64_t *starts,
                      const int64_t *counts, int64_t nc,
                      const double *accel_or_null, double fnstep, int has_yp,
                      void *stream);

/* ---- device-resident engine (flat SoA + cell index) ---------------------- */

/* One mover step for `nsp` species, fused: gather E, kick (or Boris), drift,
 * cell transfer with the reference floor/carry/mod rules
 * (pkg/src/picmc/mover.py:136-163), absorbing-wall removal, and the
 * fixed-point deposit of the post-move positions into `bins`
 * ([ndep][2][nc] uint64: R then C).  e_nodes has nc+1 entries (required for
 * KICK/BORIS species).  Errors are recorded in *status (device). */
int pb_push_deposit(const pb_species *sp, int nsp, const double *e_nodes,
                    int64_t nc, int particle_bc, uint64_t *bins,
                    pb_status *status, void *stream);

/* Rebuild cell8 / chunk_base of a species from its cell array (slots
 * [0, sp->n)). */
int pb_cell8_build(const pb_species *sp, void *stream);

/* Name of the mover kernel the last pb_push_deposit / pb_deposit_only call
 * launched (k_push_split, k_push_quad, k_push_ring, ...). */
const char *pb_last_mover_kernel(void);

/* Standalone fixed-point deposit of current positions (step-0 deposit and
 * inactive charged species). */
int pb_deposit_only(const pb_species *sp, int nsp, int64_t nc, uint64_t *bins,
                    pb_status *status, void *stream);

/* Weighted partials and stitched density from fixed-point bins:
 * left = sum_s coef_s * L_s, right likewise, in species order
 * (pkg/src/picmc/fields.py:67-77), rho per stitch_rho/deposit_charge
 * (fields.py:81-92, :115-117).  coef is a host array of ndep doubles.
 * Bin overflow: a cell holding >= 2^(64-PB_DEPOSIT_FRAC_BITS) = 65536
 * particles of one species cannot be represented; if status is non-NULL
 * such a cell sets status->code = PB_ERR_OVERFLOW (if still PB_OK) and
 * status->overflow = the largest count seen. */
int pb_rho_epilogue(const uint64_t *bins, const double *coef, int ndep,
                    int64_t nc, int field_bc, double *left, double *right,
                    double *rho, pb_status *status_or_null, void *stream);

/* The engine's per-step form of pb_rho_epilogue (two kernels): weighted
 * partials per cell, after which `bins` itself is zeroed (a bin set is clean
 * again once its density has been taken), then the stitch into rho.  If
 * non-NULL, `bins_next` (the other ping-pong set) is zeroed too.  Because it
 * never touches the set the next mover deposits into, it may run
 * concurrently with that pb_push_deposit.  Overflow as pb_rho_epilogue. */
int pb_density_step(uint64_t *bins, uint64_t *bins_next,
                    pb_status *status_or_null, const double *coef, int ndep,
                    int64_t nc, int field_bc, double *left, double *right,
                    double *rho, void *stream);

/* Fill the holes left by absorbed particles from the tail (warp-ballot
 * stream compaction); updates *n_dev.  `scratch` needs
 * pb_compact_scratch_bytes(n) bytes. */
/* stitch_rho (fields.py:81-92): rho[g] = R[g-1] + L[g]; periodic ends
 * rho[0] = rho[nc] = R[nc-1] + L[0], else rho[0] = L[0], rho[nc] = R[nc-1]
 * (no wall doubling: that is deposit_charge's, done by pb_density_step /
 * pb_rho_from_partials). */
int pb_stitch_rho(const double *left, const double *right, int64_t nc,
                  int periodic, double *rho, void *stream);

size_t pb_compact_scratch_bytes(int64_t n);
int pb_compact(const pb_species *sp, int nsp, pb_status *status,
               void *scratch, size_t scratch_bytes, void *stream);

/* Periodic sort by cell: counting sort (cell histogram, exclusive scan,
 * scatter of every field) into the `dst` species buffers (ping-pong).  Order
 * within a cell is arbitrary (the engine's physics is order independent).
 * With src->n_dev set (absorbing species) the live count is read on device
 * and src->n is only its upper bound.  `scratch` needs pb_sort_scratch_bytes(n, nc) bytes. */
size_t pb_sort_scratch_bytes(int64_t n, int64_t nc);
int pb_sort_by_cell(const pb_species *src, const pb_species *dst, int64_t nc,
                    void *scratch, size_t scratch_bytes, void *stream);

/* Field pipeline (replicated on every GPU; config 3/4 and field_solve runs).
 * smooth_density (fields.py:121-135), solve_poisson (fields.py:156-202),
 * compute_efield (fields.py:205-218).  `scratch` needs
 * pb_field_scratch_bytes(nc) bytes. */
size_t pb_field_scratch_bytes(int64_t nc);
int pb_smooth_density(const double *rho, double *out, int64_t nc, int passes,
                      void *scratch, void *stream);
int pb_solve_poisson(const double *rho, double *phi, int64_t nc, double dx,
                     double eps0, int field_bc, double phi_left,
                     double phi_right, void *scratch, void *stream);
/* Same system in parallel: its Green's-function form (the closed-form
 * Thomas pivots telescoped through both sweeps) needs ONE prefix scan of
 * (sum r, sum (k+1) r) over 512-unknown tiles plus the totals (periodic: the
 * mean enters in closed form); ~1e-14 max|phi| from a long-double
 * elimination at 1e5 unknowns.  Three launches (tile aggregates, tile
 * prefixes, tile solves).  Used for large field grids. */
int pb_solve_poisson_scan(const double *rho, double *phi, int64_t nc,
                          double dx, double eps0, int field_bc,
                          double phi_left, double phi_right, void *scratch,
                          void *stream);
int pb_compute_efield(const double *phi, double *e, int64_t nc, double dx,
                      int field_bc, void *stream);
/* pb_compute_efield, then zero nwords words of clr_a and clr_b (either may
 * be NULL): the serial field-solve cycle clears the bins read by
 * pb_rho_epilogue here. */
int pb_compute_efield_clear(const double *phi, double *e, int64_t nc,
                            double dx, int field_bc, uint64_t *clr_a,
                            uint64_t *clr_b, int64_t nwords, void *stream);


/* The whole replicated field step of a field-solve run: pb_rho_epilogue
 * (weighted partials, stitched rho, overflow check) + pb_smooth_density
 * (`passes` 1-2-1 passes into rho_s) + pb_solve_poisson_scan (on rho_s) +
 * pb_compute_efield_clear (E, then zero nwords words of clr_a / clr_b; both
 * may be NULL), bitwise those four calls, in ONE launch (k_field_fused:
 * every tile forms its density window and local scan, one grid-wide
 * arrival count, then the solve and E) when passes <= 4 and the
 * ceil((nc-1)/512) tiles fit co-resident on the device, else as kernels.
 * `scratch` needs pb_field_scratch_bytes(nc) bytes, ZEROED before its first
 * use (its two counter words return to zero after every launch); left /
 * right may be NULL.  compact_sp / compact_nsp (NULL / 0: none): also
 * pb_compact those species (the previous step's absorbing-wall holes;
 * compact_scratch as pb_compact's) -- extra blocks of the same launch,
 * independent of the field work. */
int pb_field_cycle(const uint64_t *bins, const double *coef, int ndep,
                   int64_t nc, int field_bc, int passes, double dx,
                   double eps0, double phi_left, double phi_right,
                   double *left, double *right, double *rho, double *rho_s,
                   double *phi, double *e, uint64_t *clr_a, uint64_t *clr_b,
                   int64_t nwords, pb_status *status_or_null, void *scratch,
                   const pb_species *compact_sp, int compact_nsp,
                   void *compact_scratch, size_t compact_scratch_bytes,
                   void *stream);

/* Roofline probe: streams the mover's exact read/write bytes per species with
 * a trivial update (no physics, no deposit).  Destroys particle state. */
int pb_stream_sol(const pb_species *sp, int nsp, void *stream);

/* Device init_plasma (pkg/src/picmc/core.py:292-352): ppc0 particles per
 * cell for cells [cell_lo, cell_hi) with the reference splitmix64 streams.
 * Positions are bit-exact; velocities use CUDA log/sin/cos (ulp-close). */
int pb_init_species(pb_species *sp, uint64_t species_key, int64_t cell_lo,
                    int64_t cell_hi, int64_t ppc0, double vstd, void *stream);

/* ---- canonical slot order + collisions -------------
 * In canonical mode every species is a flat SoA in the reference's exact
 * cell-major slot order (the live slots of CellSortedStore concatenated over
 * cells, pkg/src/picmc/core.py:100-181) with per-cell offs[nc+1] and
 * counts[nc] (int64).  The slot order is what the reference's collision
 * streams are indexed by (pkg/src/picmc/collisions.py:195-219). */

/* Build offs/counts of a cell-sorted species (load time).  Returns
 * PB_ERR_CONTRACT if `cell` is not in cell-major order.  Synchronises the
 * stream.  `scratch` needs pb_layout_scratch_bytes(nc) bytes. */
size_t pb_layout_scratch_bytes(int64_t nc);
int pb_cell_layout(const int32_t *cell, int64_t n, int64_t nc, int64_t *offs,
                   int64_t *counts, void *scratch, size_t scratch_bytes,
                   void *stream);

typedef struct pb_collide_params {
  uint64_t step_key;      /* stream(seed, STREAM_COLLIDE, step), collisions.py:92-93 */
  int64_t global_offset;  /* global index of local cell 0 (collide_block)   */
  double w_over_dx;       /* neutral macro weight / dx (collisions.py:239)  */
  double dt;              /* consts.dt_s                                    */
  double rate_elastic, rate_excitation, rate_ionization; /* m^3/s          */
  double threshold_j;     /* excitation_threshold_ev * ELEMENTARY_CHARGE    */
  double mass_e;          /* electron mass_kg                               */
  double dx_over_dt;      /* grid.dx_m / consts.dt_s                        */
} pb_collide_params;

/* collision_phase (pkg/src/picmc/collisions.py:310-351) over all cells:
 * elastic / excitation / ionization with the reference splitmix64 streams,
 * the dt-halving guard, and swap_remove of the ionized neutral
 * (core.py:205-218): n_counts is updated to the live neutral count, the
 * vacated neutral slots get cell = -1.  Newborn pairs (ion, electron) are
 * appended at e->n + t and ion->n + t with cell set, newborn_k[t] = event
 * index within the cell, newborn_per_cell[j] = pairs born in cell j.
 * counters (device u64[6]): elastic, excitation, ionization, suppressed,
 * newborns, overflow (zeroed by the call). */
int pb_collide(const pb_species *e, const pb_species *neutral,
               const pb_species *ion, const int64_t *e_offs,
               const int64_t *e_counts, const int64_t *n_offs,
               int64_t *n_counts, int64_t nc, const pb_collide_params *params,
               int64_t *newborn_per_cell, int32_t *newborn_k,
               int64_t newborn_cap, uint64_t *counters, void *stream);

typedef struct pb_canon {
  int64_t n_old;      /* slots [0, n_old): pre-step store (cell -1 = vacated) */
  int64_t n_tail;     /* slots [n_old, n_old+n_tail): newborns               */
  int64_t *offs;      /* in: slot offsets of the pre-step store; out: new   */
  int64_t *counts;    /* in: live counts after removals; out: new counts    */
  const int64_t *newborn_per_cell; /* nc, or NULL when n_tail == 0          */
  const int32_t *newborn_k;        /* n_tail, or NULL                        */
} pb_canon;

/* One mover step of one species in canonical order: reference push
 * (kick/drift, Boris, yp) + resort_collect transfer + commit order
 * (survivors in slot order, then newborns, then incomers by (src_cell,
 * src_slot); pkg/src/picmc/mover.py:113-195, collisions.py:286-289), written
 * into `dst` (ping-pong buffers).  New live count = offs[nc]. */
size_t pb_canonical_scratch_bytes(int64_t n_cap, int64_t nc);
int pb_canonical_resort(const pb_species *src, const pb_species *dst,
                        const pb_canon *cv, const double *e_nodes, int64_t nc,
                        int particle_bc, int species_id, pb_status *status,
                        void *scratch, size_t scratch_bytes, void *stream);

/* Multi-GPU canonical order, first half of a species' step: push +
 * transfer in place and write int64 keys[0, n_old + n_tail) = (dest cell,
 * moved, rank_offset + canonical rank) packed over rank_bits (all ones for
 * vacated / absorbed slots).  The caller exchanges the particles whose dest
 * cell another rank owns and orders its union by key. */
int pb_canonical_keys(const pb_species *src, const pb_canon *cv,
                      const double *e_nodes, int64_t nc, int particle_bc,
                      int species_id, pb_status *status, int64_t rank_offset,
                      int rank_bits, int64_t *keys, void *scratch,
                      size_t scratch_bytes, void *stream);

/* pb_canonical_resort for species 0..nsp-1 (cv[k], species id k) in one
 * call, then the new live counts (offs[nc] of each) into the host array
 * n_new[nsp].  Synchronises the stream. */
/* Stores of at least n particles take the scatter resort in
 * pb_canonical_step (default 2^20; smaller stores keep the full key sort,
 * bitwise the same result).  Process-wide. */
int pb_set_canonical_scatter_min(int64_t n);

int pb_canonical_step(const pb_species *src, const pb_species *dst,
                      const pb_canon *cv, int nsp, const double *e_nodes,
                      int64_t nc, int particle_bc, pb_status *status,
                      void *scratch, size_t scratch_bytes, int64_t *n_new,
                      void *stream);

/* Weighted partials + stitched rho from fp64 per-species partials
 * raw[ndep][2][nc] (L then R, as pb_deposit_partials produces them):
 * bitwise deposit_partials_range + stitch_rho (fields.py:55-92). */
int pb_rho_from_partials(const double *raw, const double *coef, int ndep,
                         int64_t nc, int field_bc, double *left,
                         double *right, double *rho, void *stream);

/* ---- Mover API on the reference's cell-segmented store ------------------
 * CellSortedStore (pkg/src/picmc/core.py:100-264): per cell j, live slots
 * [offs[j], offs[j]+counts[j]) of packed float64 field arrays, free space
 * zeroed.  Field 0 is x; the others (vx, vy, vz[, yp]) in the store's order.
 * These back the twin of pkg/src/picmc/mover.py (paper_2404_10270_b200.mover). */
#define PB_CS_MAX_FIELDS 5

typedef struct pb_cell_fields {
  double *field[PB_CS_MAX_FIELDS];
  int nf;
  const int64_t *offs;
  int64_t *counts;
  int64_t nc;
} pb_cell_fields;

/* Movers (mover.py:74-110): dest, src_cell, src_slot and the fields, x
 * already normalised to the destination cell. */
typedef struct pb_movers {
  double *field[PB_CS_MAX_FIELDS];
  int64_t *dest;
  int64_t *src_cell;
  int64_t *src_slot;
} pb_movers;

/* Scratch for pb_push_velocity / pb_resort_count. */
size_t pb_cs_scratch_bytes(int64_t nc);

/* push_velocity (mover.py:43-54): vx[live k] += coef * e_p[k], e_p in live
 * (cell-major) order. */
int pb_push_velocity(const double *e_p, double coef, double *vx,
                     const int64_t *offs, const int64_t *counts, int64_t nc,
                     void *scratch, size_t scratch_bytes, void *stream);

/* resort_collect, pass 1 (mover.py:136-148): movers per cell into
 * mover_counts[nc+1] (last entry 0), their exclusive scan into
 * mover_base[nc+1] (mover_base[nc] = total), and the slot of the first
 * particle whose displacement reaches across nc_global cells into *cfl_slot
 * (UINT64_MAX when none). */
int pb_resort_count(const double *x, const int64_t *offs, const int64_t *counts,
                    int64_t nc, int64_t nc_global, int64_t *mover_counts,
                    int64_t *mover_base, uint64_t *cfl_slot, void *scratch,
                    size_t scratch_bytes, void *stream);

/* resort_collect, pass 2 (mover.py:149-181): movers written in (src_cell,
 * src_slot) order at mover_base, dest wrapped into [0, nc_global) with the
 * carry rule, survivors compacted in slot order, vacated slots zeroed,
 * counts updated.  `lo` is the store's global cell offset. */
int pb_resort_collect(const pb_cell_fields *s, const pb_movers *m, int64_t lo,
                      int64_t nc_global, const int64_t *mover_base, void *stream);

/* commit_incomers (mover.py:185-195): mover order[t] goes to slot
 * offs[j] + counts[j] + rank[t] of its destination cell j = dest - lo;
 * `order` is lexsort(dest, src_cell, src_slot).  Capacity is the caller's
 * (grow first); counts are not updated here. */
int pb_commit_place(const pb_cell_fields *s, const pb_movers *m,
                    const int64_t *order, const int64_t *rank, int64_t n,
                    int64_t lo, void *stream);

/* Copy live segments to new per-cell offsets (capacity growth,
 * core.py:220-240); dst must be zeroed. */
int pb_repack(const double *src, double *dst, const int64_t *offs_old,
              const int64_t *offs_new, const int64_t *counts, int64_t nc,
              void *stream);

/* ---- Multi-GPU density exchange over peer memory --------------------------
 * The per-step density allreduce fused with the epilogue: one kernel per
 * rank sums its slice of the fixed-point bins out of every rank's memory
 * (CUDA IPC mappings over NVLink; exact integer sums), computes
 * left/right/rho there and stores the slice into every rank's buffers, with
 * flag barriers in peer memory.  Replaces reduce_bins (the NCCL allreduce)
 * + pb_density_step; bitwise the same result.  All ranks call it with the
 * same epoch sequence (1, 2, ... or a device counter), grid and nc. */
#define PB_MAX_RANKS 8
#define PB_PEER_HANDLE_BYTES 64 /* sizeof(cudaIpcMemHandle_t) */

typedef struct pb_peer_density {
  uint64_t *bins[PB_MAX_RANKS];  /* every rank's current bin set (this rank's: its own) */
  double *left[PB_MAX_RANKS];
  double *right[PB_MAX_RANKS];
  double *rho[PB_MAX_RANKS];
  uint64_t *flags[PB_MAX_RANKS]; /* PB_PEER_FLAG_WORDS zeroed words per rank:
                                    arrive epochs, done counts, error word */
  int rank;
  int world;
  uint64_t epoch;                /* 1, 2, ... one per call (when epoch_dev is NULL) */
  uint64_t *epoch_dev;           /* or: a zeroed device counter of this rank, read as
                                    epoch - 1 and advanced after the exchange, so the
                                    call can be captured in a CUDA graph */
  uint64_t timeout_ns;           /* barrier wait bound (0 = 60 s); on timeout the
                                    failing epoch is published to every rank, and
                                    every rank flags PB_ERR_PEER (sticky) */
} pb_peer_density;
#define PB_PEER_FLAG_WORDS (2 * PB_MAX_RANKS + 1)

/* cudaMalloc + zero + IPC handle (PB_PEER_HANDLE_BYTES) for a buffer peers map. */
int pb_peer_alloc(size_t bytes, void **ptr, void *handle_out);
/* Map a peer's buffer from its handle. */
int pb_peer_open(const void *handle, void **ptr);
/* Unmap (owned = 0) or free (owned = 1). */
int pb_peer_close(void *ptr, int owned);
/* One density exchange + epilogue (see above); bins_next (optional) is
 * zeroed as well, like pb_density_step's.  A timeout or a peer's failure
 * sets PB_ERR_PEER in *status on every rank and leaves the bins uncleared;
 * bin overflow as pb_rho_epilogue.  PB_ERR_INVALID if the grid could not be
 * co-resident. */
int pb_peer_density_step(const pb_peer_density *p, uint64_t *bins_next,
                         const double *coef, int ndep, int64_t nc,
                         int field_bc, pb_status *status, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PICMC_B200_H */
