/*
 * dg.h -- C ABI of libdg, the B200 (sm_100a) fp64 dGSEM right-hand side of
 * the tree-based AMR method of arXiv 2404.16648 ("Comparison of adaptive mesh
 * refinement techniques for numerical weather prediction").
 *
 * Citations: PAPER.md lines (section) and readings Rnn of DESIGN.md section 3.
 * No CUDA or torch types appear here: device buffers are plain pointers,
 * streams are `void*` holding a cudaStream_t (NULL = legacy default stream).
 *
 * Data layout (R27, R28):
 *   state q[e*elem_stride + f*Np + n], e = element in upload order,
 *   f = field (2D: rho, rho*u, rho*w, rho*theta; 3D: rho, rho*u, rho*v, rho*w,
 *   rho*theta), n = i + (N+1) j (+ (N+1)^2 k), x fastest; Np = (N+1)^dim.
 *   elem_stride >= F*Np doubles, a multiple of 16 doubles (128 B) so every
 *   element row starts on a cache line.  Padding doubles are never read.
 *   The vertical (gravity) axis is the last one: z = axis dim-1.
 *
 * Ownership: host arrays are copied during the call; device buffers are
 * caller-owned, must stay alive until the stream work completes, and are never
 * freed by the library.  The context owns its device tables (element
 * descriptors, mortar lists, operators, background copy, scratch) and frees
 * them in dg_destroy.
 *
 * Asynchrony: kernel calls are stream ordered and neither allocate nor
 * synchronise, except where stated (mesh upload, integrals, *_host variants).
 *
 * Errors: every entry point returns a dg_status; on failure a thread-local
 * message is available from dg_last_error().  Argument and precondition
 * failures are detected on the host before any launch.  Asynchronous device
 * faults surface at the caller's next synchronisation.
 *
 * Thread safety: one host thread per context at a time.
 */
#ifndef DG_H_
#define DG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dg_ctx dg_ctx;

typedef enum {
  DG_OK = 0,
  DG_ERR_ARG = -1,          /* bad argument (null pointer, range, dt <= 0, bad stage, aliasing) */
  DG_ERR_UNSUPPORTED = -2,  /* dim/order not compiled in                                         */
  DG_ERR_MESH = -3,         /* leaf overlap, gap, duplicate, out-of-range anchor, no mesh yet    */
  DG_ERR_UNBALANCED = -4,   /* a face joins leaves more than one level apart (R15; not fixed up) */
  DG_ERR_STATE = -5,        /* background table missing or wrong size                            */
  DG_ERR_CUDA = -6,         /* CUDA runtime error (message in dg_last_error)                     */
  DG_ERR_OOM = -7           /* device allocation failed                                          */
} dg_status;

typedef struct {
  int32_t dim, order;          /* dim 2 (x,z) or 3 (x,y,z); LGL order N in 1..8                   */
  int32_t root[3];             /* root-grid cells per axis (unused axes ignored)                  */
  double lo[3], hi[3];         /* domain box [m]                                                  */
  int32_t periodic[3];         /* 1 periodic, 0 no-flux wall at both ends (R9, R10)               */
  int32_t max_level;           /* deepest refinement level allowed, 0..8                           */
  double gamma, R, cp, p0, g;  /* EOS constants and gravity (R4)                */
} dg_params;

/* Create a context: validates params and builds the 1D LGL operator set
 * (nodes, weights, D, and the mortar/transfer projections P_b = M^-1 S_b,
 * R_b = 1/2 M^-1 S_b^T of PAPER.md:290-310).  Does not touch the GPU. */
dg_status dg_create(const dg_params* params, dg_ctx** out);
void dg_destroy(dg_ctx* ctx);
const char* dg_last_error(void);

/* Host-only connectivity build from a leaf list: level[n]
 * (0..max_level) and anchor[n*dim] (integer cell coordinates at the leaf's
 * own level).  Checks duplicates, overlaps, gaps (DG_ERR_MESH) and face 2:1
 * balance including periodic seams (DG_ERR_UNBALANCED), then builds the
 * canonical face lists (R29) and per-element face descriptors. */
dg_status dg_mesh_build(dg_ctx* ctx, int64_t n_leaves, const int8_t* level, const int32_t* anchor);

/* dg_mesh_build + upload of the device tables on `stream`; synchronises the
 * stream before returning (it replaces device tables in use). */
dg_status dg_mesh_upload(dg_ctx* ctx, int64_t n_leaves, const int8_t* level, const int32_t* anchor,
                         void* stream);

/* Canonical face lists (R29), host output buffers sized from the counts:
 *   conf    [n_conf][4]          eL, fL, eR, fR  (owner eL = minus side, emitted from its + face)
 *   nonconf [n_nonconf][2+2*2^(dim-1)]  eC, fC, (eF, fF) x 2^(dim-1) ordered by b_t1 + 2 b_t2
 *   bnd     [n_bnd][2]           e, f
 * Local faces f = 2*axis + (side > 0).  Any output pointer may be NULL. */
dg_status dg_mesh_face_counts(const dg_ctx* ctx, int64_t* n_conf, int64_t* n_nonconf, int64_t* n_bnd);
dg_status dg_mesh_faces(const dg_ctx* ctx, int32_t* conf, int32_t* nonconf, int32_t* bnd);

dg_status dg_state_layout(const dg_ctx* ctx, int64_t* n_elem, int32_t* n_fields, int32_t* n_nodes,
                          int64_t* elem_stride);
/* Convenience allocation of one state array (n_elem * elem_stride doubles). */
dg_status dg_state_alloc(const dg_ctx* ctx, double** out, void* stream);
dg_status dg_state_free(double* q, void* stream);

/* Hydrostatic background table (R3), device
 * pointer, rows (rho_bar, Theta_bar, P_bar) ordered (level, iz, k):
 * row(level, iz, k) = sum_{l<level} root_z 2^l (N+1) + iz (N+1) + k.
 * n_rows must equal sum_{l<=max_level} root_z 2^l (N+1).  Copied (async). */
dg_status dg_set_background(dg_ctx* ctx, const double* table, int64_t n_rows, void* stream);

/* Strong-form dGSEM right-hand side dq/dt = L(q):
 * volume flux divergence with the LGL D matrix, gravity source -rho' g,
 * Rusanov fluxes on conforming, wall and periodic faces, mortar fluxes on
 * 2:1 faces, lifted at the face nodes.  q, dqdt: device,
 * dqdt must not alias q. */
dg_status dg_rhs(dg_ctx* ctx, const double* q, double* dqdt, void* stream);

/* One SSP-RK3 Shu-Osher stage fused with the RHS (R17):
 *   q_out = q_n + b_s ((q_in - q_n) + dt L(q_in)),  b = {1, 1/4, 2/3}
 * (stage 0: q_out = q_in + dt L(q_in); q_n is not read).  q_out must not
 * alias q_in or q_n (neighbours read q_in traces); q_n == q_in allowed only at
 * stage 0.  dt must be finite and > 0. */
dg_status dg_rk_stage(dg_ctx* ctx, int32_t stage, double dt, const double* q_n, const double* q_in,
                      double* q_out, void* stream);

/* dg_rhs / dg_rk_stage restricted to a list of local elements (NEXT-4 overlap, §3.1):
 * elems[0 .. n) (device, int32, distinct rows < n_local) are computed with exactly the
 * arithmetic of the full call -- the union of disjoint lists gives the full call's result
 * bitwise; rows not listed are not written.  A partitioned rank computes its interior
 * elements (no face neighbour in another part) while the halo exchange is in flight, then
 * the boundary elements.  Errors as dg_rhs / dg_rk_stage; DG_ERR_ARG for n < 0 or a null
 * list with n > 0; DG_ERR_UNSUPPORTED with viscosity (mu > 0). */
dg_status dg_rhs_elems(dg_ctx* ctx, const double* q, double* dqdt, int64_t n, const int32_t* elems, void* stream);
dg_status dg_rk_stage_elems(dg_ctx* ctx, int32_t stage, double dt, const double* q_n, const double* q_in,
                            double* q_out, int64_t n, const int32_t* elems, void* stream);

/* Conservative transfer (R16), device index arrays:
 * refine:  children child0_dst[i] .. +2^dim-1 (child id b = bx + 2by + 4bz)
 *          = (kron_axis P_{b_axis}) q_src[parent_src[i]]
 * coarsen: q_dst[parent_dst[i]] = sum_b (kron_axis R_{b_axis}) q_src[child0_src[i] + b]
 * Both arrays use this context's elem_stride. q_dst must not alias q_src. */
dg_status dg_amr_project_refine(const dg_ctx* ctx, int64_t n, const int32_t* parent_src,
                                const int32_t* child0_dst, const double* q_src, double* q_dst, void* stream);
dg_status dg_amr_project_coarsen(const dg_ctx* ctx, int64_t n, const int32_t* child0_src,
                                 const int32_t* parent_dst, const double* q_src, double* q_dst, void* stream);
/* q_dst[dst[i]] = q_src[src[i]] (whole elements; device index arrays). */
dg_status dg_copy_elements(const dg_ctx* ctx, int64_t n, const int32_t* src, const int32_t* dst,
                           const double* q_src, double* q_dst, void* stream);

/* out_host[f] = sum_e prod_d (h_d/2) sum_n w_n q_f,n (R20): per-element sums
 * on the device, Neumaier-compensated sum over elements on the host.
 * Synchronises the stream. */
dg_status dg_integrals(const dg_ctx* ctx, const double* q, double* out_host, void* stream);

/* State health scan (TYPE ElementField: "rho > 0 at every
 * node (positivity monitored, violation is a diagnostic event)"; SPEC.md:740:
 * exit 3 on numerical failure / NaN).  Not part of the hot path: a monitor the
 * caller runs between steps.  q: device state (this context's layout); reads
 * the n_elem own rows once (8 B per DOF).  out_host[4] (host, int64):
 *   [0] number of non-finite values (NaN, +-Inf) over all E*F*Np DOF,
 *   [1] number of nodes with rho <= 0 (IEEE compare: NaN is not <= 0),
 *   [2] number of nodes with rho*theta <= 0 (last field),
 *   [3] smallest element index with any of [0]-[2], -1 if none.
 * Counts are exact integers (bit-exact with any correct scan).  Uses 32 B of
 * context-owned device scratch (allocated on first use).  Synchronises the
 * stream.  Errors: DG_ERR_ARG (null pointer), DG_ERR_MESH (no mesh). */
dg_status dg_check_state(dg_ctx* ctx, const double* q, int64_t* out_host, void* stream);

/* End-to-end variants on HOST buffers in the compact layout [E][F][Np]
 * (pinned memory recommended): host->device copy, the device computation in
 * context-owned scratch (allocated on first use), device->host copy, then a
 * stream synchronisation.
 *   dg_rhs_host:       dqdt_host = L(q_host)
 *   dg_rk3_step_host:  q_host <- n_steps SSP-RK3 steps of size dt (in place) */
dg_status dg_rhs_host(dg_ctx* ctx, const double* q_host, double* dqdt_host, void* stream);
dg_status dg_rk3_step_host(dg_ctx* ctx, double dt, int32_t n_steps, double* q_host, void* stream);

/* ---------------------------------------------------------------- NEXT-1 regrid
 * Dynamic regrid step (§3.2.1; readings
 * R37-R39 of DESIGN.md).  A regrid is: dg_amr_indicator on the device, a plan
 * on the host from the indicator, then dg_mesh_upload of the plan's leaves and
 * the plan's maps through dg_amr_project_refine / dg_amr_project_coarsen /
 * dg_copy_elements from the old state to a new one (new state sized by the new
 * element count; same elem_stride).
 *
 * Indicator: eta[e] = max over the nodes of element e of
 *   kind 0: |Theta/rho - Theta_bar/rho_bar|   (potential-temperature perturbation)
 *   kind 1: |rho - rho_bar|                   (density perturbation)
 * with the background row of each node.  q device state, eta device double[E].
 * Needs the mesh and background table; stream ordered, no synchronisation. */
dg_status dg_amr_indicator(const dg_ctx* ctx, int32_t kind, const double* q, double* eta, void* stream);

/* Host-only plan from the context's current leaf list (which must be in Morton
 * order, as every plan's output is) and eta_host[E]:
 *   feature cells eta > refine_above, dilated by `buffer` rounds of face
 *   neighbours (each round sweeps x, then y, then z; one interior cell with
 *   buffer 2 -> the 5x5(x5) block around it, R37), refined below max_level with
 *   the 2:1 ripple; families whose children all have eta < coarsen_below and lie
 *   outside the buffered set merge (finest level first) unless that breaks 2:1
 *   balance (R38).  At most one level of change per leaf per regrid.
 * Outputs (dg_regrid_plan_get, caller-sized from dg_regrid_plan_sizes; any
 * pointer may be NULL): the new leaves level[n_leaves], anchor[n_leaves*dim] in
 * Morton order; refine maps (old parent -> new first child), coarsen maps (old
 * first child -> new parent), copy maps (old -> new) -- all int32 element
 * indices.  Errors: DG_ERR_MESH when the old order keeps siblings apart.
 * The plan owns its arrays; free with dg_regrid_plan_destroy. */
typedef struct dg_regrid_plan dg_regrid_plan;
dg_status dg_regrid_plan_create(const dg_ctx* ctx, const double* eta_host, double refine_above, double coarsen_below,
                                int32_t buffer, dg_regrid_plan** out);
dg_status dg_regrid_plan_sizes(const dg_regrid_plan* plan, int64_t* n_leaves, int64_t* n_refine, int64_t* n_coarsen,
                               int64_t* n_copy);
dg_status dg_regrid_plan_get(const dg_regrid_plan* plan, int8_t* level, int32_t* anchor, int32_t* refine_parent,
                             int32_t* refine_child0, int32_t* coarsen_child0, int32_t* coarsen_parent,
                             int32_t* copy_src, int32_t* copy_dst);
void dg_regrid_plan_destroy(dg_regrid_plan* plan);

/* ---------------------------------------------------------------- NEXT-4 partition
 * Domain decomposition for one process per GPU.  Every
 * rank passes the same global leaf list (Morton order); it is split into n_parts
 * contiguous ranges (global elements [n*k/n_parts, n*(k+1)/n_parts) for part k --
 * a space-filling-curve partition) and this context keeps part `part` plus its
 * halo: the remote elements its kernels read (face neighbours, the fine elements
 * of its coarse faces, the coarse element of its fine faces).
 *
 * Local row order: the part's own elements (global order), then the halo grouped
 * by owning part k ascending, each group in global order.  dg_state_layout then
 * reports n_elem = n_local + n_halo rows (allocate that many); dg_rhs /
 * dg_rk_stage / dg_integrals / dg_amr_indicator compute the n_local own rows and
 * READ the halo rows, which the caller must refresh from the owners before every
 * RHS evaluation (each RK stage input): rows received from part k go to
 * n_local + sum_{j<k} recv_count[j] ... (+ recv_count[k]); the rows to send to part k
 * are send_idx[sum_{j<k} send_count[j] ...] (local indices).  Face adjacency is
 * mutual, so part r's send list to k is, row for row, k's halo group from r.
 * dg_integrals returns this part's sums (the caller reduces over parts).
 * The *_host variants and the regrid planner reject partitioned contexts.
 * dg_mesh_build_part is the host-only build (no device tables). */
dg_status dg_mesh_build_part(dg_ctx* ctx, int64_t n_leaves, const int8_t* level, const int32_t* anchor,
                             int32_t n_parts, int32_t part);
dg_status dg_mesh_upload_part(dg_ctx* ctx, int64_t n_leaves, const int8_t* level, const int32_t* anchor,
                              int32_t n_parts, int32_t part, void* stream);
dg_status dg_part_info(const dg_ctx* ctx, int32_t* n_parts, int32_t* part, int64_t* n_local, int64_t* n_halo,
                       int64_t* global_begin);
/* send_count[n_parts], recv_count[n_parts] (0 for the own part), send_idx[sum send_count]. */
dg_status dg_part_exchange_lists(const dg_ctx* ctx, int64_t* send_count, int64_t* recv_count, int32_t* send_idx);
/* Face-trace exchange (the kernels read only the face nodes of a remote element that touch this part):
 * per peer k the (local element, face) pairs to send -- this part's elements with a neighbour across
 * the face in part k -- and the (local halo row, face) pairs to receive, element then face ascending
 * on both sides.  send_pairs[2 * sum send_count], recv_pairs[2 * sum recv_count].  dg_pack_faces
 * gathers the F x Nf face-node values of each pair of q into buf[n][F][Nf]; dg_unpack_faces scatters
 * buf back into the halo rows (device arrays; pairs as int32 (element, face)). */
dg_status dg_part_face_lists(const dg_ctx* ctx, int64_t* send_count, int64_t* recv_count, int32_t* send_pairs,
                             int32_t* recv_pairs);
dg_status dg_pack_faces(const dg_ctx* ctx, int64_t n, const int32_t* pairs, const double* q, double* buf, void* stream);
dg_status dg_unpack_faces(const dg_ctx* ctx, int64_t n, const int32_t* pairs, const double* buf, double* q,
                          void* stream);

/* ---------------------------------------------------------------- NEXT-3 baseline
 * Treatment of 2:1 faces by dg_rhs / dg_rk_stage: mode 0 (default) the mortar method
 * (conservative); mode 1 the paper's comparison baseline, pointwise
 * interpolation (reading R41): each coarse face node takes the containing
 * fine sub-face's trace interpolated at that point; the fine side is unchanged.  Mode 1
 * is NOT conservative (that is its purpose: reproducing the paper's comparison).  For 3D
 * N = 7 it runs on the generic tile kernel (the specialised N = 7 kernel has mortars only). */
dg_status dg_set_nonconforming(dg_ctx* ctx, int32_t mode);

/* NEXT-3 artificial viscosity ("artificial viscosity of mu = 1.5 m^2/s";
 * reading R42): with mu > 0, dg_rhs and dg_rk_stage add V = mu div grad u' of the
 * perturbation vector u' = (rho', U, Theta'), BR1 in strong form with central face values
 * (walls: no diffusive flux; 2:1 faces through the mortars, conservative).  Two extra
 * kernels per RHS evaluation plus context-owned scratch (dim + 1 state arrays, allocated
 * on first use).  mu = 0 (default) turns it off.  Not on partitioned contexts
 * (DG_ERR_UNSUPPORTED: needs a gradient halo exchange). */
dg_status dg_set_viscosity(dg_ctx* ctx, double mu);

/* NEXT-3 kinematic tracer (the paper's LeVeque test, §4.2; reading R43):
 * dC/dt + div(C u) = 0 with a prescribed wind.  Arrays use this context's state layout:
 * field 0 = C, fields 1..dim = the wind at the nodes (the caller writes it for each stage
 * time), other fields unused.  Upwind faces, impermeable walls (F*.n = 0), 2:1 faces by
 * the mortar method or the pointwise baseline (dg_set_nonconforming).
 *   dg_tracer_rhs:      out field 0 = dC/dt
 *   dg_tracer_rk_stage: out field 0 = SSP-RK3 stage (R17) of C; fields 1..dim copied from s_in
 * Device pointers; out must not alias the inputs. */
dg_status dg_tracer_rhs(dg_ctx* ctx, const double* s, double* out, void* stream);
dg_status dg_tracer_rk_stage(dg_ctx* ctx, int32_t stage, double dt, const double* s_n, const double* s_in,
                             double* s_out, void* stream);

/* NEXT-3 passive tracer of the Euler flow (PAPER.md:73-89 eq. eulervector: C = rho c with flux
 * C U / rho and no source; reading R45).  C rides beside the Euler state (one-way coupling): the
 * Rusanov flux F*.n = 1/2 (C- u-.n + C+ u+.n) + 1/2 lambda (C- - C+) with the Euler faces' wave
 * speed lambda (R6), mirror walls (zero flux), 2:1 faces by the mortar method (conservative).
 * Arrays use this context's state rows, field 0 = C (other fields untouched; device pointers):
 *   dg_passive_rhs:      dcdt field 0 = dC/dt for the Euler state q
 *   dg_passive_rk_stage: c_out field 0 = SSP-RK3 stage (R17) of C, with q_in the Euler stage's input
 *                        (call it beside dg_rk_stage with the same q_in); c_n read for stages 1, 2.
 * c_out / dcdt must not alias an input.  DG_ERR_UNSUPPORTED with the pointwise 2:1 mode. */
dg_status dg_passive_rhs(dg_ctx* ctx, const double* q, const double* c, double* dcdt, void* stream);
dg_status dg_passive_rk_stage(dg_ctx* ctx, int32_t stage, double dt, const double* q_in, const double* c_n,
                              const double* c_in, double* c_out, void* stream);

/* Number of CUDA kernels launched by this context since creation (for the
 * bench's gpu_launches accounting). */
int64_t dg_launch_count(const dg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DG_H_ */
