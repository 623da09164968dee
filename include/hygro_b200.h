/*
 * hygro_b200.h — C ABI of the B200-native Dufort–Frankel (DF) wall solver.
 *
 * This is the drop-in boundary for the reference's DF hot path
 * (reference: /root/reference/proj, "hygrosim").  The reference exposes the
 * path as per-wall, per-step C++ calls; on a GPU one launch per wall-step is
 * meaningless, so the boundary moves one level up to a batched, multi-step
 * context that owns the device-resident state of many walls (and zones):
 *
 *   reference call (file:line)                         replaced by
 *   -------------------------------------------------  -------------------------
 *   df_step_coupled(f,grid,p,L,R,dt)  wall.hpp:81-82   hyg_advance  (constant walls)
 *   df_step_nonlinear(...)            wall.hpp:88-90   hyg_advance  (HYG_COEFF_ANALYTIC_D)
 *   euler_explicit_step(...)          wall.hpp:95-97   hyg_bootstrap(HYG_BOOT_EXPLICIT)
 *   bootstrap_first_layer(...)        wall.hpp:119-122 hyg_bootstrap(HYG_BOOT_IMPLICIT)
 *   step_implicit (DF bootstrap)      building.hpp:75  hyg_bootstrap(HYG_BOOT_IMPLICIT)
 *   step_explicit(model,state)        building.hpp:69  hyg_advance  (zones present)
 *   run(model,cadence,partial)        building.hpp:101 hyg_run
 *   check_bounded / max_abs_field     building.cpp:282-300, wall.cpp:579-587
 *                                                      fused guard -> HYG_EDIVERGED
 *   BuildingModel / BuildingWall      building.hpp:24-53  hyg_model_desc
 *   WallField (u/v prev/curr, t_star) wall.hpp:23-29   hyg_set_state / hyg_get_state
 *   Signal::operator()(t)             signal.hpp:39-50 hyg_signal (host-evaluated
 *                                                      per time layer, uploaded as tables)
 *
 * Errors: every call returns an int code.  The codes map one-to-one onto the
 * reference's exception taxonomy (errors.hpp:8-45); include/hygro_b200.hpp
 * rethrows them as the matching C++ exception types.
 *
 * Layout of host state arrays: wall-major, [n_walls][n_nodes] doubles.
 * Plain pointers and sizes only; no CUDA or torch types cross this boundary.
 */
#ifndef HYGRO_B200_H
#define HYGRO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HYG_ABI_VERSION 3

/* ---- return codes (errors.hpp:8-45) ------------------------------------ */
enum {
    HYG_OK = 0,
    HYG_EINVAL = 1,     /* std::invalid_argument   wall.cpp:14,19,519; building.cpp:295 */
    HYG_ESCHEMA = 2,    /* hygro::schema_error     building.cpp:12-52 (validate)        */
    HYG_EDIVERGED = 3,  /* hygro::numerical_error  building.cpp:282-300 (check_bounded) */
    HYG_EDOMAIN = 4,    /* hygro::domain_error     wall.cpp:105-126 (strict StarTables) */
    HYG_ECONVERGE = 5,  /* hygro::convergence_error wall.cpp:538-543, building.cpp:249  */
    HYG_ESCALING = 6,   /* hygro::scaling_error    scaling.cpp:9-16                     */
    HYG_ECUDA = 7,      /* device / driver failure (no reference equivalent)            */
    HYG_ENOTSUP = 8     /* configuration outside what this build implements             */
};

/* ---- dimensionless parameter blocks (scaling.hpp, wall.hpp) ------------ */
typedef struct { double Fo_M, Fo_TT, Fo_TM, gamma; } hyg_wall_groups; /* WallGroups scaling.hpp:20-25 */
typedef struct { double Bi_M, Bi_TT, Bi_TM; } hyg_face_biot;          /* FaceBiot   scaling.hpp:28-32 */
typedef struct { double u_inf, v_inf, g_inf, q_inf; } hyg_ambient;    /* ambient part of FaceValues wall.hpp:32-36 */

/* ---- forcing signals (signal.hpp:13-86) -------------------------------- */
enum { HYG_SIG_CONSTANT = 0, HYG_SIG_SIN = 1, HYG_SIG_SIN2 = 2 };
typedef struct { double from, to, value; } hyg_window; /* Signal::Window signal.hpp:19-21 */
typedef struct {
    int32_t form;            /* HYG_SIG_*                                  */
    int32_t n_windows;       /* additive piecewise-constant schedule       */
    double base, amplitude, period, phase;
    const hyg_window* windows;
} hyg_signal;

/* An exterior forcing channel: the four ambient signals of a face
 * (FaceAttachment::u_inf/v_inf/g_inf/q_inf, building.hpp:17-20). */
typedef struct { hyg_signal u_inf, v_inf, g_inf, q_inf; } hyg_channel;

/* Zone source schedules (ZoneDimensionless::g_o/q_o/q_h, scaling.hpp:63). */
typedef struct { hyg_signal g_o, q_o, q_h; } hyg_zone_sources;

/* ---- topology ----------------------------------------------------------- */
enum { HYG_FACE_EXTERIOR = 0, HYG_FACE_ZONE = 1 };
typedef struct {
    int32_t kind;   /* HYG_FACE_EXTERIOR: index = forcing channel; HYG_FACE_ZONE: index = zone */
    int32_t index;
} hyg_face_attach;   /* FaceAttachment building.hpp:13-21 */

typedef struct {
    int32_t wall, face;                     /* ZoneWallLink zone.hpp:24-29 */
    double Bi_M, Bi_TT, Bi_TM, theta_T, theta_M;
} hyg_zone_wall_link;

typedef struct {
    int32_t peer;                           /* ZoneInterzoneLink zone.hpp:32-35 */
    double g_inz, q_inz1, q_inz2;
} hyg_interzone_link;

enum { HYG_MOISTURE_AS_PRINTED = 0, HYG_MOISTURE_FLUX_CONSISTENT = 1 }; /* zone.hpp:21 */

/* Long-wave exchange between two wall surfaces bounding a zone: the flux
 * s*eps*sigma*(T_e^4 - T_r^4) [W/m2] is added to the receiver face's imposed
 * heat flux, scaled by L/(T_i k_TT0) of the receiving wall (RadiationLink
 * zone.hpp:39-45, radiative_flux zone.cpp:55-67, radiation_fluxes
 * building.cpp:88-105). */
typedef struct {
    int32_t emitter_wall, receiver_wall;
    double view_factor, emissivity;
} hyg_radiation_link;

typedef struct {
    double kappa_a_tt1, g_v, q_v1, q_v2;    /* ZoneDimensionless scaling.hpp:61-67 */
    int32_t sources;                        /* index into hyg_model_desc::zone_sources */
    int32_t moisture_sign;                  /* HYG_MOISTURE_*                          */
    int32_t n_walls;
    const hyg_zone_wall_link* walls;
    int32_t n_interzone;
    const hyg_interzone_link* interzone;
    int32_t n_radiation;                    /* ABI 2: ZoneConfig::radiation            */
    const hyg_radiation_link* radiation;
} hyg_zone_desc;                            /* ZoneConfig zone.hpp:47-54 */

/* ---- coefficient models (CoefficientModel wall.hpp:41-60) -------------- */
enum {
    HYG_COEFF_CONSTANT = 0,   /* CoefficientModel::constant(): all six starred coefficients 1 */
    /* Device functor (API extension; the reference can only express it through
     * the test oracle's StarFn callback, tests/support/df_oracle.hpp:19):
     *   k_M*(u,v) = 1 + p0*v + p1*exp(-p2*(v - p3)^2), other five starred coefficients 1 */
    HYG_COEFF_ANALYTIC_D = 1,
    /* CoefficientModel::material (wall.cpp:33-58): the load-bearing material
     * correlations (MaterialModel::evaluate materials.cpp:91-114, default
     * PhysicalConstants materials.hpp:7-15) at (u*T_i, v*P_vi), divided by the
     * wall's reference set.  Strict in DF steps (box violation -> HYG_EDOMAIN
     * naming wall and node / half node, wall.cpp:99-126), clamped in the
     * starting steps (evaluate_clamped materials.cpp:116-121).  Per wall through
     * hyg_model_desc::wall_coeff (constant walls keep df_step_coupled,
     * building.cpp:172-176). */
    HYG_COEFF_MATERIAL = 2
};

/* CoefficientSet materials.hpp:21-28 */
typedef struct { double c_M, k_M, c_TT, k_TT, c_TM, k_TM; } hyg_coeff_set;

enum { HYG_F64 = 0, HYG_F32 = 1 };
enum { HYG_BOOT_IMPLICIT = 0, HYG_BOOT_EXPLICIT = 1 };

typedef struct {
    int32_t n_walls;
    int32_t n_nodes;          /* Grid1D::n, shared by every wall of a model (wall.hpp:12-19) */
    double dx;                /* Grid1D::dx                                              */
    int32_t precision;        /* HYG_F64, or HYG_F32 (fp32 state + fp64 boundary fluxes)  */
    int32_t coeff_kind;       /* HYG_COEFF_*                                             */
    double coeff_params[4];
    const hyg_wall_groups* groups;    /* [n_walls]                                       */
    const hyg_face_biot* biot;        /* [n_walls][2]; [0] is x*=0, [1] is x*=1          */
    const hyg_face_attach* attach;    /* [n_walls][2]                                    */
    int32_t n_channels;
    const hyg_channel* channels;      /* [n_channels]                                    */
    int32_t n_zones;
    const hyg_zone_desc* zones;       /* [n_zones]                                       */
    int32_t n_zone_sources;
    const hyg_zone_sources* zone_sources;
    hyg_signal outdoor_u, outdoor_v;  /* BuildingModel::outdoor_u/v building.hpp:41-42  */
    double dt;                        /* BuildingModel::dt                               */
    double divergence_norm;           /* BuildingModel::divergence_norm (default 1e3)    */
    double eta_factor;                /* BuildingModel::eta_factor (implicit bootstrap)  */
    int32_t max_subiters;             /* BuildingModel::max_subiters                     */
    int32_t device;                   /* CUDA ordinal                                    */
    /* ---- ABI 2: material walls and radiation -------------------------------- */
    double T_i, P_vi;                 /* ScalingContext (scaling.hpp:11-16)              */
    const int32_t* wall_coeff;        /* [n_walls] HYG_COEFF_CONSTANT / _MATERIAL when
                                         coeff_kind == HYG_COEFF_MATERIAL; NULL: all material */
    const hyg_coeff_set* wall_reference; /* [n_walls] CoefficientModel::reference_ of
                                         material walls (NULL only without material walls) */
    const double* wall_thickness;     /* [n_walls] BuildingWall::thickness (radiation)   */
    const double* wall_k_TT0;         /* [n_walls] BuildingWall::k_TT0     (radiation)   */
} hyg_model_desc;

typedef struct {
    int32_t code;            /* HYG_*                                          */
    int32_t wall;            /* first failing wall (lowest index), -1 if none  */
    int32_t zone;            /* failing zone, -1 if none                       */
    int32_t subiterations;   /* implicit bootstrap passes (StepReport)         */
    int64_t layer;           /* time-layer index after the failing step        */
    double t_star;           /* numerical_error::t_star                         */
    double residual;         /* convergence_error::residual                    */
    int32_t node;            /* ABI 2, HYG_EDOMAIN: node j, or half node j+1/2  */
    int32_t half;            /*   when half == 1 (StarTables wall.cpp:105-126)  */
    char message[256];
} hyg_status;

typedef struct hyg_ctx hyg_ctx;

int hyg_abi_version(void);
const char* hyg_strerror(int code);

/* Validates (BuildingModel::validate building.cpp:12-52), uploads parameters,
 * allocates device state.  State starts uniform at 1 (WallField::uniform). */
int hyg_create(const hyg_model_desc* desc, hyg_ctx** out, hyg_status* status);
void hyg_destroy(hyg_ctx* ctx);

/* Host <-> device state.  Arrays are [n_walls*n_nodes] wall-major; zone
 * arrays are [n_zones] (may be NULL when n_zones == 0).  t_star is the
 * time of layer "curr" (BuildingState::t).  `layer` is the integer index of
 * layer curr (0 after initialisation). */
int hyg_set_state(hyg_ctx* ctx, const double* u_prev, const double* u_curr,
                  const double* v_prev, const double* v_curr,
                  const double* zone_u, const double* zone_v, double t_star, int64_t layer);
int hyg_get_state(hyg_ctx* ctx, double* u_prev, double* u_curr, double* v_prev,
                  double* v_curr, double* zone_u, double* zone_v, double* t_star,
                  int64_t* layer);

/* Sub-range access for halo exchange between shards (fp64 models).  Cells
 * are the flattened wall-major index w*n_nodes + j; any pointer may be NULL
 * to skip that layer.  Zones [zone0, zone0+count).  Pointers may be host
 * (pageable or pinned) or device memory of any GPU (cudaMemcpyDefault over
 * UVA): shards exchange halos device to device, e.g. straight into NCCL
 * buffers, with no host staging.  Each call returns after the copy. */
int hyg_get_cells(hyg_ctx* ctx, int64_t cell0, int64_t count, double* u_prev, double* u_curr,
                  double* v_prev, double* v_curr);
int hyg_set_cells(hyg_ctx* ctx, int64_t cell0, int64_t count, const double* u_prev,
                  const double* u_curr, const double* v_prev, const double* v_curr);
int hyg_get_zones(hyg_ctx* ctx, int32_t zone0, int32_t count, double* zone_u, double* zone_v);
int hyg_set_zones(hyg_ctx* ctx, int32_t zone0, int32_t count, const double* zone_u,
                  const double* zone_v);
/* Stream-ordered halo payloads (multi-GPU shards): pack the cells [cell0,
 * cell0+count) of the four layers into buf[4][count] (device memory of the
 * context's GPU), or unpack buf into them; zones into/from buf[2][count]
 * (zone_u then zone_v).  Enqueued on the context's stream with no host
 * synchronisation: a caller that hands the context its communication stream
 * (hyg_set_stream) orders NCCL sends/receives of buf behind and ahead of them
 * by stream order alone.  One launch per call. */
/* The pack / unpack calls below run on `stream` (a cudaStream_t) instead of the
 * context's stream; NULL: on the context's stream again.  No implicit ordering:
 * the caller orders the two streams with events (shard.py: the exchange stream
 * waits for the interval's compute, hyg_advance_overlapped takes the event
 * recorded behind the unpack). */
int hyg_set_exchange_stream(hyg_ctx* ctx, void* stream);
int hyg_pack_cells(hyg_ctx* ctx, int64_t cell0, int64_t count, double* buf);
int hyg_unpack_cells(hyg_ctx* ctx, int64_t cell0, int64_t count, const double* buf);
int hyg_pack_zones(hyg_ctx* ctx, int32_t zone0, int32_t count, double* buf);
int hyg_unpack_zones(hyg_ctx* ctx, int32_t zone0, int32_t count, const double* buf);
/* Launch everything on `stream` (a cudaStream_t of the context's device;
 * NULL: the context's own stream), ordered after the work already issued. */
int hyg_set_stream(hyg_ctx* ctx, void* stream);

/* Restricts the divergence guard and the implicit starting step's
 * fixed-point residual to the cells [cell0, cell1) and zones [zone0, zone1)
 * a shard owns (its halo copies are excluded), and reduces the residual
 * across shards through `reduce` (max; NULL = local only).  Default: all. */
typedef double (*hyg_reduce_fn)(void* user, double local_max);
int hyg_set_owned(hyg_ctx* ctx, int64_t cell0, int64_t cell1, int32_t zone0, int32_t zone1,
                  hyg_reduce_fn reduce, void* user);

/* Device-resident checkpoint of the complete resumable state (both time
 * layers of every wall, zone states, t_star, layer index — the state a DF
 * march needs, wall.hpp:23-29 + building.hpp:55-59).  hyg_snapshot copies
 * the current state into the context's snapshot buffer; hyg_restore copies
 * it back.  Device-to-device only. */
int hyg_snapshot(hyg_ctx* ctx);
int hyg_restore(hyg_ctx* ctx);

/* Overrides channel `channel` with explicit ambient values for time layers
 * [first_layer, first_layer + n_layers): the value used by the step that
 * starts at layer n (forcing at layer-n time, building.cpp:153,168-169) and by
 * the implicit bootstrap into layer n (t^{n+1} forcing, building.cpp:196). */
int hyg_set_channel_table(hyg_ctx* ctx, int32_t channel, int64_t first_layer,
                          int64_t n_layers, const hyg_ambient* values);

/* Per-layer overrides of the zone source schedules (source `source`:
 * values [n_layers][3] = g_o, q_o, q_h) and of the outdoor signals
 * (values [n_layers][2] = u, v), same layer convention as channel tables.
 * With these, a caller holding opaque Signal objects (signal.hpp exposes only
 * operator()(t)) evaluates them itself at the layer times. */
int hyg_set_source_table(hyg_ctx* ctx, int32_t source, int64_t first_layer, int64_t n_layers,
                         const double* values);
int hyg_set_outdoor_table(hyg_ctx* ctx, int64_t first_layer, int64_t n_layers, const double* values);

/* One starting step producing layer 1 from layer 0 (run() counts it as step 1,
 * building.cpp:317-323).  Guarded like every step. */
int hyg_bootstrap(hyg_ctx* ctx, int32_t kind, hyg_status* status);

/* nsteps DF steps with time step dt (dt <= 0: the model dt), each followed by
 * the divergence guard.  On HYG_EDIVERGED the state is left at the last
 * layer that passed the guard for every wall and status names the first
 * failing layer and the lowest failing wall index. */
int hyg_advance(hyg_ctx* ctx, int64_t nsteps, double dt, hyg_status* status);
/* hyg_advance for a shard whose halo cells are being refreshed on ANOTHER stream
 * (shard.py: pack -> NCCL -> unpack behind the previous interval): `event` is a
 * cudaEvent_t recorded on that stream after the refresh of the first edge_lo and
 * the last edge_hi cells of the context.  On the long-wall path (K3w) the windows
 * of the first launch that read none of those cells are launched at once — they
 * march while the exchange is in flight — and the remaining windows, the face
 * windows and every later launch follow behind the event in stream order; on
 * every other path the context's stream waits for the event first.  Same results
 * as hyg_advance after the refresh.  event == NULL: hyg_advance. */
int hyg_advance_overlapped(hyg_ctx* ctx, int64_t nsteps, double dt, int64_t edge_lo, int64_t edge_hi, void* event,
                           hyg_status* status);

/* run() building.cpp:303-356: nsteps = lround(horizon/dt); DF bootstrap
 * (`boot_kind`) counted as step 1; frames every lround(cadence/dt) steps and
 * at the end through `frame` (may be NULL), which may call hyg_get_state. */
typedef void (*hyg_frame_fn)(void* user, int64_t layer, double t_star, hyg_ctx* ctx);
int hyg_run(hyg_ctx* ctx, double horizon, double cadence, int32_t boot_kind,
            hyg_frame_fn frame, void* user, hyg_status* status);

/* run() for each of the reference's schemes (Scheme wall.hpp:62, building.cpp:303-356):
 * DF (implicit start + DF steps), EulerImplicit (step_implicit every step, the
 * paper's comparison baseline) and EulerExplicit (step_explicit with
 * euler_explicit_step walls).  `report` (may be NULL) receives
 * SimulationResult's counters. */
enum { HYG_SCHEME_DF = 0, HYG_SCHEME_EULER_IMPLICIT = 1, HYG_SCHEME_EULER_EXPLICIT = 2 };
typedef struct {
    int64_t steps;
    int32_t bootstrap_subiters;
    int32_t max_subiters_seen;
    double mean_subiters;
} hyg_run_report;   /* SimulationResult building.hpp:86-93 */
int hyg_run_scheme(hyg_ctx* ctx, int32_t scheme, double horizon, double cadence, hyg_frame_fn frame,
                   void* user, hyg_run_report* report, hyg_status* status);


/* df_step_linear (wall.hpp:73-74, wall.cpp:60-71; the single-field DF form of
 * the paper's Eq. 8, boundary nodes copied) applied `steps` times, with the
 * layer rotation of wall.cpp:80-83, to n_fields independent fields of n nodes
 * on the device: prev/curr ([n_fields][n], host or device pointers) hold
 * layers n-1 and n on entry and the last two layers on return.  The
 * reference's property tests use this form (test_wall.cpp:43-61, 171-194). */
int hyg_df_march_linear(int32_t device, int32_t n_fields, int32_t n, double lambda, int64_t steps,
                        double* prev, double* curr);

/* ---- host-side setup: dimensionless groups (scaling.cpp, materials.cpp) -
 * Coefficient sets are {c_M, k_M, c_TT, k_TT, c_TM, k_TM} (CoefficientSet,
 * materials.hpp:21-28).  Scaling context from (T_i [K], phi_i, t_0 [s]),
 * ScalingContext::from_state scaling.cpp:20-28. */
int hyg_saturation_pressure(double T, double* out);                         /* materials.cpp:33-40 */
/* MaterialModel::evaluate / evaluate_clamped (materials.cpp:91-121) on the
 * host: e.g. the reference set of a material wall, evaluate(T_i, P_vi)
 * (scenario.cpp:178).  HYG_EDOMAIN outside the admissible box. */
int hyg_material_evaluate(double T, double P_v, int32_t clamped, hyg_coeff_set* out);
int hyg_scale_wall(const double reference[6], double L, double h_T0, double h_M0, double h_T1,
                   double h_M1, double T_i, double phi_i, double t_0, hyg_wall_groups* groups,
                   hyg_face_biot face[2]);                                   /* scaling.cpp:30-58 */
/* out = {kappa_a_tt1, g_v, q_v1, q_v2, g_o per kg/s, q_o per kg/s, q_h per W} */
int hyg_scale_zone(double volume, double rho_a, double c_pa, double c_pv, double ventilation_ach,
                   double T_i, double phi_i, double t_0, double out[7]);     /* scaling.cpp:60-83 */
/* out = {theta_T, theta_M} */
int hyg_attach_wall_to_zone(const double reference[6], double area, double L, double volume,
                            double rho_a, double c_pa, double T_i, double phi_i, double t_0,
                            double out[2]);                                  /* scaling.cpp:85-90 */
/* out = {g_inz, q_inz1, q_inz2} */
int hyg_scale_interzone(double ach, double volume, double rho_a, double c_pa, double c_pv,
                        double T_i, double phi_i, double t_0, double out[3]); /* scaling.cpp:92-101 */

/* ---- measurement hooks (bench.py) --------------------------------------- */
int hyg_synchronize(hyg_ctx* ctx);
int hyg_host_register(void* ptr, size_t bytes);   /* cudaHostRegister (pinned H2D/D2H) */
int hyg_host_unregister(void* ptr);
/* CUDA events on the context's stream; slot in [0, 16). */
int hyg_event_record(hyg_ctx* ctx, int32_t slot);
int hyg_event_elapsed_ms(hyg_ctx* ctx, int32_t slot_a, int32_t slot_b, double* ms);
/* Per-kernel launch accounting (CUDA events around every launch while on). */
int hyg_set_profiling(hyg_ctx* ctx, int32_t on);
int hyg_kernel_stats_count(hyg_ctx* ctx);
int hyg_kernel_stats(hyg_ctx* ctx, int32_t i, const char** name, int64_t* launches,
                     double* total_ms, double* node_updates);
int hyg_reset_kernel_stats(hyg_ctx* ctx);
/* Number of kernels this context has launched since creation. */
int64_t hyg_launch_count(hyg_ctx* ctx);

/* Launch-shape knobs (an extension; the reference has no launch shapes).
 * HYG_TUNE_RING_GRID: cap on the persistent zone-ring kernel's grid (K4r,
 * k_ring_reg.cuh; 0 = one CTA per SM).  A cap below the number of zone blocks
 * makes every CTA walk several blocks, so small rings under test run the
 * next-block prefetch path the full-size ring runs (for K6 it caps the walls
 * kernel's grid, so every warp walks several wall pairs).  HYG_TUNE_RING_KERNEL
 * picks the zone-ring kernel: 0 = automatic (K6 k_ring_split.cuh where it
 * applies: zone air + wall cones first, then every wall in registers), 1 = K4r
 * (k_ring_reg.cuh), 2 = K4 (k_ring.cuh), 3 = K5 (k_ring_pipe.cuh: S = 12,
 * trimmed halo, named-barrier hand-off), 4 = K6; all bitwise equal, for A/B
 * measurement and cross-checks.  HYG_TUNE_MATERIAL_EXACT = 1 evaluates
 * the load-bearing material with the accurate exp/log/pow of hyg_crmath.cuh
 * (glibc's roundings in all but rare cases), the reference's expressions and
 * IEEE divisions — ~8x slower than the default (0) table-driven evaluation with
 * reciprocal quotients, which is a few ulp per coefficient.  Both agree with
 * the reference within its own conditioning: on the ill-conditioned
 * wall_nonlinear fixture (a 1-ulp change of one initial value moves the
 * reference by 8e-10) they differ from it by 9.6e-10 (exact) and 1.7e-9
 * (default); on the other fixtures and tests by ~1e-14.  HYG_TUNE_RING_DEPTH = m (1..3) makes K6's
 * walls kernel march m x 8 steps per launch, fed by m cone launches (the later
 * ones on tails a stub kernel marches ahead); bitwise equal for every m.
 * HYG_TUNE_TILED_LOAD picks how the long-wall
 * kernel K3w stages its windows and K6's walls kernel its wall pairs: 0 = 2-D
 * tiles on the TMA engine through tensor maps of the state arrays
 * (k_dv_tiled_tma; k_ring_walls<.., true>), 1 = per-lane cp.async copies
 * (k_dv_tiled_stream) / 1-D bulk copies with rotated shared accesses; bitwise equal.  HYG_EINVAL for an unknown knob or a
 * negative value. */
enum { HYG_TUNE_RING_GRID = 1, HYG_TUNE_RING_KERNEL = 2, HYG_TUNE_MATERIAL_EXACT = 3, HYG_TUNE_TILED_LOAD = 4,
       HYG_TUNE_RING_DEPTH = 5 };
int hyg_set_tuning(hyg_ctx* ctx, int32_t knob, int64_t value);

/* Device FP64 FMA throughput probe (DFMA loop), TFLOP/s counting FMA = 2. */
int hyg_probe_fp64_peak(int32_t device, double* tflops, double* sm_clock_mhz);
/* Self-test of the device exp/reciprocal used by the d(v) rows
 * (hyg_fastmath.cuh): exp_out[i] = exp(x[i]), rcp_out[i] = 1/x[i] on the device. */
int hyg_selftest_fastmath(int32_t device, int32_t n, const double* x, double* exp_out, double* rcp_out);
/* The d(v) half node's exp and the v row's two-FMA reciprocal (fexp_addend, frcp2):
 * exp_out[i] = exp(-|x[i]|) for |x[i]| <= 700, rcp_out[i] ~ 1/x[i] (relative error
 * below 1.1e-12, towards zero). */
int hyg_selftest_dvmath(int32_t device, int32_t n, const double* x, double* exp_out, double* rcp_out);
/* Self-test of the device log of the material correlations (flog_pos,
 * hyg_fastmath.cuh; positive normal x): log_out[i] = ln x[i] on the device. */
int hyg_selftest_fastlog(int32_t device, int32_t n, const double* x, double* log_out);
/* Self-test of the accurate device exp/log/log10/pow of the material parity
 * path (hyg_crmath.cuh): out[0..n) = exp(x), [n..2n) = log(x), [2n..3n) =
 * log10(x), [3n..4n) = pow(x, y), computed on the device. */
int hyg_selftest_crmath(int32_t device, int32_t n, const double* x, const double* y, double* out);
/* Device FP32 FMA throughput probe (FFMA loop), TFLOP/s counting FMA = 2. */
int hyg_probe_fp32_peak(int32_t device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* HYGRO_B200_H */
