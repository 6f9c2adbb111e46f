/*
 * links_b200.h — C ABI of the B200-native LINKS hot path (sm_100a).
 *
 * The reference (`linkatlas`, /root/reference/pkg/src/linkatlas) is pure
 * Python: its "interface" for this path is a set of Python functions, not an
 * FFI.  Each entry point below replaces the numpy body of one of them; the
 * Python mirror in paper_2208_14567_b200/ keeps the reference signatures and
 * binds these symbols with ctypes (see INTEGRATION.md for the stub a
 * maintainer would add to linkatlas itself).
 *
 * ABI contract
 *   - The caller owns every buffer; pointers marked (device) are CUDA device
 *     pointers, the library allocates nothing persistent.
 *   - Calls are stream-ordered on `stream` (a cudaStream_t passed as void*),
 *     reentrant across streams/devices; no global mutable state.
 *   - Return 0 on success, a negative LA_E* code for an invalid argument, or a
 *     positive cudaError_t.  la_last_error() returns a thread-local message.
 *   - Do not fork() after the first call (CUDA context).
 */
#ifndef LINKS_B200_H
#define LINKS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LA_ABI_VERSION 4
#define LA_MAX_JOINTS 20   /* joints per mechanism (generator.py n_max default) */
#define LA_MAX_STEPS 18    /* dyad steps per plan: n - |fixed| - 1 <= 18       */
#define LA_MAX_TOPK 32

/* error codes (negative) */
#define LA_EINVAL (-1)     /* bad argument / shape                              */
#define LA_ERANGE (-2)     /* size beyond a compiled limit                      */
#define LA_EWS (-3)        /* workspace too small                               */
#define LA_EHOST (-4)      /* host-side failure (allocation, thread creation)   */

/* ---------------------------------------------------------------- plans
 * One compiled solve order (solver.py:26-46 SolutionPlan, built by
 * compile_plan solver.py:71-102 on the host).  64 bytes.                   */
typedef struct la_plan {
  int16_t n;                       /* joints                                   */
  int16_t nsteps;                  /* S = len(plan.steps)                      */
  uint32_t fixed_mask;             /* bit j set: joint j is Fixed              */
  int8_t step[LA_MAX_STEPS][3];    /* (target, a, b) per PlanStep              */
  int8_t _pad[2];
} la_plan;

/* flags for la_simulate */
#define LA_SIM_WRITE_TRAJ 1u       /* write (T,2) f32 paths of every joint     */
#define LA_SIM_FP64 2u             /* evaluate every angle in f64 (no fp32)    */
#define LA_SIM_GATE_ONLY 4u        /* two-fidelity gate: skip exact first lock
                                      search for coarse-locked candidates      */
#define LA_SIM_NO_COARSE 8u        /* disable the coarse-first angle order     */
#define LA_SIM_TRAJ_F64 16u        /* traj holds f64 (T,2) rows instead of f32 */
#define LA_SIM_DEFER 32u           /* screen only: coarse survivors are left
                                      undecided, first_t = LA_PENDING         */
#define LA_SIM_SCATTER 64u         /* flags written at the candidate index
                                      cand[i] instead of the work item i      */
#define LA_SIM_WRITE_ONLY 128u     /* no screening: all T angles in f64 in
                                      natural order, exact first lock, paths
                                      written (needs LA_SIM_WRITE_TRAJ)       */
#define LA_SIM_EXACT64 256u        /* f64 rounds (writes, fix-up replays,
                                      LA_SIM_FP64) in numpy's operation order
                                      with IEEE ops + glibc hypot: paths and
                                      flags bit-identical to simulate_batch.
                                      Without it the f64 rounds use DFMA and
                                      Newton rsqrt (a few ulp; ~2x faster)   */
#define LA_SIM_LANE_SCREEN 512u   /* screen with the lane-per-candidate kernel
                                      (screen.cu) instead of the
                                      warp-per-candidate one (lanes = angles) */
#define LA_SIM_STATIC_GRID 1024u  /* deal the candidates to the warps round-robin
                                      (four waves of CTAs) instead of through
                                      the persistent grid's work queue        */
#define LA_PENDING (-3)            /* first_t of a deferred coarse survivor    */

/* Batched replay of compiled plans over (candidate x crank angle).
 * Replaces simulate_batch (solver.py:172-239) and, with coarse-first order,
 * the two-fidelity gate of check_feasible / find_valid_variant
 * (solver.py:242-249, generator.py:241-283).  Mixed topologies per launch.  */
typedef struct la_sim_args {
  const double* pos0;         /* (device) [B][pos_stride][2] initial poses    */
  const int32_t* topo;        /* (device) [B] plan index, or NULL => plan 0   */
  const la_plan* plans;       /* (device) [G]                                 */
  const double* crank_cs;     /* (device) [T][2] cos, sin of 2*pi*t/T          */
  int64_t B;
  int32_t G;
  int32_t pos_stride;         /* joints per pose row (>= every plan's n)      */
  int32_t T;                  /* crank angles per revolution (<= 2048)        */
  int32_t traj_stride;        /* joint rows per candidate in traj             */
  void* traj;                 /* (device) [rows][T][2] f32 (f64 with
                                 LA_SIM_TRAJ_F64), or NULL                    */
  const int64_t* traj_row;    /* (device) [B] first row of work item i, or
                                 NULL => i * traj_stride                      */
  const int64_t* cand;        /* (device, optional) [n_cand] candidate index
                                 of work item i (gather); outputs are indexed
                                 by i                                        */
  int64_t n_cand;             /* entries of cand (work items when cand set)   */
  const int64_t* cand_count;  /* (device, optional) number of valid entries of
                                 cand (<= n_cand), read on device: no host
                                 sync                                         */
  int32_t* first_t;           /* (device, optional with cand) [B] first
                                 locking angle, T if valid; -1 (with joint
                                 -2) if the plan has more joints than
                                 pos_stride or LA_MAX_JOINTS                  */
  int32_t* first_joint;       /* (device, optional with cand) [B] target joint
                                 of the first locking dyad, -1 if valid       */
  int32_t* low_t;             /* (device, optional) [B] lock step of the T/4
                                 coarse sweep (T_low semantics), -1 if none   */
  int32_t* low_joint;         /* (device, optional) [B]                       */
  unsigned long long* counters; /* (device, optional) [8] accumulated:
                                 0 f64 fix-up lane-angles, 1 warp lane-slots
                                 (32 x rounds), 2 warp dyad-slots (32 x rounds
                                 x S), 3 candidates, 4 rounds with an f64
                                 replay, 5 active lane-angles of fp32
                                 rounds, 6 fp32 dyads executed (to the
                                 first lock), 7 reserved                      */
  float fixup_tau;            /* fp32 screen: an angle is redone in f64
                                 when a dyad's margin min(ra+rb-d, d-|ra-rb|)
                                 is within tau + 3 E of a lock, E a running
                                 first-order bound on the fp32 position
                                 error (input rounding, per-dyad rounding,
                                 amplification |x|(1+|x|/d)/h by flat
                                 dyads); tau is the floor (default 2e-6).
                                 Trajectory rounds always run in f64        */
  uint32_t flags;             /* LA_SIM_*                                     */
  void* traj2;                /* (device, optional) split rows: with it the
                                 write pass stores dyad-target rows in traj
                                 and the other joints' rows (static joints,
                                 crank tip) in traj2, ascending joint order  */
  const int64_t* traj_row2;   /* (device) [B] first traj2 row of item i      */
  int32_t screen_refill;      /* lane screen: refill free lanes once at least
                                 this many are free (0 => 8)                 */
  int32_t screen_replay;      /* lane screen: replay parked (ambiguous)
                                 angles in f64 once at least this many lanes
                                 are parked (0 => 4)                         */
} la_sim_args;

int la_simulate(const la_sim_args* args, void* stream);

/* Per-candidate step geometry r_a, r_b, branch in f64
 * (plan_geometry, solver.py:105-120).  Outputs [B][LA_MAX_STEPS].          */
int la_plan_geometry(const double* pos0, const int32_t* topo, const la_plan* plans,
                     int64_t B, int32_t G, int32_t pos_stride,
                     double* r_a, double* r_b, double* branch, void* stream);

/* Element-wise f64 circle-circle intersection (dyad_solve, solver.py:123-139).
 * pa, pb: [n][2]; out: [n][2]; ok: [n] 1 solved / 0 no intersection.       */
int la_dyad_solve(const double* pa, const double* pb, const double* r_a,
                  const double* r_b, const double* branch, int64_t n,
                  double* out, int32_t* ok, void* stream);

/* Ordered stream compaction of valid candidates (first_t == T):
 * valid_idx[0..count) ascending.  count is written to *valid_count (device). */
size_t la_compact_workspace(int64_t B);
int la_compact_valid(const int32_t* first_t, int64_t B, int32_t T,
                     int64_t* valid_idx, int64_t* valid_count,
                     void* ws, size_t ws_bytes, void* stream);

/* The same selection with dense path rows: selected item k (candidate
 * idx[k]) starts at row row_off[k] = sum of plans[topo[idx[j]]].n over
 * j < k; *row_total (device) = rows of all selected items.  With
 * la_sim_args.traj_row = row_off a write pass stores (T,2) paths for the
 * real joints only (no padding rows up to traj_stride).                    */
size_t la_compact_rows_workspace(int64_t B);
/* Split rows: per selected item its dyad-target rows (plan nsteps) and its
 * other rows (static joints + crank tip, n - nsteps), two running sums; the
 * write pass stores them to traj / traj2 (la_sim_args.traj2).             */
size_t la_compact_rows_split_workspace(int64_t B);
int la_compact_rows_split(const int32_t* first_t, int64_t B, int32_t T, const int32_t* topo, const la_plan* plans,
                          int64_t* idx, int64_t* target_row, int64_t* other_row, int64_t* count,
                          int64_t* target_total, int64_t* other_total, void* ws, size_t ws_bytes, void* stream);
int la_compact_rows(const int32_t* first_t, int64_t B, int32_t T, const int32_t* topo,
                    const la_plan* plans, int64_t* idx, int64_t* row_off, int64_t* count,
                    int64_t* row_total, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- curves
 * Batched farthest-pair normalisation (normalize, curves.py:45-71) fused
 * with is_circle (curves.py:95-101) and the frame-stability predicate.     */
typedef struct la_norm_args {
  const void* paths;          /* (device) [rows][P][2] f32 or f64             */
  int32_t in_f64;
  const int64_t* src_row;     /* (device, optional) [M] row of path m         */
  int64_t M;
  int32_t P;
  void* out;                  /* (device) [M][P][2] f32 or f64                */
  int32_t out_f64;
  int32_t* pair;              /* (device, optional) [M][2] farthest pair i<j  */
  double* diameter;           /* (device, optional) [M]                       */
  uint8_t* is_circle;         /* (device, optional) [M]                       */
  double* circle_var;         /* (device, optional) [M]                       */
  uint8_t* unstable;          /* (device, optional) [M] frame not unique      */
  int32_t* status;            /* (device) [M] 0 ok, 1 degenerate (d <= 0)     */
  double* bbox;               /* (device, optional) [M][4] input lo_x, lo_y,
                                 hi_x, hi_y (is_normalized, curves.py:74-84) */
  double rel_tol;             /* near-tie tolerance on the diameter (1e-6)    */
  double y_tol;               /* |y0 - 0.5| flip-boundary tolerance (1e-6)   */
} la_norm_args;

int la_normalize(const la_norm_args* args, void* stream);

/* is_circle statistic of already-normalised paths (curves.py:95-101):
 * population variance of hypot(x-0.5, y-0.5); flag = var < 5e-4.          */
int la_circle_stats(const void* paths, int32_t in_f64, int64_t M, int32_t P,
                    double* var, uint8_t* flag, void* stream);

/* ---------------------------------------------------------------- chamfer
 * Bi-directional mean chamfer of every database curve against each query
 * (chamfer curves.py:123-129, _chamfer_block atlas.py:45-55), fused with the
 * shuffle-and-scan selection of Atlas.retrieve (atlas.py:179-236):
 *   top_*: best k non-hits (d >= threshold) by (d, scan position)
 *   hit_*: first k hits (d < threshold) by scan position
 * Exhaustive top-k is threshold = 0.                                        */
#define LA_CH_EXPANSION 1u   /* |a|^2+|q|^2-2a.q inner loop (FFMA2) with a
                                per-curve rounding bound; curves whose bound
                                exceeds fixup_below are redone with direct
                                differences                                  */
#define LA_CH_SCALAR_PIPE 2u /* one-lane FFMA/FADD inner loop instead of the
                                f32x2 (FFMA2/FADD2) forms                    */
#define LA_CH_TENSOR 8u      /* squared distances on tcgen05 (3xTF32 split,
                                direct-difference recheck of small minima)   */
#define LA_CH_NO_PRUNE 16u   /* disable the exact lower-bound pruning of the
                                top-k scan (every curve fully evaluated)     */
#define LA_CH_SEED_SCAN 32u  /* pruned scan: seed the running k-th bound with
                                the exact k-th of a 1/128 prefix scan first  */
#define LA_CH_NO_MQ 64u      /* pruned scan with NQ >= 2: one CTA set per query
                                instead of the multi-query kernel (groups of
                                queries share each streamed curve)           */
#define LA_CH_NO_INDEX 256u  /* ignore la_chamfer_args.cells                  */
#define LA_CH_INDEX_MQ 512u  /* use la_chamfer_args.cells for NQ >= 2 too:
                                multi-query seed, bound step for every
                                (query, curve), per-query survivor scans.
                                Off by default: against the multi-query
                                kernel it wins for few queries on a large
                                database (10M x 4: 16.6 vs 23.3 ms) and
                                loses for many on a small one (616k x 64:
                                40.6 vs 17.0 ms)                             */
#define LA_CH_MQ_FINE 128u   /* multi-query kernel: 64x64 common grid for the
                                stage-0 bound instead of 32x32               */

typedef struct la_chamfer_args {
  const float* db;            /* (device) [N][P][2] f32 normalised curves     */
  int64_t N;
  int32_t P;
  const float* queries;       /* (device) [NQ][Q][2] f32                      */
  int32_t NQ;
  int32_t Q;
  const int64_t* order;       /* (device, optional) [N] record at scan pos    */
  int64_t pos_begin;          /* scan-position range [pos_begin, pos_end)     */
  int64_t pos_end;
  int64_t id_base;            /* added to record ids in outputs (sharding)    */
  int64_t pos_base;           /* reported scan position = pos + pos_base ...  */
  const int64_t* pos_map;     /* (device, optional) ... or pos_map[pos]       */
  int32_t k;                  /* 0..LA_MAX_TOPK                               */
  float threshold;
  int64_t exclude_id;         /* record skipped entirely (self hit), -1 none  */
  float* top_d; int64_t* top_id; int64_t* top_pos;   /* [NQ][k]               */
  float* hit_d; int64_t* hit_id; int64_t* hit_pos;   /* [NQ][k]               */
  int64_t* n_hits;            /* (device, optional) [NQ] total hits           */
  float* all_d;               /* (device, optional) [NQ][N] by record index   */
  void* ws;
  size_t ws_bytes;
  uint32_t flags;             /* LA_CH_*                                      */
  float fixup_below;          /* expansion mode: max tolerated error bound on a
                                 curve's distance (e.g. 5e-5) before the
                                 direct-difference recomputation             */
  int64_t* n_full;            /* (device, optional) [NQ] += curves evaluated in
                                 full (the rest were pruned by their bound)  */
  int64_t* n_stage;           /* (device, optional) [5] += (query, curve) pairs
                                 surviving the multi-query kernel's bounds:
                                 box/gap-table column term, common-grid row
                                 term, 4-corner row term, 50-point and
                                 10-point run-box column terms               */
  const uint16_t* cells;      /* (device, optional) [N][LA_INDEX_ROW(P)] cell index of db from
                                 la_chamfer_index: single-query pruned scans
                                 first bound every curve from its 2-byte
                                 cells against the k-th best of a seed scan
                                 and scan only the survivors (same lists);
                                 n_stage[0] += survivors                     */
  const uint8_t* coarse;      /* (device, optional, with cells) [N][256] coarse
                                 distance tables of db from la_chamfer_index:
                                 adds the column term to the bound step (the
                                 query's 16 x 16 cell histogram against each
                                 curve's bytes)                              */
  const uint8_t* fine;        /* (device, optional, with coarse) [N][1024]: the
                                 32 x 32 tables, read for the bound step's
                                 survivors only (second level; n_stage[1] +=
                                 its survivors)                              */
} la_chamfer_args;

#define LA_INDEX_ROW(P) (((P) + 15) & ~15) /* cells per index row (32-byte sectors) */
/* Cell index of a curve database for la_chamfer_args.cells: cells[i][j] =
 * cell of point j of curve i on the fixed 64 x 64 grid over the unit square
 * padded by 1/32 (outside points clamp into the border cells), numbered
 * ix * 66 + iy (table rows padded against bank conflicts); entries j >= P
 * of a row hold the null cell 64.  cells: [N][LA_INDEX_ROW(P)].  Built once
 * per database (Atlas build / load); 2 bytes per point.
 * coarse (optional): [N][256] bytes, coarse[i][cx * 16 + cy] = floor(160 x
 * distance from cell (cx, cy) of the 16 x 16 grid over the same square to
 * curve i's nearest point), saturated at 255.  fine (optional): [N][1024],
 * the same on the 32 x 32 grid.                                            */
int la_chamfer_index(const float* db, int64_t N, int32_t P, uint16_t* cells, uint8_t* coarse, uint8_t* fine,
                     void* stream);

size_t la_chamfer_workspace(const la_chamfer_args* args);
int la_chamfer_topk(const la_chamfer_args* args, void* stream);

/* Merge of the per-shard (NQ x k) lists every rank all-gathered (multi-GPU
 * retrieval): gathered = (device) [world][NQ][6k+1] int64
 * rows (top_d float bits, top_id, top_pos, hit_d float bits, hit_id,
 * hit_pos, n_hits); outputs (device) [NQ][k] as la_chamfer_topk's, non-hits
 * by (d, scan position), hits by scan position, n_hits summed.  Replaces the
 * scan-order bookkeeping of Atlas.retrieve (atlas.py:207-235) across
 * shards.                                                                 */
int la_merge_shard_lists(const int64_t* gathered, int32_t world, int32_t NQ, int32_t k, float* top_d,
                         int64_t* top_id, int64_t* top_pos, float* hit_d, int64_t* hit_id, int64_t* hit_pos,
                         int64_t* n_hits, void* stream);

/* ---------------------------------------------------------------- generator
 * Host (CPU, multi-threaded) reproduction of the reference's candidate
 * streams: group g draws n = integers(n_lo, n_hi + 1) and its topology from
 * default_rng([seed, g0 + g, 0]) (sample_topology, generator.py:200-222) and
 * its poses from default_rng([seed, g0 + g, 1]) (_sample_positions_batch,
 * generator.py:234-238) — numpy's SeedSequence / PCG64 / Generator
 * restated bit for bit.                                                     */
int la_sample_topologies(int64_t seed, int64_t g0, int64_t G, int32_t n_lo, int32_t n_hi, double ng_prob,
                         int32_t retries, int32_t threads, la_plan* plans, int8_t* types /* [G][20] */,
                         uint8_t* adj /* [G][20][20] or NULL */, int32_t* n_out);
/* One sample_topology(rng, n, ng_probability, retries) draw on a caller's
 * numpy PCG64 state (generator.py:200-222): st = {state hi, lo, inc hi, lo},
 * buf = {has_uint32, uinteger}, advanced in place; LA_ERANGE when every
 * retry fails (the reference raises GenerationError).                    */
int la_sample_topology_rng(uint64_t* st, uint32_t* buf, int32_t n, double ng_prob, int32_t retries,
                           la_plan* plan, int8_t* types /* [20] */, uint8_t* adj /* [20][20] */);
int la_sample_poses(int64_t seed, int64_t g0, int64_t G, int32_t per_group, const int32_t* n_of_group,
                    int32_t stride, int32_t threads, double* pos /* [G*per_group][stride][2] host */);
/* Coarse prefilter (Atlas.coarse_filter, atlas.py:153-177).
 * la_coarse_descriptors: paths [M][P][2] f64 -> desc [M][18] f64 = radial
 *   histogram (16 bins over edges[0..16], host array = np.linspace(0, .75,
 *   17), np.histogram semantics, / P) + bbox extent; bit-identical to
 *   Atlas._descriptor (atlas.py:167-172).
 * la_coarse_select: L1 distance to qdesc (device [18]) in numpy's summation
 *   order, keeps the min(budget, M) smallest by (distance, index) and writes
 *   them to out in scan order (order[] filtered; order NULL = identity);
 *   optional dist_out [M].  Workspace from la_coarse_workspace(M).        */
int la_coarse_descriptors(const double* paths, int64_t M, int32_t P, const double* edges /* host [17] */,
                          double* desc, void* stream);
size_t la_coarse_workspace(int64_t M);
int la_coarse_select(const double* desc, int64_t M, const double* qdesc, int64_t budget, const int64_t* order,
                     int64_t* out, double* dist_out, void* ws, size_t ws_bytes, void* stream);

/* Curation keep rule (curation_keep, curves.py:104-110) for a batch of
 * curve records on the device: keep[i] = !flagged[i] ||
 * default_rng([seed, mech_ids[i], joint_ids[i]]).random() < keep_rate
 * (ids >= 0).                                                            */
int la_curation_keep(const int64_t* mech_ids, const int64_t* joint_ids, const uint8_t* flagged, int64_t n,
                     int64_t seed, double keep_rate, uint8_t* keep, void* stream);

/* Dataset-generation engine (GenerationRun / _generate_slot /
 * find_valid_variant, generator.py:241-375): a caller-owned host object that
 * holds every slot's topology / pose / negative PCG64 streams and replays the
 * reference control flow exactly; the GPU answers the two-fidelity gate for
 * look-ahead windows (la_simulate with LA_SIM_GATE_ONLY and low_t).       */
typedef struct la_gen_cfg {
  int64_t seed;
  int32_t n_min, n_max;
  double ng_prob;
  int32_t variants, T_low, T_high, max_attempts, retries, batch;
  double negative_rate;
  int32_t threads; /* host threads for window layout / flag walks (0: 1) */
  int32_t _pad;
} la_gen_cfg;
void* la_gen_create(const la_gen_cfg* cfg, int64_t slot0, int64_t n_slots);
void la_gen_destroy(void* engine);
int64_t la_gen_window(void* engine, int32_t lookahead, int64_t cap, int32_t threads, double* pos /* [cap][20][2] */,
                      int32_t* cand_plan /* [cap] */, la_plan* plans /* [n_slots] */, int32_t* n_plans);
/* Device-drawn window: one descriptor per reference batch; candidate c of
 * the batch is the c-th pose of the stream starting at `state`.          */
typedef struct la_gen_batch {
  uint64_t state_hi, state_lo, inc_hi, inc_lo; /* PCG64 128-bit state / increment */
  int64_t first;                               /* first candidate index in window  */
  int32_t k, n, plan, _pad;
} la_gen_batch;
int64_t la_gen_window_dev(void* engine, int32_t lookahead, int64_t cap, la_gen_batch* batches /* host */,
                          int64_t max_batches, int64_t* n_batches, la_plan* plans, int32_t* n_plans);
/* device kernel: poses [cand][stride][2] f64 (pivot/tip pinned, NaN beyond
 * n) and plan index per candidate, from device-resident descriptors       */
int la_gen_poses(const la_gen_batch* batches, int64_t n_batches, int32_t stride, double* pos, int32_t* topo,
                 void* stream);
/* pos may be NULL for device-drawn windows (poses of accepted / negative
 * candidates are redrawn on the host from the batch stream state)         */
int la_gen_consume(void* engine, const double* pos, const int32_t* first_t, const int32_t* low_t);
int64_t la_gen_count(void* engine, int32_t what /* 0 records, 1 negatives */);
int la_gen_records(void* engine, int64_t* meta /* [R][4] */, double* pos, la_plan* plans, uint8_t* adj,
                   int8_t* types);
int la_gen_negatives(void* engine, int64_t* meta /* [R][3] */, double* pos, uint8_t* adj, int8_t* types);
int la_gen_stats(void* engine, int64_t* by_n /* [21][2] */, int64_t* discarded);

/* moving-joint curves of a generated block in cli.normalize order
 * (cli.py:124-136): rows into the packed trajectory block, mech ids
 * slot * variants + variant, joint ids, is_arc (curves.py:87-92).  Host
 * function; outputs NULL -> count only.  Returns the curve count.        */
int64_t la_moving_joints(const int64_t* meta, const int8_t* types, const uint8_t* adj, const int64_t* row0,
                         int64_t R, int32_t variants, int64_t* rows, int64_t* mech_ids, int64_t* joint_ids,
                         uint8_t* is_arc);

/* raw PCG64 stream of default_rng(entropy[:n_ent]): kind 0 -> random(),
 * kind 1 -> integers(0, bound)                                              */
int la_rng_draw(const int64_t* entropy, int32_t n_ent, int32_t kind, int64_t bound, int64_t count,
                double* out_d, int64_t* out_i);

/* ---------------------------------------------------------------- misc */
int la_abi_version(void);
const char* la_last_error(void);
/* number of SMs of the current device (grid sizing helper), or <0 */
int la_device_sm_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LINKS_B200_H */
