/*
 * guidefill_b200.h -- C ABI of the B200-native Guidefill fill engine.
 *
 * Plain pointers and sizes only; every device pointer is CUDA global memory
 * on the current device, every call is stream-ordered on `stream`
 * (a cudaStream_t, NULL = legacy default stream) and re-entrant: there is no
 * global mutable state, all scratch lives in the caller's workspace.
 * Functions return GF_OK (0) or a negative GF_E* code; gf_last_error()
 * returns a thread-local message for the last failure on the calling thread.
 *
 * The reference (arXiv 1611.05319, /root/reference/pkg) is pure Python with
 * no FFI; each entry point below replaces one of its Python operators, cited
 * as file:line under pkg/src/guidefill/.  INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 */
#ifndef GUIDEFILL_B200_H
#define GUIDEFILL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GF_ABI_VERSION 2

/* status codes */
#define GF_OK 0
#define GF_E_INVALID (-1)   /* bad argument (maps to the reference's ValueError) */
#define GF_E_CUDA (-2)      /* CUDA runtime failure */
#define GF_E_WORKSPACE (-3) /* workspace too small */
#define GF_E_UNSUPPORTED (-4)

/* element types */
#define GF_F32 0
#define GF_F64 1

/* FillParams.order (engine.py:28) */
#define GF_ORDER_ONION 0
#define GF_ORDER_SMART 1
#define GF_ORDER_SMART_DATA 2
/* FillParams.neighborhood (engine.py:29) */
#define GF_BALL_ROTATED 0
#define GF_BALL_AXIS 1
/* guide source (engine.py:234-242): g = 0, FillParams.g_fixed, or a per-pixel field */
#define GF_G_ZERO 0
#define GF_G_FIXED 1
#define GF_G_FIELD 2

/* largest supported ball radius (disk of r = 12 has K = 440 samples) */
#define GF_MAX_RADIUS 12

/* per-frame statistics written by gf_fill (int32 each) */
#define GF_STAT_ITERATIONS 0    /* FillReport.iterations   engine.py:96   */
#define GF_STAT_FILLED 1        /* FillReport.filled       engine.py:97   */
#define GF_STAT_DEADLOCK 2      /* FillReport.deadlock_fills engine.py:98 */
#define GF_STAT_UNFILLABLE 3    /* 1: frontier emptied (or guard found no
                                   readable neighbour) with Inpaint pixels
                                   left; the caller runs the nearest-readable
                                   fallback of engine.py:270-283 */
#define GF_STAT_REMAINING 4     /* Inpaint pixels left unfilled */
#define GF_STAT_INPAINT 5       /* |D| of the frame */
#define GF_STAT_ROWS_OVERFLOW 6 /* 1 if iterations > rows_cap */
#define GF_STAT_LAST_FRONTIER 7 /* frontier size of the shell that ended the
                                   loop unfilled (0 when the fill completed) */
#define GF_STAT_BAD_LABELS 8    /* 1 if a label is not 0 / 128 / 255 (the
                                   caller raises grid.py:36-46's ValueError;
                                   the fill result is then meaningless) */
#define GF_STATS 9

/* FillParams (engine.py:33-60), minus the coherence-transport knobs */
typedef struct gf_fill_params {
  int32_t r;            /* ball radius epsilon in pixels: 1..GF_MAX_RADIUS for
                           gf_fill* / gf_coherence_fill, any r >= 1 for
                           gf_sample_points (tables in device memory)      */
  double mu;            /* guidance strength, >= 0, +inf allowed           */
  double c;             /* smart-order confidence threshold                */
  double c2;            /* data-term threshold                             */
  int32_t order;        /* GF_ORDER_*                                      */
  int32_t neighborhood; /* GF_BALL_*                                       */
  int32_t g_mode;       /* GF_G_*                                          */
  double g_fixed[2];    /* used when g_mode == GF_G_FIXED                  */
  int32_t periodic_x;   /* wrap the x axis                                 */
  int32_t tracked;      /* 1: frontier tracking (tracker.py:143-172),
                           0: full-lattice rescan every shell (engine.py:357-360) */
} gf_fill_params;

/* A batch of equally sized frames, each filled independently (video). */
typedef struct gf_frames {
  int32_t n_frames;
  int32_t height;
  int32_t width;
  int32_t channels;      /* 1..4 */
  int32_t dtype;         /* GF_F32 or GF_F64, for both image and out   */
  const void* image;     /* [n_frames][H][W][C], values in [0, 1]        */
  const uint8_t* labels; /* [n_frames][H][W], 0 / 128 / 255              */
  const double* guide;   /* [n_frames][H][W][2] if g_mode == GF_G_FIELD  */
  void* out;             /* [n_frames][H][W][C]                          */
} gf_frames;

typedef struct gf_fill_outputs {
  int32_t* frame_stats; /* device [n_frames][GF_STATS]                        */
  int32_t* rows;        /* device [n_frames][rows_cap][2]: (frontier_size, filled)
                           per shell -- FillReport.rows columns 1 and 4        */
  int32_t rows_cap;
  int32_t* enter;       /* optional device [n_frames][H][W]: shell at which the
                           pixel joined the frontier, -1 never (order log)     */
  int32_t* fillshell;   /* optional device [n_frames][H][W]: shell in which the
                           pixel was filled, -1 never                           */
  uint64_t* shell_trace; /* optional device [trace_cap][8], zero-initialised:
                           profiling record per shell -- globaltimer ns at shell
                           start, end of the fill phase (latest block), after
                           its grid barrier, end of the frontier update (latest
                           block), after its barrier; the number of frontier
                           items; the longest single-item evaluation (ns) on
                           the lattice (g = 0) path and on the rotated-ball
                           path                                               */
  int32_t trace_cap;
} gf_fill_outputs;

/* Splines flattened to polylines on the host (Spline.polyline,
 * splines.py:42-73), for every frame of a batch.  All device pointers. */
typedef struct gf_splines {
  int32_t n_seg;
  const double* seg;         /* [n_seg][4] = (ax, ay, bx, by), polyline order */
  const int32_t* seg_spline; /* [n_seg] owning spline index, non-decreasing  */
  int32_t n_splines;
  const double* dirs;        /* [n_splines][2] spline directions             */
  double eta;                /* falloff scale, guide.py:28                   */
  const int32_t* frame_seg;  /* optional [n_frames + 1]: frame f uses segments
                                [frame_seg[f], frame_seg[f+1]); NULL = every
                                frame uses all segments                      */
} gf_splines;

/* Bytes of device workspace gf_fill / gf_fill_splines need for this batch
 * (splines may be NULL). */
size_t gf_fill_workspace_bytes(const gf_frames* frames, const gf_fill_params* params);
size_t gf_fill_splines_workspace_bytes(const gf_frames* frames, const gf_fill_params* params,
                                       const gf_splines* splines);

/*
 * Fill every Inpaint pixel of every frame: Algorithm 1 with Eq. 3.2 weights,
 * ghost-pixel rotated balls, onion/smart/data-term order, deadlock guard and
 * the final value-hull clip.  Replaces engine._fill_loop (engine.py:286-376)
 * and its tracker hook (tracker.py:161-170) -- the seam both
 * engine.inpaint (engine.py:379-408) and tracker.run_tracked
 * (tracker.py:143-172) call.  Outputs match the reference bit for bit on the
 * fill order and within 1e-4 on values (fp32 colour path, fp64 decisions).
 */
int gf_fill(const gf_frames* frames, const gf_fill_params* params,
            const gf_fill_outputs* outputs, void* workspace, size_t workspace_bytes,
            void* stream);

/*
 * gf_fill with the guide field rastered from splines inside the fill's
 * first pass -- the CLI / project path build_guide_field + run_tracked
 * (cli.py:106-112, project.py:193-202) as one call, without materialising
 * the dense (H, W, 2) field.  g_mode is ignored (the rastered field is the
 * guide).  Fill results are identical to gf_guide_field followed by gf_fill.
 */
int gf_fill_splines(const gf_frames* frames, const gf_fill_params* params,
                    const gf_splines* splines, const gf_fill_outputs* outputs,
                    void* workspace, size_t workspace_bytes, void* stream);

/*
 * Guide-field rasteriser: g(x) = dir_s * exp(-d^2 / (2 eta^2)) for the
 * nearest spline s (first on ties), 0 beyond 3 eta and outside the Inpaint
 * set.  Replaces guide.build_guide_field + _segment_min_distance
 * (guide.py:286-327).  Splines arrive already flattened to polylines
 * (Spline.polyline, splines.py:42-73, stays on the host):
 *   seg[n_seg][4] = (ax, ay, bx, by) in polyline order,
 *   seg_spline[n_seg] = owning spline index (non-decreasing),
 *   dirs[n_splines][2] = spline directions.
 * out_field: device [H][W][2] float64, fully written.
 */
int gf_guide_field(int32_t height, int32_t width, const uint8_t* labels,
                   int32_t n_seg, const double* seg, const int32_t* seg_spline,
                   int32_t n_splines, const double* dirs, double eta,
                   double* out_field, void* stream);

/*
 * Ball sampler at arbitrary points: readable weight mass, total weight mass
 * and weighted average colour.  Replaces engine._BallSampler.gather
 * (engine.py:175-199) as used by engine.confidence / engine.fill_color
 * (engine.py:202-221).  image: device float64 [H][W][C]; points: device
 * [n][2] (x, y); g: device [n][2].  Outputs: rw[n], tw[n], vals[n][C].
 */
int gf_sample_points(int32_t height, int32_t width, int32_t channels,
                     const double* image, const uint8_t* labels,
                     int32_t n, const double* points, const double* g,
                     const gf_fill_params* params,
                     double* rw, double* tw, double* vals, void* stream);

/*
 * Strict bilinear ghost sampling at points (grid.bilinear_gather,
 * grid.py:158-211).  Outputs vals[n][C] (zero where not readable), ok[n].
 */
int gf_bilinear_gather(int32_t height, int32_t width, int32_t channels,
                       const double* image, const uint8_t* labels,
                       int32_t n, const double* X, const double* Y, int32_t periodic_x,
                       double* vals, uint8_t* ok, void* stream);

/*
 * Boundary masks of a label lattice (grid.py:84-106): active (Inpaint with
 * a Readable 8-neighbour), inner (Inpaint with a non-Inpaint 8-neighbour),
 * outer (non-Inpaint with an Inpaint 8-neighbour).  Any output may be NULL.
 */
int gf_boundary_masks(int32_t height, int32_t width, const uint8_t* labels,
                      int32_t periodic_x, uint8_t* active, uint8_t* inner,
                      uint8_t* outer, void* stream);

/*
 * Output delta for host-side results.  A fill returns every Readable pixel
 * bit for bit as it came in (engine.py:364-376 only writes u[filled] and
 * clips to the Readable hull), so a host caller can DMA the INPUT into its
 * pinned result buffer while the frame uploads and then call this after the
 * fill: every pixel whose output differs bitwise from the input is written
 * into host_out (pinned, mapped: cudaHostAlloc / cudaHostRegister memory).
 * input/output: device [n_px][channels] of dtype GF_F32/GF_F64.
 * n_changed (device, nullable) is incremented by the pixels written.
 * Stream-ordered: host_out must already hold the input copy on `stream`.
 * No reference counterpart (the reference returns a fresh numpy array,
 * engine.py:289,376); it is the transfer half of the drop-in fill.
 */
int gf_output_delta(int64_t n_px, int32_t channels, int32_t dtype, const void* input,
                    const void* output, void* host_out, unsigned long long* n_changed,
                    void* stream);

/*
 * The upload half of the same path: copies nbytes host_src -> dev_dst on
 * `stream` in `chunk`-byte pieces and, as each piece lands, copies it back
 * dev_dst -> host_mirror on `side_stream` (the link's two directions run
 * concurrently).  host_src and host_mirror must be pinned for the copies to
 * be asynchronous.  The caller joins side_stream into its stream before
 * gf_output_delta.
 */
int gf_upload_mirrored(const void* host_src, void* dev_dst, void* host_mirror, int64_t nbytes,
                       int64_t chunk, void* stream, void* side_stream);

/*
 * Unfillable fallback on the device (engine.py:270-283): every stranded
 * pixel (Inpaint with fillshell < 0) takes the colour, in `out`, of its
 * nearest readable pixel (Readable, or Inpaint with fillshell >= 0) as
 * scipy.ndimage.distance_transform_edt(~readable, return_indices=True)
 * picks it, ties included; 0.5 in every channel when nothing is readable.
 * One frame: labels [H][W] u8, fillshell [H][W] int32 (gf_fill_outputs),
 * out [H][W][C] of dtype GF_F32/GF_F64, updated in place.  n_painted
 * (device, nullable) is incremented by the stranded pixel count.
 * workspace: gf_paint_unfillable_workspace_bytes(H, W) device bytes.
 */
size_t gf_paint_unfillable_workspace_bytes(int32_t height, int32_t width);
int gf_paint_unfillable(int32_t height, int32_t width, int32_t channels, int32_t dtype,
                        const uint8_t* labels, const int32_t* fillshell, void* out,
                        void* workspace, size_t workspace_bytes, int32_t* n_painted,
                        void* stream);

/*
 * Coherence-transport guide directions (g_source "modified_structure_tensor"):
 * replaces guide.coherence_directions (guide.py:330-355) as called per shell
 * by engine._resolve_g (engine.py:243-249).  The masked structure tensor of
 * guide._tensor_field (guide.py:91-120) over image [H][W][C] float64 with
 * readable = (labels == 0), evaluated at the n flat pixel indices idx
 * (device int64), eigen split as guide.eigen_2x2 (guide.py:123-136):
 * g[n][2] = tanh((hi - lo) / lam) * minor eigenvector, 0 where the rho
 * window holds no readable mass.  sigma / rho: Gaussian scales (truncate 2,
 * radius int(2 s + 0.5) <= 63).  2 <= H <= 65535, W >= 2 (np.gradient needs
 * 2 samples).
 * points (nullable): device [n][2] float64, receives (x, y) = (i, j) of each
 * query, ready for gf_sample_points.
 * workspace: gf_coherence_workspace_bytes(H, W, C) device bytes.
 */
size_t gf_coherence_workspace_bytes(int32_t height, int32_t width, int32_t channels);
int gf_coherence_directions(int32_t height, int32_t width, int32_t channels,
                            const double* image, const uint8_t* labels, int32_t n,
                            const int64_t* idx, double sigma, double rho, double lam,
                            double* g, double* points, void* workspace, size_t workspace_bytes,
                            void* stream);

/*
 * Tracked frontier update of one shell (tracker._update_arrays,
 * tracker.py:59-79), for a frontier of n sorted flat indices with fill[n]
 * (u8) after the filled pixels were relabelled Readable in labels.  Writes
 * mark[p] = 1 for every candidate (a surviving frontier pixel, or an
 * in-lattice / x-periodic Inpaint 8-neighbour of a filled one) and 2 for a
 * candidate that passes _active_filter.  mark: device [H][W] u8, zeroed by
 * the caller; the sorted nonzero positions are np.unique(pool).
 */
int gf_frontier_candidates(int32_t height, int32_t width, const uint8_t* labels,
                           int32_t periodic_x, int32_t n, const int64_t* frontier,
                           const uint8_t* fill, uint8_t* mark, void* stream);

/*
 * Decision and scatter of one shell (engine.py:317-356), after
 * gf_sample_points at the n frontier pixels: conf = rw / tw; ready_mode 0 =
 * onion (all ready), 1 = conf > c, 2 = (hypot(g) > c2) & (conf > c) (the
 * data-term order while its latch is live; g: device [n][2]);
 * fill[k] = ready & (rw > 0).  Filled pixels get image[p] = vals[k] (float64
 * [H][W][C]), labels[p] = 0 (Readable) and fillshell[p] = shell; *count
 * (device int32, zeroed by the caller) += the number filled.  A shell with
 * no fill is the caller's deadlock guard (engine.py:334-348).
 */
int gf_commit_shell(int32_t channels, int32_t n, const int64_t* frontier, const double* rw,
                    const double* tw, const double* vals, const double* g, int32_t ready_mode,
                    double c, double c2, int32_t shell, double* image, uint8_t* labels,
                    int32_t* fillshell, uint8_t* fill, int32_t* count, void* stream);

/*
 * The whole coherence-transport fill (engine._fill_loop, engine.py:286-376,
 * with g_source = "modified_structure_tensor": guide.coherence_directions,
 * guide.py:330-355) in one persistent kernel launch: image / labels (device,
 * f64 [H][W][C] / uint8 [H][W]) are filled and relabelled in place;
 * fillshell receives each pixel's shell (-1 if never filled), enter (optional)
 * the shell it joined the frontier (-1 never), rows[rows_cap][5] the report rows
 * (iteration, frontier size, candidates, threads, filled) and report[4] =
 * (done: 0 finished / 2 unfillable / 3 capacity exceeded, iterations,
 * deadlock fills, filled).  The image is clipped to the readable hull
 * (engine.py:375-376) unless the fill ended unfillable: then the caller paints
 * the stranded pixels and clips (engine.py:370-376).  capacity bounds the
 * frontier (>= the Inpaint pixel count; H * W always works).
 * params->tracked picks the frontier tracker; params->r / mu / neighborhood /
 * periodic_x the ball.
 */
size_t gf_coherence_fill_workspace_bytes(int32_t height, int32_t width, int32_t channels,
                                         int64_t capacity);
int gf_coherence_fill(int32_t height, int32_t width, int32_t channels, double* image,
                      uint8_t* labels, const gf_fill_params* params, double sigma, double rho,
                      double lam, int64_t capacity, int32_t* fillshell, int32_t* enter,
                      int64_t* rows, int32_t rows_cap, int32_t* report, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Thread-local message for the last failing call on this thread. */
const char* gf_last_error(void);
int gf_abi_version(void);
/* Kernels launched by this library so far (process-wide, all devices): the
 * launch evidence bench.py reports as gpu_launches.  A CUDA-graph capture of
 * an entry counts once, at capture; replays are counted by the caller. */
int64_t gf_launch_count(void);

/* Host-side builds of the exact-math primitives the kernels use (same
 * source, gf_math.cuh), exported so CPU tests can pin them to numpy. */
void gf_host_exp(const double* x, double* y, int64_t n);
void gf_host_hypot(const double* x, const double* y, double* out, int64_t n);
double gf_host_pairwise_sum(const double* a, int32_t n);
/* numpy's float64 arctan2 / tanh (SVML __svml_atan28_ha / __svml_tanh8) and
 * sin / cos (glibc libm, |x| <= 2.426) as the coherence kernels compute them
 * (gf_npmath.cuh): guide.eigen_2x2, guide.py:123-136. */
void gf_host_atan2(const double* y, const double* x, double* out, int64_t n);
void gf_host_tanh(const double* x, double* y, int64_t n);
void gf_host_sincos(const double* x, double* s, double* c, int64_t n);
/* The same four on the device, element-wise over n device doubles:
 * op 0 out = atan2(a, b), 1 tanh(a), 2 sin(a), 3 cos(a). */
int gf_npmath_eval(int32_t op, int64_t n, const double* a, const double* b, double* out,
                   void* stream);

/*
 * The plain / masked structure tensor's eigen split at the n queries, as
 * gf_coherence_directions but returning eig[n][8] = (vx, vy, coh, a, b, c,
 * mass, 0): the minor eigenvector (guide.eigen_2x2, guide.py:123-136),
 * tanh((hi - lo) / lam), the normalised tensor [[a, b], [b, c]] and the rho
 * window's mass (ZeroMassError when <= 0, guide.py:164-166).
 * With labels all 0 (every pixel readable) this is guide.structure_tensor
 * (guide.py:139-156) as make_spline uses it (guide.py:221-223).
 */
int gf_structure_eigen(int32_t height, int32_t width, int32_t channels, const double* image,
                       const uint8_t* labels, int32_t n, const int64_t* idx, double sigma,
                       double rho, double lam, double* eig, void* workspace,
                       size_t workspace_bytes, void* stream);

/*
 * Edge seeds of automatic spline detection (guide.detect_edge_seeds,
 * guide.py:177-197, before the clustering): the measurement ring
 * (compute_ring, guide.py:65-88: Readable pixels at chessboard distance
 * ceil(2 sigma + 2 rho) + 1 from D u B), Canny restricted to the annulus
 * around it (scikit-image's canny restated: masked Gaussian with bleed-over,
 * Sobel, bilinear non-maximum suppression, hysteresis with low / high), and
 * the ring pixels on an edge with strength hypot(np.gradient(gauss(gray))).
 * Replaces guide.py:183-196.  Synchronous on `stream` (hysteresis passes
 * until a fixpoint).  Up to cap hits: hit_idx (device int64 flat indices,
 * unordered), hit_strength (device float64); *n_hits (HOST int32) = total
 * hits (may exceed cap).  ring_out / edges_out (nullable, device [H][W] u8):
 * the ring mask and the edge flags (bit 2 = edge).
 * workspace: gf_detect_workspace_bytes(H, W) device bytes.
 */
size_t gf_detect_workspace_bytes(int32_t height, int32_t width);
int gf_detect_edges(int32_t height, int32_t width, int32_t channels, const double* image,
                    const uint8_t* labels, double sigma, double rho, double low, double high,
                    int32_t cap, int64_t* hit_idx, double* hit_strength, int32_t* n_hits,
                    uint8_t* ring_out, uint8_t* edges_out, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * make_spline's ray search and extension (guide.py:231-259) for n seeds
 * (device [n][2] (i, j) float64) along unit directions v (device [n][2]):
 * out[n][3] = (sign, t_entry, t_end), sign +1 (along v), -1 (along -v) or 0
 * (no entry within `budget`, the seed yields no spline).
 */
int gf_trace_rays(int32_t height, int32_t width, const uint8_t* labels, int32_t n,
                  const double* seeds, const double* v, double budget, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GUIDEFILL_B200_H */
