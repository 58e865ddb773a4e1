/*
 * ralpb.h — C ABI of libralpb200.so, the B200-native execution backend for the
 * resource-aware layer-placement (RALP) training step of arXiv 1901.05803.
 *
 * The reference (`ralp`, pkg/src/ralp) has no FFI: its drop-in surface is the
 * Python package API (pkg/src/ralp/__init__.py:3-91).  The execution entry it
 * offers is `simulate_run(Scenario) -> SimReport` (pkg/src/ralp/simulator.py:743-770),
 * whose per-job schedule is `_JobRun._ralp_worker/_ralp_ps`
 * (simulator.py:669-715) and `_baseline_worker/_baseline_ps` (simulator.py:637-665).
 * This library executes that schedule for real; the Python package
 * `paper_1901_05803_b200` binds it with ctypes.
 *
 * Conventions: every function returns 0 on success and a nonzero code on
 * failure; ralpb_last_error() returns a thread-local message.  Pointers are
 * device pointers unless a parameter name says `host_`.  `stream` is a
 * cudaStream_t (NULL = legacy default stream).  No torch types cross the ABI.
 */
#ifndef RALPB_H_
#define RALPB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status */
const char* ralpb_last_error(void);
int ralpb_version(void);

/* ------------------------------------------------------------ kernels
 * Dense contraction on tcgen05 tensor cores (bf16 operands, fp32 accumulate).
 *   out[m*s_m + n*s_n] = epi( sum_k A[m,k] * B[n,k] )
 * A is [a_rows][a_cols] row-major with leading dim a_ld; a_mn=0 means rows=M, cols=K
 * (K-major), a_mn=1 means rows=K, cols=M (MN-major).  Same for B with N.
 * out_kind: 0 = bf16 store, 1 = fp32 store, 2 = fp32 atomic add (allows k_splits).
 * bias (fp32, per n) and relu apply before the store; mask (bf16, mask[m*mask_s+n] > 0)
 * multiplies by the ReLU derivative.  k_splits=0 picks a split for the atomic epilogue;
 * block_n=0 picks the N tile.  Replaces the FC forward/backward compute the
 * reference models as `back_batch_s` (simulator.py:542) and infer_fc (layers.py:117-123). */
int ralpb_gemm_bf16(const void* a, long long a_rows, long long a_cols, long long a_ld, int a_mn,
                    const void* b, long long b_rows, long long b_cols, long long b_ld, int b_mn,
                    int M, int N, long long K, void* out, int out_kind, long long s_m,
                    long long s_n, const float* bias, int relu, const void* mask, long long mask_s,
                    int k_splits, int block_n, void* stream);

/* Implicit-GEMM convolution (stride 1, k = 2*pad+1) over the padded NHWC layout
 * [n][h+2pad][w+2pad][c] bf16 with zero borders.  Implements infer_conv
 * (layers.py:87-103) with ReLU fused.  Outputs are written on interior
 * pixels only: allocate output buffers with zero borders.
 *   w:  [cout][k*k][cin] bf16      wd: [cin][k*k][cout] bf16 (tap-reversed transpose)
 *   dw: [cout][k*k][cin] fp32 and db: [cout] fp32 (may be NULL), accumulated (caller zeroes).
 *   colsum (dgrad, may be NULL): colsum[ci] += sum over pixels of the stored bf16 dx -- the bias
 *   gradient of the convolution that produced the masked activation, fused into this producer. */
int ralpb_conv_fwd(const void* x_pad, const void* w, const float* bias, void* y_pad, int n, int h,
                   int w_, int cin, int cout, int k, int pad, int relu, void* stream);
/* conv_fwd plus the 2x2/2 max pool of its output (max_pool2d, layers.py:106-114) written to
 * pool_out [n][h/2+2pp][w/2+2pp][cout] (interior), fused into the epilogue: the pool reads no
 * activation back from HBM.  h, w even; errors where the slab kernels do not apply.
 * pool_idx (may be NULL): uint8 [n][h/2][w/2][cout], the window position (0..3 row-major) of the
 * first max, 255 where the max is not > 0 -- input of ralpb_maxpool_bwd_idx. */
int ralpb_conv_fwd_pool(const void* x_pad, const void* w, const float* bias, void* y_pad, void* pool_out,
                        int pool_pad, void* pool_idx, int n, int h, int w_, int cin, int cout, int k, int pad,
                        int relu, void* stream);
/* 2x2/2 max-pool backward from those argmax bytes: dx (interior of [n][2oh+2pi][2ow+2pi][c]) gets
 * dy at the recorded position, 0 elsewhere (ReLU mask included); colsum as ralpb_maxpool_bwd. */
int ralpb_maxpool_bwd_idx(const void* idx, const void* dy, int n, int oh, int ow, int c, int pad_out, int pad_in,
                          void* dx, float* colsum, void* stream);
int ralpb_conv_dgrad(const void* dy_pad, const void* wd, const void* mask_pad, void* dx_pad, float* colsum,
                     int n, int h, int w_, int cin, int cout, int k, int pad, void* stream);
int ralpb_conv_wgrad(const void* x_pad, const void* dy_pad, float* dw, float* db, int n, int h, int w_,
                     int cin, int cout, int k, int pad, void* stream);

/* First (RGB) convolution fused with its im2col (3x3, stride 1, pad 1, 3 -> 64 channels,
 * h % 8 == 0, w % 16 == 0): the patch rows are built on chip from the fp32 NHWC image.
 *   wf: [64][32] bf16, columns (r*3+s)*3+ch, column 27 = bias;  y_pad/dy_pad: [n][h+2p][w+2p][64]
 *   (y written on interior pixels, ReLU fused);  dw: [64][32] fp32 accumulated (column 27 = db).
 * Returns an error for other shapes (the im2col GEMM path, ralpb_pack_im2col + ralpb_gemm, covers
 * them). */
int ralpb_conv_first_fwd(const float* img, int n, int h, int w, const void* wf, void* y_pad, int pad_out,
                         void* stream);
int ralpb_conv_first_wgrad(const float* img, int n, int h, int w, const void* dy_pad, int pad_out, float* dw,
                           void* stream);

/* fp32 NHWC images -> bf16 padded NHWC with cp >= c channels (zero fill). */
int ralpb_pack_input(const float* x, int n, int h, int w, int c, void* out, int cp, int pad,
                     void* stream);
/* im2col patch matrix of fp32 NHWC images for a first (RGB) convolution: rows = the conv's
 * padded output grid [n][ho+2po][wo+2po], columns j = (r*k+s)*c+ch, column k*k*c = 1 (bias),
 * zero elsewhere and on border rows; kpad >= k*k*c+1, multiple of 8. */
int ralpb_pack_im2col(const float* x, int n, int h, int w, int c, int k, int stride, int pad, int ho, int wo,
                      int po, int kpad, void* out, void* stream);
/* Max pool (infer_pool, layers.py:106-114; stride defaults to window). */
int ralpb_maxpool_fwd(const void* x, int n, int h, int w, int c, int pad_in, int k, int stride,
                      void* y, int pad_out, void* stream);
/* Pool forward that also records, per output element, the window position (ky*k+kx) of the first
 * max (255 where it is not > 0), and the backward that gathers from those bytes -- any window and
 * stride, e.g. AlexNet's overlapping 3/2 pools (the input is not re-read). */
int ralpb_maxpool_fwd_idx(const void* x, int n, int h, int w, int c, int pad_in, int k, int stride, void* y,
                          int pad_out, void* idx, void* stream);
int ralpb_maxpool_bwd_gather(const void* idx, const void* dy, int n, int h, int w, int c, int pad_in, int k,
                             int stride, int pad_out, void* dx, float* colsum, void* stream);
/* colsum (may be NULL, c <= 1024): colsum[ch] += sum of the stored dx (bias gradient of the conv
 * feeding the pool, fused into the pool backward). */
int ralpb_maxpool_bwd(const void* x, const void* dy, int n, int h, int w, int c, int pad_in, int k,
                      int stride, int pad_out, void* dx, float* colsum, void* stream);
/* Softmax cross-entropy (the LOSS layer, layers.py:161-163): per-row loss and
 * dlogits = (softmax - onehot) * scale (bf16). */
int ralpb_softmax_xent(const float* logits, int rows, int classes, long long ld,
                       const int32_t* labels, float scale, float* row_loss, void* dlogits,
                       long long ld_d, void* stream);
/* SGD with momentum, PyTorch form: v = mu*v + gscale*g; p -= lr*v. */
int ralpb_sgd_momentum(float* p, float* v, const float* g, long long n, float lr, float mu,
                       float gscale, void* stream);
/* db[c] += sum_r dy[r*ld + c] (bf16 in, fp32 atomics). */
int ralpb_colsum_bf16(const void* dy, long long rows, int c, long long ld, float* db, void* stream);
/* fp32 [co][taps][ci] -> bf16 forward copy and bf16 [ci][taps-1-t][co] dgrad copy (wd may be NULL). */
int ralpb_conv_weight_prep(const float* w, int co, int taps, int ci, void* wf, void* wd, void* stream);
int ralpb_cast_bf16(const float* x, long long n, void* y, void* stream);

/* ------------------------------------------------------------ executor
 * One ralpb_model per rank (one process per GPU).  The layer table is the
 * reference ModelGraph (pkg/src/ralp/layers.py:204-267) lowered by the Python
 * package; `split` is the 1-based cut index chosen by profile()/find_split()
 * (profiler.py:101-134,187-227); the strategy mirrors StrategyKind
 * (costmodel.py:34-37): RALP = conv front replicated + FC tail on the PS rank,
 * BASELINE_PS = every layer on every worker, all parameters through the PS. */
/* Layer kinds.  BLOCK: a ResNet bottleneck block (1x1 -> 3x3 (stride) -> 1x1, batch norm after
 * every convolution, ReLU, identity or 1x1-projection shortcut; the catalog's linearised
 * s?b?_{a,b,c,down} entries, pkg/tools/build_catalog.py:286-333).  APOOL: global average pool.
 * MODULE: a branch group (an Inception / GoogLeNet module, or a single convolution of any window,
 * stride and padding): the nodes [node_begin, node_begin + node_count) of the node table passed to
 * ralpb_model_create_graph, whose output nodes are concatenated along channels (the catalog's
 * linearised "<group>_<branch>" entries, the last one carrying the merged group output;
 * pkg/tools/build_catalog.py:115-285). */
enum { RALPB_CONV = 0, RALPB_POOL = 1, RALPB_FC = 2, RALPB_BLOCK = 3, RALPB_APOOL = 4, RALPB_MODULE = 5 };

/* A node of a MODULE.  CONV: kh x kw window, stride, zero padding (pad_h, pad_w), cout output
 * channels, then batch norm (bn = 1: training-mode batch statistics, learnable scale / shift, no
 * bias) or a bias (bn = 0), then ReLU.  MAXPOOL: first maximum of the window, padding never wins.
 * AVGPOOL: mean over the window's in-image elements (padding excluded from the count).  input: the
 * node it reads (an earlier node of the same module; -1 = the module input).  output = 1: part of
 * the module output (outputs concatenate in node order; an output node feeds no other node). */
enum { RALPB_NODE_CONV = 0, RALPB_NODE_MAXPOOL = 1, RALPB_NODE_AVGPOOL = 2 };
typedef struct {
  int op;
  int input;
  int kh, kw, stride, pad_h, pad_w;
  int cout;
  int bn;
  int output;
} ralpb_node_desc;
/* BASELINE: StrategyKind.BASELINE_PS (every layer on every worker, all parameters through the
 * sharded PS).  RALP: StrategyKind.RALP.  RING: StrategyKind.RING_ALLREDUCE (simulator.py:719-737)
 * with the hand-written reduce-scatter + SGD + all-gather over NVLink; RING_EXTERNAL: the same
 * but the step stops after the backward so the caller all-reduces the gradient buffer (e.g. with
 * NCCL, the comparison baseline) and then calls ralpb_model_apply. */
/* RALP_MPS: layer-placed with the FC tail sharded over every GPU (the paper's
 * multi-PS future work; the reference forbids ps_count != 1 for RALP, costmodel.py:75-76): the
 * first FC layer column-parallel, the second row-parallel (partial sums reduced on rank 0), later
 * FC layers on rank 0; cuts all-gathered, the cut gradient reduce-scattered back. */
/* BASELINE_LAYER_SHARDS: BASELINE with the reference's own PS shard layout -- whole weighted
 * layers assigned round-robin to the W shards (simulator.py:551-563: "PS frameworks place whole
 * variables"), so under parameter skew one shard carries most of the model (VGG-16: fc1) -- instead
 * of equal contiguous byte shards.  Same logical bytes (volume_baseline), a different hot spot. */
enum { RALPB_STRATEGY_BASELINE = 0, RALPB_STRATEGY_RALP = 1, RALPB_STRATEGY_RING = 2, RALPB_STRATEGY_RING_EXTERNAL = 3,
       RALPB_STRATEGY_RALP_MPS = 4, RALPB_STRATEGY_BASELINE_LAYER_SHARDS = 5 };

typedef struct {
  int kind;            /* RALPB_CONV / RALPB_POOL / RALPB_FC / RALPB_BLOCK / RALPB_APOOL */
  int k, stride, pad;  /* window geometry (conv / pool; block: stride of its 3x3 convolution) */
  int h, w, cin;       /* per-sample input shape (fc: cin = input features, h = w = 0) */
  int cout;            /* conv / block output channels, fc output features */
  int relu;            /* ReLU after the layer (conv, fc except the last) */
  int bn;              /* conv: batch norm (training-mode batch statistics, scale + shift) before
                          the ReLU, no bias */
  int width;           /* block: bottleneck width (the 1x1 / 3x3 convolutions' channels) */
  int downsample;      /* block: 1x1 projection shortcut (else identity) */
  int node_begin;      /* module: its nodes in the node table (ralpb_model_create_graph) */
  int node_count;
} ralpb_layer_desc;

typedef struct {
  double loss;                 /* mean cross-entropy over the job's W*b samples (ps_rank -- rank 0 for
                                  RALP_MPS / RING; NaN elsewhere) */
  long long logical_bytes;     /* descriptor-unit (elem_bytes) bytes of the transfers THIS rank issued
                                  this step, counted where it issues them, at the reference's count_wire
                                  sites (simulator.py:647,663,677,689,707,713): worker act + grad, PS
                                  actgrad + pull (per sync shard it owns).  Summed over the ranks it is
                                  the job's volume_*() (costmodel.py:107-162). */
  long long physical_bytes;    /* bytes this rank moved over NVLink this step (out + in) */
  int launches;                /* kernels this rank launched in the step */
  float ms_step;               /* device time of the whole step on this rank (CUDA events) */
  float ms_front_fwd;          /* worker front forward */
  float ms_back;               /* PS back segment incl. waiting for cut activations */
  float ms_front_bwd;          /* worker front backward incl. waiting for the act-grad */
  float ms_sync;               /* parameter synchronisation (sharded PS) + weight re-layout */
  float ms_gemm;               /* sum of tcgen05 GEMM-engine launch durations (profiling mode only) */
  int gemm_launches;           /* GEMM-engine launches timed (profiling mode only) */
  long long nvlink_out_bytes;  /* ... of physical_bytes: stored to peers (cut / act-grad pushes, pulls) */
  long long nvlink_in_bytes;   /* ... loaded from peers (sharded-PS gradient reads) */
} ralpb_step_stats;

typedef struct ralpb_model ralpb_model;

/* Arithmetic of the step.  BF16: bf16 operands / activations, fp32 accumulation, fp32 master
 * parameters (the throughput mode).  FP32: the parity mode north_star pins to the fp32 oracle --
 * every activation, activation gradient and GEMM operand is carried as three bf16 pieces
 * (hi, mid, lo; their sum is the fp32 value exactly) and every contraction runs on the same tcgen05
 * GEMM engine over the pieces (all 9 piece products, fp32 accumulation), so results match plain
 * fp32 arithmetic to ~1e-5 relative (reference unit: elem_bytes=4, layers.py:238-250). */
enum { RALPB_PRECISION_BF16 = 0, RALPB_PRECISION_FP32 = 1 };

/* Replaces JobSpec + _JobRun.__init__ (costmodel.py:64-86, simulator.py:517-567).
 * workers: ranks that run a conv front.  workers == world is the colocated placement (the PS role on
 * ps_rank, which is also a worker); workers == world - 1 (RALP only) is the paper's RALP-N placement
 * (costmodel.py:244-245, gpu_assignments): ps_rank is a dedicated PS GPU that runs only the back
 * segment, the other ranks are workers 0..W-1 in rank order. */
int ralpb_model_create(const ralpb_layer_desc* layers, int n_layers, int split, int batch, int strategy,
                       int rank, int world, int ps_rank, int elem_bytes, int precision, int workers,
                       ralpb_model** out);
/* ralpb_model_create for a layer table with MODULE layers: `nodes` (n_nodes entries) is the node
 * table the modules index.  ralpb_model_create(...) == ralpb_model_create_graph(..., NULL, 0, ...). */
int ralpb_model_create_graph(const ralpb_layer_desc* layers, int n_layers, const ralpb_node_desc* nodes,
                             int n_nodes, int split, int batch, int strategy, int rank, int world, int ps_rank,
                             int elem_bytes, int precision, int workers, ralpb_model** out);
void ralpb_model_destroy(ralpb_model* m);
/* 64-byte CUDA IPC handle of this rank's exchange arena; ralpb_model_ipc_open takes
 * world*64 bytes (rank-major) and maps the peers. */
int ralpb_model_ipc_handle(ralpb_model* m, void* out64);
int ralpb_model_ipc_open(ralpb_model* m, const void* handles);
/* Host (on_host=1) or device fp32 parameters of layer `layer` (0-based):
 * conv w [cout][k][k][cin], b [cout] (bn conv: b = [gamma (cout) | beta (cout)]);
 * fc w [out][in] (in = HWC-flattened), b [out];
 * block: w = every parameter of the block, in order wa [width][cin], wb [width][3][3][width],
 * wc [cout][width] (, wd [cout][cin]), b = [gamma_a | beta_a | gamma_b | beta_b | gamma_c | beta_c
 * (| gamma_d | beta_d)];
 * module: w = its convolution nodes' filters [cout][kh][kw][cin] back to back in node order,
 * b = their [gamma | beta] (bn) or bias [cout] in the same order. */
int ralpb_model_set_params(ralpb_model* m, int layer, const float* w, const float* b, int on_host);
int ralpb_model_get_params(ralpb_model* m, int layer, float* w, float* b, int on_host);
/* This rank's parameter gradient of `layer` from the last step (same layout as get_params; host or
 * device destination): the front's summed over this rank's batch before the sharded-PS reduction,
 * the FC tail's over the PS's rows.  Inspection for the per-layer parity tests. */
int ralpb_model_get_grads(ralpb_model* m, int layer, float* w, float* b);
/* One training step of this rank's worker batch: images [b][h][w][c] fp32 NHWC, labels [b] int32,
 * host or device memory.  Executes _ralp_worker/_ralp_ps (simulator.py:669-715) or
 * _baseline_worker/_baseline_ps (simulator.py:637-665).  Asynchronous: host inputs are copied on
 * a copy stream into one of two device staging buffers, so the copy of step t+1 overlaps step t
 * (pinned host buffers must stay unchanged until that step's loss has been read; pageable ones
 * are staged before the call returns). */
int ralpb_model_step(ralpb_model* m, const void* images, const int32_t* labels, int on_host, float lr,
                     float mu);
/* Synchronises the model stream and reports the last step. */
int ralpb_model_stats(ralpb_model* m, ralpb_step_stats* out);
/* Loss of the step issued `lag` steps ago (0 = latest, lag < 4), copied to pinned host memory at
 * the end of that step; waits for that step only (NaN on ranks without the FC tail). */
int ralpb_model_read_loss(ralpb_model* m, int lag, float* out);
void* ralpb_model_stream(ralpb_model* m);
/* Inspection: copies one of the last step's device buffers to host_out (may be NULL to query) and
 * returns its element count, or -1.  Layouts (BF16 precision; FP32 precision: every bf16 buffer is
 * stored as three pieces -- per pixel / row the hi channels, then the mid, then the lo channels --
 * and the byte size triples; the element count returned is the value count):
 *   ACT i / ACT_GRAD i   bf16 padded NHWC input of front layer i / its gradient
 *   LOGITS               fp32 [rows][ld]            DLOGITS          bf16 [rows][ld]
 *   FC_OUT i             bf16 [rows][ld] output of hidden FC layer i (ReLU applied)
 *   FC_OUT_GRAD i        bf16 [rows][ld] gradient w.r.t. FC layer i's output (ReLU-masked)
 *   FC_WEIGHT i          bf16 [out][in] operand copy of FC layer i
 *   CUT_ROWS / CUT_GRAD_ROWS  bf16 [rows][cut] the PS's exchanged cut rows (every worker's cut --
 *                        layer split-1's output in its padded layout; at the FC boundary the HWC
 *                        flatten) / their gradient;  CUT_GRAD  bf16 [b][cut] the act-grad this rank
 *                        received;  FC_IN / FC_IN_GRAD  bf16 [rows][fc_in] the FC tail's input rows /
 *                        their gradient (== CUT_ROWS / CUT_GRAD_ROWS without a conv back segment);
 *                        MPS_PARTIAL  fp32 [rows][ld] (RALP_MPS) */
enum {
  RALPB_DBG_ACT = 0, RALPB_DBG_ACT_GRAD = 1, RALPB_DBG_LOGITS = 2, RALPB_DBG_FC_OUT = 3,
  RALPB_DBG_MPS_PARTIAL = 4, RALPB_DBG_FC_WEIGHT = 5, RALPB_DBG_DLOGITS = 6, RALPB_DBG_FC_OUT_GRAD = 7,
  RALPB_DBG_CUT_ROWS = 8, RALPB_DBG_CUT_GRAD_ROWS = 9, RALPB_DBG_CUT_GRAD = 10, RALPB_DBG_FC_IN = 11,
  RALPB_DBG_FC_IN_GRAD = 12
};
long long ralpb_model_debug_buffer(ralpb_model* m, int i, int which, void* host_out);
/* RING_EXTERNAL: the fp32 gradient vector (all parameters, device memory, `*n` floats) the caller
 * all-reduces (sum over ranks) after ralpb_model_step, and the update that follows
 * (SGD-momentum + bf16 re-layout) on the model stream. */
int ralpb_model_grad_buffer(ralpb_model* m, float** ptr, long long* n);
int ralpb_model_apply(ralpb_model* m, float lr, float mu);
/* Profiling mode: bracket every tensor-core launch with CUDA events (reported in stats). */
int ralpb_model_set_profiling(ralpb_model* m, int on);
/* Per-launch records of the last profiled step: kind = 0 conv fwd/dgrad (single CTA), 1 conv
 * fwd/dgrad (CTA pair), 2 conv wgrad (CTA pair), 3 conv wgrad (single CTA), 4 first-conv fwd,
 * 5 first-conv wgrad, 6 GEMM, 7 peer push (cut gather / act-grad scatter), 8 sharded-PS update,
 * 9 max-pool backward, 10 SGD-momentum; ms = CUDA-event duration on the launching stream;
 * flops = algorithmic FLOPs (7, 8: bytes moved over NVLink per direction); bytes = algorithmic
 * DRAM bytes (7, 8: NVLink bytes per direction).  Returns the number of records (writes at most
 * cap) or -1. */
typedef struct {
  int kind;
  float ms;
  double flops;
  double bytes;        /* algorithmic DRAM bytes (push / shard update: NVLink bytes per direction) */
  float t0;            /* start, ms after the step's first event (a per-rank timeline) */
  int stream;          /* 0 main, 1 aux (FC update / filter copies), 2 comm (act-grad scatter), 3 sync (bucket) */
} ralpb_launch_rec;
int ralpb_model_timed_launches(ralpb_model* m, ralpb_launch_rec* out, int cap);

#ifdef __cplusplus
}
#endif

#endif /* RALPB_H_ */
