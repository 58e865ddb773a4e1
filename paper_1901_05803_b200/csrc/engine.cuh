// Native executor of one job's training step under a placement strategy.
// See engine.cu for the schedule; the C ABI (ralpb_model_*) is in api_engine.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <string>
#include <vector>
#include "../../include/ralpb.h"
#include "conv.cuh"
#include "exchange.cuh"

namespace ralpb {

using bf16 = __nv_bfloat16;

struct ActBuf {
  bf16* ptr = nullptr;
  int n = 0, h = 0, w = 0, c = 0, pad = 0;
  long long rows() const { return static_cast<long long>(n) * (h + 2 * pad) * (w + 2 * pad); }
  long long elems() const { return rows() * c; }
};

// A ResNet bottleneck block's operands and saved tensors (block.cu).  Forward:
//   a_pre = x Wa^T; a = relu(bn_a(a_pre)) (padded); b_pre = conv3x3_s(a, Wb); b = relu(bn_b(b_pre));
//   c_pre = b Wc^T; y = relu(bn_c(c_pre) + (downsample ? bn_d(subsample_s(x) Wd^T) : x)).
struct BlockBufs {
  int cin = 0, width = 0, cout = 0, stride = 1, down = 0;
  int n = 0, h = 0, w = 0, ho = 0, wo = 0;
  int groups = 1;                 // batch-norm statistics per image group (the PS's back segment:
                                  // one group per worker's b rows)
  long long wa_off = 0, ga_off = 0, wb_off = 0, gb_off = 0, wc_off = 0, gc_off = 0, wd_off = 0, gd_off = 0;
  __nv_bfloat16 *wa = nullptr, *wbf = nullptr, *wbd = nullptr, *wc = nullptr, *wd = nullptr;
  __nv_bfloat16 *a_pre = nullptr, *a = nullptr, *b_pre = nullptr, *b = nullptr, *c_pre = nullptr, *d_in = nullptr,
                *d_pre = nullptr, *col = nullptr;
  __nv_bfloat16 *dc_pre = nullptr, *dz = nullptr, *db = nullptr, *db_pre = nullptr, *dil = nullptr, *da = nullptr,
                *da_pre = nullptr, *dd_pre = nullptr, *dxs = nullptr;
  float* stats = nullptr;   // [4][2][cmax]: mean / rstd of bn a, b, c, d
  uint8_t *ma = nullptr, *mb = nullptr, *mc = nullptr;   // ReLU masks (bits) of a, b and the output
  int cmax = 0;
};

// A branch group (RALPB_MODULE, graph.cu): nodes in topological order, output nodes
// concatenated along channels into the module output [n][ho][wo][cout] (unpadded NHWC).
struct ModNode {
  ralpb_node_desc d{};
  int cin = 0, h = 0, w = 0, ho = 0, wo = 0;   // per-sample input / output geometry
  int out_off = 0;             // output node: channel offset in the module output
  int consumers = 0;           // nodes reading this node's output
  bool direct = false;         // conv 1x1 / stride 1 / no padding: a GEMM over the input rows
  bool same = false;           // conv 3x3 / 5x5, stride 1, "same" padding p, channels % 16: the
  int p = 0;                   // implicit-GEMM conv kernels (conv.cuh) over padded copies
  int crop = 0;                // same, 'valid' node (pad 0): its outputs are the same conv's cropped by p
  int cpad = 0;                // same: input channels as the implicit kernels see them (cin, or cin
                               // zero-extended to the channel alignment)
  float* gw = nullptr;         // same, cpad > cin: the padded filters (fp32, prep) / their gradient
  __nv_bfloat16* xp = nullptr;        // same: the input, padded by p (zero borders)
  __nv_bfloat16* dzp = nullptr;       // same: gradient w.r.t. the pre-activation, padded
  __nv_bfloat16* dxp = nullptr;       // same: gradient w.r.t. the input, padded
  __nv_bfloat16* wdb = nullptr;       // same: backward-data filters [cin][taps reversed][cout]
  long long w_off = -1, b_off = -1;   // conv: filters [cout][kh*kw*cin], then gamma|beta or bias
  __nv_bfloat16* wbf = nullptr;       // conv: bf16 copy of the filters
  __nv_bfloat16* z = nullptr;         // bn conv: output before the batch norm (same: padded; bias
                                      // conv: the same path's padded output)
  __nv_bfloat16* y = nullptr;         // non-output node: its output
  __nv_bfloat16* dy = nullptr;        // non-output node: gradient w.r.t. its output
  uint8_t* idx = nullptr;             // max pool: window position of the first max (255: not > 0)
  float* stats = nullptr;             // bn conv: [2][cout] mean / rstd
  uint8_t* mask = nullptr;            // bn conv: ReLU mask bits of its output [rows][cout/8]
  int grp = -1, grp_col = 0;          // sibling group (ModGroup) and this node's first column in it
  long long K() const { return static_cast<long long>(d.kh) * d.kw * cin; }
};
// Sibling 1x1 convolutions (batch-normalised, same input): one GEMM over the concatenated
// filters [ncat][cin] (their parameters are laid out back to back), one statistics pass over the
// concatenated pre-activations, one backward-filter and one backward-data GEMM over the
// concatenated gradient (the sum over the siblings' input gradients falls out of the contraction).
struct ModGroup {
  std::vector<int> members;           // node indices, ascending
  int ncat = 0;                       // sum of the members' output channels
  long long w_off = -1;               // the members' filters, contiguous [ncat][cin]
  __nv_bfloat16* wbf = nullptr;       // bf16 copy
  __nv_bfloat16* z = nullptr;         // pre-batch-norm outputs [rows][ncat]
  __nv_bfloat16* dz = nullptr;        // gradient w.r.t. them [rows][ncat]
  float* stats = nullptr;             // [groups][2][ncat] mean / rstd
};
struct ModuleBufs {
  int n = 0, h = 0, w = 0, cin = 0, ho = 0, wo = 0, cout = 0;
  int groups = 1;                 // batch-norm statistics per image group (see BlockBufs)
  std::vector<ModNode> nodes;
  std::vector<ModGroup> sib;      // sibling 1x1 groups (RALPB_MODULE_FUSE=0: none)
  __nv_bfloat16* col = nullptr;   // im2col patches / their gradient (largest conv node)
  __nv_bfloat16* dz = nullptr;    // gradient w.r.t. a conv node's pre-activation (largest node)
  long long col_elems = 0, dz_elems = 0;
};

struct FrontLayer {
  int kind = 0;                // RALPB_CONV / RALPB_POOL / RALPB_BLOCK / RALPB_APOOL
  ConvGeom g{};                // conv geometry (cin padded to 16)
  int cin_real = 0;
  int k = 0, stride = 0;       // pool window
  int relu = 1;
  long long w_off = 0, b_off = 0;  // offsets (floats) into the flat parameter vector
  long long w_count = 0;           // cout*k*k*cin_pad
  bf16* wf = nullptr;          // forward filter [cout][k*k][cin]
  bf16* wd = nullptr;          // backward-data filter [cin][k*k][cout]
  bool im2col = false;         // first conv as a GEMM over the im2col patch matrix acts[0]
  int kpad = 0;                // im2col row width (k*k*cin + 1 bias column, padded)
  bool fused = false;          // im2col layer run by the fused first-conv kernels (conv_first.cu):
                               // patches built on chip from the fp32 image, acts[0] unused
  bool fused_fwd = false;      // pool computed in the preceding conv's epilogue
  uint8_t* idx = nullptr;      // ... with argmax bytes [n][oh][ow][c] for its backward
  int pool_pad = 0;            // pool: zero padding (ResNet's 3x3/2 pad 1)
  bool bn = false;             // conv: batch norm (+ReLU) after it, no bias; b_off = gamma, beta follows
  __nv_bfloat16* pre = nullptr;     // bn conv: its output before the batch norm
  __nv_bfloat16* dpre = nullptr;    // ... and the gradient w.r.t. it
  float* bn_stats = nullptr;        // bn conv: [2][cout] mean / rstd
  uint8_t* bn_mask = nullptr;       // bn conv: ReLU mask bits of its output [rows][cout/8]
  int blk = -1;                // RALPB_BLOCK: index into Model::blocks
  int mod = -1;                // RALPB_MODULE: index into Model::modules
};

struct FcLayer {
  int in = 0, out = 0, relu = 1;
  int ld_out = 0;                  // padded row stride (elements) of this layer's output
  long long w_off = 0, b_off = 0;
  bf16* wbf = nullptr;             // [lout][lin] (pair precision: the forward pair operand)
  bf16* wbd = nullptr;             // pair precision: the backward-data pair operand
  int lout = 0, lin = 0;           // this rank's weight block: [out][in], or a slice (RALP_MPS:
                                   // layer 0 rows [r*s0, (r+1)*s0), layer 1 columns of that range)
};

struct Model {
  // configuration
  int rank = 0, world = 1, ps_rank = 0, device = 0;
  int batch = 0, split = 0, strategy = RALPB_STRATEGY_RALP, elem_bytes = 4;
  int precision = RALPB_PRECISION_BF16;
  int pieces = 1;                  // bf16 pieces per value (parity precision: 3, pair.cuh)
  int workers = 1;                 // ranks that run a conv front (world, or world - 1 for RALP-N)
  bool dedicated_ps = false;       // RALP-N: ps_rank runs only the back segment
  bool is_worker = true;           // this rank runs a conv front
  int widx = 0;                    // this rank's worker index (rank order, the dedicated PS skipped)
  std::vector<int> worker_ranks;   // worker index -> rank
  bool layer_shards = false;          // BASELINE_LAYER_SHARDS: whole layers round-robin over the shards
  int bucket_k = -1;                  // sync bucket: layers [bucket_k, split) are synchronised on
  long long bucket_lo = 0;            // sync_stream under the remaining backward; their parameters
  bool bucket_forked = false;         // are [bucket_lo, n_front); forked in the current step body
  cudaStream_t sync_stream = nullptr;
  cudaEvent_t ev_b1 = nullptr, ev_b1_done = nullptr;
  float step_lr = 0.f, step_mu = 0.f; // hyper-parameters of the step being issued
  std::vector<std::vector<std::pair<long long, long long>>> shard_ranges;   // per shard: [lo, hi) floats
  std::vector<long long> shard_real;  // real (descriptor) parameters in each sync shard, for the
                                      // logical byte count of the pull / ring sites
  std::vector<ralpb_layer_desc> desc;
  std::vector<FrontLayer> front;
  std::vector<BlockBufs> blocks;   // RALPB_BLOCK layers
  std::vector<ModuleBufs> modules; // RALPB_MODULE layers
  bool branchy = false;            // the model has blocks / batch-normalised convolutions
  float* bn_work = nullptr;        // kBnWorkFloats batch-norm reduction scratch (resnet.cuh)
  std::vector<FcLayer> back;
  std::vector<ActBuf> acts;        // acts[i] = input of front layer i; acts.back() = cut (local)
  int in_h = 0, in_w = 0, in_c = 0, in_cp = 0;
  int cut_elems = 0;               // per-sample elements of the FC tail's input (HWC-flattened pool output)
  int nconv = 0;                   // conv / pool layers before the FC tail
  bool bseg = false;               // split < nconv: layers [split, nconv) run on the PS over W*b rows
  long long real_bseg = 0;         // descriptor parameters of that conv back segment (PS-local)
  long long bseg_end = 0;          // its parameters occupy [n_front, bseg_end) of the flat vector
  int xch_elems = 0;               // per-sample bf16 elements of the exchanged cut (layer split-1's
                                   // output in its padded layout; == cut_elems at the FC boundary)
  long long xch_logical = 0;       // ... its descriptor elements (h*w*c)
  ActBuf bin;                      // PS: the back segment's input, every worker's cut rows (= xin)
  int rows_back = 0;               // rows the back segment processes on this rank
  bool holds_back = false;         // this rank runs the FC tail
  long long n_front = 0, n_total = 0;  // floats in the flat parameter vector (front prefix, total)
  long long real_front = 0, real_total = 0;  // logical parameter counts (unpadded)

  // device memory
  cudaStream_t stream = nullptr;
  void* arena = nullptr;           // IPC-exported allocation
  size_t arena_bytes = 0;
  std::vector<void*> owned;        // other allocations
  uint32_t* flags = nullptr;       // in arena
  uint32_t* counters = nullptr;    // local
  float* P = nullptr;              // params (arena)
  float* G = nullptr;              // grads (arena)
  float* V = nullptr;              // momentum (local)
  bf16* xin = nullptr;             // exchanged cut rows [rows_back][xch_elems] (arena; PS reads)
  bf16* dxin = nullptr;            // their gradient [rows_back][xch_elems] (PS; scattered back)
  bf16* x_fc = nullptr;            // FC tail input [rows_back][cut_elems] (== xin without a conv back
                                   // segment)
  int32_t* labels_all = nullptr;   // [rows_back] (arena, PS)
  bf16* dcut = nullptr;            // cut gradient received from the PS [batch][xch_elems] (arena)
  bf16* dx_fc = nullptr;           // FC tail input gradient [rows_back][cut_elems] (PS; == dxin
                                   // without a conv back segment)
  std::vector<bf16*> hid;          // FC outputs (bf16) for hidden layers
  float* logits = nullptr;
  float* fc_scratch = nullptr;     // split-K accumulators for FC GEMMs with few rows
  bf16* dlogits = nullptr;
  std::vector<bf16*> dyb;          // dyb[j] = gradient w.r.t. FC layer j's output (j < last; the
                                   // last layer's is dlogits), kept for the deferred wgrads
  cudaStream_t aux_stream = nullptr;   // PS: FC weight gradients + SGD, concurrent with the
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // front backward
  cudaEvent_t ev_wd_fork = nullptr, ev_wd_join = nullptr;  // backward-data filter copies (aux stream)
  cudaStream_t comm_stream = nullptr;  // PS: the act-grad scatter, concurrent with the FC weight
  cudaEvent_t ev_comm_fork = nullptr, ev_comm_join = nullptr;  // gradients and the front backward
  float* row_loss = nullptr;
  float* loss = nullptr;           // [4]: the reported loss (mean over the job's samples), [1] this
                                   // rank's own-row sum (baseline / ring: pushed to ps_rank's slot)
  std::vector<bf16*> gacts;        // gacts[i] = gradient w.r.t. acts[i] (dedicated, zero borders)
  // host inputs: double-buffered device staging filled on a copy stream, so the copy of step
  // t+1 overlaps the compute of step t (buffer b is reused once step t-1 has consumed it)
  float* img_dev[2] = {nullptr, nullptr};
  int32_t* lab_dev[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {}, ev_consumed[2] = {};
  const float* step_img = nullptr; // this step's fp32 image batch (device) -- fused first conv
  // per-step loss copied to pinned host memory (ring), readable without draining the stream
  static constexpr int kLossRing = 4;
  float* loss_host = nullptr;
  cudaEvent_t ev_loss[kLossRing] = {};
  uint32_t loss_seq[kLossRing] = {};
  size_t arena_off_flags = 0, arena_off_P = 0, arena_off_G = 0, arena_off_xfc = 0, arena_off_lab = 0,
         arena_off_dcut = 0, arena_off_loss = 0;

  // peers (IPC-mapped base pointers of every rank's arena; self = arena)
  std::vector<char*> peer_base;
  bool peers_open = false;

  // pair precision (RALPB_PRECISION_FP32, pair.cuh): fp32 scratch of the contractions
  float* pair_acc = nullptr;
  float* pair_s = nullptr;
  size_t pair_acc_floats = 0, pair_s_floats = 0;

  // RALP_MPS (FC tail sharded over the ranks)
  bool mps = false;
  int s0 = 0, ld_s0 = 0;           // first FC layer's output slice per rank (and its padded stride)
  bf16* h0s = nullptr;             // [R][ld_s0] this rank's slice of FC-0's output
  bf16* dh0s = nullptr;            // [R][ld_s0] its gradient
  float* p1_local = nullptr;       // [R][ld1] this rank's partial FC-1 pre-activation
  float* dxp = nullptr;            // [R][cut] this rank's partial cut gradient
  size_t arena_off_p1 = 0, arena_off_dh1 = 0, arena_off_dxpart = 0;

  // step state
  uint32_t seq = 0;                // host mirror of *seq_dev (steps issued)
  uint32_t* seq_dev = nullptr;     // device step counter: flag value of the exchange kernels
  // CUDA graph of the step body (everything after the input upload), re-captured when the
  // input pointers or hyper-parameters change; disabled while profiling or RALPB_GRAPH=0
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    const void* img = nullptr;
    const void* lab = nullptr;
    float lr = 0.f, mu = 0.f;
    int launches = 0;
    long long phys = 0, nvl_out = 0, nvl_in = 0, logical = 0;
    uint64_t used = 0;
  };
  GraphEntry graphs[2];            // one per staging buffer (or caller buffers)
  uint64_t graph_clock = 0;
  int launches = 0;
  long long phys_bytes = 0;        // NVLink bytes this rank moved (out + in)
  long long nvl_out = 0, nvl_in = 0;  // ... stored to / loaded from peers
  long long logical = 0;           // descriptor-unit bytes of this rank's count_wire sites
  cudaEvent_t ev[6] = {};
  bool profiling = false;
  GemmTimer timer;
  bool stats_valid = false;
};

int model_create(const ralpb_layer_desc* layers, int n_layers, const ralpb_node_desc* nodes, int n_nodes, int split,
                 int batch, int strategy,
                 int rank, int world, int ps_rank, int elem_bytes, int precision, int workers, Model** out,
                 std::string* why);
void model_destroy(Model* m);
int model_step(Model* m, const void* images, const int32_t* labels, int on_host, float lr, float mu,
               std::string* why);
int model_stats(Model* m, ralpb_step_stats* st, std::string* why);
int model_read_loss(Model* m, int lag, float* out, std::string* why);
int model_set_params(Model* m, int layer, const float* w, const float* b, int on_host, std::string* why);
int model_get_params(Model* m, int layer, float* w, float* b, int on_host, std::string* why);
int model_get_grads(Model* m, int layer, float* w, float* b, std::string* why);
int model_ipc_handle(Model* m, void* out, std::string* why);
int model_ipc_open(Model* m, const void* handles, std::string* why);
int model_set_profiling(Model* m, int on, std::string* why);
int model_timed_launches(Model* m, ralpb_launch_rec* out, int cap, int* n, std::string* why);
int model_grad_buffer(Model* m, float** ptr, long long* n, std::string* why);
int model_apply(Model* m, float lr, float mu, std::string* why);

}  // namespace ralpb
