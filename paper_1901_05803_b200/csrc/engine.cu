// Executor of the layer-placed (RALP) and all-on-PS (baseline) training step.
//
// Per rank (one process per GPU), one CUDA stream, step sequence number `seq`:
//
//   worker front  : pack images -> [conv (implicit GEMM, bias+ReLU) | maxpool]* -> cut
//   cut exchange  : the PS rank's own cut is written straight into the FC input
//                   matrix; every other worker pushes its cut (+labels) into the PS
//                   rank's FC input rows with 128-bit peer stores and raises a flag
//   PS back       : FC fwd (bias+ReLU) -> softmax-CE -> FC wgrad/dgrad/bias-grad over
//                   all W*b rows at once -> FC SGD-momentum (local, never synchronised)
//                   -> push each worker's rows of the cut gradient back + flag
//   worker back   : maxpool bwd (ReLU mask) / conv wgrad (split-K) + bias colsum +
//                   dgrad with the ReLU mask fused into the epilogue
//   sync          : sharded PS over NVLink: every rank owns 1/W of the front
//                   parameter vector; reduce-scatter (peer loads) + SGD-momentum +
//                   all-gather (peer stores) in one kernel, flag barriers around it
//   re-layout     : fp32 master -> bf16 forward / backward-data filter copies
//
// Baseline (StrategyKind.BASELINE_PS): every worker runs every layer on its own batch
// and the whole parameter vector goes through the sharded PS.
//
// Reference: simulator.py:669-715 (RALP worker/PS), :637-665 (baseline), the step
// semantics of SURVEY.md §7.4 (mean loss over W*b, SGD v=mu*v+g, p-=lr*v, HWC flatten).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include "elementwise.cuh"
#include "engine.cuh"
#include "gemm_host.cuh"
#include "pair.cuh"
#include "block.cuh"
#include "graph.cuh"
#include "resnet.cuh"

namespace ralpb {

namespace {

bool fuse_pool_enabled() {
  const char* e = getenv("RALPB_FUSE_POOL");
  return e == nullptr || e[0] != '0';
}

constexpr int kFlagAct = 0;       // [8]  PS: worker r's cut landed
constexpr int kFlagActGrad = 8;   // [1]  worker: act-grad landed
constexpr int kFlagGrad = 16;     // [8]  rank r finished its backward
constexpr int kFlagDone = 24;     // [8]  rank r finished its shard update
constexpr int kFlagP1 = 32;       // [8]  RALP_MPS, rank 0: rank r's FC-1 partial landed
constexpr int kFlagDh1 = 40;      // [1]  RALP_MPS: FC-1 output gradient landed
constexpr int kFlagDcut = 48;     // [8]  RALP_MPS: rank r's partial of this rank's cut gradient landed
constexpr int kFlagLoss = 56;     // [7]  ps_rank: worker w's own-row loss sum landed (baseline / ring)
constexpr int kFlagPsFree = 64;   // [1]  worker: the dedicated PS finished the previous step
constexpr int kFlagGradB = 80;    // [8]  rank r finished the backward of the sync bucket's layers
constexpr int kFlagDoneB = 88;    // [8]  rank r finished its shard of the sync bucket
constexpr int kNumFlags = 96;
constexpr int kCtrScatter = 48;   // [8]  per-destination counters of the fused act-grad scatter
// The parameter vector is padded to a multiple of 4 * lcm(1..8) floats, so every sync group size
// (world, or world - 1 workers with a dedicated PS) splits it into float4-aligned equal shards.
constexpr long long kShardAlign = 4 * 840;
constexpr int kNumCounters = 64;  // last-CTA counters (local)

long long align_up(long long x, long long a) { return (x + a - 1) / a * a; }

#define RALPB_TRY(expr)                                   \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) {                              \
      if (why->empty()) *why = std::string(#expr);        \
      *why += std::string(": ") + cudaGetErrorString(_e); \
      return 1;                                           \
    }                                                     \
  } while (0)

template <class T>
T* alloc(Model* m, size_t count, std::string* why) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(count * sizeof(T), 16)) != cudaSuccess) {
    *why = "cudaMalloc failed (" + std::to_string(count * sizeof(T)) + " bytes)";
    return nullptr;
  }
  m->owned.push_back(p);
  return static_cast<T*>(p);
}


char* peer(Model* m, int r) { return m->peer_base[r]; }
template <class T>
T* at(Model* m, int r, size_t off) { return reinterpret_cast<T*>(peer(m, r) + off); }

bool pair_mode(const Model* m);
int pair_relayout(Model* m, bool front, bool fc, cudaStream_t s, std::string* why);

}  // namespace

int model_create(const ralpb_layer_desc* layers, int n_layers, const ralpb_node_desc* nodes, int n_nodes, int split,
                 int batch, int strategy, int rank, int world, int ps_rank, int elem_bytes, int precision, int workers,
                 Model** out, std::string* why) {
  if (n_layers < 2 || batch < 1 || world < 1 || world > kMaxRanks || rank < 0 || rank >= world ||
      ps_rank < 0 || ps_rank >= world) {
    *why = "bad model configuration";
    return 1;
  }
  if (batch % 4 != 0) { *why = "batch must be a multiple of 4"; return 1; }
  if (strategy < RALPB_STRATEGY_BASELINE || strategy > RALPB_STRATEGY_BASELINE_LAYER_SHARDS) { *why = "unknown strategy"; return 1; }
  const bool layer_shards = strategy == RALPB_STRATEGY_BASELINE_LAYER_SHARDS;
  if (layer_shards) strategy = RALPB_STRATEGY_BASELINE;   // the baseline with whole-layer PS shards
  if (precision != RALPB_PRECISION_BF16 && precision != RALPB_PRECISION_FP32) { *why = "unknown precision"; return 1; }
  if (workers != world && !(workers == world - 1 && workers >= 1 && strategy == RALPB_STRATEGY_RALP)) {
    *why = "workers must equal world, or world - 1 (RALP-N: a dedicated PS rank, RALP strategy only)";
    return 1;
  }
  if (precision == RALPB_PRECISION_FP32 && strategy == RALPB_STRATEGY_RALP_MPS) {
    *why = "the sharded FC tail (RALP_MPS) runs in bf16 precision only";
    return 1;
  }
  auto m = new Model();
  m->layer_shards = layer_shards;
  m->rank = rank; m->world = world; m->ps_rank = ps_rank; m->batch = batch;
  m->strategy = strategy; m->elem_bytes = elem_bytes;
  m->precision = precision;
  m->workers = workers;
  m->dedicated_ps = workers < world;
  for (int r = 0; r < world; ++r)
    if (!(m->dedicated_ps && r == ps_rank)) m->worker_ranks.push_back(r);
  m->is_worker = !(m->dedicated_ps && rank == ps_rank);
  m->widx = 0;
  for (int i = 0; i < workers; ++i)
    if (m->worker_ranks[i] == rank) m->widx = i;
  m->desc.assign(layers, layers + n_layers);
  cudaGetDevice(&m->device);
  auto fail = [&](const std::string& w) { *why = w; model_destroy(m); return 1; };

  int nconv = 0;
  while (nconv < n_layers && layers[nconv].kind != RALPB_FC) ++nconv;
  if (nconv == 0 || nconv == n_layers) return fail("model needs a conv/pool front and an FC tail");
  for (int i = nconv; i < n_layers; ++i)
    if (layers[i].kind != RALPB_FC) return fail("only FC layers may follow the first FC layer");
  const bool layer_placed = strategy == RALPB_STRATEGY_RALP || strategy == RALPB_STRATEGY_RALP_MPS;
  m->mps = strategy == RALPB_STRATEGY_RALP_MPS;
  // split = 1-based cut index of the partitioner (profiler.py:101-134): layers [0, split) are the
  // replicated worker front; conv / pool layers [split, nconv) -- a conv back segment -- run on the
  // PS over the W*b gathered rows together with the FC tail (layer-placed, single PS, bf16)
  if (layer_placed && (split < 1 || split > nconv))
    return fail("the split must cut inside the conv/pool front or at the FC boundary (1.." + std::to_string(nconv) + ")");
  if (layer_placed && split < nconv && (strategy != RALPB_STRATEGY_RALP || precision != RALPB_PRECISION_BF16))
    return fail("a conv back segment (split before the FC tail) runs with the single PS in bf16 precision");
  m->nconv = nconv;
  m->split = layer_placed ? split : nconv;
  m->bseg = m->split < nconv;
  m->holds_back = strategy != RALPB_STRATEGY_RALP || rank == ps_rank;   // RALP_MPS: every rank
  m->rows_back = layer_placed ? workers * batch : batch;
  if (m->mps) {
    if (n_layers - nconv < 2) return fail("RALP_MPS needs at least two FC layers");
    if (ps_rank != 0) return fail("RALP_MPS keeps the FC tail's head on rank 0");
    const int out0 = layers[nconv].cout;
    if (out0 % world != 0 || (out0 / world) % 8 != 0) return fail("RALP_MPS: first FC width must split into multiples of 8");
    m->s0 = out0 / world;
    m->ld_s0 = m->s0;
  }

  // ---- front geometry
  const ralpb_layer_desc& l0 = layers[0];
  if (l0.kind != RALPB_CONV) return fail("first layer must be a convolution");
  m->in_h = l0.h; m->in_w = l0.w; m->in_c = l0.cin;
  m->in_cp = static_cast<int>(align_up(l0.cin, 16));
  // A first convolution over a few input channels (RGB) runs as an im2col GEMM: acts[0] is
  // then the [rows of the conv's padded output grid][kpad] patch matrix with a ones column
  // that carries the bias (so bias and its gradient come out of the GEMMs themselves).
  const bool first_im2col = l0.cin <= 4;
  ActBuf a0;
  a0.n = batch; a0.h = l0.h; a0.w = l0.w; a0.c = m->in_cp; a0.pad = l0.pad;
  if (first_im2col) {
    const int kk1 = l0.k * l0.k * l0.cin + 1;
    a0.h = (l0.h + 2 * l0.pad - l0.k) / l0.stride + 1;
    a0.w = (l0.w + 2 * l0.pad - l0.k) / l0.stride + 1;
    a0.c = static_cast<int>(kk1 <= 32 ? 32 : align_up(kk1, 64));
    a0.pad = (nconv > 1 && layers[1].kind == RALPB_CONV) ? layers[1].pad : 0;
  }
  m->acts.push_back(a0);
  long long off = 0;
  std::vector<std::pair<long long, long long>> real_runs;  // (offset, floats) of descriptor parameters
  const int rows_bseg = workers * batch;   // the PS's back segment runs over every worker's rows
  for (int i = 0; i < nconv; ++i) {
    const ralpb_layer_desc& d = layers[i];
    if (i == m->split && m->bseg) {  // the synchronised front ends here
      m->n_front = align_up(off, kShardAlign);
      off = m->n_front;
    }
    const int nb = i >= m->split ? rows_bseg : batch;
    ActBuf in = m->acts.back();
    in.n = nb;
    ActBuf o;
    o.n = nb;
    FrontLayer f;
    f.kind = d.kind;
    if (i == 0 && first_im2col) {
      if (!d.relu || d.cout % 16 != 0) return fail("first conv: needs ReLU and cout % 16 == 0");
      f.im2col = true;
      {
        const char* fe = getenv("RALPB_FIRST");
        f.fused = precision == RALPB_PRECISION_BF16 && conv_first_ok(d.h, d.w, d.cin, d.cout, d.k, d.stride, d.pad) &&
                  !(fe != nullptr && std::strcmp(fe, "im2col") == 0);
      }
      f.kpad = in.c;
      f.cin_real = d.cin;
      f.g = ConvGeom{batch, in.h, in.w, in.c, d.cout, d.k, d.pad};  // h/w = output grid
      f.k = d.k;
      f.stride = d.stride;
      f.w_count = static_cast<long long>(d.cout) * f.kpad;
      f.w_off = off;
      f.b_off = -1;  // folded into column k*k*cin of the filter
      f.bn = d.bn != 0;
      if (f.bn) {
        // batch-normalised stem (ResNet): no bias -- the patch rows carry no ones column -- and
        // gamma / beta after the filter
        if (precision != RALPB_PRECISION_BF16 || f.fused) return fail("a batch-normalised first conv runs as a bf16 im2col GEMM");
        if (in.pad != 0) return fail("a batch-normalised first conv must feed a pool or block");
        for (int oc = 0; oc < d.cout; ++oc)
          real_runs.emplace_back(f.w_off + static_cast<long long>(oc) * f.kpad, d.k * d.k * d.cin);
        off = align_up(off + f.w_count, 4);
        f.b_off = off;
        real_runs.emplace_back(f.b_off, 2LL * d.cout);
        off = align_up(off + 2LL * d.cout, 4);
        m->real_front += static_cast<long long>(d.cout) * d.k * d.k * d.cin + 2LL * d.cout;
        m->branchy = true;
      } else {
        for (int oc = 0; oc < d.cout; ++oc)
          real_runs.emplace_back(f.w_off + static_cast<long long>(oc) * f.kpad, d.k * d.k * d.cin + 1);
        off = align_up(off + f.w_count, 4);
        m->real_front += static_cast<long long>(d.cout) * d.k * d.k * d.cin + d.cout;
      }
      o.h = in.h; o.w = in.w; o.c = d.cout; o.pad = in.pad;
      m->front.push_back(f);
      m->acts.push_back(o);
      continue;
    }
    if (d.h != in.h || d.w != in.w) return fail("layer " + std::to_string(i) + ": input shape mismatch");
    if (d.kind == RALPB_CONV) {
      if (d.stride != 1 || d.k != 2 * d.pad + 1) return fail("conv layer " + std::to_string(i) + ": only stride-1 'same' convolutions are implemented");
      if (d.pad != in.pad) return fail("conv layer " + std::to_string(i) + ": padding differs from its input buffer");
      if (!d.relu) return fail("conv layers must be followed by ReLU");
      if (d.cout % 16 != 0) return fail("conv output channels must be a multiple of 16");
      f.cin_real = d.cin;
      f.k = d.k;
      f.stride = 1;
      f.g = ConvGeom{nb, d.h, d.w, in.c, d.cout, d.k, d.pad};
      f.relu = 1;
      f.w_count = static_cast<long long>(d.cout) * d.k * d.k * in.c;
      f.w_off = off;
      off = align_up(off + f.w_count, 4);
      f.b_off = off;
      off = align_up(off + d.cout, 4);
      if (i < m->split) {  // synchronised front parameters
        for (long long ot = 0; ot < static_cast<long long>(d.cout) * d.k * d.k; ++ot)
          real_runs.emplace_back(f.w_off + ot * in.c, d.cin);
        real_runs.emplace_back(f.b_off, d.cout);
        m->real_front += static_cast<long long>(d.cout) * d.k * d.k * d.cin + d.cout;
      } else {
        m->real_bseg += static_cast<long long>(d.cout) * d.k * d.k * d.cin + d.cout;
      }
      o.h = d.h; o.w = d.w; o.c = d.cout; o.pad = d.pad;
    } else if (d.kind == RALPB_POOL) {
      f.k = d.k;
      f.stride = d.stride > 0 ? d.stride : d.k;
      f.pool_pad = d.pad;
      if (d.pad > 0 && (in.pad != 0 || precision != RALPB_PRECISION_BF16))
        return fail("a padded pool reads an unpadded bf16 activation");
      o.h = (d.h + 2 * d.pad - f.k) / f.stride + 1;
      o.w = (d.w + 2 * d.pad - f.k) / f.stride + 1;
      o.c = in.c;
      o.pad = (i + 1 < nconv && layers[i + 1].kind == RALPB_CONV) ? layers[i + 1].pad : 0;
      if (in.c % 8 != 0) return fail("pool channels must be a multiple of 8");
    } else if (d.kind == RALPB_MODULE) {
      if (precision != RALPB_PRECISION_BF16) return fail("modules run in bf16 precision");
      if (in.pad != 0) return fail("layer " + std::to_string(i) + ": a module reads an unpadded activation");
      if (d.node_begin < 0 || d.node_count < 1 || d.node_begin + d.node_count > n_nodes)
        return fail("layer " + std::to_string(i) + ": node range outside the node table");
      m->branchy = true;
      ModuleBufs k;
      std::vector<std::pair<long long, long long>> runs;
      long long count = 0;
      const long long first = off;
      std::string w2;
      if (module_build(k, nodes + d.node_begin, d.node_count, nb, d.h, d.w, in.c, &off, &runs, &count, &w2))
        return fail("layer " + std::to_string(i) + ": " + w2);
      k.groups = i >= m->split ? workers : 1;   // the PS's back segment: per-worker statistics
      if (d.cout != k.cout) return fail("layer " + std::to_string(i) + ": module output channels differ from its nodes'");
      if (i < m->split) {
        for (auto& r : runs) real_runs.push_back(r);
        m->real_front += count;
      } else {
        m->real_bseg += count;
      }
      f.w_off = first;
      f.w_count = off - first;
      f.mod = static_cast<int>(m->modules.size());
      o.h = k.ho; o.w = k.wo; o.c = k.cout; o.pad = 0;
      m->modules.push_back(std::move(k));
    } else if (d.kind == RALPB_BLOCK || d.kind == RALPB_APOOL) {
      if (precision != RALPB_PRECISION_BF16) return fail("bottleneck blocks run in bf16 precision");
      if (in.pad != 0) return fail("layer " + std::to_string(i) + ": a block / average pool reads an unpadded activation");
      m->branchy = true;
      if (d.kind == RALPB_APOOL) {
        f.k = d.h;
        o.h = 1; o.w = 1; o.c = in.c; o.pad = 0;
      } else {
        if (d.stride != 1 && d.stride != 2) return fail("block stride must be 1 or 2");
        if (d.width % 64 != 0 || d.cout % 64 != 0 || in.c % 64 != 0) return fail("block channels must be multiples of 64");
        if (!d.downsample && (d.stride != 1 || d.cin != d.cout)) return fail("an identity shortcut needs stride 1 and cin == cout");
        BlockBufs k;
        k.cin = in.c; k.width = d.width; k.cout = d.cout; k.stride = d.stride; k.down = d.downsample;
        k.n = nb; k.h = d.h; k.w = d.w; k.ho = d.h / d.stride; k.wo = d.w / d.stride;
        k.groups = i >= m->split ? workers : 1;   // the PS's back segment: per-worker statistics
        auto take_params = [&](long long count) { const long long o2 = off; off = align_up(off + count, 4); return o2; };
        k.wa_off = take_params(static_cast<long long>(k.width) * k.cin);
        k.ga_off = take_params(2LL * k.width);
        k.wb_off = take_params(9LL * k.width * k.width);
        k.gb_off = take_params(2LL * k.width);
        k.wc_off = take_params(static_cast<long long>(k.cout) * k.width);
        k.gc_off = take_params(2LL * k.cout);
        if (k.down) {
          k.wd_off = take_params(static_cast<long long>(k.cout) * k.cin);
          k.gd_off = take_params(2LL * k.cout);
        }
        const long long count = static_cast<long long>(k.width) * k.cin + 9LL * k.width * k.width +
                                static_cast<long long>(k.cout) * k.width + 2LL * (2 * k.width + k.cout) +
                                (k.down ? static_cast<long long>(k.cout) * k.cin + 2LL * k.cout : 0);
        if (i < m->split) {
          real_runs.emplace_back(k.wa_off, off - k.wa_off);   // the block's parameters are contiguous
          m->real_front += count;
        } else {
          m->real_bseg += count;
        }
        f.w_off = k.wa_off;
        f.w_count = off - k.wa_off;
        f.blk = static_cast<int>(m->blocks.size());
        m->blocks.push_back(k);
        o.h = k.ho; o.w = k.wo; o.c = k.cout; o.pad = 0;
      }
    } else {
      return fail("unsupported front layer kind");
    }
    m->front.push_back(f);
    m->acts.push_back(o);
  }
  const ActBuf& cut = m->acts.back();
  if (cut.pad != 0) return fail("the FC tail's input must be a pooling output");
  for (int i : {m->split - 1, nconv - 1})   // the backward of these layers needs their stored output
    if (i >= 0 && (m->front[i].kind == RALPB_BLOCK || m->front[i].kind == RALPB_MODULE || m->front[i].bn))
      return fail("a cut must follow a pool or the average pool, not a block / module / batch-normalised conv");
  m->cut_elems = cut.h * cut.w * cut.c;
  if (!m->bseg) m->n_front = align_up(off, kShardAlign);
  m->bseg_end = align_up(off, 4);
  off = align_up(off, kShardAlign);
  m->real_total = m->real_front + m->real_bseg;
  // sync bucket (layer-placed, W > 1, bf16): the smallest cut k whose earlier layers still hold
  // >= 30 % of the front's forward FLOPs (their backward hides the bucket's update) while layers
  // [k, split) hold >= half of the synchronised parameters.  RALPB_SYNC_BUCKET=0: one sync after
  // the whole backward.
  {
    const char* be = getenv("RALPB_SYNC_BUCKET");
    const bool want = !(be != nullptr && be[0] == '0') && layer_placed && workers > 1 &&
                      precision == RALPB_PRECISION_BF16 && !m->layer_shards;
    if (want) {
      std::vector<double> fl(m->split, 0.0);
      double total = 0.0;
      for (int i = 0; i < m->split; ++i) {
        const ralpb_layer_desc& d = layers[i];
        const FrontLayer& f = m->front[i];
        const ActBuf& o = m->acts[i + 1];
        if (d.kind == RALPB_CONV) {
          fl[i] = 2.0 * d.k * d.k * d.cin * d.cout * o.h * o.w;
        } else if (d.kind == RALPB_BLOCK) {
          const BlockBufs& k = m->blocks[f.blk];
          fl[i] = 2.0 * (static_cast<double>(k.h) * k.w * k.cin * k.width + 9.0 * k.ho * k.wo * k.width * k.width +
                         static_cast<double>(k.ho) * k.wo * k.width * k.cout +
                         (k.down ? static_cast<double>(k.ho) * k.wo * k.cin * k.cout : 0.0));
        } else if (d.kind == RALPB_MODULE) {
          for (const ModNode& q : m->modules[f.mod].nodes)
            if (q.d.op == RALPB_NODE_CONV) fl[i] += 2.0 * q.K() * q.d.cout * q.ho * q.wo;
        }
        total += fl[i];
      }
      double before = 0.0;
      for (int i = 0; i < m->split; ++i) {
        const FrontLayer& f = m->front[i];
        const bool has_params = f.kind == RALPB_CONV || f.kind == RALPB_BLOCK || f.kind == RALPB_MODULE;
        if (i > 0 && has_params && before >= 0.3 * total && 2 * (m->n_front - f.w_off) >= m->n_front) {
          m->bucket_k = i;
          m->bucket_lo = f.w_off;
          break;
        }
        before += fl[i];
      }
    }
  }
  {  // the exchanged cut: layer split-1's output (padded when a conv of the back segment reads it)
    const ActBuf& x = m->acts[m->split];
    m->xch_elems = (x.h + 2 * x.pad) * (x.w + 2 * x.pad) * x.c;
    m->xch_logical = static_cast<long long>(x.h) * x.w * x.c;
    m->bin = x;
    m->bin.n = rows_bseg;
  }
  int prev = m->cut_elems;
  for (int i = nconv; i < n_layers; ++i) {
    const ralpb_layer_desc& d = layers[i];
    if (d.cin != prev) return fail("fc layer " + std::to_string(i) + ": input width mismatch");
    FcLayer f;
    f.in = d.cin; f.out = d.cout;
    f.lout = d.cout; f.lin = d.cin;
    if (m->mps && i == nconv) f.lout = m->s0;           // column-parallel: rows of W0
    if (m->mps && i == nconv + 1) f.lin = m->s0;        // row-parallel: columns of W1
    f.relu = i + 1 < n_layers ? 1 : 0;
    if ((i + 1 < n_layers) != (d.relu != 0)) return fail("ReLU must follow every FC layer except the last");
    if (i + 1 < n_layers && d.cout % 8 != 0) return fail("hidden FC widths must be multiples of 8");
    f.ld_out = static_cast<int>(align_up(d.cout, 8));
    f.w_off = off;
    off = align_up(off + static_cast<long long>(f.lout) * f.lin, 4);
    f.b_off = off;
    off = align_up(off + f.lout, 4);
    m->real_total += static_cast<long long>(d.cout) * d.cin + d.cout;
    m->back.push_back(f);
    prev = d.cout;
  }
  m->n_total = align_up(off, kShardAlign);
  // real (descriptor) parameters per sync shard: the logical byte count of the pull / ring sites
  {
    const bool placed = strategy == RALPB_STRATEGY_RALP || strategy == RALPB_STRATEGY_RALP_MPS;
    if (!placed)
      for (const FcLayer& f : m->back) {
        real_runs.emplace_back(f.w_off, static_cast<long long>(f.out) * f.in);
        real_runs.emplace_back(f.b_off, f.out);
      }
    const long long n = placed ? m->n_front : m->n_total;
    const int groups = strategy == RALPB_STRATEGY_RALP ? workers : world;
    const long long shard = n / groups;
    m->shard_ranges.assign(groups, {});
    if (m->layer_shards) {
      // the reference's PS layout: weighted layer k (in model order) -> shard k mod W, a layer's
      // parameters being the contiguous span up to the next weighted layer's first tensor
      std::vector<long long> starts;
      for (const FrontLayer& f : m->front)
        if (f.kind == RALPB_CONV || f.kind == RALPB_BLOCK || f.kind == RALPB_MODULE)
          starts.push_back(f.b_off >= 0 ? std::min(f.w_off, f.b_off) : f.w_off);
      for (const FcLayer& f : m->back) starts.push_back(std::min(f.w_off, f.b_off));
      for (size_t k = 0; k < starts.size(); ++k) {
        const long long hi = k + 1 < starts.size() ? starts[k + 1] : n;
        auto& rg = m->shard_ranges[k % groups];
        if (!rg.empty() && rg.back().second == starts[k]) rg.back().second = hi;   // merge adjacent (W = 1)
        else rg.emplace_back(starts[k], hi);
      }
      for (const auto& rg : m->shard_ranges)
        if (static_cast<int>(rg.size()) > kMaxShardRanges) return fail("too many layers per PS shard");
    } else {
      for (int g = 0; g < groups; ++g) m->shard_ranges[g].emplace_back(shard * g, shard * (g + 1));
    }
    m->shard_real.assign(groups, 0);
    for (const auto& run : real_runs)
      for (int g = 0; g < groups; ++g)
        for (const auto& r : m->shard_ranges[g]) {
          const long long lo = std::max(run.first, r.first), hi = std::min(run.first + run.second, r.second);
          if (hi > lo) m->shard_real[g] += hi - lo;
        }
  }

  // ---- exchange arena (identical layout on every rank)
  size_t ao = 0;
  auto take = [&](size_t bytes) { size_t o2 = ao; ao = align_up(static_cast<long long>(ao + bytes), 256); return o2; };
  m->arena_off_flags = take(kNumFlags * sizeof(uint32_t));
  m->arena_off_P = take(m->n_total * sizeof(float));
  m->arena_off_G = take(m->n_total * sizeof(float));
  // parity precision: P bf16 pieces per value (pair.cuh; RALPB_PIECES=2 for the coarser split)
  if (precision == RALPB_PRECISION_FP32) {
    const char* pe = getenv("RALPB_PIECES");
    m->pieces = pe != nullptr && atoi(pe) == 2 ? 2 : 3;
  }
  const int pm = precision == RALPB_PRECISION_FP32 ? m->pieces : 1;  // bf16 elements per value
  m->arena_off_xfc = take(static_cast<size_t>(m->rows_back) * m->xch_elems * sizeof(bf16) * pm);
  m->arena_off_lab = take(static_cast<size_t>(m->rows_back) * sizeof(int32_t));
  m->arena_off_dcut = take(static_cast<size_t>(batch) * m->xch_elems * sizeof(bf16) * pm);
  m->arena_off_loss = take(kMaxRanks * 4 * sizeof(float));   // [worker][4] own-row loss sums
  if (m->mps) {
    const int ld1 = static_cast<int>(align_up(layers[nconv + 1].cout, 8));
    m->arena_off_p1 = take(static_cast<size_t>(world) * m->rows_back * ld1 * sizeof(float));
    m->arena_off_dh1 = take(static_cast<size_t>(m->rows_back) * ld1 * sizeof(bf16));
    m->arena_off_dxpart = take(static_cast<size_t>(world) * batch * m->cut_elems * sizeof(float));
  }
  m->arena_bytes = ao;
  if (cudaMalloc(&m->arena, m->arena_bytes) != cudaSuccess) return fail("cudaMalloc(arena) failed");
  cudaMemset(m->arena, 0, m->arena_bytes);
  char* base = static_cast<char*>(m->arena);
  m->flags = reinterpret_cast<uint32_t*>(base + m->arena_off_flags);
  m->P = reinterpret_cast<float*>(base + m->arena_off_P);
  m->G = reinterpret_cast<float*>(base + m->arena_off_G);
  m->xin = reinterpret_cast<bf16*>(base + m->arena_off_xfc);
  m->x_fc = m->xin;
  m->bin.ptr = m->xin;
  m->labels_all = reinterpret_cast<int32_t*>(base + m->arena_off_lab);
  m->dcut = reinterpret_cast<bf16*>(base + m->arena_off_dcut);
  m->peer_base.assign(world, nullptr);
  m->peer_base[rank] = base;

  // ---- local buffers
  std::string w2;
  if (!(m->V = alloc<float>(m, m->n_total, why))) return fail(*why);
  cudaMemset(m->V, 0, m->n_total * sizeof(float));
  if (!(m->counters = alloc<uint32_t>(m, kNumCounters, why))) return fail(*why);
  cudaMemset(m->counters, 0, kNumCounters * sizeof(uint32_t));
  m->seq_dev = m->counters + kNumCounters - 1;
  // Every activation and activation-gradient buffer is dedicated and zeroed once: the conv
  // kernels write interior pixels only, so the padding borders stay zero for the job's life.
  // Workers hold acts[0..split] (batch rows); the PS of a conv back segment acts[split+1..nconv]
  // (W*b rows; its input is the arena's xin).
  m->gacts.assign(m->acts.size(), nullptr);
  for (size_t i = 0; i < m->acts.size(); ++i) {
    const bool mine = static_cast<int>(i) <= m->split ? m->is_worker : (m->bseg && m->holds_back);
    if (!mine) continue;
    const size_t bytes = static_cast<size_t>(m->acts[i].elems()) * sizeof(bf16) * pm;
    if (!(m->acts[i].ptr = alloc<bf16>(m, m->acts[i].elems() * pm, why))) return fail(*why);
    cudaMemset(m->acts[i].ptr, 0, bytes);
    if (i > 0 && i + 1 < m->acts.size() && static_cast<int>(i) != m->split) {
      if (!(m->gacts[i] = alloc<bf16>(m, m->acts[i].elems() * pm, why))) return fail(*why);
      cudaMemset(m->gacts[i], 0, bytes);
    }
  }
  // 2x2/2 pools fused into the preceding conv's epilogue.  With RALPB_POOL_IDX=1 those after a
  // conv with cin >= 128 also record argmax bytes so their backward does not re-read the conv
  // output; measured: the backward saves what the forward epilogue loses (-0.22 / +0.28 ms per
  // VGG-16 step), so it is off by default
  for (size_t i = 0; i + 1 < m->front.size(); ++i) {
    FrontLayer& c = m->front[i];
    FrontLayer& pl = m->front[i + 1];
    if (c.kind == RALPB_CONV && !c.im2col && pl.kind == RALPB_POOL && pl.k == 2 && pl.stride == 2 &&
        static_cast<int>(i) + 1 != m->split &&
        conv_fwd_pool_ok(c.g) && fuse_pool_enabled() && precision == RALPB_PRECISION_BF16) {
      pl.fused_fwd = true;
      const ActBuf& po = m->acts[i + 2];
      const char* ie = getenv("RALPB_POOL_IDX");
      if (ie != nullptr && ie[0] == '1' && c.g.cin >= 128 && m->acts[i + 1].ptr != nullptr &&
          !(pl.idx = alloc<uint8_t>(m, static_cast<size_t>(po.n) * po.h * po.w * po.c, why)))
        return fail(*why);
    }
  }
  // stand-alone pools (overlapping windows, or after a non-slab conv) record argmax bytes in their
  // forward and gather the backward from them (maxpool_bwd_gather)
  for (size_t i = 0; i < m->front.size(); ++i) {
    FrontLayer& pl = m->front[i];
    if (pl.kind != RALPB_POOL || pl.fused_fwd || pl.k * pl.k > 255) continue;
    if (!(static_cast<int>(i) < m->split ? m->is_worker : (m->bseg && m->holds_back))) continue;
    const ActBuf& po = m->acts[i + 1];
    if (!(pl.idx = alloc<uint8_t>(m, static_cast<size_t>(po.n) * po.h * po.w * po.c, why))) return fail(*why);
  }
  for (size_t i = 0; i < m->front.size(); ++i) {
    FrontLayer& f = m->front[i];
    const bool mine = static_cast<int>(i) < m->split ? m->is_worker : (m->bseg && m->holds_back);
    if (f.kind != RALPB_CONV || !mine) continue;
    // pair precision: [2co][taps][2ci] operand copies (pair.cuh)
    if (!(f.wf = alloc<bf16>(m, f.w_count * pm * pm, why))) return fail(*why);
    if (!f.im2col && !(f.wd = alloc<bf16>(m, f.w_count * pm * pm, why))) return fail(*why);
  }
  // branchy layers: the blocks' operands and saved tensors, the stem's pre-batch-norm output
  if (m->branchy) {   // zeroed once: every reduction leaves its accumulators and ticket zero
    if (!(m->bn_work = alloc<float>(m, kBnWorkFloats, why))) return fail(*why);
    if (cudaMemset(m->bn_work, 0, kBnWorkFloats * sizeof(float)) != cudaSuccess) return fail("bn scratch memset");
  }
  for (size_t i = 0; i < m->front.size(); ++i) {
    FrontLayer& f = m->front[i];
    const bool mine = static_cast<int>(i) < m->split ? m->is_worker : (m->bseg && m->holds_back);
    if (!mine) continue;
    if (f.kind == RALPB_BLOCK) {
      if (block_alloc(m, m->blocks[f.blk], why)) return fail(*why);
      if (m->blocks[f.blk].cmax > 2048) return fail("block channels above 2048");
    } else if (f.kind == RALPB_MODULE) {
      if (module_alloc(m, m->modules[f.mod], why)) return fail(*why);
      for (const ModNode& q : m->modules[f.mod].nodes)
        if (q.d.op == RALPB_NODE_CONV && q.d.cout > 2048) return fail("module conv channels above 2048");
    } else if (f.bn) {
      const size_t rows = static_cast<size_t>(m->acts[i + 1].rows());
      if (!(f.pre = alloc<bf16>(m, rows * f.g.cout, why)) || !(f.dpre = alloc<bf16>(m, rows * f.g.cout, why)) ||
          !(f.bn_stats = alloc<float>(m, 2 * static_cast<size_t>(f.g.cout), why)) ||
          !(f.bn_mask = alloc<uint8_t>(m, rows * f.g.cout / 8, why)))
        return fail(*why);
    }
  }
  const int R = m->rows_back;
  if (m->mps) {
    const int ld1 = m->back[1].ld_out;
    if (!(m->h0s = alloc<bf16>(m, static_cast<size_t>(R) * m->ld_s0, why))) return fail(*why);
    if (!(m->dh0s = alloc<bf16>(m, static_cast<size_t>(R) * m->ld_s0, why))) return fail(*why);
    if (!(m->p1_local = alloc<float>(m, static_cast<size_t>(R) * ld1, why))) return fail(*why);
    if (!(m->dxp = alloc<float>(m, static_cast<size_t>(R) * m->cut_elems, why))) return fail(*why);
  }
  for (size_t j = 0; j < m->back.size(); ++j) {
    auto& f = m->back[j];
    if (pm > 1) {  // piece operands [P*ld_out][P*in] for the forward and the backward-data GEMMs
      const size_t n4 = static_cast<size_t>(pm) * pm * f.ld_out * f.lin;
      if (!(f.wbf = alloc<bf16>(m, n4, why)) || !(f.wbd = alloc<bf16>(m, n4, why))) return fail(*why);
      cudaMemset(f.wbf, 0, n4 * sizeof(bf16));
      cudaMemset(f.wbd, 0, n4 * sizeof(bf16));
      m->pair_s_floats = std::max(m->pair_s_floats, n4);
      m->pair_acc_floats = std::max(m->pair_acc_floats, static_cast<size_t>(pm) * R * std::max(f.ld_out, f.lin));
    } else if (!(f.wbf = alloc<bf16>(m, static_cast<size_t>(f.lout) * f.lin, why))) {
      return fail(*why);
    }
    if (j + 1 < m->back.size()) {
      bf16* h = alloc<bf16>(m, static_cast<size_t>(R) * f.ld_out * pm, why);
      if (!h) return fail(*why);
      m->hid.push_back(h);
    }
  }
  int widest = m->cut_elems;
  for (auto& f : m->back) widest = std::max(widest, f.ld_out);
  const FcLayer& last = m->back.back();
  if (!(m->logits = alloc<float>(m, static_cast<size_t>(R) * last.ld_out, why))) return fail(*why);
  if (!(m->dlogits = alloc<bf16>(m, static_cast<size_t>(R) * last.ld_out * pm, why))) return fail(*why);
  cudaMemset(m->dlogits, 0, static_cast<size_t>(R) * last.ld_out * sizeof(bf16) * pm);
  for (size_t j = 0; j + 1 < m->back.size(); ++j) {
    bf16* d = alloc<bf16>(m, static_cast<size_t>(R) * m->back[j].ld_out * pm, why);
    if (!d) return fail(*why);
    m->dyb.push_back(d);
  }
  if (!(m->dx_fc = alloc<bf16>(m, static_cast<size_t>(R) * m->cut_elems * pm, why))) return fail(*why);
  m->dxin = m->dx_fc;
  if (m->bseg && m->holds_back) {
    // the conv back segment: FC input rows and the cut gradient rows are separate buffers
    if (!(m->x_fc = alloc<bf16>(m, static_cast<size_t>(R) * m->cut_elems, why))) return fail(*why);
    if (!(m->dxin = alloc<bf16>(m, static_cast<size_t>(R) * m->xch_elems, why))) return fail(*why);
    cudaMemset(m->dxin, 0, static_cast<size_t>(R) * m->xch_elems * sizeof(bf16));
  }
  if (pm > 1) {
    // scratch of the piece contractions: the fp32 [rows][P*N] outputs before their finishing pass
    // and the [P*M][T][P*C] weight-gradient blocks
    for (size_t i = 0; i < m->front.size(); ++i) {
      const FrontLayer& f = m->front[i];
      if (f.kind != RALPB_CONV) continue;
      const ActBuf& in = m->acts[i];
      m->pair_acc_floats = std::max(m->pair_acc_floats, static_cast<size_t>(in.rows()) * pm * std::max(f.g.cout, f.g.cin));
      m->pair_s_floats = std::max(m->pair_s_floats, static_cast<size_t>(pm) * pm * static_cast<size_t>(f.w_count));
    }
    if (!(m->pair_acc = alloc<float>(m, m->pair_acc_floats, why))) return fail(*why);
    if (!(m->pair_s = alloc<float>(m, m->pair_s_floats, why))) return fail(*why);
  }
  if (!(m->fc_scratch = alloc<float>(m, static_cast<size_t>(R) * std::max(widest, m->cut_elems), why))) return fail(*why);
  if (!(m->row_loss = alloc<float>(m, R, why))) return fail(*why);
  if (!(m->loss = alloc<float>(m, 4, why))) return fail(*why);
  for (int i = 0; i < 2; ++i) {
    if (m->is_worker &&
        !(m->img_dev[i] = alloc<float>(m, static_cast<size_t>(batch) * m->in_h * m->in_w * m->in_c, why)))
      return fail(*why);
    if (!(m->lab_dev[i] = alloc<int32_t>(m, batch, why))) return fail(*why);
    cudaEventCreateWithFlags(&m->ev_copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&m->ev_consumed[i], cudaEventDisableTiming);
  }
  if (cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking) != cudaSuccess) return fail("stream");
  if (cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking) != cudaSuccess) return fail("stream");
  if (cudaStreamCreateWithFlags(&m->aux_stream, cudaStreamNonBlocking) != cudaSuccess) return fail("stream");
  if (cudaStreamCreateWithFlags(&m->comm_stream, cudaStreamNonBlocking) != cudaSuccess) return fail("stream");
  if (cudaStreamCreateWithFlags(&m->sync_stream, cudaStreamNonBlocking) != cudaSuccess) return fail("stream");
  cudaEventCreateWithFlags(&m->ev_b1, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_b1_done, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_comm_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_comm_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_wd_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_wd_join, cudaEventDisableTiming);
  for (auto& e : m->ev) cudaEventCreate(&e);
  if (cudaMallocHost(&m->loss_host, sizeof(float) * Model::kLossRing) != cudaSuccess) return fail("cudaMallocHost");
  for (auto& e : m->ev_loss) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail("device error during model creation");
  *out = m;
  return 0;
}

void model_destroy(Model* m) {
  if (!m) return;
  cudaDeviceSynchronize();
  for (auto& g : m->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (int i = 0; i < 2; ++i) {
    if (m->ev_copied[i]) cudaEventDestroy(m->ev_copied[i]);
    if (m->ev_consumed[i]) cudaEventDestroy(m->ev_consumed[i]);
  }
  for (auto& e : m->ev_loss)
    if (e) cudaEventDestroy(e);
  if (m->loss_host) cudaFreeHost(m->loss_host);
  if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
  if (m->aux_stream) cudaStreamDestroy(m->aux_stream);
  if (m->comm_stream) cudaStreamDestroy(m->comm_stream);
  if (m->sync_stream) cudaStreamDestroy(m->sync_stream);
  if (m->ev_b1) cudaEventDestroy(m->ev_b1);
  if (m->ev_b1_done) cudaEventDestroy(m->ev_b1_done);
  if (m->ev_comm_fork) cudaEventDestroy(m->ev_comm_fork);
  if (m->ev_comm_join) cudaEventDestroy(m->ev_comm_join);
  if (m->ev_fork) cudaEventDestroy(m->ev_fork);
  if (m->ev_join) cudaEventDestroy(m->ev_join);
  if (m->ev_wd_fork) cudaEventDestroy(m->ev_wd_fork);
  if (m->ev_wd_join) cudaEventDestroy(m->ev_wd_join);
  for (int r = 0; r < static_cast<int>(m->peer_base.size()); ++r)
    if (r != m->rank && m->peer_base[r] != nullptr) cudaIpcCloseMemHandle(m->peer_base[r]);
  for (void* p : m->owned) cudaFree(p);
  if (m->arena) cudaFree(m->arena);
  for (auto& e : m->ev)
    if (e) cudaEventDestroy(e);
  if (m->timer.ev) {
    for (int i = 0; i < 2 * m->timer.cap; ++i) cudaEventDestroy(m->timer.ev[i]);
    delete[] m->timer.kind;
    delete[] m->timer.flops;
    delete[] m->timer.bytes;
    delete[] m->timer.stream;
    delete[] m->timer.ev;
  }
  if (m->stream) cudaStreamDestroy(m->stream);
  delete m;
}

int model_ipc_handle(Model* m, void* out, std::string* why) {
  cudaIpcMemHandle_t h;
  RALPB_TRY(cudaIpcGetMemHandle(&h, m->arena));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::memcpy(out, &h, 64);
  return 0;
}

int model_ipc_open(Model* m, const void* handles, std::string* why) {
  const char* hs = static_cast<const char*>(handles);
  for (int r = 0; r < m->world; ++r) {
    if (r == m->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hs + 64 * r, 64);
    void* p = nullptr;
    RALPB_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    m->peer_base[r] = static_cast<char*>(p);
  }
  m->peers_open = true;
  for (auto& g : m->graphs)  // peer pointers are baked into captured steps
    if (g.exec) { cudaGraphExecDestroy(g.exec); g = Model::GraphEntry{}; }
  return 0;
}

// ------------------------------------------------------------------ parameters
int model_set_params(Model* m, int layer, const float* w, const float* b, int on_host, std::string* why) {
  if (layer < 0 || layer >= static_cast<int>(m->desc.size())) { *why = "layer out of range"; return 1; }
  const auto kind = cudaMemcpyDefault;
  (void)on_host;
  if (layer < m->nconv && m->front[layer].kind == RALPB_BLOCK) {
    // w: wa, wb, wc(, wd) back to back; b: the batch-norm scale / shift pairs in the same order
    BlockBufs& k = m->blocks[m->front[layer].blk];
    const long long sw[4] = {static_cast<long long>(k.width) * k.cin, 9LL * k.width * k.width,
                             static_cast<long long>(k.cout) * k.width, static_cast<long long>(k.cout) * k.cin};
    const long long ow[4] = {k.wa_off, k.wb_off, k.wc_off, k.wd_off};
    const long long sg[4] = {2LL * k.width, 2LL * k.width, 2LL * k.cout, 2LL * k.cout};
    const long long og[4] = {k.ga_off, k.gb_off, k.gc_off, k.gd_off};
    long long pw = 0, pg = 0;
    for (int q = 0; q < (k.down ? 4 : 3); ++q) {
      RALPB_TRY(cudaMemcpy(m->P + ow[q], w + pw, sw[q] * sizeof(float), kind));
      RALPB_TRY(cudaMemcpy(m->P + og[q], b + pg, sg[q] * sizeof(float), kind));
      pw += sw[q];
      pg += sg[q];
    }
    if (k.wa != nullptr && block_prep(m, k, m->stream, why)) return 1;
    RALPB_TRY(cudaStreamSynchronize(m->stream));
    return 0;
  }
  if (layer < m->nconv && m->front[layer].kind == RALPB_MODULE) {
    // w: the conv nodes' filters back to back; b: their gamma|beta or bias in the same order
    ModuleBufs& k = m->modules[m->front[layer].mod];
    std::vector<std::pair<long long, long long>> wr, br;
    module_param_runs(k, &wr, &br);
    long long pw = 0, pb = 0;
    for (size_t q = 0; q < wr.size(); ++q) {
      RALPB_TRY(cudaMemcpy(m->P + wr[q].first, w + pw, wr[q].second * sizeof(float), kind));
      RALPB_TRY(cudaMemcpy(m->P + br[q].first, b + pb, br[q].second * sizeof(float), kind));
      pw += wr[q].second;
      pb += br[q].second;
    }
    if (module_prep(m, k, m->stream, why)) return 1;
    RALPB_TRY(cudaStreamSynchronize(m->stream));
    return 0;
  }
  if (layer < m->nconv) {
    FrontLayer& f = m->front[layer];
    if (f.kind != RALPB_CONV) { *why = "layer has no parameters"; return 1; }
    const int co = f.g.cout, taps = f.k * f.k, cr = f.cin_real;
    const int kk = taps * cr;
    std::vector<float> host(static_cast<size_t>(co) * kk), hb(f.bn ? 2 * co : co), packed(f.w_count, 0.f);
    RALPB_TRY(cudaMemcpy(host.data(), w, host.size() * sizeof(float), kind));
    RALPB_TRY(cudaMemcpy(hb.data(), b, hb.size() * sizeof(float), kind));
    if (f.im2col) {  // [co][kpad]: taps*cin filter columns, then the bias column (bn: gamma | beta after)
      for (int o = 0; o < co; ++o) {
        for (int j = 0; j < kk; ++j) packed[static_cast<size_t>(o) * f.kpad + j] = host[static_cast<size_t>(o) * kk + j];
        if (!f.bn) packed[static_cast<size_t>(o) * f.kpad + kk] = hb[o];
      }
      if (f.bn) RALPB_TRY(cudaMemcpy(m->P + f.b_off, hb.data(), hb.size() * sizeof(float), cudaMemcpyHostToDevice));
    } else {  // [co][taps][cin_pad], padded input channels are zero
      const int cp = f.g.cin;
      for (int o = 0; o < co; ++o)
        for (int t = 0; t < taps; ++t)
          for (int c = 0; c < cr; ++c)
            packed[(static_cast<size_t>(o) * taps + t) * cp + c] = host[(static_cast<size_t>(o) * taps + t) * cr + c];
      RALPB_TRY(cudaMemcpyAsync(m->P + f.b_off, hb.data(), co * sizeof(float), cudaMemcpyHostToDevice, m->stream));
    }
    RALPB_TRY(cudaMemcpyAsync(m->P + f.w_off, packed.data(), packed.size() * sizeof(float), cudaMemcpyHostToDevice, m->stream));
    if (f.wf == nullptr || pair_mode(m)) {
      // layers this rank does not run keep no operand copies; pairs: pair_relayout below
    } else if (f.im2col) {
      RALPB_TRY(cast_bf16(m->P + f.w_off, f.w_count, f.wf, m->stream));
    } else {
      RALPB_TRY(conv_weight_prep(m->P + f.w_off, co, taps, f.g.cin, f.wf, f.wd, m->stream));
    }
  } else {
    const int j = layer - m->nconv;
    FcLayer& f = m->back[j];
    if (m->mps && j == 0) {          // column-parallel: this rank's rows
      const size_t r0 = static_cast<size_t>(m->rank) * m->s0;
      RALPB_TRY(cudaMemcpyAsync(m->P + f.w_off, w + r0 * f.in, static_cast<size_t>(f.lout) * f.in * sizeof(float), kind,
                                m->stream));
      RALPB_TRY(cudaMemcpyAsync(m->P + f.b_off, b + r0, f.lout * sizeof(float), kind, m->stream));
    } else if (m->mps && j == 1) {   // row-parallel: this rank's columns (bias applied on rank 0)
      RALPB_TRY(cudaMemcpy2DAsync(m->P + f.w_off, f.lin * sizeof(float), w + static_cast<size_t>(m->rank) * m->s0,
                                  f.in * sizeof(float), f.lin * sizeof(float), f.out, kind, m->stream));
      RALPB_TRY(cudaMemcpyAsync(m->P + f.b_off, b, f.out * sizeof(float), kind, m->stream));
    } else {
      RALPB_TRY(cudaMemcpyAsync(m->P + f.w_off, w, static_cast<size_t>(f.out) * f.in * sizeof(float), kind, m->stream));
      RALPB_TRY(cudaMemcpyAsync(m->P + f.b_off, b, f.out * sizeof(float), kind, m->stream));
    }
    if (!pair_mode(m)) RALPB_TRY(cast_bf16(m->P + f.w_off, static_cast<long long>(f.lout) * f.lin, f.wbf, m->stream));
  }
  if (pair_mode(m) && pair_relayout(m, layer < m->nconv, layer >= m->nconv, m->stream, why)) return 1;
  RALPB_TRY(cudaStreamSynchronize(m->stream));
  return 0;
}

// Reads layer `layer`'s fp32 parameters (off = arena_off_P) or this step's gradients (arena_off_G)
// in the caller's layout (get_params / get_grads).
static int read_layer(Model* m, int layer, float* w, float* b, size_t off, std::string* why) {
  if (layer < 0 || layer >= static_cast<int>(m->desc.size())) { *why = "layer out of range"; return 1; }
  const float* self = at<float>(m, m->rank, off);
  RALPB_TRY(cudaStreamSynchronize(m->stream));
  if (layer < m->nconv && m->front[layer].kind == RALPB_BLOCK) {
    BlockBufs& k = m->blocks[m->front[layer].blk];
    const long long sw[4] = {static_cast<long long>(k.width) * k.cin, 9LL * k.width * k.width,
                             static_cast<long long>(k.cout) * k.width, static_cast<long long>(k.cout) * k.cin};
    const long long ow[4] = {k.wa_off, k.wb_off, k.wc_off, k.wd_off};
    const long long sg[4] = {2LL * k.width, 2LL * k.width, 2LL * k.cout, 2LL * k.cout};
    const long long og[4] = {k.ga_off, k.gb_off, k.gc_off, k.gd_off};
    long long pw = 0, pg = 0;
    for (int q = 0; q < (k.down ? 4 : 3); ++q) {
      RALPB_TRY(cudaMemcpy(w + pw, self + ow[q], sw[q] * sizeof(float), cudaMemcpyDefault));
      RALPB_TRY(cudaMemcpy(b + pg, self + og[q], sg[q] * sizeof(float), cudaMemcpyDefault));
      pw += sw[q];
      pg += sg[q];
    }
    return 0;
  }
  if (layer < m->nconv && m->front[layer].kind == RALPB_MODULE) {
    std::vector<std::pair<long long, long long>> wr, br;
    module_param_runs(m->modules[m->front[layer].mod], &wr, &br);
    long long pw = 0, pb = 0;
    for (size_t q = 0; q < wr.size(); ++q) {
      RALPB_TRY(cudaMemcpy(w + pw, self + wr[q].first, wr[q].second * sizeof(float), cudaMemcpyDefault));
      RALPB_TRY(cudaMemcpy(b + pb, self + br[q].first, br[q].second * sizeof(float), cudaMemcpyDefault));
      pw += wr[q].second;
      pb += br[q].second;
    }
    return 0;
  }
  if (layer < m->nconv) {
    FrontLayer& f = m->front[layer];
    if (f.kind != RALPB_CONV) { *why = "layer has no parameters"; return 1; }
    const int co = f.g.cout, taps = f.k * f.k, cr = f.cin_real;
    const int kk = taps * cr;
    std::vector<float> packed(f.w_count), host(static_cast<size_t>(co) * kk), hb(co);
    RALPB_TRY(cudaMemcpy(packed.data(), self + f.w_off, packed.size() * sizeof(float), cudaMemcpyDeviceToHost));
    if (f.im2col && f.bn) {
      for (int o = 0; o < co; ++o)
        for (int j = 0; j < kk; ++j) host[static_cast<size_t>(o) * kk + j] = packed[static_cast<size_t>(o) * f.kpad + j];
      hb.resize(2 * co);
      RALPB_TRY(cudaMemcpy(hb.data(), self + f.b_off, 2 * co * sizeof(float), cudaMemcpyDeviceToHost));
    } else if (f.im2col) {
      for (int o = 0; o < co; ++o) {
        for (int j = 0; j < kk; ++j) host[static_cast<size_t>(o) * kk + j] = packed[static_cast<size_t>(o) * f.kpad + j];
        hb[o] = packed[static_cast<size_t>(o) * f.kpad + kk];
      }
    } else {
      const int cp = f.g.cin;
      for (int o = 0; o < co; ++o)
        for (int t = 0; t < taps; ++t)
          for (int c = 0; c < cr; ++c)
            host[(static_cast<size_t>(o) * taps + t) * cr + c] = packed[(static_cast<size_t>(o) * taps + t) * cp + c];
      RALPB_TRY(cudaMemcpy(hb.data(), self + f.b_off, co * sizeof(float), cudaMemcpyDeviceToHost));
    }
    RALPB_TRY(cudaMemcpy(w, host.data(), host.size() * sizeof(float), cudaMemcpyDefault));
    RALPB_TRY(cudaMemcpy(b, hb.data(), hb.size() * sizeof(float), cudaMemcpyDefault));
  } else {
    const int j = layer - m->nconv;
    FcLayer& f = m->back[j];
    if (m->mps && j <= 1) {
      // gather every rank's slice through the peer mappings (rank 0's own for W = 1)
      if (m->world > 1 && !m->peers_open) { *why = "RALP_MPS get_params needs the peers mapped"; return 1; }
      for (int q = 0; q < m->world; ++q) {
        const float* pq = at<float>(m, q, off);
        if (j == 0) {
          const size_t r0 = static_cast<size_t>(q) * m->s0;
          RALPB_TRY(cudaMemcpy(w + r0 * f.in, pq + f.w_off, static_cast<size_t>(f.lout) * f.in * sizeof(float), cudaMemcpyDefault));
          RALPB_TRY(cudaMemcpy(b + r0, pq + f.b_off, f.lout * sizeof(float), cudaMemcpyDefault));
        } else {
          RALPB_TRY(cudaMemcpy2D(w + static_cast<size_t>(q) * m->s0, f.in * sizeof(float), pq + f.w_off,
                                 f.lin * sizeof(float), f.lin * sizeof(float), f.out, cudaMemcpyDefault));
        }
      }
      if (j == 1)  // FC-1's bias is updated on rank 0
        RALPB_TRY(cudaMemcpy(b, at<float>(m, 0, off) + f.b_off, f.out * sizeof(float), cudaMemcpyDefault));
    } else {
      // RALP_MPS: later FC layers live on rank 0
      const float* src = m->mps && (m->world == 1 || m->peers_open) ? at<float>(m, 0, off) : self;
      RALPB_TRY(cudaMemcpy(w, src + f.w_off, static_cast<size_t>(f.out) * f.in * sizeof(float), cudaMemcpyDefault));
      RALPB_TRY(cudaMemcpy(b, src + f.b_off, f.out * sizeof(float), cudaMemcpyDefault));
    }
  }
  return 0;
}

int model_get_params(Model* m, int layer, float* w, float* b, int on_host, std::string* why) {
  (void)on_host;
  return read_layer(m, layer, w, b, m->arena_off_P, why);
}

// The gradient the last step computed for `layer` (summed over this rank's batch; the FC tail's on
// the rank that holds it), before any cross-rank reduction.
int model_get_grads(Model* m, int layer, float* w, float* b, std::string* why) {
  return read_layer(m, layer, w, b, m->arena_off_G, why);
}

// ------------------------------------------------------------------ step
namespace {

// An FC GEMM with a bias / ReLU / ReLU-mask epilogue.  With few rows (e.g. W = 1, R = b) the
// output tile grid cannot fill 148 SMs, so K is split across CTAs with fp32 atomics into a
// scratch buffer and gemm_finalize applies the epilogue.
int fc_gemm(Model* m, GemmDesc d, long long ld_out, const float* bias, int relu, const bf16* mask,
            long long ld_mask, bf16* out_bf16, float* out_f32, std::string* why) {
  const int bn = d.N >= 256 ? 256 : (d.N > 64 ? 128 : (d.N > 32 ? 64 : 32));
  const long long tiles = static_cast<long long>((d.M + 127) / 128) * ((d.N + bn - 1) / bn);
  if (tiles * 2 >= num_sms()) {
    d.epi = out_bf16 != nullptr ? EPI_BF16 : EPI_F32;
    d.out = out_bf16 != nullptr ? static_cast<void*>(out_bf16) : static_cast<void*>(out_f32);
    d.s_m = ld_out;
    d.bias = bias;
    d.relu = relu;
    d.mask = mask;
    d.mask_s = ld_mask;
    RALPB_TRY(gemm_launch(d, m->stream, why));
    ++m->launches;
    return 0;
  }
  RALPB_TRY(cudaMemsetAsync(m->fc_scratch, 0, sizeof(float) * d.M * ld_out, m->stream));
  d.epi = EPI_F32_ATOMIC;
  d.k_splits = 0;
  d.out = m->fc_scratch;
  d.s_m = ld_out;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  RALPB_TRY(gemm_finalize(m->fc_scratch, d.M, d.N, ld_out, bias, relu, mask, ld_mask, out_bf16, out_f32, ld_out,
                          m->stream));
  m->launches += 2;
  return 0;
}

int launch_fc_forward(Model* m, const bf16* in, int R, std::string* why) {
  const bf16* x = in;
  long long ldx = m->cut_elems;
  for (size_t j = 0; j < m->back.size(); ++j) {
    FcLayer& f = m->back[j];
    GemmDesc d;
    d.M = R; d.N = f.out; d.K = f.in;
    d.a = Operand2D{x, R, f.in, ldx};
    d.b = Operand2D{f.wbf, f.out, f.in, f.in};
    const bool hidden = j + 1 < m->back.size();
    if (fc_gemm(m, d, f.ld_out, m->P + f.b_off, hidden ? 1 : 0, nullptr, 0, hidden ? m->hid[j] : nullptr,
                hidden ? nullptr : m->logits, why))
      return 1;
    x = j + 1 < m->back.size() ? m->hid[j] : nullptr;
    ldx = f.ld_out;
  }
  return 0;
}

// FC backward from dlogits; writes the cut gradient for all R rows into dx_out.
// FC backward from dlogits; writes the cut gradient for all R rows into dx_out.  With
// `update` (the RALP PS: the FC tail is never synchronised) the weight-gradient GEMM applies
// SGD-momentum in its epilogue (EPI_SGD) -- after the layer's dgrad has consumed the old bf16
// weights -- so FC gradients never round-trip through HBM.
// FC backward-data chain: dyb[j-1] = (dyb[j] . W_j) * relu'(h_{j-1}); the first layer's dx is the
// cut gradient.  Runs on the main stream (its result is what the workers wait for).
int launch_fc_backward_data(Model* m, const bf16* in, int R, bf16* dx_out, std::string* why) {
  const int nb = static_cast<int>(m->back.size());
  for (int j = nb - 1; j >= 0; --j) {
    FcLayer& f = m->back[j];
    const bf16* dy = j == nb - 1 ? m->dlogits : m->dyb[j];
    const long long lddy = f.ld_out;
    const long long ldx = j == 0 ? m->cut_elems : m->back[j - 1].ld_out;
    bf16* dst = j == 0 ? dx_out : m->dyb[j - 1];
    GemmDesc d;
    d.M = R; d.N = f.in; d.K = f.out;
    d.a_mode = LD_K; d.a = Operand2D{dy, R, f.out, lddy};
    d.b_mode = LD_MN; d.b = Operand2D{f.wbf, f.out, f.in, f.in};
    const bool masked = j > 0 && m->back[j - 1].relu;
    if (fc_gemm(m, d, ldx, nullptr, 0, masked ? m->hid[j - 1] : nullptr, ldx, dst, nullptr, why)) return 1;
  }
  return 0;
}

// FC weight/bias gradients into G (dW = dy^T x, db = colsum dy) and, when `update`, the PS-local
// SGD-momentum step with the bf16 weight copy the next forward reads.  Issued on `s`: the aux
// stream for the layer-placed step (it overlaps the front backward), the main stream otherwise.
int launch_fc_backward_weights(Model* m, const bf16* in, int R, bool update, float lr, float mu, cudaStream_t s,
                               cudaStream_t s_update, std::string* why) {
  const int nb = static_cast<int>(m->back.size());
  for (int j = nb - 1; j >= 0; --j) {
    FcLayer& f = m->back[j];
    const bf16* dy = j == nb - 1 ? m->dlogits : m->dyb[j];
    const long long lddy = f.ld_out;
    const bf16* x = j == 0 ? in : m->hid[j - 1];
    const long long ldx = j == 0 ? m->cut_elems : m->back[j - 1].ld_out;
    RALPB_TRY(cudaMemsetAsync(m->G + f.b_off, 0, f.out * sizeof(float), s));
    RALPB_TRY(colsum_bf16(dy, R, f.out, lddy, m->G + f.b_off, s));
    GemmDesc w;
    w.M = f.out; w.N = f.in; w.K = R;
    w.a_mode = LD_MN; w.a = Operand2D{dy, R, f.out, lddy};
    w.b_mode = LD_MN; w.b = Operand2D{x, R, f.in, ldx};
    w.s_m = f.in; w.s_n = 1;
    w.epi = EPI_F32; w.out = m->G + f.w_off;
    RALPB_TRY(gemm_launch(w, s, why));
    m->launches += 2;
  }
  if (update) {
    if (s_update != s) {
      RALPB_TRY(cudaEventRecord(m->ev_fork, s));
      RALPB_TRY(cudaStreamWaitEvent(s_update, m->ev_fork, 0));
    }
    for (auto& f : m->back) {
      const long long nw = static_cast<long long>(f.out) * f.in;
      RALPB_TRY(sgd_momentum_bf16(m->P + f.w_off, m->V + f.w_off, m->G + f.w_off, nw, lr, mu, 1.f, f.wbf, s_update));
      RALPB_TRY(sgd_momentum(m->P + f.b_off, m->V + f.b_off, m->G + f.b_off, f.out, lr, mu, 1.f, s_update));
      m->launches += 2;
    }
  }
  return 0;
}

// RALP_MPS back segment (every rank): cut all-gather -> FC-0 column-parallel -> FC-1 row-parallel
// partials reduced on rank 0 -> rank 0 runs the rest of the tail and the loss -> FC-1 output
// gradient broadcast -> FC-1 / FC-0 backward on every rank -> cut-gradient partials
// reduce-scattered to their workers.  The weight updates of each rank's FC slices run on the aux
// stream.  Extension of the reference's single PS.
int mps_back_segment(Model* m, const int32_t* lab, const bf16* cut_local, float lr, float mu, const bf16** dcut_out,
                     bool* forked, std::string* why) {
  cudaStream_t s = m->stream;
  const uint32_t* seq = m->seq_dev;
  const int W = m->world, R = m->rows_back, r = m->rank, b = m->batch, nb = static_cast<int>(m->back.size());
  const int cut = m->cut_elems;
  const size_t cut_bytes = static_cast<size_t>(b) * cut * sizeof(bf16);
  FcLayer& f0 = m->back[0];
  FcLayer& f1 = m->back[1];
  const int ld1 = f1.ld_out;
  // 1. labels to rank 0, cut all-gather into every rank's FC input rows
  int32_t* lab0 = at<int32_t>(m, 0, m->arena_off_lab) + static_cast<size_t>(r) * b;
  if (r == 0) {
    RALPB_TRY(cudaMemcpyAsync(lab0, lab, sizeof(int32_t) * b, cudaMemcpyDeviceToDevice, s));
  } else {
    PeerSignal none{};
    RALPB_TRY(push_and_signal(lab0, lab, static_cast<long long>(b) * 4 / 16, none, seq, m->counters + 1, s));
    ++m->launches;
    m->nvl_out += sizeof(int32_t) * b;
  }
  for (int q = 0; q < W; ++q) {
    if (q == r) continue;
    PeerSignal sig{};
    sig.n = 1;
    sig.flag[0] = at<uint32_t>(m, q, m->arena_off_flags) + kFlagAct + r;
    RALPB_TRY(push_and_signal(at<bf16>(m, q, m->arena_off_xfc) + static_cast<size_t>(r) * b * cut, cut_local,
                              static_cast<long long>(cut_bytes / 16), sig, seq, m->counters + 16 + q, s));
    ++m->launches;
    m->nvl_out += cut_bytes;
    m->logical += static_cast<long long>(b) * cut * m->elem_bytes;   // cut all-gather
  }
  {
    PeerSignal own{};
    own.n = 1;
    own.flag[0] = m->flags + kFlagAct + r;
    RALPB_TRY(signal_only(own, seq, s));
    RALPB_TRY(wait_flags(m->flags + kFlagAct, W, seq, s));
    m->launches += 2;
  }
  // 2. FC-0, column-parallel: h0s = relu(X . W0s^T + b0s)  [R][s0]
  {
    GemmDesc d;
    d.M = R; d.N = m->s0; d.K = f0.in;
    d.a = Operand2D{m->x_fc, R, f0.in, f0.in};
    d.b = Operand2D{f0.wbf, m->s0, f0.in, f0.in};
    if (fc_gemm(m, d, m->ld_s0, m->P + f0.b_off, 1, nullptr, 0, m->h0s, nullptr, why)) return 1;
  }
  // 3. FC-1, row-parallel partial: h0s . W1s^T  [R][out1] fp32 -> rank 0's slot r
  float* p1_slots = at<float>(m, 0, m->arena_off_p1);
  {
    GemmDesc d;
    d.M = R; d.N = f1.out; d.K = m->s0;
    d.a = Operand2D{m->h0s, R, m->s0, m->ld_s0};
    d.b = Operand2D{f1.wbf, f1.out, m->s0, m->s0};
    float* dst = r == 0 ? p1_slots : m->p1_local;
    if (fc_gemm(m, d, ld1, nullptr, 0, nullptr, 0, nullptr, dst, why)) return 1;
    if (r != 0) {
      PeerSignal sig{};
      sig.n = 1;
      sig.flag[0] = at<uint32_t>(m, 0, m->arena_off_flags) + kFlagP1 + r;
      const size_t bytes = static_cast<size_t>(R) * ld1 * sizeof(float);
      RALPB_TRY(push_and_signal(p1_slots + static_cast<size_t>(r) * R * ld1, m->p1_local,
                                static_cast<long long>(bytes / 16), sig, seq, m->counters + 24, s));
      ++m->launches;
      m->nvl_out += bytes;
      m->logical += static_cast<long long>(R) * f1.out * m->elem_bytes;   // FC-1 partial to rank 0
    }
  }
  // 4. rank 0: reduce the partials (+ b1, ReLU), the rest of the tail, the loss, and the gradient
  //    w.r.t. FC-1's pre-activation; broadcast it
  const bf16* dz1 = nullptr;
  if (r == 0) {
    if (W > 1) {
      RALPB_TRY(wait_flags(m->flags + kFlagP1 + 1, W - 1, seq, s));
      ++m->launches;
    }
    PartialSum ps{};
    ps.n = W;
    for (int q = 0; q < W; ++q) ps.part[q] = p1_slots + static_cast<size_t>(q) * R * ld1;
    const FcLayer& last = m->back.back();
    if (nb == 2) {
      RALPB_TRY(sum_partials(ps, R, f1.out, ld1, m->P + f1.b_off, 0, nullptr, m->logits, last.ld_out, s));
    } else {
      RALPB_TRY(sum_partials(ps, R, f1.out, ld1, m->P + f1.b_off, 1, m->hid[1], nullptr, ld1, s));
      // FC layers 2..: forward on rank 0
      const bf16* x = m->hid[1];
      long long ldx = ld1;
      for (int j = 2; j < nb; ++j) {
        FcLayer& f = m->back[j];
        GemmDesc d;
        d.M = R; d.N = f.out; d.K = f.in;
        d.a = Operand2D{x, R, f.in, ldx};
        d.b = Operand2D{f.wbf, f.out, f.in, f.in};
        const bool hidden = j + 1 < nb;
        if (fc_gemm(m, d, f.ld_out, m->P + f.b_off, hidden ? 1 : 0, nullptr, 0, hidden ? m->hid[j] : nullptr,
                    hidden ? nullptr : m->logits, why))
          return 1;
        if (hidden) { x = m->hid[j]; ldx = f.ld_out; }
      }
    }
    ++m->launches;
    const float scale = 1.f / static_cast<float>(W * b);
    RALPB_TRY(softmax_xent(m->logits, R, last.out, last.ld_out, m->labels_all, scale, m->row_loss, m->dlogits,
                           last.ld_out, s));
    RALPB_TRY(reduce_sum(m->row_loss, R, 1.f / static_cast<float>(R), m->loss, s));
    m->launches += 2;
    // backward-data through layers nb-1 .. 2 down to dz1 = dL/d(FC-1 pre-activation)
    for (int j = nb - 1; j >= 2; --j) {
      FcLayer& f = m->back[j];
      const bf16* dy = j == nb - 1 ? m->dlogits : m->dyb[j];
      GemmDesc d;
      d.M = R; d.N = f.in; d.K = f.out;
      d.a_mode = LD_K; d.a = Operand2D{dy, R, f.out, f.ld_out};
      d.b_mode = LD_MN; d.b = Operand2D{f.wbf, f.out, f.in, f.in};
      const long long ldx = m->back[j - 1].ld_out;
      if (fc_gemm(m, d, ldx, nullptr, 0, m->hid[j - 1], ldx, m->dyb[j - 1], nullptr, why)) return 1;
    }
    dz1 = nb == 2 ? m->dlogits : m->dyb[1];
    for (int q = 1; q < W; ++q) {
      PeerSignal sig{};
      sig.n = 1;
      sig.flag[0] = at<uint32_t>(m, q, m->arena_off_flags) + kFlagDh1;
      const size_t bytes = static_cast<size_t>(R) * ld1 * sizeof(bf16);
      RALPB_TRY(push_and_signal(at<bf16>(m, q, m->arena_off_dh1), dz1, static_cast<long long>(bytes / 16), sig, seq,
                                m->counters + 32 + q, s));
      ++m->launches;
      m->nvl_out += bytes;
      m->logical += static_cast<long long>(R) * f1.out * m->elem_bytes;   // FC-1 output gradient back
    }
  } else {
    RALPB_TRY(wait_flags(m->flags + kFlagDh1, 1, seq, s));
    ++m->launches;
    dz1 = reinterpret_cast<const bf16*>(static_cast<char*>(m->arena) + m->arena_off_dh1);
  }
  // 5. FC-1 backward (row-parallel slice): dW1s = dz1^T h0s, dh0s = (dz1 . W1s) * relu'(h0s)
  {
    GemmDesc d;
    d.M = R; d.N = m->s0; d.K = f1.out;
    d.a_mode = LD_K; d.a = Operand2D{dz1, R, f1.out, ld1};
    d.b_mode = LD_MN; d.b = Operand2D{f1.wbf, f1.out, m->s0, m->s0};
    if (fc_gemm(m, d, m->ld_s0, nullptr, 0, m->h0s, m->ld_s0, m->dh0s, nullptr, why)) return 1;
    GemmDesc w;
    w.M = f1.out; w.N = m->s0; w.K = R;
    w.a_mode = LD_MN; w.a = Operand2D{dz1, R, f1.out, ld1};
    w.b_mode = LD_MN; w.b = Operand2D{m->h0s, R, m->s0, m->ld_s0};
    w.s_m = m->s0; w.s_n = 1;
    w.epi = EPI_F32; w.out = m->G + f1.w_off;
    RALPB_TRY(gemm_launch(w, s, why));
    ++m->launches;
  }
  // 6. FC-0 backward (column-parallel slice): db0s, dW0s = dh0s^T X, partial dX = dh0s . W0s
  {
    RALPB_TRY(cudaMemsetAsync(m->G + f0.b_off, 0, m->s0 * sizeof(float), s));
    RALPB_TRY(colsum_bf16(m->dh0s, R, m->s0, m->ld_s0, m->G + f0.b_off, s));
    GemmDesc w;
    w.M = m->s0; w.N = f0.in; w.K = R;
    w.a_mode = LD_MN; w.a = Operand2D{m->dh0s, R, m->s0, m->ld_s0};
    w.b_mode = LD_MN; w.b = Operand2D{m->x_fc, R, f0.in, f0.in};
    w.s_m = f0.in; w.s_n = 1;
    w.epi = EPI_F32; w.out = m->G + f0.w_off;
    RALPB_TRY(gemm_launch(w, s, why));
    GemmDesc d;
    d.M = R; d.N = f0.in; d.K = m->s0;
    d.a_mode = LD_K; d.a = Operand2D{m->dh0s, R, m->s0, m->ld_s0};
    d.b_mode = LD_MN; d.b = Operand2D{f0.wbf, m->s0, f0.in, f0.in};
    if (fc_gemm(m, d, f0.in, nullptr, 0, nullptr, 0, nullptr, m->dxp, why)) return 1;
    m->launches += 2;
  }
  // 7. reduce-scatter of the cut gradient: rows of worker q go to q's partial slot r
  {
    float* parts = reinterpret_cast<float*>(static_cast<char*>(m->arena) + m->arena_off_dxpart);
    const size_t blk = static_cast<size_t>(b) * cut;
    for (int q = 0; q < W; ++q) {
      if (q == r) continue;
      PeerSignal sig{};
      sig.n = 1;
      sig.flag[0] = at<uint32_t>(m, q, m->arena_off_flags) + kFlagDcut + r;
      RALPB_TRY(push_and_signal(at<float>(m, q, m->arena_off_dxpart) + static_cast<size_t>(r) * blk,
                                m->dxp + static_cast<size_t>(q) * blk, static_cast<long long>(blk * sizeof(float) / 16),
                                sig, seq, m->counters + 40 + q, s));
      ++m->launches;
      m->nvl_out += blk * sizeof(float);
      m->logical += static_cast<long long>(b) * cut * m->elem_bytes;   // cut-gradient reduce-scatter
    }
    PeerSignal own{};
    own.n = 1;
    own.flag[0] = m->flags + kFlagDcut + r;
    RALPB_TRY(signal_only(own, seq, s));
    RALPB_TRY(wait_flags(m->flags + kFlagDcut, W, seq, s));
    PartialSum ps{};
    ps.n = W;
    for (int q = 0; q < W; ++q) ps.part[q] = q == r ? m->dxp + static_cast<size_t>(r) * blk : parts + static_cast<size_t>(q) * blk;
    RALPB_TRY(sum_partials(ps, b, cut, cut, nullptr, 0, m->dcut, nullptr, cut, s));
    m->launches += 3;
  }
  *dcut_out = m->dcut;
  // 8. FC updates (this rank's slices; rank 0 also FC-1's bias and the layers after it) on the aux
  //    stream: their weight gradients first (rank 0, layers >= 2), then SGD with the bf16 copies
  if (r == 0) {
    RALPB_TRY(cudaMemsetAsync(m->G + f1.b_off, 0, f1.out * sizeof(float), s));
    RALPB_TRY(colsum_bf16(dz1, R, f1.out, ld1, m->G + f1.b_off, s));
    ++m->launches;
    for (int j = 2; j < nb; ++j) {
      FcLayer& f = m->back[j];
      const bf16* dy = j == nb - 1 ? m->dlogits : m->dyb[j];
      RALPB_TRY(cudaMemsetAsync(m->G + f.b_off, 0, f.out * sizeof(float), s));
      RALPB_TRY(colsum_bf16(dy, R, f.out, f.ld_out, m->G + f.b_off, s));
      GemmDesc w;
      w.M = f.out; w.N = f.in; w.K = R;
      w.a_mode = LD_MN; w.a = Operand2D{dy, R, f.out, f.ld_out};
      w.b_mode = LD_MN; w.b = Operand2D{m->hid[j - 1], R, f.in, m->back[j - 1].ld_out};
      w.s_m = f.in; w.s_n = 1;
      w.epi = EPI_F32; w.out = m->G + f.w_off;
      RALPB_TRY(gemm_launch(w, s, why));
      m->launches += 2;
    }
  }
  RALPB_TRY(cudaEventRecord(m->ev_fork, s));
  RALPB_TRY(cudaStreamWaitEvent(m->aux_stream, m->ev_fork, 0));
  cudaStream_t su = m->aux_stream;
  for (int j = 0; j < nb; ++j) {
    FcLayer& f = m->back[j];
    if (j >= 2 && r != 0) break;
    const long long nw = static_cast<long long>(f.lout) * f.lin;
    RALPB_TRY(sgd_momentum_bf16(m->P + f.w_off, m->V + f.w_off, m->G + f.w_off, nw, lr, mu, 1.f, f.wbf, su));
    ++m->launches;
    if (j != 1 || r == 0) {
      RALPB_TRY(sgd_momentum(m->P + f.b_off, m->V + f.b_off, m->G + f.b_off, f.lout, lr, mu, 1.f, su));
      ++m->launches;
    }
  }
  RALPB_TRY(cudaEventRecord(m->ev_join, su));
  *forked = true;
  return 0;
}

// Backward through conv/pool layers [lo, hi), from `cur` = the gradient w.r.t. layer hi-1's output
// (for a conv: already ReLU-masked).  Layer lo's input is *in_lo (acts[lo] if null) and its
// gradient goes to dst_lo (gacts[lo] if null); dgrad_lo: produce that gradient (the worker's
// layer 0 needs none; the PS's back segment returns it to the workers).  gacts[i] receives the
// gradient w.r.t. the input of layer i.
int sync_bucket_fork(Model* m, float lr, float mu, std::string* why);

int launch_conv_backward(Model* m, int lo, int hi, const bf16* cur, const ActBuf* in_lo, bf16* dst_lo, bool dgrad_lo,
                         std::string* why) {
  bool db_done = false;  // the bias gradient of the layer `cur` belongs to is already summed
  for (int i = hi - 1; i >= lo; --i) {
    // the worker front's backward: layers [bucket_k, split) are done -> their sync forks off
    if (lo == 0 && hi == m->split && i == m->bucket_k - 1 && m->bucket_k > 0 && m->is_worker &&
        sync_bucket_fork(m, m->step_lr, m->step_mu, why))
      return 1;
    FrontLayer& f = m->front[i];
    const ActBuf& in = i == lo && in_lo != nullptr ? *in_lo : m->acts[i];
    const ActBuf& out = m->acts[i + 1];
    bf16* dst_i = i == lo && dst_lo != nullptr ? dst_lo : m->gacts[i];
    if (f.kind == RALPB_BLOCK) {
      const bool need = i > lo || dgrad_lo;
      if (block_backward(m, m->blocks[f.blk], in.ptr, out.ptr, cur, need ? dst_i : nullptr, why)) return 1;
      cur = dst_i;
      db_done = false;
      continue;
    }
    if (f.kind == RALPB_MODULE) {
      const bool need = i > lo || dgrad_lo;
      if (module_backward(m, m->modules[f.mod], in.ptr, out.ptr, cur, need ? dst_i : nullptr, why)) return 1;
      cur = dst_i;
      db_done = false;
      continue;
    }
    if (f.kind == RALPB_APOOL) {
      RALPB_TRY(avgpool_bwd(cur, in.n, in.h, in.w, in.c, MutAct4{dst_i, in.pad}, m->stream));
      ++m->launches;
      cur = dst_i;
      db_done = false;
      continue;
    }
    if (f.kind == RALPB_POOL && f.pool_pad > 0) {
      RALPB_TRY(maxpool_pad_bwd(f.idx, Act4{cur, out.pad}, in.n, in.h, in.w, in.c, f.k, f.stride, f.pool_pad, out.h, out.w,
                                MutAct4{dst_i, in.pad}, m->stream));
      ++m->launches;
      cur = dst_i;
      db_done = false;
      continue;
    }
    if (f.bn) {
      if (bn_stem_backward(m, f, in, out, cur, why)) return 1;
      continue;
    }
    // bias gradient of a (non-im2col) conv i-1 of this segment is summed by the kernel that
    // produces its dY
    float* prev_db = (i > lo && m->front[i - 1].kind == RALPB_CONV && !m->front[i - 1].im2col && !m->front[i - 1].bn &&
                      m->front[i - 1].g.cout <= 512)
                         ? m->G + m->front[i - 1].b_off
                         : nullptr;
    if (f.kind == RALPB_POOL) {
      bf16* dst = dst_i;
      if (f.idx != nullptr && f.fused_fwd)
        RALPB_TRY(maxpool_bwd_idx(f.idx, cur, in.n, out.h, out.w, in.c, out.pad, in.pad, dst, prev_db, m->stream));
      else if (f.idx != nullptr)
        RALPB_TRY(maxpool_bwd_gather(f.idx, cur, in.n, in.h, in.w, in.c, in.pad, f.k, f.stride, out.pad, dst, prev_db,
                                     m->stream));
      else
        RALPB_TRY(maxpool_bwd(in.ptr, cur, in.n, in.h, in.w, in.c, in.pad, f.k, f.stride, out.pad, dst, prev_db,
                              m->stream));
      ++m->launches;
      cur = dst;
      db_done = prev_db != nullptr;
    } else if (f.fused) {
      RALPB_TRY(conv_first_wgrad(m->step_img, in.n, m->in_h, m->in_w, m->in_c, cur, out.pad, m->G + f.w_off, m->stream,
                                 why));
      ++m->launches;
    } else if (f.im2col) {
      // dW[co][j] += sum_rows dY[row][co] * patches[row][j]  (j = kpad incl. the bias column)
      GemmDesc d;
      d.M = f.g.cout; d.N = f.kpad; d.K = in.rows();
      d.a_mode = LD_MN; d.a = Operand2D{cur, out.rows(), f.g.cout, f.g.cout};
      d.b_mode = LD_MN; d.b = Operand2D{in.ptr, in.rows(), f.kpad, f.kpad};
      d.k_splits = 0;
      d.epi = EPI_F32_ATOMIC; d.out = m->G + f.w_off; d.s_m = f.kpad; d.s_n = 1;
      RALPB_TRY(gemm_launch(d, m->stream, why));
      ++m->launches;
    } else {
      // db of this layer: already summed by the producer of `cur` unless `cur` is the segment's
      // incoming gradient
      RALPB_TRY(conv_wgrad(f.g, in.ptr, cur, m->G + f.w_off, db_done ? nullptr : m->G + f.b_off, m->stream, why));
      ++m->launches;
      if (i > lo || dgrad_lo) {
        bf16* dst = dst_i;
        const bool mask = i > 0 && m->front[i - 1].kind == RALPB_CONV;
        RALPB_TRY(conv_dgrad(f.g, cur, f.wd, mask ? in.ptr : nullptr, dst, prev_db, m->stream, why));
        ++m->launches;
        cur = dst;
        db_done = prev_db != nullptr;
      }
    }
  }
  return 0;
}

int launch_front_backward(Model* m, const bf16* dcut, std::string* why) {
  return launch_conv_backward(m, 0, m->split, dcut, nullptr, nullptr, false, why);
}

// Forward through conv/pool layers [lo, hi): layer lo reads *in_lo (acts[lo] if null), layer hi-1
// writes out_last (a following 2x2/2 max pool is fused into the conv epilogue where set up).
int launch_conv_forward(Model* m, int lo, int hi, const float* img, const ActBuf* in_lo, bf16* out_last,
                        std::string* why) {
  cudaStream_t s = m->stream;
  for (int i = lo; i < hi; ++i) {
    FrontLayer& f = m->front[i];
    const ActBuf& in = i == lo && in_lo != nullptr ? *in_lo : m->acts[i];
    ActBuf out = m->acts[i + 1];
    if (i + 1 == hi) out.ptr = out_last;
    if (f.kind == RALPB_BLOCK) {
      if (block_forward(m, m->blocks[f.blk], in.ptr, out.ptr, why)) return 1;
      continue;
    }
    if (f.kind == RALPB_MODULE) {
      if (module_forward(m, m->modules[f.mod], in.ptr, out.ptr, why)) return 1;
      continue;
    }
    if (f.kind == RALPB_APOOL) {
      RALPB_TRY(avgpool_fwd(Act4{in.ptr, in.pad}, in.n, in.h, in.w, in.c, out.ptr, s));
      ++m->launches;
      continue;
    }
    if (f.kind == RALPB_POOL && f.pool_pad > 0) {
      RALPB_TRY(maxpool_pad_fwd(Act4{in.ptr, in.pad}, in.n, in.h, in.w, in.c, f.k, f.stride, f.pool_pad,
                                MutAct4{out.ptr, out.pad}, out.h, out.w, f.idx, s));
      ++m->launches;
      continue;
    }
    if (f.bn) {
      if (bn_stem_forward(m, f, in, out, why)) return 1;
      continue;
    }
    if (f.fused) {
      RALPB_TRY(conv_first_fwd(img, in.n, m->in_h, m->in_w, m->in_c, f.wf, out.ptr, out.pad, s, why));
    } else if (f.im2col) {
      // y = relu(patches . W^T) on the padded output grid (bias rides in the ones column)
      GemmDesc d;
      d.M = static_cast<int>(in.rows()); d.N = f.g.cout; d.K = f.kpad;
      d.kb = std::min(64, f.kpad);
      d.a = Operand2D{in.ptr, in.rows(), f.kpad, f.kpad};
      d.b = Operand2D{f.wf, f.g.cout, f.kpad, f.kpad};
      d.epi = EPI_BF16; d.relu = 1; d.out = out.ptr; d.s_m = f.g.cout;
      d.border = 1; d.img_rows = (out.h + 2 * out.pad) * (out.w + 2 * out.pad); d.wp = out.w + 2 * out.pad;
      d.pad = out.pad; d.h = out.h; d.w = out.w;
      RALPB_TRY(gemm_launch(d, s, why));
    } else if (f.kind == RALPB_CONV) {
      const bool pool_next = i + 1 < hi && m->front[i + 1].fused_fwd;
      if (pool_next) {
        const ActBuf& pooled = m->acts[i + 2];
        bf16* pdst = i + 2 == hi ? out_last : pooled.ptr;
        RALPB_TRY(conv_fwd_pool(f.g, in.ptr, f.wf, m->P + f.b_off, out.ptr, 1, pdst, pooled.pad, s, why,
                                m->front[i + 1].idx));
        ++m->launches;
        ++i;  // the pool layer is done
        continue;
      }
      RALPB_TRY(conv_fwd(f.g, in.ptr, f.wf, m->P + f.b_off, out.ptr, 1, s, why));
    } else {
      RALPB_TRY(maxpool_fwd(in.ptr, in.n, in.h, in.w, in.c, in.pad, f.k, f.stride, out.ptr, out.pad, s, f.idx));
    }
    ++m->launches;
  }
  return 0;
}

// bf16 filter copies from the fp32 masters, batched into one launch per kMaxPrepJobs layers:
// forward copies (wf, needed by the next step's first kernel) and/or the tap-reversed
// transposes the backward-data kernels read (wd).
int prep_filters(Model* m, bool forward, bool dgrad, cudaStream_t s, std::string* why, int lo = 0, int hi = -1) {
  WeightPrepJob jobs[kMaxPrepJobs];
  int nj = 0;
  std::vector<CastJob> casts;   // plain filter casts (branch-group nodes, im2col layers): one launch
  if (hi < 0) hi = static_cast<int>(m->front.size());
  for (size_t i = lo; i < static_cast<size_t>(hi); ++i) {
    FrontLayer& f = m->front[i];
    if (f.kind == RALPB_BLOCK) {   // all of a block's operand copies with the forward ones
      if (forward && m->blocks[f.blk].wa != nullptr) {
        std::vector<WeightPrepJob> bj;
        if (block_prep(m, m->blocks[f.blk], s, why, &casts, &bj)) return 1;
        for (const WeightPrepJob& j : bj) {
          if (nj == kMaxPrepJobs) {
            RALPB_TRY(conv_weight_prep_batch(jobs, nj, s));
            ++m->launches;
            nj = 0;
          }
          jobs[nj++] = j;
        }
      }
      continue;
    }
    if (f.kind == RALPB_MODULE) {
      if (forward && module_prep(m, m->modules[f.mod], s, why, &casts)) return 1;
      continue;
    }
    if (f.kind != RALPB_CONV || f.wf == nullptr) continue;   // (layers this rank does not run)
    if (f.im2col) {
      if (forward) casts.push_back(CastJob{m->P + f.w_off, f.wf, f.w_count});
      continue;
    }
    if (!forward && i == 0) continue;   // no backward-data for the first layer
    if (nj == kMaxPrepJobs) {
      RALPB_TRY(conv_weight_prep_batch(jobs, nj, s));
      ++m->launches;
      nj = 0;
    }
    WeightPrepJob& j = jobs[nj++];
    j = WeightPrepJob{};
    j.w = m->P + f.w_off; j.wf = forward ? f.wf : nullptr; j.wd = dgrad && i > 0 ? f.wd : nullptr;
    j.co = f.g.cout; j.taps = f.g.taps(); j.ci = f.g.cin;
  }
  if (nj > 0) {
    RALPB_TRY(conv_weight_prep_batch(jobs, nj, s));
    ++m->launches;
  }
  if (!casts.empty()) {
    RALPB_TRY(cast_bf16_batch(casts.data(), static_cast<int>(casts.size()), s));
    m->launches += (static_cast<int>(casts.size()) + kMaxCastJobs - 1) / kMaxCastJobs;
  }
  return 0;
}

// After a parameter update: the forward copies on the model stream; the backward-data
// transposes are rebuilt at the start of the next step on the aux stream, overlapping the
// forward pass (step_body), so only `dgrad_now` callers need them here.
int relayout_weights(Model* m, bool fc_too, std::string* why, bool dgrad_now = false) {
  if (prep_filters(m, true, dgrad_now, m->stream, why)) return 1;
  if (fc_too) {
    for (auto& f : m->back) {
      RALPB_TRY(cast_bf16(m->P + f.w_off, static_cast<long long>(f.lout) * f.lin, f.wbf, m->stream));
      ++m->launches;
    }
  }
  return 0;
}

// Sharded-PS synchronisation of params[0, n) over the worker group (every rank, or the workers only
// with a dedicated PS rank): worker w owns shard w.  Logical bytes at the reference's sites: this
// worker's gradient push ("grad"/"push", simulator.py:647,689: every real parameter of [0, n)) and
// the pull of the shard it owns to every worker ("pull", simulator.py:663,713); the ring strategy
// counts its reduce-scatter + all-gather share 2*(W-1)*shard (ring_shares, simulator.py:726).
int sync_range(Model* m, long long lo, long long hi, int fg, int fd, uint32_t* counter, cudaStream_t s, float lr,
               float mu, std::string* why);

// The sync bucket (layers [bucket_k, split) -- the late, parameter-heavy layers whose backward is
// done first): forked onto sync_stream right after layer bucket_k's backward-filter, its sharded
// update over [bucket_lo, n_front) runs while this rank's backward of the early layers continues;
// the update kernels are small (no shared memory) and co-reside with the persistent conv kernels.
int sync_bucket_fork(Model* m, float lr, float mu, std::string* why) {
  RALPB_TRY(cudaEventRecord(m->ev_b1, m->stream));
  RALPB_TRY(cudaStreamWaitEvent(m->sync_stream, m->ev_b1, 0));
  if (sync_range(m, m->bucket_lo, m->n_front, kFlagGradB, kFlagDoneB, m->counters + 4, m->sync_stream, lr, mu, why))
    return 1;
  RALPB_TRY(cudaEventRecord(m->ev_b1_done, m->sync_stream));
  m->bucket_forked = true;
  return 0;
}

int sync_params(Model* m, long long n, float lr, float mu, std::string* why) {
  const int W = m->workers;
  const long long eb = m->elem_bytes;
  const bool ring = m->strategy == RALPB_STRATEGY_RING || m->strategy == RALPB_STRATEGY_RING_EXTERNAL;
  long long real_n = 0;
  for (long long v : m->shard_real) real_n += v;
  if (ring)
    m->logical += 2LL * (W - 1) * m->shard_real[m->widx] * eb;
  else
    m->logical += real_n * eb + static_cast<long long>(W) * m->shard_real[m->widx] * eb;
  if (W == 1) {
    RALPB_TRY(sgd_momentum(m->P, m->V, m->G, n, lr, mu, 1.f, m->stream));
    ++m->launches;
    return 0;
  }
  // a sync bucket (the late layers, updated under the remaining backward by sync_bucket_fork):
  // here only [0, bucket_lo), then wait for the bucket's shards of every worker
  const bool bucket = m->bucket_forked;
  if (bucket) n = m->bucket_lo;
  if (sync_range(m, 0, n, kFlagGrad, kFlagDone, m->counters + 0, m->stream, lr, mu, why)) return 1;
  if (bucket) {
    RALPB_TRY(cudaStreamWaitEvent(m->stream, m->ev_b1_done, 0));
    RALPB_TRY(wait_flags(m->flags + kFlagDoneB, W, m->seq_dev, m->stream));
    ++m->launches;
    m->bucket_forked = false;
  }
  return 0;
}

// One sharded-PS update of params[lo, hi) on stream s: signal this rank's gradient ready (flag
// base fg) on every worker, wait for all, update this rank's shard (whole-layer ranges with
// layer_shards), store it into every worker, signal done (flag base fd).
int sync_range(Model* m, long long lo, long long hi, int fg, int fd, uint32_t* counter, cudaStream_t s, float lr,
               float mu, std::string* why) {
  const int W = m->workers;
  const long long n = hi - lo;
  const uint32_t* seq = m->seq_dev;
  PeerSignal all_grad{}, all_done{};
  all_grad.n = all_done.n = W;
  for (int w = 0; w < W; ++w) {
    uint32_t* fl = at<uint32_t>(m, m->worker_ranks[w], m->arena_off_flags);
    all_grad.flag[w] = fl + fg + m->widx;
    all_done.flag[w] = fl + fd + m->widx;
  }
  RALPB_TRY(signal_only(all_grad, seq, s));
  RALPB_TRY(wait_flags(m->flags + fg, W, seq, s));
  ShardUpdate u{};
  u.nranks = W;
  u.self = m->widx;
  // equal shards, multiples of 4 floats (the last one takes the remainder)
  const long long shard = ((n + 4LL * W - 1) / (4LL * W)) * 4;
  u.begin = std::min(hi, lo + shard * m->widx);
  u.end = std::min(hi, u.begin + shard);
  if (m->widx == W - 1) u.end = hi;
  long long mine = u.end - u.begin;
  if (m->layer_shards) {   // whole-layer shards (the reference's PS layout)
    const auto& rg = m->shard_ranges[m->widx];
    u.nr = static_cast<int>(rg.size());
    mine = 0;
    for (int k = 0; k < u.nr; ++k) {
      u.rb[k] = rg[k].first;
      u.re[k] = rg[k].second;
      mine += rg[k].second - rg[k].first;
    }
    if (u.nr == 0) { u.nr = 1; u.rb[0] = u.re[0] = 0; }   // a shard without layers (W > weighted layers)
  }
  u.lr = lr; u.mu = mu; u.gscale = 1.f;
  u.momentum = m->V;
  for (int w = 0; w < W; ++w) {
    u.grads[w] = at<float>(m, m->worker_ranks[w], m->arena_off_G);
    u.params[w] = at<float>(m, m->worker_ranks[w], m->arena_off_P);
  }
  RALPB_TRY(shard_update(u, all_done, seq, counter, s));
  if (fd == kFlagDone) RALPB_TRY(wait_flags(m->flags + fd, W, seq, s));   // (the bucket's wait: in sync_params)
  m->launches += fd == kFlagDone ? 4 : 3;
  const long long peer = static_cast<long long>(W - 1) * mine * static_cast<long long>(sizeof(float));
  m->nvl_in += peer;   // gradient shards of the other workers
  m->nvl_out += peer;  // the updated shard to the other workers
  return 0;
}

}  // namespace

namespace {

// Event record that also works as a graph node while the stream is being captured.
cudaError_t mark(Model* m, int i, bool capturing) {
  return capturing ? cudaEventRecordWithFlags(m->ev[i], m->stream, cudaEventRecordExternal)
                   : cudaEventRecord(m->ev[i], m->stream);
}

// ------------------------------------------------------------------ pair precision
// The parity precision (RALPB_PRECISION_FP32): the same schedule, every activation / gradient an
// fp32-accurate (hi, lo) bf16 pair, every contraction the tcgen05 GEMM engine over the pairs with
// an fp32 result finished by pair.cu (layouts in pair.cuh).

bool pair_mode(const Model* m) { return m->precision == RALPB_PRECISION_FP32; }

// K-block (elements) of a K-major piece operand: the largest of 64 / 32 / 16 dividing its width.
int kb_for(long long k) { return k % 64 == 0 ? 64 : (k % 32 == 0 ? 32 : 16); }

// FC layer j's input as (groups, channels): the cut (HWC pixels x channels) or a hidden row.
void fc_in_geom(const Model* m, int j, int* groups, int* c) {
  if (j == 0) {
    const ActBuf& cut = m->acts.back();
    *groups = cut.h * cut.w;
    *c = cut.c;
  } else {
    *groups = 1;
    *c = m->back[j].in;
  }
}

// Pair operand copies of every parameter from the fp32 masters.
int pair_relayout(Model* m, bool front, bool fc, cudaStream_t s, std::string* why) {
  if (front && m->is_worker) {
    for (auto& f : m->front) {
      if (f.kind != RALPB_CONV) continue;
      if (f.im2col)
        RALPB_TRY(pair_prep_mat(m->P + f.w_off, f.g.cout, f.g.cout, 1, f.kpad, f.wf, nullptr, m->pieces, s));
      else
        RALPB_TRY(pair_prep_conv(m->P + f.w_off, f.g.cout, f.g.taps(), f.g.cin, f.wf, f.wd, m->pieces, s));
      ++m->launches;
    }
  }
  if (fc) {
    for (size_t j = 0; j < m->back.size(); ++j) {
      FcLayer& f = m->back[j];
      int groups = 0, c = 0;
      fc_in_geom(m, static_cast<int>(j), &groups, &c);
      RALPB_TRY(pair_prep_mat(m->P + f.w_off, f.out, f.ld_out, groups, c, f.wbf, f.wbd, m->pieces, s));
      ++m->launches;
    }
  }
  return 0;
}

// out[M][N] (+)= A . B^T on the GEMM engine with an fp32 result (atomic: split-K, caller zeroes).
int pair_gemm(Model* m, GemmDesc d, void* out, long long s_m, long long s_n, bool atomic, std::string* why) {
  d.epi = atomic ? EPI_F32_ATOMIC : EPI_F32;
  d.k_splits = atomic ? 0 : 1;
  d.out = out;
  d.s_m = s_m;
  d.s_n = s_n;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  ++m->launches;
  return 0;
}

void set_border(GemmDesc* d, const ActBuf& a) {
  d->border = 1;
  d->img_rows = (a.h + 2 * a.pad) * (a.w + 2 * a.pad);
  d->wp = a.w + 2 * a.pad;
  d->pad = a.pad;
  d->h = a.h;
  d->w = a.w;
}

PairFinish finish_for(const ActBuf& a, const float* acc, int n, const float* bias, int relu, const bf16* mask,
                      bf16* out2, int P) {
  PairFinish f{};
  f.pieces = P;
  f.acc = acc;
  f.rows = a.rows();
  f.n = n;
  f.ld = n;
  f.bias = bias;
  f.relu = relu;
  f.mask = mask;
  f.out2 = out2;
  f.border = 1;
  f.img_rows = (a.h + 2 * a.pad) * (a.w + 2 * a.pad);
  f.wp = a.w + 2 * a.pad;
  f.pad = a.pad;
  f.h = a.h;
  f.w = a.w;
  return f;
}

int pair_front_forward(Model* m, const float* img, bf16* cut_dst, std::string* why) {
  const int P = m->pieces;
  cudaStream_t s = m->stream;
  const int b = m->batch;
  for (size_t i = 0; i < m->front.size(); ++i) {
    FrontLayer& f = m->front[i];
    const ActBuf& in = m->acts[i];
    ActBuf out = m->acts[i + 1];
    if (i + 1 == m->front.size()) out.ptr = cut_dst;
    if (f.im2col) {
      const FrontLayer& f0 = m->front[0];
      RALPB_TRY(pair_pack_im2col(img, b, m->in_h, m->in_w, m->in_c, f0.k, f0.stride, m->desc[0].pad, in.h, in.w, in.pad,
                                 f0.kpad, in.ptr, P, s));
      ++m->launches;
      GemmDesc d;
      d.M = static_cast<int>(in.rows()); d.N = P * f.g.cout; d.K = P * f.kpad;
      d.kb = kb_for(P * f.kpad);
      d.a = Operand2D{in.ptr, in.rows(), P * f.kpad, P * f.kpad};
      d.b = Operand2D{f.wf, P * f.g.cout, P * f.kpad, P * f.kpad};
      set_border(&d, out);
      if (pair_gemm(m, d, m->pair_acc, P * f.g.cout, 1, false, why)) return 1;
      RALPB_TRY(pair_finish(finish_for(out, m->pair_acc, f.g.cout, nullptr, 1, nullptr, out.ptr, P), s));
      ++m->launches;
    } else if (f.kind == RALPB_CONV) {
      const ConvGeom& g = f.g;
      GemmDesc d;
      d.M = static_cast<int>(g.q()); d.N = P * g.cout;
      d.kb = kb_for(P * g.cin);
      d.K = static_cast<long long>(g.taps()) * P * g.cin;
      d.a_mode = LD_K_CONV;
      d.a = Operand2D{in.ptr, g.q(), P * g.cin, P * g.cin};
      d.cblks = P * g.cin / d.kb;
      d.b = Operand2D{f.wf, P * g.cout, d.K, d.K};
      d.taps = g.taps();
      for (int r = 0; r < g.k; ++r)
        for (int c = 0; c < g.k; ++c) d.tap_off[r * g.k + c] = (r - g.pad) * g.wp() + (c - g.pad);
      set_border(&d, out);
      if (pair_gemm(m, d, m->pair_acc, P * g.cout, 1, false, why)) return 1;
      RALPB_TRY(pair_finish(finish_for(out, m->pair_acc, g.cout, m->P + f.b_off, 1, nullptr, out.ptr, P), s));
      ++m->launches;
    } else {
      RALPB_TRY(pair_maxpool_fwd(in.ptr, in.n, in.h, in.w, in.c, in.pad, f.k, f.stride, out.ptr, out.pad, f.idx, P, s));
      ++m->launches;
    }
  }
  return 0;
}

// FC tail forward + loss over R rows of x_fc: logits (fp32), dlogits (pair), loss share.
int pair_fc_forward_loss(Model* m, int R, float scale, std::string* why) {
  const int P = m->pieces;
  cudaStream_t s = m->stream;
  const bf16* x = m->x_fc;
  long long in2 = static_cast<long long>(P) * m->cut_elems;
  const int nb = static_cast<int>(m->back.size());
  for (int j = 0; j < nb; ++j) {
    FcLayer& f = m->back[j];
    GemmDesc d;
    d.M = R; d.N = P * f.ld_out; d.K = in2;
    d.a = Operand2D{x, R, in2, in2};
    d.b = Operand2D{f.wbf, P * f.ld_out, in2, in2};
    RALPB_TRY(cudaMemsetAsync(m->pair_acc, 0, sizeof(float) * R * P * f.ld_out, s));
    if (pair_gemm(m, d, m->pair_acc, P * f.ld_out, 1, true, why)) return 1;
    PairFinish fin{};
    fin.pieces = P;
    fin.acc = m->pair_acc; fin.rows = R; fin.n = f.out; fin.ld = f.ld_out; fin.bias = m->P + f.b_off;
    const bool hidden = j + 1 < nb;
    fin.relu = hidden ? 1 : 0;
    fin.out2 = hidden ? m->hid[j] : nullptr;
    fin.out_f32 = hidden ? nullptr : m->logits;
    fin.ld_f32 = f.ld_out;
    RALPB_TRY(pair_finish(fin, s));
    m->launches += 2;
    x = hidden ? m->hid[j] : nullptr;
    in2 = static_cast<long long>(P) * f.ld_out;
  }
  const FcLayer& last = m->back.back();
  RALPB_TRY(pair_softmax_xent(m->logits, R, last.out, last.ld_out, m->labels_all, scale, m->row_loss, m->dlogits, P, s));
  RALPB_TRY(reduce_sum(m->row_loss, R, scale, m->loss, s));
  m->launches += 2;
  return 0;
}

// FC backward-data chain down to the cut gradient rows (pairs in the cut's pixel-group layout).
int pair_fc_backward_data(Model* m, int R, bf16* dx_out, std::string* why) {
  const int P = m->pieces;
  cudaStream_t s = m->stream;
  const int nb = static_cast<int>(m->back.size());
  for (int j = nb - 1; j >= 0; --j) {
    FcLayer& f = m->back[j];
    const bf16* dy = j == nb - 1 ? m->dlogits : m->dyb[j];
    int groups = 0, c = 0;
    fc_in_geom(m, j, &groups, &c);
    const long long in2 = static_cast<long long>(P) * groups * c;
    GemmDesc d;
    d.M = R; d.N = static_cast<int>(in2); d.K = P * f.ld_out;
    d.a_mode = LD_K; d.a = Operand2D{dy, R, P * f.ld_out, P * f.ld_out};
    d.b_mode = LD_MN; d.b = Operand2D{f.wbd, P * f.ld_out, in2, in2};
    RALPB_TRY(cudaMemsetAsync(m->pair_acc, 0, sizeof(float) * R * in2, s));
    if (pair_gemm(m, d, m->pair_acc, in2, 1, true, why)) return 1;
    PairFinishGroups fin{};
    fin.pieces = P;
    fin.acc = m->pair_acc; fin.rows = R; fin.groups = groups; fin.c = c;
    fin.mask = j > 0 ? m->hid[j - 1] : nullptr;
    fin.out2 = j > 0 ? m->dyb[j - 1] : dx_out;
    RALPB_TRY(pair_finish_groups(fin, s));
    m->launches += 2;
  }
  return 0;
}

// FC weight / bias gradients into G, and (update) the PS-local SGD with the pair re-layout.
int pair_fc_backward_weights(Model* m, int R, bool update, float lr, float mu, std::string* why) {
  const int P = m->pieces;
  cudaStream_t s = m->stream;
  const int nb = static_cast<int>(m->back.size());
  for (int j = nb - 1; j >= 0; --j) {
    FcLayer& f = m->back[j];
    const bf16* dy = j == nb - 1 ? m->dlogits : m->dyb[j];
    const bf16* x = j == 0 ? m->x_fc : m->hid[j - 1];
    int groups = 0, c = 0;
    fc_in_geom(m, j, &groups, &c);
    const long long in2 = static_cast<long long>(P) * groups * c;
    RALPB_TRY(cudaMemsetAsync(m->G + f.b_off, 0, f.out * sizeof(float), s));
    RALPB_TRY(pair_colsum(dy, R, f.out, f.ld_out, m->G + f.b_off, P, s));
    GemmDesc w;
    w.M = P * f.ld_out; w.N = static_cast<int>(in2); w.K = R;
    w.a_mode = LD_MN; w.a = Operand2D{dy, R, P * f.ld_out, P * f.ld_out};
    w.b_mode = LD_MN; w.b = Operand2D{x, R, in2, in2};
    RALPB_TRY(cudaMemsetAsync(m->pair_s, 0, sizeof(float) * P * f.ld_out * in2, s));
    if (pair_gemm(m, w, m->pair_s, in2, 1, true, why)) return 1;
    RALPB_TRY(pair_reduce_wgrad(m->pair_s, f.ld_out, f.out, groups, c, m->G + f.w_off, static_cast<long long>(groups) * c, P, s));
    m->launches += 3;
  }
  if (update) {
    for (auto& f : m->back) {
      RALPB_TRY(sgd_momentum(m->P + f.w_off, m->V + f.w_off, m->G + f.w_off, static_cast<long long>(f.out) * f.in, lr, mu,
                             1.f, s));
      RALPB_TRY(sgd_momentum(m->P + f.b_off, m->V + f.b_off, m->G + f.b_off, f.out, lr, mu, 1.f, s));
      m->launches += 2;
    }
    if (pair_relayout(m, false, true, s, why)) return 1;
  }
  return 0;
}

int pair_front_backward(Model* m, const bf16* dcut, std::string* why) {
  const int P = m->pieces;
  cudaStream_t s = m->stream;
  const bf16* cur = dcut;
  for (int i = static_cast<int>(m->front.size()) - 1; i >= 0; --i) {
    FrontLayer& f = m->front[i];
    const ActBuf& in = m->acts[i];
    const ActBuf& out = m->acts[i + 1];
    if (f.kind == RALPB_POOL) {
      RALPB_TRY(pair_maxpool_bwd(f.idx, cur, in.n, in.h, in.w, in.c, in.pad, f.k, f.stride, out.pad, m->gacts[i], nullptr,
                                 P, s));
      ++m->launches;
      cur = m->gacts[i];
      continue;
    }
    if (f.im2col) {
      // dW[co][j] = sum over the output grid of dY[row][co] * patches[row][j] (bias in column k*k*cin)
      GemmDesc d;
      d.M = P * f.g.cout; d.N = P * f.kpad; d.K = in.rows();
      d.a_mode = LD_MN; d.a = Operand2D{cur, out.rows(), P * f.g.cout, P * f.g.cout};
      d.b_mode = LD_MN; d.b = Operand2D{in.ptr, in.rows(), P * f.kpad, P * f.kpad};
      RALPB_TRY(cudaMemsetAsync(m->pair_s, 0, sizeof(float) * P * P * f.g.cout * f.kpad, s));
      if (pair_gemm(m, d, m->pair_s, P * f.kpad, 1, true, why)) return 1;
      RALPB_TRY(pair_reduce_wgrad(m->pair_s, f.g.cout, f.g.cout, 1, f.kpad, m->G + f.w_off, f.kpad, P, s));
      ++m->launches;
      continue;
    }
    const ConvGeom& g = f.g;
    // bias gradient: sum of the (masked) output gradient
    RALPB_TRY(pair_colsum(cur, out.rows(), g.cout, g.cout, m->G + f.b_off, P, s));
    // weight gradient: S[(a,co)][t][(b,ci)] = sum_q dy_a[q][co] x_b[q + off(t)][ci]
    {
      GemmDesc d;
      d.M = g.taps() * P * g.cin; d.N = P * g.cout; d.K = g.q();
      d.a_mode = LD_MN_CONV; d.a = Operand2D{in.ptr, g.q(), P * g.cin, P * g.cin}; d.a_cin = P * g.cin;
      d.b_mode = LD_MN; d.b = Operand2D{cur, g.q(), P * g.cout, P * g.cout};
      d.taps = g.taps();
      for (int r = 0; r < g.k; ++r)
        for (int c = 0; c < g.k; ++c) d.tap_off[r * g.k + c] = (r - g.pad) * g.wp() + (c - g.pad);
      const int n2 = P * g.cout;
      d.block_n = n2 >= 256 ? 256 : (n2 >= 128 ? 128 : (n2 >= 64 ? 64 : 32));
      RALPB_TRY(cudaMemsetAsync(m->pair_s, 0, sizeof(float) * P * P * f.w_count, s));
      if (pair_gemm(m, d, m->pair_s, 1, static_cast<long long>(g.taps()) * P * g.cin, true, why)) return 1;
      RALPB_TRY(pair_reduce_wgrad(m->pair_s, g.cout, g.cout, g.taps(), g.cin, m->G + f.w_off,
                                  static_cast<long long>(g.taps()) * g.cin, P, s));
      m->launches += 2;
    }
    if (i > 0) {
      // backward-data: out[q][(a,ci)] = sum dy[q + off'][(b,co)] wd_a; masked by the producer's ReLU
      GemmDesc d;
      d.M = static_cast<int>(g.q()); d.N = P * g.cin;
      d.kb = kb_for(P * g.cout);
      d.K = static_cast<long long>(g.taps()) * P * g.cout;
      d.a_mode = LD_K_CONV; d.a = Operand2D{cur, g.q(), P * g.cout, P * g.cout};
      d.cblks = P * g.cout / d.kb;
      d.b = Operand2D{f.wd, P * g.cin, d.K, d.K};
      d.taps = g.taps();
      for (int r = 0; r < g.k; ++r)
        for (int c = 0; c < g.k; ++c) d.tap_off[r * g.k + c] = (r - g.pad) * g.wp() + (c - g.pad);
      set_border(&d, in);
      if (pair_gemm(m, d, m->pair_acc, P * g.cin, 1, false, why)) return 1;
      const bool mask = m->front[i - 1].kind == RALPB_CONV;
      RALPB_TRY(pair_finish(finish_for(in, m->pair_acc, g.cin, nullptr, 0, mask ? in.ptr : nullptr, m->gacts[i], P), s));
      ++m->launches;
      cur = m->gacts[i];
    }
  }
  return 0;
}

__global__ void combine_loss_kernel(const float* slots, int n, int self, float* out) {
  // out[0] = own share + the other workers' shares (slots[w * 4], w != self), fixed order
  if (threadIdx.x == 0) {
    float acc = 0.f;
    for (int w = 0; w < n; ++w) acc += w == self ? out[0] : slots[4 * w];
    out[0] = acc;
  }
}

// The step's mean loss on the reporting rank when every rank computes the loss of its own rows
// (baseline / ring): the others push their share (16 bytes) into its arena slot; it sums them in
// worker order.  Called where the reporting rank already waits for every rank (after the sync).
int push_loss_share(Model* m, std::string* why) {
  if (m->workers == 1 || m->rank == m->ps_rank) return 0;
  PeerSignal sig{};
  sig.n = 1;
  sig.flag[0] = at<uint32_t>(m, m->ps_rank, m->arena_off_flags) + kFlagLoss + m->widx;
  float* slot = at<float>(m, m->ps_rank, m->arena_off_loss) + 4 * m->widx;
  RALPB_TRY(push_and_signal(slot, m->loss, 1, sig, m->seq_dev, m->counters + 3, m->stream));
  ++m->launches;
  m->nvl_out += 16;
  return 0;
}

int combine_loss(Model* m, std::string* why) {
  if (m->workers == 1 || m->rank != m->ps_rank) return 0;
  const int W = m->workers;
  // flags kFlagLoss + w for every other worker w (this rank's own slot is never signalled: wait on
  // the two contiguous ranges around it)
  if (m->widx > 0) RALPB_TRY(wait_flags(m->flags + kFlagLoss, m->widx, m->seq_dev, m->stream));
  if (m->widx + 1 < W) RALPB_TRY(wait_flags(m->flags + kFlagLoss + m->widx + 1, W - m->widx - 1, m->seq_dev, m->stream));
  combine_loss_kernel<<<1, 32, 0, m->stream>>>(reinterpret_cast<const float*>(static_cast<char*>(m->arena) + m->arena_off_loss),
                                               W, m->widx, m->loss);
  RALPB_TRY(cudaGetLastError());
  m->launches += 3;
  return 0;
}

// Everything of one step after the inputs are resident in HBM: bump the device step
// counter, front forward, cut exchange, back segment, front backward, sync, re-layout.
// Logical bytes are counted where each transfer is issued, at the reference's count_wire sites
// (simulator.py:677 act, :707 actgrad, :689 grad, :713 pull; :647/:663 baseline push/pull).
int step_body(Model* m, const float* img, const int32_t* lab, float lr, float mu, bool capturing,
              std::string* why) {
  const uint32_t* seq = m->seq_dev;
  const int b = m->batch;
  const int W = m->workers;
  const long long eb = m->elem_bytes;
  const bool ralp = m->strategy == RALPB_STRATEGY_RALP;
  cudaStream_t s = m->stream;
  bool fc_forked = false;
  m->step_lr = lr;
  m->step_mu = mu;
  m->bucket_forked = false;
  RALPB_TRY(bump_counter(m->seq_dev, s));
  ++m->launches;
  const long long cut_logical = static_cast<long long>(b) * m->xch_logical * eb;  // one worker's cut
  const bool pairs = pair_mode(m);
  // bf16 elements per sample of the exchanged cut (padded when a conv back segment reads it)
  const size_t cut_row = static_cast<size_t>(m->xch_elems) * (pairs ? m->pieces : 1);
  const size_t cut_bytes = static_cast<size_t>(b) * cut_row * sizeof(bf16);
  const int slot = ralp || m->mps ? m->widx : 0;   // this worker's row block in the PS input
  const bf16* cut_local = nullptr;
  bool scatter_forked = false;

  if (m->is_worker && pairs) {
    bf16* cut_dst = m->acts.back().ptr;
    if (m->holds_back) cut_dst = m->xin + static_cast<size_t>(slot) * b * cut_row;
    if (pair_front_forward(m, img, cut_dst, why)) return 1;
    cut_local = cut_dst;
  } else if (m->is_worker) {
    // backward-data filter copies from this step's masters, on the aux stream under the forward
    RALPB_TRY(cudaEventRecord(m->ev_wd_fork, s));
    RALPB_TRY(cudaStreamWaitEvent(m->aux_stream, m->ev_wd_fork, 0));
    if (prep_filters(m, false, true, m->aux_stream, why)) return 1;
    RALPB_TRY(cudaEventRecord(m->ev_wd_join, m->aux_stream));

    // ---------------- worker front forward
    const FrontLayer& f0 = m->front[0];
    const ActBuf& a0 = m->acts[0];
    m->step_img = img;
    if (f0.fused) {
      // patches are built on chip by conv_first_fwd / conv_first_wgrad
    } else if (f0.im2col) {
      RALPB_TRY(pack_im2col(img, b, m->in_h, m->in_w, m->in_c, f0.k, f0.stride, m->desc[0].pad, a0.h, a0.w, a0.pad,
                            f0.kpad, a0.ptr, s));
      ++m->launches;
      if (f0.bn) {  // a batch-normalised stem has no bias: clear the patch rows' ones column
        const int kk = f0.k * f0.k * f0.cin_real;
        RALPB_TRY(cudaMemset2DAsync(a0.ptr + kk, static_cast<size_t>(f0.kpad) * sizeof(bf16), 0, sizeof(bf16),
                                    static_cast<size_t>(a0.rows()), s));
      }
    } else {
      RALPB_TRY(pack_input(img, b, m->in_h, m->in_w, m->in_c, a0.ptr, m->in_cp, a0.pad, s));
      ++m->launches;
    }
    bf16* cut_dst = m->acts[m->split].ptr;
    if (m->holds_back) cut_dst = m->xin + static_cast<size_t>(slot) * b * cut_row;
    if (launch_conv_forward(m, 0, m->split, img, nullptr, cut_dst, why)) return 1;
    cut_local = cut_dst;
  }
  RALPB_TRY(mark(m, 1, capturing));

  // ---------------- cut exchange + PS back segment
  const bf16* dcut = nullptr;
  if (m->mps) {
    if (mps_back_segment(m, lab, cut_local, lr, mu, &dcut, &fc_forked, why)) return 1;
  } else if (m->holds_back) {
    if (m->is_worker) {
      RALPB_TRY(cudaMemcpyAsync(m->labels_all + static_cast<size_t>(slot) * b, lab, sizeof(int32_t) * b,
                                cudaMemcpyDeviceToDevice, s));
      if (ralp) m->logical += cut_logical;   // "act": this colocated worker's cut, written in place
    }
    if (ralp && m->world > 1) {   // cuts arrive from peers (colocated W > 1, or a dedicated PS)
      if (m->is_worker) {
        PeerSignal own{};
        own.n = 1;
        own.flag[0] = m->flags + kFlagAct + m->widx;
        RALPB_TRY(signal_only(own, seq, s));
        ++m->launches;
      }
      RALPB_TRY(wait_flags(m->flags + kFlagAct, W, seq, s));
      ++m->launches;
    }
  } else {
    // a remote worker: push labels then the cut into the PS rank's rows, raise act_ready there.
    // With a dedicated PS the rows are free only once the PS has finished the previous step.
    if (m->dedicated_ps) {
      RALPB_TRY(wait_flags(m->flags + kFlagPsFree, 1, m->seq_dev - 1, s));
      ++m->launches;
    }
    int32_t* lab_ps = at<int32_t>(m, m->ps_rank, m->arena_off_lab) + static_cast<size_t>(slot) * b;
    bf16* x_ps = at<bf16>(m, m->ps_rank, m->arena_off_xfc) + static_cast<size_t>(slot) * b * cut_row;
    PeerSignal none{};
    RALPB_TRY(push_and_signal(lab_ps, lab, static_cast<long long>(b) * 4 / 16, none, seq, m->counters + 1, s));
    PeerSignal sig{};
    sig.n = 1;
    sig.flag[0] = at<uint32_t>(m, m->ps_rank, m->arena_off_flags) + kFlagAct + m->widx;
    RALPB_TRY(push_and_signal(x_ps, cut_local, static_cast<long long>(cut_bytes / 16), sig, seq, m->counters + 2, s));
    m->launches += 2;
    m->nvl_out += cut_bytes + sizeof(int32_t) * b;
    m->logical += cut_logical;   // "act" (simulator.py:677)
  }
  if (m->mps) {
    // the sharded FC tail ran in mps_back_segment
  } else if (m->holds_back) {
    const int R = m->rows_back;
    const bf16* in = m->x_fc;
    const float scale = 1.f / static_cast<float>(W * b);
    // conv back segment: layers [split, nconv) over every worker's cut rows, into the FC input
    if (m->bseg && launch_conv_forward(m, m->split, m->nconv, nullptr, &m->bin, m->x_fc, why)) return 1;
    if (pairs) {
      if (pair_fc_forward_loss(m, R, scale, why)) return 1;
    } else {
      if (launch_fc_forward(m, in, R, why)) return 1;
      const FcLayer& last = m->back.back();
      RALPB_TRY(softmax_xent(m->logits, R, last.out, last.ld_out, m->labels_all, scale, m->row_loss, m->dlogits, last.ld_out, s));
      // this rank's rows' share of the job's mean loss (RALP: all W*b rows are here)
      RALPB_TRY(reduce_sum(m->row_loss, R, scale, m->loss, s));
      m->launches += 2;
    }
    if (!ralp && push_loss_share(m, why)) return 1;
    if (pairs ? pair_fc_backward_data(m, R, m->dx_fc, why) : launch_fc_backward_data(m, in, R, m->dx_fc, why)) return 1;
    if (m->bseg) {
      // ... back through the conv back segment to the cut gradient rows (dxin), then its PS-local
      // SGD update (like the FC tail's, never synchronised) and the operand re-layout
      const long long nb = m->bseg_end - m->n_front;
      RALPB_TRY(cudaMemsetAsync(m->G + m->n_front, 0, nb * sizeof(float), s));
      if (launch_conv_backward(m, m->split, m->nconv, m->dx_fc, &m->bin, m->dxin, true, why)) return 1;
      RALPB_TRY(sgd_momentum(m->P + m->n_front, m->V + m->n_front, m->G + m->n_front, nb, lr, mu, 1.f, s));
      ++m->launches;
      if (prep_filters(m, true, true, s, why, m->split, m->nconv)) return 1;
    }
    if (ralp) {
      // return every remote worker's rows of the cut gradient first, then the FC tail's
      // weight gradients and its (PS-local, never synchronised) update run on the aux
      // stream, overlapping this rank's front backward
      // (one launch for all peers; RALPB_SCATTER_FUSED=0: one push launch per peer)
      m->logical += static_cast<long long>(W) * cut_logical;   // "actgrad" (simulator.py:707)
      const char* sf = getenv("RALPB_SCATTER_FUSED");
      if (sf != nullptr && sf[0] == '0') {
        for (int w = 0; w < W; ++w) {
          const int r = m->worker_ranks[w];
          if (r == m->rank) continue;
          PeerSignal sig{};
          sig.n = 1;
          sig.flag[0] = at<uint32_t>(m, r, m->arena_off_flags) + kFlagActGrad;
          RALPB_TRY(push_and_signal(at<bf16>(m, r, m->arena_off_dcut), m->dxin + static_cast<size_t>(w) * b * cut_row,
                                    static_cast<long long>(cut_bytes / 16), sig, seq, m->counters + kCtrScatter + w, s));
          ++m->launches;
          m->nvl_out += cut_bytes;
        }
      } else if (m->world > 1) {
        // on the comm stream: the 128-bit peer copies to the workers run concurrently with this
        // rank's FC weight gradients and front backward (RALPB_SCATTER_STREAM=0: in order)
        const char* ss = getenv("RALPB_SCATTER_STREAM");
        const bool own_stream = !(ss != nullptr && ss[0] == '0');
        cudaStream_t sx = own_stream ? m->comm_stream : s;
        if (own_stream) {
          RALPB_TRY(cudaEventRecord(m->ev_comm_fork, s));
          RALPB_TRY(cudaStreamWaitEvent(sx, m->ev_comm_fork, 0));
        }
        PeerScatter sc{};
        PeerSignal sig{};
        for (int w = 0; w < W; ++w) {
          const int r = m->worker_ranks[w];
          if (r == m->rank) continue;
          sc.dst[sc.n] = at<bf16>(m, r, m->arena_off_dcut);
          sc.src[sc.n] = m->dxin + static_cast<size_t>(w) * b * cut_row;
          ++sc.n;
          sig.flag[sig.n++] = at<uint32_t>(m, r, m->arena_off_flags) + kFlagActGrad;
          m->nvl_out += cut_bytes;
        }
        RALPB_TRY(scatter_and_signal(sc, static_cast<long long>(cut_bytes / 16), sig, seq, m->counters + kCtrScatter, sx));
        ++m->launches;
        if (own_stream) {
          RALPB_TRY(cudaEventRecord(m->ev_comm_join, sx));
          scatter_forked = true;
        }
      }
      // weight gradients on this stream (tensor/HBM work that would contend with the persistent
      // conv kernels), the HBM-bound update on the aux stream, overlapping the front backward
      // (RALPB_FC_OVERLAP=0: everything in order on one stream)
      const char* ov = getenv("RALPB_FC_OVERLAP");
      const bool overlap = !(ov != nullptr && ov[0] == '0') && m->is_worker && !pairs;
      cudaStream_t su = overlap ? m->aux_stream : s;
      if (pairs) {
        if (pair_fc_backward_weights(m, R, true, lr, mu, why)) return 1;
      } else if (launch_fc_backward_weights(m, in, R, true, lr, mu, s, su, why)) {
        return 1;
      }
      if (overlap) {
        RALPB_TRY(cudaEventRecord(m->ev_join, m->aux_stream));
        fc_forked = true;
      }
    } else {
      if (pairs ? pair_fc_backward_weights(m, R, false, lr, mu, why) : launch_fc_backward_weights(m, in, R, false, lr, mu, s, s, why))
        return 1;
    }
    if (m->is_worker) dcut = m->dxin + static_cast<size_t>(slot) * b * cut_row;
  } else {
    RALPB_TRY(wait_flags(m->flags + kFlagActGrad, 1, seq, s));
    ++m->launches;
    dcut = m->dcut;
  }
  RALPB_TRY(mark(m, 2, capturing));

  // the act-grad rows (dx_fc) are rewritten next step only after the sync; join the scatter here
  if (scatter_forked && !m->is_worker) RALPB_TRY(cudaStreamWaitEvent(s, m->ev_comm_join, 0));
  if (!m->is_worker) {
    // dedicated PS (RALP-N): its step ends with the FC tail's update; release the FC input rows
    // to the workers' next cut pushes
    PeerSignal free_rows{};
    for (int w = 0; w < W; ++w) free_rows.flag[free_rows.n++] = at<uint32_t>(m, m->worker_ranks[w], m->arena_off_flags) + kFlagPsFree;
    RALPB_TRY(signal_only(free_rows, seq, s));
    ++m->launches;
    RALPB_TRY(mark(m, 3, capturing));
    return 0;
  }

  // ---------------- worker front backward
  if (!pairs) RALPB_TRY(cudaStreamWaitEvent(s, m->ev_wd_join, 0));
  RALPB_TRY(cudaMemsetAsync(m->G, 0, m->n_front * sizeof(float), s));
  if (pairs ? pair_front_backward(m, dcut, why) : launch_front_backward(m, dcut, why)) return 1;
  RALPB_TRY(mark(m, 3, capturing));

  // ---------------- parameter synchronisation + re-layout
  // join the FC tail's update before this rank signals the sync: a worker can only start the
  // next step (and push its cut into x_fc, which the FC wgrads read) after that sync
  if (fc_forked) RALPB_TRY(cudaStreamWaitEvent(s, m->ev_join, 0));
  if (scatter_forked) RALPB_TRY(cudaStreamWaitEvent(s, m->ev_comm_join, 0));
  if (m->strategy == RALPB_STRATEGY_RING_EXTERNAL) {
    // the caller all-reduces G, then ralpb_model_apply; count the ring share here
    const long long sh = m->shard_real[m->widx];
    m->logical += 2LL * (W - 1) * sh * eb;
    return combine_loss(m, why);
  }
  const bool placed = ralp || m->mps;
  if (sync_params(m, placed ? m->n_front : m->n_total, lr, mu, why)) return 1;
  if (pairs ? pair_relayout(m, true, !placed, s, why) : relayout_weights(m, !placed, why)) return 1;
  if (!ralp && !m->mps && combine_loss(m, why)) return 1;
  return 0;
}

// The rank whose m->loss holds the job's mean loss: the PS (RALP; baseline / ring after
// combine_loss), rank 0 for the sharded FC tail.
bool reports_loss(const Model* m) { return m->mps ? m->rank == 0 : m->rank == m->ps_rank; }

bool graphs_enabled() {
  const char* e = getenv("RALPB_GRAPH");
  return e == nullptr || e[0] != '0';
}

}  // namespace

int model_step(Model* m, const void* images, const int32_t* labels, int on_host, float lr, float mu,
               std::string* why) {
  if (m->world > 1 && !m->peers_open) { *why = "ralpb_model_ipc_open has not been called"; return 1; }
  const int b = m->batch;
  cudaStream_t s = m->stream;
  if (m->is_worker && (images == nullptr || labels == nullptr)) { *why = "a worker rank needs images and labels"; return 1; }
  if (!m->is_worker) on_host = 0;   // the dedicated PS receives its rows from the workers
  m->seq += 1;
  const float* img = static_cast<const float*>(images);
  const int32_t* lab = labels;
  const int buf = static_cast<int>(m->seq & 1);
  if (on_host) {
    // copy stream: wait until step seq-2 (same staging buffer) consumed it, copy, signal
    cudaStream_t c = m->copy_stream;
    RALPB_TRY(cudaStreamWaitEvent(c, m->ev_consumed[buf], 0));
    RALPB_TRY(cudaMemcpyAsync(m->img_dev[buf], images, sizeof(float) * b * m->in_h * m->in_w * m->in_c,
                              cudaMemcpyHostToDevice, c));
    RALPB_TRY(cudaMemcpyAsync(m->lab_dev[buf], labels, sizeof(int32_t) * b, cudaMemcpyHostToDevice, c));
    RALPB_TRY(cudaEventRecord(m->ev_copied[buf], c));
    RALPB_TRY(cudaStreamWaitEvent(s, m->ev_copied[buf], 0));
    img = m->img_dev[buf];
    lab = m->lab_dev[buf];
  }
  RALPB_TRY(cudaEventRecord(m->ev[0], s));
  if (m->profiling || !graphs_enabled()) {
    m->launches = 0;
    m->nvl_out = m->nvl_in = m->logical = 0;
    m->timer.n = 0;
    set_gemm_timer(m->profiling ? &m->timer : nullptr);
    struct Reset { ~Reset() { set_gemm_timer(nullptr); } } reset_timer;
    if (step_body(m, img, lab, lr, mu, false, why)) return 1;
  } else {
    // captured step bodies, keyed by (inputs, hyper-parameters); two entries cover the
    // alternating staging buffers
    Model::GraphEntry* e = nullptr;
    for (auto& g : m->graphs)
      if (g.exec != nullptr && g.img == img && g.lab == lab && g.lr == lr && g.mu == mu) e = &g;
    if (e == nullptr) {
      e = &m->graphs[0];
      for (auto& g : m->graphs)
        if (g.exec == nullptr || g.used < e->used) e = &g;
      m->launches = 0;
      m->nvl_out = m->nvl_in = m->logical = 0;
      RALPB_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      const int rc = step_body(m, img, lab, lr, mu, true, why);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(s, &g);
      if (rc) { if (g) cudaGraphDestroy(g); return 1; }
      if (ce != cudaSuccess) { *why = std::string("step capture failed: ") + cudaGetErrorString(ce); return 1; }
      bool updated = false;
      if (e->exec != nullptr) {
        cudaGraphExecUpdateResultInfo info{};
        updated = cudaGraphExecUpdate(e->exec, g, &info) == cudaSuccess;
        if (!updated) {
          cudaGetLastError();
          cudaGraphExecDestroy(e->exec);
          e->exec = nullptr;
        }
      }
      cudaError_t ie = updated ? cudaSuccess : cudaGraphInstantiate(&e->exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) { *e = Model::GraphEntry{}; *why = std::string("graph instantiate failed: ") + cudaGetErrorString(ie); return 1; }
      e->img = img; e->lab = lab; e->lr = lr; e->mu = mu;
      e->launches = m->launches;
      e->nvl_out = m->nvl_out;
      e->nvl_in = m->nvl_in;
      e->logical = m->logical;
    }
    e->used = ++m->graph_clock;
    RALPB_TRY(cudaGraphLaunch(e->exec, s));
    m->launches = e->launches;
    m->nvl_out = e->nvl_out;
    m->nvl_in = e->nvl_in;
    m->logical = e->logical;
  }
  if (on_host) RALPB_TRY(cudaEventRecord(m->ev_consumed[buf], s));
  const int slot = static_cast<int>(m->seq % Model::kLossRing);
  if (reports_loss(m))
    RALPB_TRY(cudaMemcpyAsync(m->loss_host + slot, m->loss, sizeof(float), cudaMemcpyDeviceToHost, s));
  RALPB_TRY(cudaEventRecord(m->ev_loss[slot], s));
  m->loss_seq[slot] = m->seq;
  RALPB_TRY(cudaEventRecord(m->ev[4], s));
  m->stats_valid = true;
  return 0;
}

// Loss of the step issued `lag` steps ago (0 = the latest), waiting only for that step.
int model_read_loss(Model* m, int lag, float* out, std::string* why) {
  if (lag < 0 || lag >= Model::kLossRing || static_cast<uint32_t>(lag) >= m->seq) { *why = "no such step"; return 1; }
  const uint32_t want = m->seq - static_cast<uint32_t>(lag);
  const int slot = static_cast<int>(want % Model::kLossRing);
  if (m->loss_seq[slot] != want) { *why = "step no longer in the loss ring"; return 1; }
  RALPB_TRY(cudaEventSynchronize(m->ev_loss[slot]));
  *out = reports_loss(m) ? m->loss_host[slot] : NAN;
  return 0;
}

int model_stats(Model* m, ralpb_step_stats* st, std::string* why) {
  RALPB_TRY(cudaStreamSynchronize(m->stream));
  std::memset(st, 0, sizeof(*st));
  if (!m->stats_valid) { *why = "no step has run"; return 1; }
  float loss = NAN;
  if (reports_loss(m)) RALPB_TRY(cudaMemcpy(&loss, m->loss, sizeof(float), cudaMemcpyDeviceToHost));
  st->loss = loss;
  st->logical_bytes = m->logical;
  st->nvlink_out_bytes = m->nvl_out;
  st->nvlink_in_bytes = m->nvl_in;
  st->physical_bytes = m->nvl_out + m->nvl_in;
  st->launches = m->launches;
  cudaEventElapsedTime(&st->ms_step, m->ev[0], m->ev[4]);
  cudaEventElapsedTime(&st->ms_front_fwd, m->ev[0], m->ev[1]);
  cudaEventElapsedTime(&st->ms_back, m->ev[1], m->ev[2]);
  cudaEventElapsedTime(&st->ms_front_bwd, m->ev[2], m->ev[3]);
  cudaEventElapsedTime(&st->ms_sync, m->ev[3], m->ev[4]);
  st->gemm_launches = 0;
  st->ms_gemm = 0.f;
  for (int i = 0; m->profiling && i < m->timer.n; ++i) {
    if (m->timer.kind[i] > KIND_GEMM) continue;   // tensor-core launches only
    float ms = 0.f;
    cudaEventElapsedTime(&ms, m->timer.ev[2 * i], m->timer.ev[2 * i + 1]);
    st->ms_gemm += ms;
    ++st->gemm_launches;
  }
  return 0;
}

int model_grad_buffer(Model* m, float** ptr, long long* n, std::string* why) {
  if (m->strategy != RALPB_STRATEGY_RING_EXTERNAL) { *why = "only for RALPB_STRATEGY_RING_EXTERNAL"; return 1; }
  *ptr = m->G;
  *n = m->n_total;
  return 0;
}

// Update after the caller's gradient all-reduce (RING_EXTERNAL): SGD-momentum over every
// parameter, then the bf16 re-layouts the next step reads.
int model_apply(Model* m, float lr, float mu, std::string* why) {
  if (m->strategy != RALPB_STRATEGY_RING_EXTERNAL) { *why = "only for RALPB_STRATEGY_RING_EXTERNAL"; return 1; }
  RALPB_TRY(sgd_momentum(m->P, m->V, m->G, m->n_total, lr, mu, 1.f, m->stream));
  if (relayout_weights(m, true, why)) return 1;
  return 0;
}

// Per-launch records of the last profiled step (kind, CUDA-event time, algorithmic FLOPs).
int model_timed_launches(Model* m, ralpb_launch_rec* out, int cap, int* n, std::string* why) {
  RALPB_TRY(cudaStreamSynchronize(m->stream));
  *n = m->profiling ? m->timer.n : 0;
  for (int i = 0; i < *n && i < cap; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, m->timer.ev[2 * i], m->timer.ev[2 * i + 1]);
    out[i].kind = m->timer.kind[i];
    out[i].ms = ms;
    out[i].flops = m->timer.flops[i];
    out[i].bytes = m->timer.bytes[i];
    float t0 = 0.f;
    cudaEventElapsedTime(&t0, m->ev[0], m->timer.ev[2 * i]);
    out[i].t0 = t0;
    const cudaStream_t st = m->timer.stream[i];
    out[i].stream = st == m->stream ? 0 : st == m->aux_stream ? 1 : st == m->comm_stream ? 2 : st == m->sync_stream ? 3 : -1;
  }
  return 0;
}

int model_set_profiling(Model* m, int on, std::string* why) {
  if (on && m->timer.ev == nullptr) {
    m->timer.cap = 512;
    m->timer.ev = new cudaEvent_t[2 * m->timer.cap];
    m->timer.kind = new int[m->timer.cap];
    m->timer.flops = new double[m->timer.cap];
    m->timer.bytes = new double[m->timer.cap];
    m->timer.stream = new cudaStream_t[m->timer.cap];
    for (int i = 0; i < 2 * m->timer.cap; ++i) RALPB_TRY(cudaEventCreate(&m->timer.ev[i]));
  }
  m->profiling = on != 0;
  return 0;
}

}  // namespace ralpb
