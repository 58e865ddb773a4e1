// C ABI of the executor (ralpb_model_*), see include/ralpb.h.
#include <string>
#include "engine.cuh"
#include "status.cuh"

using namespace ralpb;

struct ralpb_model {
  Model* impl;
};

extern "C" {

int ralpb_model_create_graph(const ralpb_layer_desc* layers, int n_layers, const ralpb_node_desc* nodes,
                             int n_nodes, int split, int batch, int strategy, int rank, int world, int ps_rank,
                             int elem_bytes, int precision, int workers, ralpb_model** out) {
  std::string why;
  Model* m = nullptr;
  if (model_create(layers, n_layers, nodes, n_nodes, split, batch, strategy, rank, world, ps_rank, elem_bytes, precision,
                   workers, &m, &why))
    return set_error("ralpb_model_create: " + why);
  *out = new ralpb_model{m};
  return 0;
}

int ralpb_model_create(const ralpb_layer_desc* layers, int n_layers, int split, int batch, int strategy,
                       int rank, int world, int ps_rank, int elem_bytes, int precision, int workers,
                       ralpb_model** out) {
  return ralpb_model_create_graph(layers, n_layers, nullptr, 0, split, batch, strategy, rank, world, ps_rank, elem_bytes,
                                  precision, workers, out);
}

void ralpb_model_destroy(ralpb_model* m) {
  if (!m) return;
  model_destroy(m->impl);
  delete m;
}

int ralpb_model_ipc_handle(ralpb_model* m, void* out64) {
  std::string why;
  return model_ipc_handle(m->impl, out64, &why) ? set_error("ralpb_model_ipc_handle: " + why) : 0;
}

int ralpb_model_ipc_open(ralpb_model* m, const void* handles) {
  std::string why;
  return model_ipc_open(m->impl, handles, &why) ? set_error("ralpb_model_ipc_open: " + why) : 0;
}

int ralpb_model_set_params(ralpb_model* m, int layer, const float* w, const float* b, int on_host) {
  std::string why;
  return model_set_params(m->impl, layer, w, b, on_host, &why) ? set_error("ralpb_model_set_params: " + why) : 0;
}

int ralpb_model_get_params(ralpb_model* m, int layer, float* w, float* b, int on_host) {
  std::string why;
  return model_get_params(m->impl, layer, w, b, on_host, &why) ? set_error("ralpb_model_get_params: " + why) : 0;
}

int ralpb_model_get_grads(ralpb_model* m, int layer, float* w, float* b) {
  std::string why;
  return model_get_grads(m->impl, layer, w, b, &why) ? set_error("ralpb_model_get_grads: " + why) : 0;
}

int ralpb_model_step(ralpb_model* m, const void* images, const int32_t* labels, int on_host, float lr,
                     float mu) {
  std::string why;
  return model_step(m->impl, images, labels, on_host, lr, mu, &why) ? set_error("ralpb_model_step: " + why) : 0;
}

int ralpb_model_stats(ralpb_model* m, ralpb_step_stats* out) {
  std::string why;
  return model_stats(m->impl, out, &why) ? set_error("ralpb_model_stats: " + why) : 0;
}

int ralpb_model_timed_launches(ralpb_model* m, ralpb_launch_rec* out, int cap) {
  std::string why;
  int n = 0;
  if (model_timed_launches(m->impl, out, cap, &n, &why)) return set_error("ralpb_model_timed_launches: " + why);
  return n;
}

int ralpb_model_grad_buffer(ralpb_model* m, float** ptr, long long* n) {
  std::string why;
  return model_grad_buffer(m->impl, ptr, n, &why) ? set_error("ralpb_model_grad_buffer: " + why) : 0;
}

int ralpb_model_apply(ralpb_model* m, float lr, float mu) {
  std::string why;
  return model_apply(m->impl, lr, mu, &why) ? set_error("ralpb_model_apply: " + why) : 0;
}

int ralpb_model_read_loss(ralpb_model* m, int lag, float* out) {
  std::string why;
  return model_read_loss(m->impl, lag, out, &why) ? set_error("ralpb_model_read_loss: " + why) : 0;
}

void* ralpb_model_stream(ralpb_model* m) { return m->impl->stream; }

int ralpb_model_set_profiling(ralpb_model* m, int on) {
  std::string why;
  return model_set_profiling(m->impl, on, &why) ? set_error("ralpb_model_set_profiling: " + why) : 0;
}

}  // extern "C"

// Debug/inspection (include/ralpb.h): copy one of the step's device buffers to host memory;
// returns its element count (host_out may be NULL to query) or -1.
extern "C" long long ralpb_model_debug_buffer(ralpb_model* m, int i, int which, void* host_out) {
  Model* mm = m->impl;
  const void* src = nullptr;
  long long n = 0;
  size_t esz = sizeof(bf16);
  const int R = mm->rows_back;
  const int nb = static_cast<int>(mm->back.size());
  switch (which) {
    case RALPB_DBG_ACT:
    case RALPB_DBG_ACT_GRAD:
      if (i < 0 || i >= static_cast<int>(mm->acts.size())) return -1;
      n = mm->acts[i].elems();
      src = which == RALPB_DBG_ACT ? static_cast<const void*>(mm->acts[i].ptr) : static_cast<const void*>(mm->gacts[i]);
      break;
    case RALPB_DBG_LOGITS:
      n = static_cast<long long>(R) * mm->back.back().ld_out;
      src = mm->logits;
      esz = sizeof(float);
      break;
    case RALPB_DBG_FC_OUT:  // hidden FC output i (RALP_MPS, i = 0: this rank's slice)
      if (i < 0 || i + 1 >= nb) return -1;
      n = static_cast<long long>(R) * (mm->mps && i == 0 ? mm->ld_s0 : mm->back[i].ld_out);
      src = mm->mps && i == 0 ? static_cast<const void*>(mm->h0s) : static_cast<const void*>(mm->hid[i]);
      break;
    case RALPB_DBG_MPS_PARTIAL:
      if (!mm->mps) return -1;
      n = static_cast<long long>(R) * mm->back[1].ld_out;
      src = static_cast<const char*>(mm->arena) + mm->arena_off_p1;
      esz = sizeof(float);
      break;
    case RALPB_DBG_FC_WEIGHT:
      if (i < 0 || i >= nb) return -1;
      n = static_cast<long long>(mm->back[i].lout) * mm->back[i].lin;
      src = mm->back[i].wbf;
      break;
    case RALPB_DBG_DLOGITS:
      n = static_cast<long long>(R) * mm->back.back().ld_out;
      src = mm->dlogits;
      break;
    case RALPB_DBG_FC_OUT_GRAD:
      if (i < 0 || i + 1 >= nb) return -1;
      n = static_cast<long long>(R) * mm->back[i].ld_out;
      src = mm->dyb[i];
      break;
    case RALPB_DBG_CUT_ROWS:   // the exchanged cut rows (layer split-1's output, padded layout)
      n = static_cast<long long>(R) * mm->xch_elems;
      src = mm->xin;
      break;
    case RALPB_DBG_CUT_GRAD_ROWS:
      n = static_cast<long long>(R) * mm->xch_elems;
      src = mm->dxin;
      break;
    case RALPB_DBG_CUT_GRAD:
      n = static_cast<long long>(mm->batch) * mm->xch_elems;
      src = mm->dcut;
      break;
    case RALPB_DBG_FC_IN:      // the FC tail's input rows (== CUT_ROWS without a conv back segment)
      n = static_cast<long long>(R) * mm->cut_elems;
      src = mm->x_fc;
      break;
    case RALPB_DBG_FC_IN_GRAD:
      n = static_cast<long long>(R) * mm->cut_elems;
      src = mm->dx_fc;
      break;
    default:
      return -1;
  }
  if (src == nullptr) return -1;
  if (mm->precision == RALPB_PRECISION_FP32 && esz == sizeof(bf16)) esz *= mm->pieces;  // bf16 pieces
  if (host_out != nullptr) {
    if (cudaStreamSynchronize(mm->stream) != cudaSuccess) return -1;
    if (cudaMemcpy(host_out, src, n * esz, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  }
  return n;
}
