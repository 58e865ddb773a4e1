// C ABI of the executor (ralpb_model_*), see include/ralpb.h.
#include <string>
#include "engine.cuh"
#include "status.cuh"

using namespace ralpb;

struct ralpb_model {
  Model* impl;
};

extern "C" {

int ralpb_model_create(const ralpb_layer_desc* layers, int n_layers, int split, int batch, int strategy,
                       int rank, int world, int ps_rank, int elem_bytes, ralpb_model** out) {
  std::string why;
  Model* m = nullptr;
  if (model_create(layers, n_layers, split, batch, strategy, rank, world, ps_rank, elem_bytes, &m, &why))
    return set_error("ralpb_model_create: " + why);
  *out = new ralpb_model{m};
  return 0;
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

// Debug/inspection: copy activation buffer acts[i] (bf16, padded layout) or, for which=1,
// the activation-gradient buffer gacts[i], into host memory; returns the element count.
extern "C" long long ralpb_model_debug_buffer(ralpb_model* m, int i, int which, void* host_out) {
  Model* mm = m->impl;
  if (which == 2) {  // logits of the last step (fp32 [rows][ld], as bf16-sized count of floats)
    const long long n = static_cast<long long>(mm->rows_back) * mm->back.back().ld_out;
    if (host_out != nullptr) {
      cudaStreamSynchronize(mm->stream);
      if (cudaMemcpy(host_out, mm->logits, n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    }
    return n;
  }
  if (which == 6) {  // dlogits (bf16 [rows][ld])
    const long long n = static_cast<long long>(mm->rows_back) * mm->back.back().ld_out;
    if (host_out != nullptr) {
      cudaStreamSynchronize(mm->stream);
      if (cudaMemcpy(host_out, mm->dlogits, n * sizeof(bf16), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    }
    return n;
  }
  if (which == 4 && mm->mps) {  // RALP_MPS: this rank's arena partial slot 0 (fp32 [rows][ld1])
    const long long n = static_cast<long long>(mm->rows_back) * mm->back[1].ld_out;
    if (host_out != nullptr) {
      cudaStreamSynchronize(mm->stream);
      const char* src = static_cast<const char*>(mm->arena) + mm->arena_off_p1;
      if (cudaMemcpy(host_out, src, n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    }
    return n;
  }
  if (which == 5 && mm->back.size() > 1) {  // FC-1 bf16 weights as stored on this rank
    const FcLayer& f = mm->back[1];
    const long long n = static_cast<long long>(f.lout) * f.lin;
    if (host_out != nullptr) {
      cudaStreamSynchronize(mm->stream);
      if (cudaMemcpy(host_out, f.wbf, n * sizeof(bf16), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    }
    return n;
  }
  if (which == 3) {  // FC-0 output of the last step (bf16 [rows][ld]; RALP_MPS: this rank's slice)
    const long long n = static_cast<long long>(mm->rows_back) * (mm->mps ? mm->ld_s0 : mm->back[0].ld_out);
    if (host_out != nullptr) {
      cudaStreamSynchronize(mm->stream);
      if (cudaMemcpy(host_out, mm->mps ? mm->h0s : mm->hid[0], n * sizeof(bf16), cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    }
    return n;
  }
  if (i < 0 || i >= static_cast<int>(mm->acts.size())) return -1;
  const long long n = mm->acts[i].elems();
  const void* src = which == 0 ? static_cast<const void*>(mm->acts[i].ptr) : static_cast<const void*>(mm->gacts[i]);
  if (src == nullptr) return -1;
  if (host_out != nullptr) {
    cudaStreamSynchronize(mm->stream);
    if (cudaMemcpy(host_out, src, n * sizeof(bf16), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  }
  return n;
}
