// Branch groups (RALPB_MODULE layers, graph.cu): Inception-v3 / GoogLeNet modules and single
// convolutions of any window, stride and padding, executed on the tcgen05 GEMM engine.
#pragma once
#include <string>
#include <utility>
#include <vector>
#include <vector>
#include "elementwise.cuh"
#include "engine.cuh"

namespace ralpb {

// Geometry, validation and parameter offsets of a module over `n` samples of [h][w][cin]:
// parameters are laid out from *off (aligned to 4 floats per tensor); appends the descriptor
// parameter runs (offset, floats) to runs and returns their total in *count.
int module_build(ModuleBufs& k, const ralpb_node_desc* nodes, int n_nodes, int n, int h, int w, int cin,
                 long long* off, std::vector<std::pair<long long, long long>>* runs, long long* count,
                 std::string* why);
int module_alloc(Model* m, ModuleBufs& k, std::string* why);
// casts: when given, the filter casts are appended (one batched launch by the caller)
int module_prep(Model* m, ModuleBufs& k, cudaStream_t s, std::string* why, std::vector<CastJob>* casts = nullptr);
// x [n][h][w][cin] -> y [n][ho][wo][cout] (unpadded NHWC)
int module_forward(Model* m, ModuleBufs& k, const __nv_bfloat16* x, __nv_bfloat16* y, std::string* why);
// dy w.r.t. y -> dx w.r.t. x (may be null); parameter gradients into G
int module_backward(Model* m, ModuleBufs& k, const __nv_bfloat16* x, const __nv_bfloat16* y,
                    const __nv_bfloat16* dy, __nv_bfloat16* dx, std::string* why);
// (offset, floats) of each conv node's filters and of its gamma|beta / bias, in node order
void module_param_runs(const ModuleBufs& k, std::vector<std::pair<long long, long long>>* w_runs,
                       std::vector<std::pair<long long, long long>>* b_runs);

}  // namespace ralpb
