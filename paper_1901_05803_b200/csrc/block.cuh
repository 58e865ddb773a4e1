// ResNet bottleneck blocks and the batch-normalised stem (block.cu), used by the executor for the
// RALPB_BLOCK layers and bn convolutions of a branchy model.
#pragma once
#include <string>
#include <vector>
#include "elementwise.cuh"
#include "engine.cuh"

namespace ralpb {

int block_alloc(Model* m, BlockBufs& k, std::string* why);
// RALPB_RES_EPI=1: a gradient summed into another in the dgrad GEMM's epilogue (GemmDesc::residual)
// instead of a separate add pass -- measured slower (the narrow-K 1x1 dgrad GEMMs are epilogue-
// bound: ResNet-50 15.80 vs 15.66 ms, Inception-v3 34.6 vs 34.2 ms, GoogLeNet 9.93 vs 9.67 ms)
bool res_epilogue();
// casts / preps: when given, the operand copies are appended for the caller's batched launches
int block_prep(Model* m, BlockBufs& k, cudaStream_t s, std::string* why, std::vector<CastJob>* casts = nullptr,
               std::vector<WeightPrepJob>* preps = nullptr);
// x [n][h][w][cin] -> y [n][ho][wo][cout] (unpadded NHWC)
int block_forward(Model* m, BlockBufs& k, const __nv_bfloat16* x, __nv_bfloat16* y, std::string* why);
// dy w.r.t. y -> dx w.r.t. x (dx may be null: no input gradient); parameter gradients into G
int block_backward(Model* m, BlockBufs& k, const __nv_bfloat16* x, const __nv_bfloat16* y, const __nv_bfloat16* dy,
                   __nv_bfloat16* dx, std::string* why);
int bn_stem_forward(Model* m, FrontLayer& f, const ActBuf& in, const ActBuf& out, std::string* why);
int bn_stem_backward(Model* m, FrontLayer& f, const ActBuf& in, const ActBuf& out, const __nv_bfloat16* dy,
                     std::string* why);

}  // namespace ralpb
