// NVLink peer-memory exchange kernels for the layer-placed step.
//
// One process per GPU; every rank maps its peers' exported arenas with CUDA IPC,
// so a peer buffer is a plain device pointer and these kernels move data with
// 128-bit loads/stores over NVLink.  Readiness is signalled with monotonically
// increasing 32-bit flags written with st.release.sys by the last CTA of the
// producing kernel and polled with ld.acquire.sys by a one-CTA wait kernel on
// the consumer's stream (the step sequence number is the flag value, so flags
// never need resetting).
//
// Reference schedule being executed (pkg/src/ralp/simulator.py:669-715):
//   worker: fwd front -> ship cut (count_wire act) -> wait act-grad -> bwd front
//           -> push grads (count_wire grad) -> wait pull
//   PS:     per arriving batch: back fwd+bwd, return act-grad; aggregate once; pull
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ralpb {

constexpr int kMaxRanks = 8;

struct PeerSignal {
  uint32_t* flag[kMaxRanks];  // flag words to set (possibly on peers); nullptr = skip
  int n;
};

struct PeerScatter {
  void* dst[kMaxRanks];
  const void* src[kMaxRanks];
  int n;
};

// dst[j] = src[j] (n16 chunks of 16 bytes each, j < sc.n) in one launch.  With sig.n == sc.n,
// sig.flag[j] is set to `value` as soon as destination j's bytes are globally visible (per-row
// last-CTA counters counter[0..sc.n)); otherwise every flag once all rows are.
cudaError_t scatter_and_signal(const PeerScatter& sc, long long n16, const PeerSignal& sig, const uint32_t* value,
                               uint32_t* counter, cudaStream_t s);

// dst = src (n16 chunks of 16 bytes), then set every flag in `sig` to `value`
// once all CTAs' stores are globally visible (system scope).  `counter` is a
// local zero-initialised word used for last-CTA detection.
cudaError_t push_and_signal(void* dst, const void* src, long long n16, const PeerSignal& sig,
                            const uint32_t* value, uint32_t* counter, cudaStream_t s);

// Set flags only (after a fence of this kernel's predecessors on the stream).
cudaError_t signal_only(const PeerSignal& sig, const uint32_t* value, cudaStream_t s);

// *counter += 1 (the per-step sequence number, first node of the step); counter[-1] = the new
// value - 1 (wait target for "the peer finished the previous step").
cudaError_t bump_counter(uint32_t* counter, cudaStream_t s);

// Flag values are read from device memory (`value` points at the rank's step counter) so a
// captured CUDA graph of the step replays correctly.
// Spin until flags[i] >= *value for i in [0, n).
cudaError_t wait_flags(const uint32_t* flags, int n, const uint32_t* value, cudaStream_t s);

// Sharded-PS aggregation over NVLink (reduce-scatter + SGD-momentum + all-gather):
// for i in this rank's shard [begin, end):
//   g = sum_r grads[r][i]; v[i] = mu*v[i] + gscale*g; p = params_local[i] - lr*v[i];
//   params[r][i] = p for every rank r
// then signals `done` flags.  grads/params are arrays of per-rank device pointers
// (peer pointers via IPC, local pointer for this rank).
constexpr int kMaxShardRanges = 32;
struct ShardUpdate {
  const float* grads[kMaxRanks];
  float* params[kMaxRanks];
  int nranks;
  int self;
  long long begin, end;  // float indices, multiples of 4
  int nr;                // > 0: the shard is these ranges instead (whole-layer shards), multiples of 4
  long long rb[kMaxShardRanges], re[kMaxShardRanges];
  float lr, mu, gscale;
  float* momentum;       // local, full-size vector (only the shard is touched)
};
cudaError_t shard_update(const ShardUpdate& u, const PeerSignal& done, const uint32_t* value,
                         uint32_t* counter, cudaStream_t s);

}  // namespace ralpb
