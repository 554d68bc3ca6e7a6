// Launch recording for the batched decode step's CUDA-graph mode
// (pkv_decode_step_graph): while a recorder is installed on the calling
// thread, the step's device work (input copies, metadata copy, aux kernel,
// decode kernel, slot event) is appended to it instead of being issued; the
// graph module replays it as one cached CUDA graph.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <vector>

namespace pkv {

struct RecordedOp {
  enum Kind { kCopyH2D = 0, kKernel = 1, kEvent = 2 } kind;
  // kCopyH2D
  void* dst = nullptr;
  const void* src = nullptr;
  size_t bytes = 0;
  // kKernel
  const void* fn = nullptr;
  dim3 grid, block;
  unsigned smem = 0, cluster = 1;
  alignas(16) unsigned char args[1024];  // >= sizeof(TcParams) (static_assert in decode_tc.cu)
  size_t arg_off[16];
  int nargs = 0;
  size_t args_used = 0;
  // kEvent
  cudaEvent_t event = nullptr;
};

struct LaunchRecorder {
  std::vector<RecordedOp> ops;
};

// the calling thread's recorder (nullptr: launch directly)
LaunchRecorder*& launch_recorder();

// copies may stay outside the graph (issued at once, in order, on the
// step's stream); see graph_copies()
bool graph_copies();

inline void record_copy(void* dst, const void* src, size_t bytes) {
  RecordedOp op;
  op.kind = RecordedOp::kCopyH2D;
  op.dst = dst;
  op.src = src;
  op.bytes = bytes;
  launch_recorder()->ops.push_back(op);
}

inline void record_event(cudaEvent_t e) {
  RecordedOp op;
  op.kind = RecordedOp::kEvent;
  op.event = e;
  launch_recorder()->ops.push_back(op);
}

// arguments are converted to the kernel's parameter types and packed the way
// cudaKernelNodeParams::kernelParams expects (one pointer per parameter)
template <typename... P, typename... A>
void record_kernel(void (*fn)(P...), dim3 grid, dim3 block, unsigned smem, unsigned cluster, A... args) {
  static_assert(sizeof...(P) == sizeof...(A), "argument count");
  RecordedOp op;
  op.kind = RecordedOp::kKernel;
  op.fn = reinterpret_cast<const void*>(fn);
  op.grid = grid;
  op.block = block;
  op.smem = smem;
  op.cluster = cluster;
  auto push = [&](const auto& v) {
    const size_t al = alignof(std::decay_t<decltype(v)>);
    size_t off = (op.args_used + al - 1) / al * al;
    std::memcpy(op.args + off, &v, sizeof(v));
    op.arg_off[op.nargs++] = off;
    op.args_used = off + sizeof(v);
  };
  (push(static_cast<P>(args)), ...);
  launch_recorder()->ops.push_back(op);
}

}  // namespace pkv
