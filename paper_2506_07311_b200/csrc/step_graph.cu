// CUDA-graph mode of the batched decode step (pkv_decode_step_graph).
//
// A serving loop calls the one-call step (pkv_decode_step, kernels.cu) every
// token with the same buffers.  Its device work is a short fixed chain: the
// input copies, the packed metadata copy, the page / mirror aux kernel (only
// on steps that grant pages) and the fused append + decode kernel.  Issued
// one by one that is three or four API calls on the critical path of every
// token.  Here the step runs with a launch recorder installed (step_graph.h):
// the host work is unchanged, the device work is recorded, and the chain is
// replayed as ONE cudaGraphLaunch.  Executable graphs are cached per
// topology (the sequence of copy endpoints / kernel functions / cluster
// sizes: in steady state one per metadata ring slot, with and without the
// aux kernel); a cached graph gets only the parameters that changed since
// its last launch (the metadata copy size, the aux kernel's arguments).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "pkv200.h"
#include "status.h"
#include "step_graph.h"

namespace pkv {

LaunchRecorder*& launch_recorder() {
  static thread_local LaunchRecorder* rec = nullptr;
  return rec;
}

bool graph_copies() {
  static const bool on = [] {
    const char* e = std::getenv("PKV_GRAPH_COPIES");
    return e && e[0] == '1';
  }();
  return on;
}

namespace {

struct RecorderScope {
  explicit RecorderScope(LaunchRecorder* r) { launch_recorder() = r; }
  ~RecorderScope() { launch_recorder() = nullptr; }
};

// node parameters of a recorded kernel (kernelParams point into op.args)
struct KernelNode {
  cudaKernelNodeParams p;
  void* argp[16];
  void fill(const RecordedOp& op) {
    for (int i = 0; i < op.nargs; ++i) argp[i] = const_cast<unsigned char*>(op.args) + op.arg_off[i];
    p = {};
    p.func = const_cast<void*>(op.fn);
    p.gridDim = op.grid;
    p.blockDim = op.block;
    p.sharedMemBytes = op.smem;
    p.kernelParams = argp;
    p.extra = nullptr;
  }
};

bool same_topology(const RecordedOp& a, const RecordedOp& b) {
  if (a.kind != b.kind) return false;
  if (a.kind == RecordedOp::kCopyH2D) return a.dst == b.dst && a.src == b.src;
  if (a.kind == RecordedOp::kKernel) return a.fn == b.fn && a.cluster == b.cluster && a.block.x == b.block.x;
  return a.event == b.event;
}

bool same_kernel_params(const RecordedOp& a, const RecordedOp& b) {
  return a.grid.x == b.grid.x && a.grid.y == b.grid.y && a.grid.z == b.grid.z && a.smem == b.smem &&
         a.args_used == b.args_used && std::memcmp(a.args, b.args, a.args_used) == 0;
}

struct GraphEntry {
  std::vector<RecordedOp> ops;  // parameters of the last launch
  std::vector<cudaGraphNode_t> nodes;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t last_use = 0;
  ~GraphEntry() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

// issue recorded ops directly on the stream (the steps that leave the graph
// path: a block-table shape change hands the launch back to the caller)
int replay_direct(const std::vector<RecordedOp>& ops, cudaStream_t stream) {
  for (const RecordedOp& op : ops) {
    cudaError_t e = cudaSuccess;
    if (op.kind == RecordedOp::kCopyH2D) {
      e = cudaMemcpyAsync(op.dst, op.src, op.bytes, cudaMemcpyHostToDevice, stream);
    } else if (op.kind == RecordedOp::kEvent) {
      e = cudaEventRecord(op.event, stream);
    } else {
      KernelNode kn;
      kn.fill(op);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = op.grid;
      cfg.blockDim = op.block;
      cfg.dynamicSmemBytes = op.smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = op.cluster;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = op.cluster > 1 ? 1 : 0;
      e = cudaLaunchKernelExC(&cfg, op.fn, kn.argp);
    }
    if (e != cudaSuccess) return fail(PKV_CUDA_ERROR, "decode step replay: %s", cuda_err_str(e));
  }
  return PKV_OK;
}

}  // namespace

struct StepGraphCache {
  std::mutex mu;
  std::vector<GraphEntry*> entries;
  uint64_t clock = 0;
  int64_t launches = 0, builds = 0;
  static constexpr size_t kMaxEntries = 16;
  ~StepGraphCache() {
    for (GraphEntry* g : entries) delete g;
  }

  // build and instantiate a linear-chain graph of the recorded ops (events
  // stay outside the graph: they are recorded after the launch)
  int build(const std::vector<RecordedOp>& ops, GraphEntry** out) {
    GraphEntry* g = new GraphEntry();
    cudaError_t e = cudaGraphCreate(&g->graph, 0);
    cudaGraphNode_t prev = nullptr;
    std::vector<KernelNode> kns(ops.size());
    for (size_t i = 0; i < ops.size() && e == cudaSuccess; ++i) {
      const RecordedOp& op = ops[i];
      cudaGraphNode_t node = nullptr;
      if (op.kind == RecordedOp::kCopyH2D) {
        e = cudaGraphAddMemcpyNode1D(&node, g->graph, prev ? &prev : nullptr, prev ? 1 : 0, op.dst, op.src,
                                     op.bytes, cudaMemcpyHostToDevice);
      } else if (op.kind == RecordedOp::kKernel) {
        kns[i].fill(op);
        e = cudaGraphAddKernelNode(&node, g->graph, prev ? &prev : nullptr, prev ? 1 : 0, &kns[i].p);
        if (e == cudaSuccess && op.cluster > 1) {
          cudaLaunchAttributeValue v = {};
          v.clusterDim.x = op.cluster;
          v.clusterDim.y = 1;
          v.clusterDim.z = 1;
          e = cudaGraphKernelNodeSetAttribute(node, cudaLaunchAttributeClusterDimension, &v);
        }
      } else {
        g->nodes.push_back(nullptr);
        continue;
      }
      g->nodes.push_back(node);
      prev = node;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) {
      delete g;
      return fail(PKV_CUDA_ERROR, "decode step graph build: %s", cuda_err_str(e));
    }
    g->ops = ops;
    ++builds;
    *out = g;
    return PKV_OK;
  }

  int launch(const std::vector<RecordedOp>& ops, cudaStream_t stream) {
    std::lock_guard<std::mutex> lock(mu);
    GraphEntry* hit = nullptr;
    for (GraphEntry* g : entries) {
      if (g->ops.size() != ops.size()) continue;
      bool same = true;
      for (size_t i = 0; i < ops.size() && same; ++i) same = same_topology(g->ops[i], ops[i]);
      if (same) {
        hit = g;
        break;
      }
    }
    if (!hit) {
      const int st = build(ops, &hit);
      if (st) return st;
      if (entries.size() >= kMaxEntries) {  // evict the least recently used
        auto lru = std::min_element(entries.begin(), entries.end(),
                                    [](GraphEntry* a, GraphEntry* b) { return a->last_use < b->last_use; });
        delete *lru;
        entries.erase(lru);
      }
      entries.push_back(hit);
    } else {
      // bring the cached graph's parameters up to date (only what changed)
      for (size_t i = 0; i < ops.size(); ++i) {
        const RecordedOp& op = ops[i];
        RecordedOp& old = hit->ops[i];
        cudaError_t e = cudaSuccess;
        if (op.kind == RecordedOp::kCopyH2D && op.bytes != old.bytes) {
          e = cudaGraphExecMemcpyNodeSetParams1D(hit->exec, hit->nodes[i], op.dst, op.src, op.bytes,
                                                  cudaMemcpyHostToDevice);
        } else if (op.kind == RecordedOp::kKernel && !same_kernel_params(op, old)) {
          KernelNode kn;
          kn.fill(op);
          e = cudaGraphExecKernelNodeSetParams(hit->exec, hit->nodes[i], &kn.p);
        }
        if (e != cudaSuccess) return fail(PKV_CUDA_ERROR, "decode step graph update: %s", cuda_err_str(e));
        old = op;
      }
    }
    hit->last_use = ++clock;
    cudaError_t e = cudaGraphLaunch(hit->exec, stream);
    if (e != cudaSuccess) return fail(PKV_CUDA_ERROR, "decode step graph launch: %s", cuda_err_str(e));
    for (const RecordedOp& op : ops)
      if (op.kind == RecordedOp::kEvent) {
        e = cudaEventRecord(op.event, stream);
        if (e != cudaSuccess) return fail(PKV_CUDA_ERROR, "decode step slot event: %s", cuda_err_str(e));
      }
    ++launches;
    return PKV_OK;
  }
};

}  // namespace pkv

using pkv::StepGraphCache;

extern "C" {

int pkv_step_graph_create(pkv_step_graph** out) {
  if (!out) return pkv::fail(PKV_VALUE_ERROR, "null output");
  *out = reinterpret_cast<pkv_step_graph*>(new StepGraphCache());
  return PKV_OK;
}

void pkv_step_graph_destroy(pkv_step_graph* g) { delete reinterpret_cast<StepGraphCache*>(g); }

int pkv_step_graph_stats(pkv_step_graph* g, int64_t* launches, int64_t* builds) {
  if (!g) return pkv::fail(PKV_VALUE_ERROR, "null graph cache");
  auto* c = reinterpret_cast<StepGraphCache*>(g);
  std::lock_guard<std::mutex> lock(c->mu);
  if (launches) *launches = c->launches;
  if (builds) *builds = c->builds;
  return PKV_OK;
}

int pkv_decode_step_graph(pkv_step_graph* g, pkv_step_stage_args* stage, pkv_attention_args* attn,
                          pkv_decode_io* io, void* stream_) {
  if (!g) return pkv::fail(PKV_VALUE_ERROR, "null graph cache");
  if (!stage || !attn) return pkv::fail(PKV_VALUE_ERROR, "null args");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  // graph mode covers the tensor-core path without a trailing copy; anything
  // else is the ordinary one-call step
  const bool tensor = attn->mode == 2 || (attn->mode == 0 && attn->kv_dtype == PKV_BF16);
  if (!tensor || (io && io->out_host) || attn->prof_start || attn->prof_stop)
    return pkv_decode_step(stage, attn, io, stream_);
  pkv::DeviceGuard guard(stream);
  pkv::LaunchRecorder rec;
  int st;
  {
    pkv::RecorderScope scope(&rec);
    st = pkv_decode_step(stage, attn, io, stream_);
  }
  if (st) return st;  // the step rolled the allocator back; nothing was issued
  if (stage->needs_resync) return pkv::replay_direct(rec.ops, stream);  // the caller launches (mirror re-export)
  return reinterpret_cast<StepGraphCache*>(g)->launch(rec.ops, stream);
}

}  // extern "C"
