// C-ABI plumbing: thread-local error text, device identity (keys the schedule
// database like cpu_identifier, reference tuning.py:73-83), the conv
// dispatcher and whole-graph CUDA-graph capture.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "neo_common.cuh"

static thread_local char g_err[1024] = "";

void neo_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int neo_conv_tc_launch(const neo_conv_params* p, cudaStream_t stream);
int neo_conv_simt_launch(const neo_conv_params* p, cudaStream_t stream);

extern "C" {

const char* neo_last_error(void) { return g_err; }

// v2: neo_conv_params gained a leading struct_size (checked by every entry
// point that takes the struct); v3: NEO_MODE_FP8 / NEO_FP8 and the e4m3
// storage scales at the end of neo_conv_params
int neo_abi_version(void) { return 3; }

int neo_conv_params_size(void) { return (int)sizeof(neo_conv_params); }

int neo_device_info(int device, char* buf, int buflen) {
  NEO_CHECK_ARG(buf && buflen > 0, NEO_ERR_INVALID_ARG, "null buffer");
  cudaDeviceProp prop;
  NEO_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  snprintf(buf, buflen, "%s|%d|%d.%d|%zu", prop.name, prop.multiProcessorCount, prop.major,
           prop.minor, (size_t)prop.totalGlobalMem);
  return NEO_OK;
}

int neo_conv2d_nchwc_fused(const neo_conv_params* p, neo_stream_t stream) {
  NEO_CHECK_ARG(p != nullptr, NEO_ERR_INVALID_ARG, "null params");
  NEO_CHECK_ARG(p->struct_size == (int)sizeof(neo_conv_params), NEO_ERR_INVALID_ARG,
                "neo_conv_params.struct_size %d != %d (ABI v%d layout)", p->struct_size,
                (int)sizeof(neo_conv_params), neo_abi_version());
  NEO_CHECK_ARG(p->x && p->w && p->out, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(p->n >= 1 && p->c >= 1 && p->h >= 1 && p->w_in >= 1 && p->k >= 1 && p->r >= 1 &&
                    p->s >= 1,
                NEO_ERR_SHAPE_MISMATCH, "non-positive conv dimension");
  NEO_CHECK_ARG(p->stride_h >= 1 && p->stride_w >= 1 && p->pad_h >= 0 && p->pad_w >= 0,
                NEO_ERR_SHAPE_MISMATCH, "bad stride/pad");
  NEO_CHECK_ARG((p->h + 2 * p->pad_h - p->r) >= 0 && (p->w_in + 2 * p->pad_w - p->s) >= 0,
                NEO_ERR_SHAPE_MISMATCH, "conv has empty output");
  // ConvSchedule.check (kernels.py:56-63)
  NEO_CHECK_ARG(p->ic_bn >= 1 && p->oc_bn >= 1, NEO_ERR_SCHEDULE_INVALID,
                "non-positive factor ic_bn=%d oc_bn=%d", p->ic_bn, p->oc_bn);
  NEO_CHECK_ARG((p->flags & NEO_FLAG_PAD_CHANNELS) || p->c % p->ic_bn == 0,
                NEO_ERR_SCHEDULE_INVALID, "ic_bn=%d does not divide C=%lld", p->ic_bn,
                (long long)p->c);
  NEO_CHECK_ARG(p->k % p->oc_bn == 0, NEO_ERR_SCHEDULE_INVALID, "oc_bn=%d does not divide K=%lld",
                p->oc_bn, (long long)p->k);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (p->mode) {
    case NEO_MODE_FP32:
      NEO_CHECK_ARG(p->pro_scale == nullptr, NEO_ERR_UNSUPPORTED,
                    "the BN-ReLU prologue runs on the tensor-core path only");
      return neo_conv_simt_launch(p, st);
    case NEO_MODE_TF32:
    case NEO_MODE_BF16:
    case NEO_MODE_FP8: return neo_conv_tc_launch(p, st);
    default: neo_set_error("unknown conv mode %d", p->mode); return NEO_ERR_INVALID_ARG;
  }
}

int neo_capture_begin(neo_stream_t stream) {
  NEO_CUDA_TRY(cudaStreamBeginCapture(static_cast<cudaStream_t>(stream),
                                      cudaStreamCaptureModeThreadLocal));
  return NEO_OK;
}

int neo_capture_end(neo_stream_t stream, void** graph_exec) {
  NEO_CHECK_ARG(graph_exec != nullptr, NEO_ERR_INVALID_ARG, "null output");
  cudaGraph_t g = nullptr;
  NEO_CUDA_TRY(cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g));
  cudaGraphExec_t ge = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  NEO_CUDA_TRY(e);
  *graph_exec = ge;
  return NEO_OK;
}

int neo_graph_launch(void* graph_exec, neo_stream_t stream) {
  NEO_CHECK_ARG(graph_exec != nullptr, NEO_ERR_INVALID_ARG, "null graph");
  NEO_CUDA_TRY(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec),
                               static_cast<cudaStream_t>(stream)));
  return NEO_OK;
}

int neo_graph_destroy(void* graph_exec) {
  if (graph_exec) NEO_CUDA_TRY(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec)));
  return NEO_OK;
}

}  // extern "C"
