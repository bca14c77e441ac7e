/*
 * clifford_b200.h -- C-ABI drop-in boundary for the B200 (sm_100a) Clifford
 * convolution / multivector activation / basic-block inference path.
 *
 * Plain pointers and sizes only: no torch or CUDA C++ types. `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/mvkernels/ unless stated):
 *
 *   cl_validate_signature  <- algebra.validate_signature          algebra.py:49-63
 *   cl_blade_product       <- algebra.blade_product                algebra.py:87-99
 *   cl_schedule_terms      <- len(specialize.schedule_for(sig))    specialize.py:49-74
 *   cl_expand_kernel       <- conv.build_expanded_kernel           conv.py:188-202
 *   cl_conv_create         <- conv.make_conv_layer                 conv.py:101-140
 *   cl_conv_forward        <- conv.conv_forward(x, layer, variant) conv.py:371-381
 *   cl_conv_forward_host   <- serve "forward" on a conv handle     serve.py:151-158
 *   cl_linear_create/forward <- linear.make_linear_layer / linear_forward  linear.py:32-102
 *   cl_act_create          <- activation.make_activation_config    activation.py:57-89
 *   cl_act_forward         <- activation.activation_forward + the
 *                             spatial fold of serve._forward       activation.py:400-416, serve.py:102-119
 *   cl_block_create/forward<- frontend/src/block.ts runBlock /
 *                             referenceBlockForward (conv->act->conv),
 *                             plus the residual of BASELINE configs 3/5   block.ts:134-148, :181-189
 *   cl_last_error          <- the "Type: message" error strings of serve.handle_request  serve.py:129-138
 *
 * Tensor layouts are the reference protocol layouts (layout.py:3-7):
 *   input (B, C_in, d_image^k, N_B), output (B, C_out, d_out^k, N_B),
 *   filters (N_B, C_in, C_out, d_filter^k), bias (N_B, C_out); activation
 *   input (B, C, N_B) or spatial (B, C, P, N_B). fp32, row-major, contiguous.
 *
 * Ownership: create() copies parameters into the handle (device memory);
 * caller owns input/output buffers; forward() is stream-ordered and
 * asynchronous; handles are immutable after create and may be used by
 * concurrent forwards on different streams.
 */
#ifndef CLIFFORD_B200_H
#define CLIFFORD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; names mirror the exception classes of errors.py:4-56. */
typedef enum {
  CL_OK = 0,
  CL_ERR_INVALID_SIGNATURE = 1,    /* InvalidSignature */
  CL_ERR_INVALID_METRIC_VALUE = 2, /* InvalidMetricValue */
  CL_ERR_DIMENSION_MISMATCH = 3,   /* DimensionMismatch */
  CL_ERR_SHAPE_MISMATCH = 4,       /* ShapeMismatch */
  CL_ERR_MODE_CONFIG_MISMATCH = 5, /* ModeConfigMismatch */
  CL_ERR_INDEX_OUT_OF_RANGE = 6,   /* IndexOutOfRange */
  CL_ERR_CONFIG_INVALID = 7,       /* ConfigInvalid */
  CL_ERR_CUDA = 8,                 /* CUDA runtime / driver failure */
  CL_ERR_UNSUPPORTED = 9           /* valid request outside what this build implements */
} cl_status;

/* Arithmetic mode of the tensor-core convolution. */
typedef enum {
  CL_PREC_FP32 = 0,   /* fp32-accurate: int8 digit slices, exact s32 accumulation
                         (max_rel_error <= 1e-4 vs the fp64 oracle) */
  CL_PREC_TF32 = 1,   /* single TF32 pass */
  CL_PREC_BF16 = 2,   /* BF16 operands, fp32 accumulate */
  CL_PREC_3XTF32 = 3  /* 3xTF32 split (hi/lo rounded to nearest tf32): the cross terms
                         accumulate in their own tensor-core accumulator, the hi*hi
                         accumulator is drained every 192 reduction elements into fp32
                         sums: fp32-accurate (max_rel_error <= 1e-4 at the BASELINE
                         configs, normwise ~1e-7) */
} cl_precision;

typedef enum { CL_PAD_VALID = 0, CL_PAD_SAME = 1 } cl_padding;

/* AggMode values are part of the reference FFI contract (activation.py:36-41). */
typedef enum { CL_AGG_LINEAR = 0, CL_AGG_SUM = 1, CL_AGG_MEAN = 2 } cl_agg_mode;

typedef struct cl_conv cl_conv;
typedef struct cl_conv cl_linear; /* a linear layer is a 1x1 conv over samples */
typedef struct cl_act cl_act;
typedef struct cl_block cl_block;

/* ---- algebra (host) ---------------------------------------------------- */
int cl_validate_signature(const int32_t* g, int k);
int cl_blade_product(int i_mask, int j_mask, const int32_t* g, int k, int* target, int* coeff);
/* number of surviving FMA terms of the signature schedule, or -status */
int cl_schedule_terms(const int32_t* g, int k);
/* change of basis used by the conv for this signature:
 * returns 1 and fills ncol, w and the 8x8 row-major transform T (x' = T x,
 * T T^T = 2 I) if the algebra is a full 2x2 matrix algebra, 0 if none, -status */
int cl_basis_info(const int32_t* g, int k, int* ncol, int* w, int8_t* T64);

/* ---- (1) on-device Clifford kernel construction ----------------------- */
/* Writes the (C_out*N_B, C_in*N_B, Q) real filter of conv.py:188-202 from
 * device filters (N_B, C_in, C_out, Q) into out_dev (device). */
int cl_expand_kernel(const int32_t* g, int k, const float* filters_dev, int C_in, int C_out,
                     int Q, float* out_dev, void* stream);

/* ---- (2) Clifford convolution ------------------------------------------ */
int cl_conv_create(const int32_t* g, int k, int C_in, int C_out, int d_image, int d_filter,
                   int padding, int precision, const float* filters_dev, const float* bias_dev,
                   void* stream, cl_conv** out);
/* FLOPs of one forward of B samples: the reference's algorithmic count
 * (conv_flops, conv.py:384-387) and the dense tensor-core GEMM actually
 * issued (half of the expanded one under a change of basis); basis = 1 if the
 * layer runs in a changed (matrix-algebra) basis */
int cl_conv_gemm_flops(const cl_conv* h, int64_t B, double* algorithmic, double* executed, int* basis);

/* Host-only planner query (no device memory, no GPU needed): the kernel
 * configuration cl_conv_create would choose. out[16] (int64): 0 basis_on,
 * 1 halo reuse, 2 2-SM pair MMA, 3 K steps per stage, 4 row groups per stage,
 * 5 filter taps per stage, 6 pipeline stages, 7 N tile, 8 N tiles, 9-11 tile
 * extent (x, y, z), 12 dynamic shared memory bytes, 13 TMA line elements per
 * pixel (0 = per-pixel lines), 14 epilogue basis class, 15 TMEM columns. */
int cl_conv_plan_info(const int32_t* g, int k, int C_in, int C_out, int d_image, int d_filter, int padding,
                      int precision, int64_t* out);
/* spatial output side d_out of the layer */
int cl_conv_out_side(const cl_conv* h, int* d_out);
/* x_dev (B, C_in, d_image^k, N_B) -> y_dev (B, C_out, d_out^k, N_B) */
int cl_conv_forward(const cl_conv* h, const float* x_dev, float* y_dev, int64_t B, void* stream);
/* explicit-workspace variant: ws (device) of >= cl_conv_workspace_bytes(h, B) bytes
 * (int8 digit planes of the input in fp32 mode, packed bf16 input in bf16 mode,
 * then 256 bytes for the tile scheduler's work counter; contents need not be
 * initialised, and concurrent calls need distinct workspaces).
 * cl_conv_forward uses a per-(handle, stream) cached workspace instead. */
size_t cl_conv_workspace_bytes(const cl_conv* h, int64_t B);
int cl_conv_forward_ws(const cl_conv* h, const float* x_dev, float* y_dev, int64_t B, void* ws,
                       size_t ws_bytes, void* stream);
/* diagnostics: prepares the operand once, then times `reps` launches of the
 * tensor-core conv kernel alone with CUDA events on `stream` */
int cl_conv_time_kernel(const cl_conv* h, const float* x_dev, float* y_dev, int64_t B, int reps,
                        void* stream, float* avg_ms);
/* host (pinned or pageable) buffers; copies in/out inside the call, chunked over the batch */
int cl_conv_forward_host(const cl_conv* h, const float* x_host, float* y_host, int64_t B,
                         void* stream);
void cl_conv_destroy(cl_conv* h);

/* ---- Clifford linear layer (linear.py:22-107) --------------- */
/* weight (N_B, C_out, C_in), bias (N_B, C_out); x (B, C_in, N_B) -> y (B, C_out, N_B) */
int cl_linear_create(const int32_t* g, int k, int C_in, int C_out, const float* weight, const float* bias,
                     int precision, void* stream, cl_linear** out);
int cl_linear_forward(const cl_linear* h, const float* x_dev, float* y_dev, int64_t B, void* stream);
int cl_linear_forward_host(const cl_linear* h, const float* x_host, float* y_host, int64_t B, void* stream);
void cl_linear_destroy(cl_linear* h);

/* ---- (3) multivector activation ---------------------------------------- */
int cl_act_create(const int32_t* g, int k, int mode, const int32_t* kernel_indices, int K, int C,
                  const float* weight_dev, const float* bias_dev, void* stream, cl_act** out);
/* x_dev (B, C, P, N_B) (P = 1 for the flat (B, C, N_B) form) -> y_dev, same shape */
int cl_act_forward(const cl_act* h, const float* x_dev, float* y_dev, int64_t B, int64_t P,
                   void* stream);
int cl_act_forward_host(const cl_act* h, const float* x_host, float* y_host, int64_t B, int64_t P,
                        void* stream);
/* pre-sigmoid gate s per (b, c, p) <- activation.gate_preactivation  activation.py:110-117
 * x_dev (B, C, P, N_B) -> s_dev (B, C, P); kernel blades in kernel_indices order */
int cl_act_preactivation(const cl_act* h, const float* x_dev, float* s_dev, int64_t B, int64_t P,
                         void* stream);
/* kernel blades of every multivector <- activation.gather_vpack  activation.py:99-107
 * x_dev (B, C, P, N_B) -> v_dev (B, C, P, K) */
int cl_act_gather(const cl_act* h, const float* x_dev, float* v_dev, int64_t B, int64_t P, void* stream);
/* K (number of kernel blades) of the handle, or -status */
int cl_act_kernel_count(const cl_act* h);
void cl_act_destroy(cl_act* h);

/* ---- (4) basic block: conv1 -> act -> conv2 [+ residual] ---------------- */
/* The activation is fused into conv1's epilogue and the residual into
 * conv2's; the block does not own the three layer handles. */
int cl_block_create(const cl_conv* conv1, const cl_act* act, const cl_conv* conv2, int residual,
                    cl_block** out);
int cl_block_forward(const cl_block* h, const float* x_dev, float* y_dev, int64_t B, void* stream);
size_t cl_block_workspace_bytes(const cl_block* h, int64_t B);
int cl_block_forward_ws(const cl_block* h, const float* x_dev, float* y_dev, int64_t B, void* ws,
                        size_t ws_bytes, void* stream);
/* host buffers, streamed through the GPU in chunks of `chunk` samples
 * (0 = automatic) with copy/compute overlap */
int cl_block_forward_host(const cl_block* h, const float* x_host, float* y_host, int64_t B,
                          int64_t chunk, void* stream);
/* diagnostics: one forward, then `reps` launches of the block's conv2 alone
 * (its fused residual included, on the operand the forward prepared), timed
 * with CUDA events on `stream`: the roofline kernel of bench.py */
int cl_block_time_conv2(const cl_block* h, const float* x_dev, float* y_dev, int64_t B, int reps, void* stream,
                        float* avg_ms);
void cl_block_destroy(cl_block* h);

/* ---- diagnostics --------------------------------------------------------- */
const char* cl_last_error(void); /* thread-local, "Type: message" */
uint64_t cl_launch_count(void);  /* kernels launched by this library so far */
const char* cl_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CLIFFORD_B200_H */
