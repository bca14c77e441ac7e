// clifford_ops.cpp -- the C-ABI of include/clifford_b200.h registered as
// PyTorch operators (torch.ops.clifford_b200.*). This is the binding the
// Python layer uses (it replaces the paper's ctypes bindings):
// tensors in, the current CUDA stream of the tensor's device, C-ABI status
// codes turned into errors whose message starts "clifford_b200[<status>] ",
// from which the Python shim re-raises the reference's exception classes
// (errors.py:4-56).
//
// The library is dlopen'ed by `load_library(path)` (the production build, or
// the diagnostic A/B build selected with CL_LIB_PATH), so this extension has
// no link-time dependency on a particular libclifford_b200 build.
//
// Handles (layer, activation, block) travel as int64 (the C pointer).
#include <dlfcn.h>

#include <ATen/ATen.h>
#include <c10/cuda/CUDAGuard.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/library.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace {

// ---- the C-ABI, resolved from the loaded library --------------------------
struct Api {
  int (*validate_signature)(const int32_t*, int);
  int (*blade_product)(int, int, const int32_t*, int, int*, int*);
  int (*schedule_terms)(const int32_t*, int);
  int (*basis_info)(const int32_t*, int, int*, int*, int8_t*);
  int (*expand_kernel)(const int32_t*, int, const float*, int, int, int, float*, void*);
  int (*conv_create)(const int32_t*, int, int, int, int, int, int, int, const float*, const float*, void*, void**);
  int (*conv_gemm_flops)(const void*, int64_t, double*, double*, int*);
  int (*conv_plan_info)(const int32_t*, int, int, int, int, int, int, int, int64_t*);
  int (*conv_out_side)(const void*, int*);
  int (*conv_forward)(const void*, const float*, float*, int64_t, void*);
  int (*conv_forward_host)(const void*, const float*, float*, int64_t, void*);
  int (*conv_time_kernel)(const void*, const float*, float*, int64_t, int, void*, float*);
  void (*conv_destroy)(void*);
  int (*linear_create)(const int32_t*, int, int, int, const float*, const float*, int, void*, void**);
  int (*act_create)(const int32_t*, int, int, const int32_t*, int, int, const float*, const float*, void*, void**);
  int (*act_forward)(const void*, const float*, float*, int64_t, int64_t, void*);
  int (*act_forward_host)(const void*, const float*, float*, int64_t, int64_t, void*);
  int (*act_preactivation)(const void*, const float*, float*, int64_t, int64_t, void*);
  int (*act_gather)(const void*, const float*, float*, int64_t, int64_t, void*);
  void (*act_destroy)(void*);
  int (*block_create)(const void*, const void*, const void*, int, void**);
  int (*block_forward)(const void*, const float*, float*, int64_t, void*);
  int (*block_forward_host)(const void*, const float*, float*, int64_t, int64_t, void*);
  void (*block_destroy)(void*);
  int (*block_time_conv2)(const void*, const float*, float*, int64_t, int, void*, float*);
  const char* (*last_error)();
  uint64_t (*launch_count)();
  const char* (*version)();
};

Api g_api{};
void* g_handle = nullptr;
std::string g_path;
std::mutex g_m;

template <class F>
bool bind(void* lib, F& fn, const char* name, std::string& missing) {
  void* p = dlsym(lib, name);
  if (!p) missing += std::string(missing.empty() ? "" : ", ") + name;
  fn = reinterpret_cast<F>(p);
  return p != nullptr;
}

const Api& api() {
  TORCH_CHECK(g_handle != nullptr, "clifford_b200[7] ConfigInvalid: libclifford_b200 not loaded "
                                   "(torch.ops.clifford_b200.load_library)");
  return g_api;
}

void check(int st) {
  if (st == 0) return;
  const int code = st < 0 ? -st : st;
  const std::string msg = api().last_error();  // the C-ABI's thread-local "Type: message"
  TORCH_CHECK(false, "clifford_b200[", code, "] ", msg);
}

std::string load_library(std::string path) {
  std::lock_guard<std::mutex> lk(g_m);
  if (g_handle) {
    TORCH_CHECK(path == g_path, "clifford_b200[7] ConfigInvalid: ", g_path, " already loaded, cannot switch to ", path);
    return g_api.version();
  }
  void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
  TORCH_CHECK(h != nullptr, "clifford_b200[7] ConfigInvalid: dlopen(", path, ") failed: ", dlerror());
  Api a{};
  std::string miss;
  bind(h, a.validate_signature, "cl_validate_signature", miss);
  bind(h, a.blade_product, "cl_blade_product", miss);
  bind(h, a.schedule_terms, "cl_schedule_terms", miss);
  bind(h, a.basis_info, "cl_basis_info", miss);
  bind(h, a.expand_kernel, "cl_expand_kernel", miss);
  bind(h, a.conv_create, "cl_conv_create", miss);
  bind(h, a.conv_gemm_flops, "cl_conv_gemm_flops", miss);
  bind(h, a.conv_plan_info, "cl_conv_plan_info", miss);
  bind(h, a.conv_out_side, "cl_conv_out_side", miss);
  bind(h, a.conv_forward, "cl_conv_forward", miss);
  bind(h, a.conv_forward_host, "cl_conv_forward_host", miss);
  bind(h, a.conv_time_kernel, "cl_conv_time_kernel", miss);
  bind(h, a.conv_destroy, "cl_conv_destroy", miss);
  bind(h, a.linear_create, "cl_linear_create", miss);
  bind(h, a.act_create, "cl_act_create", miss);
  bind(h, a.act_forward, "cl_act_forward", miss);
  bind(h, a.act_forward_host, "cl_act_forward_host", miss);
  bind(h, a.act_preactivation, "cl_act_preactivation", miss);
  bind(h, a.act_gather, "cl_act_gather", miss);
  bind(h, a.act_destroy, "cl_act_destroy", miss);
  bind(h, a.block_create, "cl_block_create", miss);
  bind(h, a.block_forward, "cl_block_forward", miss);
  bind(h, a.block_forward_host, "cl_block_forward_host", miss);
  bind(h, a.block_destroy, "cl_block_destroy", miss);
  bind(h, a.block_time_conv2, "cl_block_time_conv2", miss);
  bind(h, a.last_error, "cl_last_error", miss);
  bind(h, a.launch_count, "cl_launch_count", miss);
  bind(h, a.version, "cl_version", miss);
  if (!miss.empty()) {
    dlclose(h);
    TORCH_CHECK(false, "clifford_b200[7] ConfigInvalid: ", path, " lacks ", miss, " (stale build?)");
  }
  g_api = a;
  g_handle = h;
  g_path = path;
  return g_api.version();
}

std::string loaded_library() { return g_path; }

// ---- helpers -----------------------------------------------------------------
std::vector<int32_t> sig_of(const c10::IntArrayRef g) {
  std::vector<int32_t> v(g.begin(), g.end());
  if (v.empty()) v.push_back(0);
  return v;
}

void* stream_of(const at::Tensor& t) {
  return reinterpret_cast<void*>(c10::cuda::getCurrentCUDAStream(t.device().index()).stream());
}

void* current_stream() { return reinterpret_cast<void*>(c10::cuda::getCurrentCUDAStream().stream()); }

const float* fptr(const at::Tensor& t) { return t.numel() ? t.data_ptr<float>() : nullptr; }
float* fptr_mut(const at::Tensor& t) { return t.numel() ? t.data_ptr<float>() : nullptr; }

// device tensors: fp32, contiguous, on a CUDA device (the shape contract is the C-ABI's)
void dev_f32(const at::Tensor& t, const char* what) {
  TORCH_CHECK(t.is_cuda(), "clifford_b200[4] ShapeMismatch: ", what, " must be a CUDA tensor");
  TORCH_CHECK(t.scalar_type() == at::kFloat && t.is_contiguous(),
              "clifford_b200[4] ShapeMismatch: ", what, " must be contiguous float32");
}
void host_f32(const at::Tensor& t, const char* what) {
  TORCH_CHECK(!t.is_cuda(), "clifford_b200[4] ShapeMismatch: ", what, " must be a host (CPU) tensor");
  TORCH_CHECK(t.scalar_type() == at::kFloat && t.is_contiguous(),
              "clifford_b200[4] ShapeMismatch: ", what, " must be contiguous float32");
}
const void* H(int64_t h) { return reinterpret_cast<const void*>(static_cast<intptr_t>(h)); }
void* Hm(int64_t h) { return reinterpret_cast<void*>(static_cast<intptr_t>(h)); }

// ---- algebra -----------------------------------------------------------------
int64_t validate_signature(c10::IntArrayRef g) {
  auto v = sig_of(g);
  check(api().validate_signature(v.data(), (int)g.size()));
  return 0;
}

std::vector<int64_t> blade_product(int64_t i, int64_t j, c10::IntArrayRef g) {
  auto v = sig_of(g);
  int t = 0, c = 0;
  check(api().blade_product((int)i, (int)j, v.data(), (int)g.size(), &t, &c));
  return {t, c};
}

int64_t schedule_terms(c10::IntArrayRef g) {
  auto v = sig_of(g);
  const int n = api().schedule_terms(v.data(), (int)g.size());
  check(n < 0 ? n : 0);
  return n;
}

std::vector<int64_t> basis_info(c10::IntArrayRef g) {
  auto v = sig_of(g);
  int ncol = 0, w = 0;
  int8_t T[64] = {0};
  const int r = api().basis_info(v.data(), (int)g.size(), &ncol, &w, T);
  check(r < 0 ? r : 0);
  std::vector<int64_t> out = {r, ncol, w};
  for (int a = 0; a < 64; ++a) out.push_back(T[a]);
  return out;
}

void expand_kernel(c10::IntArrayRef g, const at::Tensor& filters, int64_t C_in, int64_t C_out, int64_t Q,
                   const at::Tensor& out) {
  dev_f32(filters, "filters");
  dev_f32(out, "out");
  TORCH_CHECK(out.numel() == (int64_t)C_out * C_in * Q * (1 << g.size()) * (1 << g.size()),
              "clifford_b200[4] ShapeMismatch: expanded kernel output has the wrong size");
  c10::cuda::CUDAGuard guard(filters.device());
  auto v = sig_of(g);
  check(api().expand_kernel(v.data(), (int)g.size(), fptr(filters), (int)C_in, (int)C_out, (int)Q, fptr_mut(out),
                            stream_of(filters)));
}

// ---- conv / linear -----------------------------------------------------------
int64_t conv_create(c10::IntArrayRef g, int64_t C_in, int64_t C_out, int64_t d_image, int64_t d_filter,
                    int64_t padding, int64_t precision, const at::Tensor& filters, const at::Tensor& bias) {
  dev_f32(filters, "filters");
  dev_f32(bias, "bias");
  c10::cuda::CUDAGuard guard(filters.device());
  auto v = sig_of(g);
  void* h = nullptr;
  check(api().conv_create(v.data(), (int)g.size(), (int)C_in, (int)C_out, (int)d_image, (int)d_filter, (int)padding,
                          (int)precision, fptr(filters), fptr(bias), stream_of(filters), &h));
  return static_cast<int64_t>(reinterpret_cast<intptr_t>(h));
}

int64_t linear_create(c10::IntArrayRef g, int64_t C_in, int64_t C_out, const at::Tensor& weight,
                      const at::Tensor& bias, int64_t precision) {
  // weight / bias: host or device (the C-ABI copies them with cudaMemcpyDefault)
  TORCH_CHECK(weight.scalar_type() == at::kFloat && weight.is_contiguous() && bias.scalar_type() == at::kFloat &&
                  bias.is_contiguous(),
              "clifford_b200[4] ShapeMismatch: weight / bias must be contiguous float32");
  auto v = sig_of(g);
  void* h = nullptr;
  check(api().linear_create(v.data(), (int)g.size(), (int)C_in, (int)C_out, fptr(weight), fptr(bias),
                            (int)precision, current_stream(), &h));
  return static_cast<int64_t>(reinterpret_cast<intptr_t>(h));
}

void conv_destroy(int64_t h) { api().conv_destroy(Hm(h)); }

void conv_forward(int64_t h, const at::Tensor& x, int64_t B, const at::Tensor& y) {
  dev_f32(x, "input");
  dev_f32(y, "out");
  c10::cuda::CUDAGuard guard(x.device());
  check(api().conv_forward(H(h), fptr(x), fptr_mut(y), B, stream_of(x)));
}

void conv_forward_host(int64_t h, const at::Tensor& x, int64_t B, const at::Tensor& y) {
  host_f32(x, "input");
  host_f32(y, "out");
  check(api().conv_forward_host(H(h), fptr(x), fptr_mut(y), B, current_stream()));
}

std::vector<double> conv_gemm_flops(int64_t h, int64_t B) {
  double a = 0, e = 0;
  int basis = 0;
  check(api().conv_gemm_flops(H(h), B, &a, &e, &basis));
  return {a, e, (double)basis};
}

std::vector<int64_t> conv_plan_info(c10::IntArrayRef g, int64_t C_in, int64_t C_out, int64_t d_image,
                                    int64_t d_filter, int64_t padding, int64_t precision) {
  auto v = sig_of(g);
  std::vector<int64_t> out(16, 0);
  check(api().conv_plan_info(v.data(), (int)g.size(), (int)C_in, (int)C_out, (int)d_image, (int)d_filter,
                             (int)padding, (int)precision, out.data()));
  return out;
}

int64_t conv_out_side(int64_t h) {
  int d = 0;
  check(api().conv_out_side(H(h), &d));
  return d;
}

double conv_time_kernel(int64_t h, const at::Tensor& x, int64_t B, int64_t reps, const at::Tensor& y) {
  dev_f32(x, "input");
  dev_f32(y, "out");
  c10::cuda::CUDAGuard guard(x.device());
  float ms = 0.f;
  check(api().conv_time_kernel(H(h), fptr(x), fptr_mut(y), B, (int)reps, stream_of(x), &ms));
  return ms;
}

// ---- activation --------------------------------------------------------------
int64_t act_create(c10::IntArrayRef g, int64_t mode, c10::IntArrayRef ki, int64_t C,
                   const std::optional<at::Tensor>& weight, const std::optional<at::Tensor>& bias) {
  auto v = sig_of(g);
  std::vector<int32_t> k(ki.begin(), ki.end());
  if (k.empty()) k.push_back(-1);
  const float* w = nullptr;
  const float* b = nullptr;
  if (weight.has_value()) {
    TORCH_CHECK(weight->scalar_type() == at::kFloat && weight->is_contiguous(),
                "clifford_b200[4] ShapeMismatch: weight must be contiguous float32");
    w = fptr(*weight);
  }
  if (bias.has_value()) {
    TORCH_CHECK(bias->scalar_type() == at::kFloat && bias->is_contiguous(),
                "clifford_b200[4] ShapeMismatch: bias must be contiguous float32");
    b = fptr(*bias);
  }
  void* h = nullptr;
  check(api().act_create(v.data(), (int)g.size(), (int)mode, k.data(), (int)ki.size(), (int)C, w, b,
                         current_stream(), &h));
  return static_cast<int64_t>(reinterpret_cast<intptr_t>(h));
}

void act_destroy(int64_t h) { api().act_destroy(Hm(h)); }

void act_forward(int64_t h, const at::Tensor& x, int64_t B, int64_t P, const at::Tensor& y) {
  dev_f32(x, "input");
  dev_f32(y, "out");
  c10::cuda::CUDAGuard guard(x.device());
  check(api().act_forward(H(h), fptr(x), fptr_mut(y), B, P, stream_of(x)));
}

void act_forward_host(int64_t h, const at::Tensor& x, int64_t B, int64_t P, const at::Tensor& y) {
  host_f32(x, "input");
  host_f32(y, "out");
  check(api().act_forward_host(H(h), fptr(x), fptr_mut(y), B, P, current_stream()));
}

void act_preactivation(int64_t h, const at::Tensor& x, int64_t B, int64_t P, const at::Tensor& s) {
  dev_f32(x, "input");
  dev_f32(s, "out");
  c10::cuda::CUDAGuard guard(x.device());
  check(api().act_preactivation(H(h), fptr(x), fptr_mut(s), B, P, stream_of(x)));
}

void act_gather(int64_t h, const at::Tensor& x, int64_t B, int64_t P, const at::Tensor& v) {
  dev_f32(x, "input");
  dev_f32(v, "out");
  c10::cuda::CUDAGuard guard(x.device());
  check(api().act_gather(H(h), fptr(x), fptr_mut(v), B, P, stream_of(x)));
}

// ---- block -------------------------------------------------------------------
int64_t block_create(int64_t c1, int64_t act, int64_t c2, bool residual) {
  void* h = nullptr;
  check(api().block_create(H(c1), H(act), H(c2), residual ? 1 : 0, &h));
  return static_cast<int64_t>(reinterpret_cast<intptr_t>(h));
}

void block_destroy(int64_t h) { api().block_destroy(Hm(h)); }

void block_forward(int64_t h, const at::Tensor& x, int64_t B, const at::Tensor& y) {
  dev_f32(x, "input");
  dev_f32(y, "out");
  c10::cuda::CUDAGuard guard(x.device());
  check(api().block_forward(H(h), fptr(x), fptr_mut(y), B, stream_of(x)));
}

void block_forward_host(int64_t h, const at::Tensor& x, int64_t B, int64_t chunk, const at::Tensor& y) {
  host_f32(x, "input");
  host_f32(y, "out");
  check(api().block_forward_host(H(h), fptr(x), fptr_mut(y), B, chunk, current_stream()));
}

double block_time_conv2(int64_t h, const at::Tensor& x, int64_t B, int64_t reps, const at::Tensor& y) {
  dev_f32(x, "input");
  dev_f32(y, "out");
  c10::cuda::CUDAGuard guard(x.device());
  float ms = 0.f;
  check(api().block_time_conv2(H(h), fptr(x), fptr_mut(y), B, (int)reps, stream_of(x), &ms));
  return ms;
}

int64_t launch_count() { return (int64_t)api().launch_count(); }
std::string version() { return api().version(); }

}  // namespace

TORCH_LIBRARY(clifford_b200, m) {
  m.def("load_library(str path) -> str", &load_library);
  m.def("loaded_library() -> str", &loaded_library);
  m.def("version() -> str", &version);
  m.def("launch_count() -> int", &launch_count);
  m.def("validate_signature(int[] g) -> int", &validate_signature);
  m.def("blade_product(int i, int j, int[] g) -> int[]", &blade_product);
  m.def("schedule_terms(int[] g) -> int", &schedule_terms);
  m.def("basis_info(int[] g) -> int[]", &basis_info);
  m.def("expand_kernel(int[] g, Tensor filters, int C_in, int C_out, int Q, Tensor(a!) out) -> ()", &expand_kernel);
  m.def("conv_create(int[] g, int C_in, int C_out, int d_image, int d_filter, int padding, int precision, "
        "Tensor filters, Tensor bias) -> int",
        &conv_create);
  m.def("linear_create(int[] g, int C_in, int C_out, Tensor weight, Tensor bias, int precision) -> int",
        &linear_create);
  m.def("conv_destroy(int h) -> ()", &conv_destroy);
  m.def("conv_forward(int h, Tensor x, int B, Tensor(a!) y) -> ()", &conv_forward);
  m.def("conv_forward_host(int h, Tensor x, int B, Tensor(a!) y) -> ()", &conv_forward_host);
  m.def("conv_gemm_flops(int h, int B) -> float[]", &conv_gemm_flops);
  m.def("conv_plan_info(int[] g, int C_in, int C_out, int d_image, int d_filter, int padding, int precision) "
        "-> int[]",
        &conv_plan_info);
  m.def("conv_out_side(int h) -> int", &conv_out_side);
  m.def("conv_time_kernel(int h, Tensor x, int B, int reps, Tensor(a!) y) -> float", &conv_time_kernel);
  m.def("act_create(int[] g, int mode, int[] kernel_indices, int C, Tensor? weight, Tensor? bias) -> int",
        &act_create);
  m.def("act_destroy(int h) -> ()", &act_destroy);
  m.def("act_forward(int h, Tensor x, int B, int P, Tensor(a!) y) -> ()", &act_forward);
  m.def("act_forward_host(int h, Tensor x, int B, int P, Tensor(a!) y) -> ()", &act_forward_host);
  m.def("act_preactivation(int h, Tensor x, int B, int P, Tensor(a!) s) -> ()", &act_preactivation);
  m.def("act_gather(int h, Tensor x, int B, int P, Tensor(a!) v) -> ()", &act_gather);
  m.def("block_create(int conv1, int act, int conv2, bool residual) -> int", &block_create);
  m.def("block_destroy(int h) -> ()", &block_destroy);
  m.def("block_forward(int h, Tensor x, int B, Tensor(a!) y) -> ()", &block_forward);
  m.def("block_forward_host(int h, Tensor x, int B, int chunk, Tensor(a!) y) -> ()", &block_forward_host);
  m.def("block_time_conv2(int h, Tensor x, int B, int reps, Tensor(a!) y) -> float", &block_time_conv2);
}
