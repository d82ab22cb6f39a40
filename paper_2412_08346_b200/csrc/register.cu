// SGD-ICP registration on the device: graspmatch::register_sgd_icp
// (optim.cpp:274-321) with both preconditioners — the fixed matrix
// (sgd_update, optim.cpp:108-114) and the damped Gauss-Newton rotation step
// (gauss_newton_rotation_step, optim.cpp:250-270) — bit-identical to the
// reference (FP64, -fmad=false, the reference's reduction orders).
//
// One CTA per registration problem runs the whole iteration loop: the loop
// is a chain of tiny dependent steps (m = 100 pairs of a 500-point cloud in
// acceptance C2), so a kernel per step would be launch-bound; batching
// independent problems across CTAs is what fills the GPU.  Per iteration:
//   1. the minibatch draw: partial Fisher-Yates over iota(n_source) with
//      std::mt19937_64 + Lemire (spatial_index.cpp:113-125, rng.hpp:32-44),
//      one thread, the array and the 312-word state in shared memory;
//   2. the FP64 nearest neighbour of every transformed batch point in the
//      reference cloud (the kd-tree's "strictly closer, else lowest index",
//      spatial_index.cpp:63-83), brute force: (pair, segment) per thread over
//      the reference staged in shared memory, segments merged in index order;
//   3. per-pair terms (squared distance, residual, the four rotation-gradient
//      dots, the 3x4 Jacobian, its 4x4 moment) written to shared memory in
//      chunks of kRegChunk pairs, then summed left to right by one thread per
//      term — exactly the reference's sequential `+=` over pairs;
//   4. the update on one thread: gradient / m, A g, the Gauss-Newton
//      rotation step (Schur-centred moment, relative damping, the shim's
//      pivot-free LDLT, oracle/shim/Eigen/Dense LdltSolver), pose update,
//      convergence test.
// The rotation_matrix unit-norm require (geometry.cpp:19) is checked every
// iteration; a violation ends the problem with status 1 and the call fails
// with the reference's message.
#include "register.cuh"

#include "dmath.cuh"
#include "mt64.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

namespace asicp {
namespace {

constexpr int kRegThreads = 256;
constexpr int kRegChunk = 128;     // pairs per accumulation round
constexpr int kTerms = 36;         // |d|^2, residual (3), gradient dots (4), Jacobian (12), moment (16)
constexpr int kTermStride = 37;    // odd stride: conflict-free per-pair rows
constexpr int kRefSmemMax = 3072;  // reference points staged in shared memory (32 B each)
constexpr int kFySmemMax = 16384;  // Fisher-Yates array in shared memory (4 B each)
constexpr int kHeadBytes = kRegChunk * kTermStride * 8 + mt::kN * 8;

struct RegCfg {
  double lr, thr, damping;
  double A[49];
  long long max_iter, mb;
  int gn;
};

struct RegArgs {
  const double* src;
  const long long* src_off;
  const double* ref;
  const long long* ref_off;
  const double* init;
  const unsigned long long* seeds;
  int* fy_global;  // per-problem Fisher-Yates arrays for clouds too large for shared memory
  double* theta;
  long long* iters;
  double* loss;
  int* conv;
  int* status;
  int ref_cap, fy_cap;  // shared-memory capacities (points / indices)
};

__device__ __forceinline__ V3 load3(const double* p, int64_t i) { return V3{p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }

struct alignas(16) P4 {
  double x, y, z, w;
};

__device__ __forceinline__ uint64_t mt_next(uint64_t* s, int* mti) {
  if (*mti >= mt::kN) {
    mt::twist_serial(s);
    *mti = 0;
  }
  return mt::temper(s[(*mti)++]);
}

// Rng::uniform_index (rng.hpp:32-44).
__device__ __forceinline__ uint64_t uniform_index(uint64_t* s, int* mti, uint64_t n) {
  uint64_t out;
  while (!mt::lemire(mt_next(s, mti), n, &out)) {
  }
  return out;
}

// gauss_newton_rotation_step (optim.cpp:250-270) from the summed per-pair
// terms: acc[8 + 3 j + r] = sum jac(r, j), acc[20 + 4 i + j] = sum (jac^T jac)(i, j).
__device__ void gn_rotation_step(const double* acc, double md, const double* g, double damping, double* dq) {
  double jm[3][4], cen[4][4];
  for (int j = 0; j < 4; ++j)
    for (int r = 0; r < 3; ++r) jm[r][j] = acc[8 + 3 * j + r] / md;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const double mom = acc[20 + 4 * i + j] / md;
      cen[i][j] = mom - ((jm[0][i] * jm[0][j] + jm[1][i] * jm[1][j]) + jm[2][i] * jm[2][j]);
    }
  const double trace = ((cen[0][0] + cen[1][1]) + cen[2][2]) + cen[3][3];
  double gc[4];
  for (int i = 0; i < 4; ++i) gc[i] = g[3 + i] - ((jm[0][i] * g[0] + jm[1][i] * g[1]) + jm[2][i] * g[2]);
  if (!(trace > 1e-12)) {
    for (int i = 0; i < 4; ++i) dq[i] = g[3 + i];
    return;
  }
  const double sd = damping * trace / 4.0;
  double a[4][4];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) a[i][j] = cen[i][j] + sd * (i == j ? 1.0 : 0.0);
  // LdltSolver::solve: A = L D L^T without pivoting, then two triangular solves.
  double l[4][4] = {{1.0, 0.0, 0.0, 0.0}, {0.0, 1.0, 0.0, 0.0}, {0.0, 0.0, 1.0, 0.0}, {0.0, 0.0, 0.0, 1.0}};
  double dv[4];
  for (int j = 0; j < 4; ++j) {
    double s = a[j][j];
    for (int k = 0; k < j; ++k) s = s - l[j][k] * l[j][k] * dv[k];
    dv[j] = s;
    for (int i = j + 1; i < 4; ++i) {
      double t = a[i][j];
      for (int k = 0; k < j; ++k) t = t - l[i][k] * l[j][k] * dv[k];
      l[i][j] = t / dv[j];
    }
  }
  double y[4];
  for (int i = 0; i < 4; ++i) {
    double s = gc[i];
    for (int k = 0; k < i; ++k) s = s - l[i][k] * y[k];
    y[i] = s;
  }
  for (int i = 0; i < 4; ++i) y[i] = y[i] / dv[i];
  for (int i = 3; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 4; ++k) s = s - l[k][i] * dq[k];
    dq[i] = s;
  }
}

__global__ void __launch_bounds__(kRegThreads) register_kernel(RegArgs a, RegCfg c) {
  const int p = blockIdx.x, tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char reg_smem[];
  double* terms = reinterpret_cast<double*>(reg_smem);
  uint64_t* mts = reinterpret_cast<uint64_t*>(terms + kRegChunk * kTermStride);
  P4* refs = reinterpret_cast<P4*>(mts + mt::kN);
  int* fy_smem = reinterpret_cast<int*>(refs + a.ref_cap);
  __shared__ double s_th[7], s_R[9], s_dR[36], s_acc[kTerms];
  __shared__ double s_nnd[kRegThreads];
  __shared__ int s_nni[kRegThreads];
  __shared__ int s_stop;

  const long long s0 = a.src_off[p], r0 = a.ref_off[p];
  const int n_src = static_cast<int>(a.src_off[p + 1] - s0), n_ref = static_cast<int>(a.ref_off[p + 1] - r0);
  const double* src = a.src + 3 * s0;
  const double* refg = a.ref + 3 * r0;
  const bool ref_in = n_ref <= a.ref_cap;
  int* fy = n_src <= a.fy_cap ? fy_smem : a.fy_global + s0;
  const long long m = c.mb < n_src ? c.mb : n_src;
  const int nterms = c.gn ? kTerms : 8;

  if (ref_in)
    for (int i = tid; i < n_ref; i += kRegThreads) refs[i] = P4{refg[3 * i], refg[3 * i + 1], refg[3 * i + 2], 0.0};
  if (tid == 0) {
    mt::seed_state(mts, a.seeds[p]);
    for (int i = 0; i < 7; ++i) s_th[i] = a.init[7 * static_cast<long long>(p) + i];
  }
  int mti = mt::kN, conv = 0, status = 0;
  long long iters = 0;
  double prev_loss = -1.0, final_loss = 0.0;

  for (long long k = 0; k < c.max_iter; ++k) {
    for (int i = tid; i < n_src; i += kRegThreads) fy[i] = i;
    __syncthreads();
    if (tid == 0) {
      s_stop = 0;
      // sample_minibatch_indices (spatial_index.cpp:113-125).
      for (int i = 0; i < m; ++i) {
        const int j = i + static_cast<int>(uniform_index(mts, &mti, static_cast<uint64_t>(n_src - i)));
        const int v = fy[i];
        fy[i] = fy[j];
        fy[j] = v;
      }
      const Q4 q{s_th[3], s_th[4], s_th[5], s_th[6]};
      if (!(fabs(sqrt(sqnorm4(q)) - 1.0) <= 1e-6)) {  // rotation_matrix's require (geometry.cpp:19)
        status = 1;
        s_stop = 1;
      } else {
        const M3 R = rotation_matrix(q);
        M3 d[4];
        rotation_matrix_derivatives(q, d);
        for (int i = 0; i < 9; ++i) {
          s_R[i] = R.m[i];
          for (int j = 0; j < 4; ++j) s_dR[9 * j + i] = d[j].m[i];
        }
      }
    }
    __syncthreads();
    if (s_stop) break;
    M3 R;
    for (int i = 0; i < 9; ++i) R.m[i] = s_R[i];
    const V3 t{s_th[0], s_th[1], s_th[2]};
    double acc = 0.0;
    for (long long c0 = 0; c0 < m; c0 += kRegChunk) {
      const int np = static_cast<int>(m - c0 < kRegChunk ? m - c0 : kRegChunk);
      const int nseg = kRegThreads / np;  // >= 2
      if (tid < np * nseg) {
        const int pi = tid % np, seg = tid / np;
        const V3 q = transform(R, t, load3(src, fy[c0 + pi]));
        const int lo = static_cast<int>(static_cast<long long>(n_ref) * seg / nseg);
        const int hi = static_cast<int>(static_cast<long long>(n_ref) * (seg + 1) / nseg);
        double best = INFINITY;
        int bi = -1;
        if (ref_in) {
#pragma unroll 4
          for (int i = lo; i < hi; ++i) {
            const P4 r = refs[i];
            const double d2 = sqnorm(sub(V3{r.x, r.y, r.z}, q));
            if (d2 < best) {
              best = d2;
              bi = i;
            }
          }
        } else {
#pragma unroll 4
          for (int i = lo; i < hi; ++i) {
            const double d2 = sqnorm(sub(load3(refg, i), q));
            if (d2 < best) {
              best = d2;
              bi = i;
            }
          }
        }
        s_nnd[tid] = best;
        s_nni[tid] = bi;
      }
      __syncthreads();
      if (tid < np) {
        // Segments hold increasing index ranges: an equal distance keeps the
        // earlier (lower-index) answer.
        double best = s_nnd[tid];
        int bi = s_nni[tid];
        for (int sg = 1; sg < nseg; ++sg)
          if (s_nnd[sg * np + tid] < best) {
            best = s_nnd[sg * np + tid];
            bi = s_nni[sg * np + tid];
          }
        if (bi < 0) bi = 0;  // unreachable for finite clouds
        const V3 s = load3(src, fy[c0 + tid]);
        const V3 q = transform(R, t, s);
        const V3 rp = ref_in ? V3{refs[bi].x, refs[bi].y, refs[bi].z} : load3(refg, bi);
        double* tm = terms + tid * kTermStride;
        const double dist = sqrt(best);
        tm[0] = dist * dist;
        const V3 res = sub(q, rp);
        tm[1] = res.x;
        tm[2] = res.y;
        tm[3] = res.z;
        V3 v[4];
        for (int j = 0; j < 4; ++j) {
          M3 dj;
          for (int i = 0; i < 9; ++i) dj.m[i] = s_dR[9 * j + i];
          v[j] = mul(dj, s);
          tm[4 + j] = dot(res, v[j]);
        }
        if (c.gn) {
          for (int j = 0; j < 4; ++j) {
            tm[8 + 3 * j] = v[j].x;
            tm[9 + 3 * j] = v[j].y;
            tm[10 + 3 * j] = v[j].z;
          }
          for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) tm[20 + 4 * i + j] = dot(v[i], v[j]);
        }
      }
      __syncthreads();
      if (tid < nterms)
        for (int i = 0; i < np; ++i) acc = acc + terms[i * kTermStride + tid];
      __syncthreads();
    }
    if (tid < nterms) s_acc[tid] = acc;
    __syncthreads();
    if (tid == 0) {
      const double md = static_cast<double>(m);
      const double loss = s_acc[0] / md;
      double g[7];
      for (int i = 0; i < 7; ++i) g[i] = s_acc[1 + i] / md;
      double pre[7];
      for (int r = 0; r < 7; ++r) {
        double s = c.A[7 * r] * g[0];
        for (int k2 = 1; k2 < 7; ++k2) s = s + c.A[7 * r + k2] * g[k2];
        pre[r] = s;
      }
      double dq[4];
      if (!c.gn) {
        for (int i = 0; i < 4; ++i) dq[i] = pre[3 + i];  // sgd_update: q - lr (A g).tail
      } else {
        gn_rotation_step(s_acc, md, g, c.damping, dq);
      }
      for (int i = 0; i < 3; ++i) s_th[i] = s_th[i] - c.lr * pre[i];
      const Q4 qn = normalized(
          Q4{s_th[3] - c.lr * dq[0], s_th[4] - c.lr * dq[1], s_th[5] - c.lr * dq[2], s_th[6] - c.lr * dq[3]});
      s_th[3] = qn.w;
      s_th[4] = qn.x;
      s_th[5] = qn.y;
      s_th[6] = qn.z;
      iters = k + 1;
      final_loss = loss;
      if (prev_loss > 0.0 && c.thr >= 0.0 && fabs(loss - prev_loss) / prev_loss <= c.thr && m == n_src) {
        conv = 1;
        s_stop = 1;
      }
      prev_loss = loss;
    }
    __syncthreads();
    if (s_stop) break;
  }
  if (tid == 0) {
    for (int i = 0; i < 7; ++i) a.theta[7 * static_cast<long long>(p) + i] = s_th[i];
    a.iters[p] = iters;
    a.loss[p] = final_loss;
    a.conv[p] = conv;
    a.status[p] = status;
  }
}

// Host restatements of SgdConfig::validate (optim.cpp:10-15) against the
// shim's isApprox / LLT (oracle/shim/Eigen/Dense).
double col_major_norm(const double* A, bool transposed) {
  auto at = [&](int i, int j) { return transposed ? A[7 * j + i] : A[7 * i + j]; };
  double s = at(0, 0) * at(0, 0);
  for (int j = 0; j < 7; ++j)
    for (int i = 0; i < 7; ++i)
      if (i != 0 || j != 0) s = s + at(i, j) * at(i, j);
  return std::sqrt(s);
}

bool sgd_symmetric(const double* A) {
  double d[49];
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) d[7 * i + j] = A[7 * i + j] - A[7 * j + i];
  return col_major_norm(d, false) <= 1e-12 * std::min(col_major_norm(A, false), col_major_norm(A, true));
}

bool sgd_llt_ok(const double* A) {
  double l[7][7];
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) l[i][j] = A[7 * i + j];
  for (int j = 0; j < 7; ++j) {
    double s = l[j][j];
    for (int k = 0; k < j; ++k) s -= l[j][k] * l[j][k];
    if (!(s > 0.0)) return false;
    const double dd = std::sqrt(s);
    l[j][j] = dd;
    for (int i = j + 1; i < 7; ++i) {
      double t = l[i][j];
      for (int k = 0; k < j; ++k) t -= l[i][k] * l[j][k];
      l[i][j] = t / dd;
    }
    for (int i = 0; i < j; ++i) l[i][j] = 0.0;
  }
  return true;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

}  // namespace

// FP64 throughput ceiling of this GPU (DFMA, 2 FLOP each): the roofline
// denominator of the registration kernel's brute-force NN, which cannot
// contract (bit-exactness) and so tops out at half of it.
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = __fma_rn(acc[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  if (s == 1234.5) out[0] = s;
}

struct RegBatch::Dev {
  int n = 0;
  RegCfg cfg{};
  int ref_cap = 0, fy_cap = 0;
  size_t smem = 0;
  DevBuf src, src_off, ref, ref_off, init, seeds, fy, theta, iters, loss, conv, status;
  // Pinned result staging.
  double* h_theta = nullptr;
  long long* h_iters = nullptr;
  double* h_loss = nullptr;
  int* h_conv = nullptr;
  int* h_status = nullptr;
  int h_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void free_host() {
    void* all[] = {h_theta, h_iters, h_loss, h_conv, h_status};
    for (void* q : all)
      if (q) cudaFreeHost(q);
    h_theta = nullptr;
    h_iters = nullptr;
    h_loss = nullptr;
    h_conv = nullptr;
    h_status = nullptr;
    h_cap = 0;
  }
  ~Dev() {
    free_host();
    DevBuf* all[] = {&src, &src_off, &ref, &ref_off, &init, &seeds, &fy, &theta, &iters, &loss, &conv, &status};
    for (DevBuf* b : all) b->release();
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }
};

RegBatch::~RegBatch() { release(); }

void RegBatch::release() {
  delete d_;
  d_ = nullptr;
}

#define REG_CUDA(expr)                                                                    \
  do {                                                                                    \
    const cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                              \
      *err = std::string(#expr) + ": " + cudaGetErrorString(e_);                          \
      return ASICP_DEVICE_ERROR;                                                          \
    }                                                                                     \
  } while (0)

int RegBatch::prepare(int64_t n, const double* sources, const int64_t* src_off, const double* references,
                      const int64_t* ref_off, const double* initial, const uint64_t* seeds,
                      const asicp_sgd_config& cfg, std::string* err) {
  auto invalid = [&](const char* msg) {
    *err = msg;
    return ASICP_INVALID_ARGUMENT;
  };
  if (n < 0) return invalid("asicp: negative problem count");
  if (cfg.max_iterations < 0 || cfg.minibatch_size < 0)
    return invalid("asicp: max_iterations and minibatch_size must be >= 0");
  if (cfg.preconditioner_mode != ASICP_PRECOND_FIXED && cfg.preconditioner_mode != ASICP_PRECOND_GAUSS_NEWTON_ROTATION)
    return invalid("asicp: unknown preconditioner_mode");
  if (n > (1ll << 31) - 1) return invalid("asicp: too many problems");
  if (n > 0 && (!src_off || !ref_off || !initial || !seeds)) return invalid("asicp: null batch array");
  int max_src = 0, max_ref = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t ns = src_off[i + 1] - src_off[i], nr = ref_off[i + 1] - ref_off[i];
    // register_sgd_icp (optim.cpp:277-290), in the reference's order.
    if (ns < 0 || nr < 0) return invalid("asicp: decreasing cloud offsets");
    if (ns == 0 || nr == 0) return invalid("register_sgd_icp: empty cloud");
    if (cfg.preconditioner_mode == ASICP_PRECOND_FIXED) {
      if (!(cfg.learning_rate > 0.0)) return invalid("SgdConfig: learning_rate must be positive");
      if (!sgd_symmetric(cfg.A)) return invalid("SgdConfig: A must be symmetric");
      if (!sgd_llt_ok(cfg.A)) return invalid("SgdConfig: A must be positive definite");
    }
    if (ns >= (1ll << 31) || nr >= (1ll << 31)) return invalid("asicp: cloud too large");
    if (cfg.max_iterations > 0) {
      if (std::min<int64_t>(cfg.minibatch_size, ns) < 1) return invalid("sample_minibatch: m out of range");
      const double* q = initial + 7 * i + 3;
      const double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
      if (!(std::abs(std::sqrt(n2) - 1.0) <= 1e-6)) return invalid("rotation_matrix: quaternion is not unit-norm");
    }
    max_src = std::max<int>(max_src, static_cast<int>(ns));
    max_ref = std::max<int>(max_ref, static_cast<int>(nr));
  }
  REG_CUDA(cudaSetDevice(device_));
  if (!d_) d_ = new Dev();
  Dev& D = *d_;
  D.n = static_cast<int>(n);
  D.cfg.lr = cfg.learning_rate;
  D.cfg.thr = cfg.convergence_threshold;
  D.cfg.damping = cfg.gn_damping;
  std::memcpy(D.cfg.A, cfg.A, sizeof(D.cfg.A));
  D.cfg.max_iter = cfg.max_iterations;
  D.cfg.mb = cfg.minibatch_size;
  D.cfg.gn = cfg.preconditioner_mode == ASICP_PRECOND_GAUSS_NEWTON_ROTATION ? 1 : 0;
  D.ref_cap = max_ref <= kRefSmemMax ? max_ref : 0;
  D.fy_cap = max_src <= kFySmemMax ? max_src : 0;
  D.smem = kHeadBytes + static_cast<size_t>(D.ref_cap) * sizeof(P4) + static_cast<size_t>(D.fy_cap) * 4;
  if (n == 0) return ASICP_OK;
  const int64_t tot_src = src_off[n] - src_off[0], tot_ref = ref_off[n] - ref_off[0];
  // Offsets are rebased to the first problem's rows.
  std::vector<long long> so(n + 1), ro(n + 1);
  for (int64_t i = 0; i <= n; ++i) {
    so[i] = src_off[i] - src_off[0];
    ro[i] = ref_off[i] - ref_off[0];
  }
  REG_CUDA(D.src.ensure(std::max<int64_t>(tot_src, 1) * 24));
  REG_CUDA(D.ref.ensure(std::max<int64_t>(tot_ref, 1) * 24));
  REG_CUDA(D.src_off.ensure((n + 1) * 8));
  REG_CUDA(D.ref_off.ensure((n + 1) * 8));
  REG_CUDA(D.init.ensure(n * 56));
  REG_CUDA(D.seeds.ensure(n * 8));
  REG_CUDA(D.fy.ensure(D.fy_cap ? 4 : std::max<int64_t>(tot_src, 1) * 4));
  REG_CUDA(D.theta.ensure(n * 56));
  REG_CUDA(D.iters.ensure(n * 8));
  REG_CUDA(D.loss.ensure(n * 8));
  REG_CUDA(D.conv.ensure(n * 4));
  REG_CUDA(D.status.ensure(n * 4));
  REG_CUDA(cudaMemcpyAsync(D.src.p, sources + 3 * src_off[0], tot_src * 24, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.ref.p, references + 3 * ref_off[0], tot_ref * 24, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.src_off.p, so.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.ref_off.p, ro.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.init.p, initial, n * 56, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.seeds.p, seeds, n * 8, cudaMemcpyHostToDevice, st_));
  if (D.h_cap < n) {
    D.free_host();
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_theta), n * 56));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_iters), n * 8));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_loss), n * 8));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_conv), n * 4));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_status), n * 4));
    D.h_cap = static_cast<int>(n);
  }
  if (!D.ev0) REG_CUDA(cudaEventCreate(&D.ev0));
  if (!D.ev1) REG_CUDA(cudaEventCreate(&D.ev1));
  REG_CUDA(cudaFuncSetAttribute(register_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(D.smem)));
  // The upload reads caller memory: finish it before returning.
  REG_CUDA(cudaStreamSynchronize(st_));
  return ASICP_OK;
}

int RegBatch::run(asicp_registration* out, std::string* err) {
  if (!d_) {
    *err = "asicp: no registration batch prepared";
    return ASICP_INVALID_ARGUMENT;
  }
  Dev& D = *d_;
  kernel_ms_ = 0.0f;
  if (D.n == 0) return ASICP_OK;
  REG_CUDA(cudaSetDevice(device_));
  RegArgs a;
  a.src = static_cast<const double*>(D.src.p);
  a.src_off = static_cast<const long long*>(D.src_off.p);
  a.ref = static_cast<const double*>(D.ref.p);
  a.ref_off = static_cast<const long long*>(D.ref_off.p);
  a.init = static_cast<const double*>(D.init.p);
  a.seeds = static_cast<const unsigned long long*>(D.seeds.p);
  a.fy_global = static_cast<int*>(D.fy.p);
  a.theta = static_cast<double*>(D.theta.p);
  a.iters = static_cast<long long*>(D.iters.p);
  a.loss = static_cast<double*>(D.loss.p);
  a.conv = static_cast<int*>(D.conv.p);
  a.status = static_cast<int*>(D.status.p);
  a.ref_cap = D.ref_cap;
  a.fy_cap = D.fy_cap;
  REG_CUDA(cudaEventRecord(D.ev0, st_));
  register_kernel<<<D.n, kRegThreads, D.smem, st_>>>(a, D.cfg);
  REG_CUDA(cudaGetLastError());
  REG_CUDA(cudaEventRecord(D.ev1, st_));
  const size_t n = static_cast<size_t>(D.n);
  REG_CUDA(cudaMemcpyAsync(D.h_theta, D.theta.p, n * 56, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_iters, D.iters.p, n * 8, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_loss, D.loss.p, n * 8, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_conv, D.conv.p, n * 4, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_status, D.status.p, n * 4, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaStreamSynchronize(st_));
  REG_CUDA(cudaEventElapsedTime(&kernel_ms_, D.ev0, D.ev1));
  for (size_t i = 0; i < n; ++i) {
    if (D.h_status[i]) {
      *err = "rotation_matrix: quaternion is not unit-norm";
      return ASICP_INVALID_ARGUMENT;
    }
  }
  if (out)
    for (size_t i = 0; i < n; ++i) {
      std::memcpy(out[i].theta, D.h_theta + 7 * i, 56);
      out[i].iterations = D.h_iters[i];
      out[i].final_loss = D.h_loss[i];
      out[i].converged = D.h_conv[i];
    }
  return ASICP_OK;
}

double run_dfma_peak(int iters) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8;
  dfma_peak_kernel<<<blocks, 256>>>(out, iters / 4, 0.999, 1e-4);  // warm-up
  cudaEventRecord(e0);
  dfma_peak_kernel<<<blocks, 256>>>(out, iters, 0.999, 1e-4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.0f) return -1.0;
  return 2.0 * 8.0 * static_cast<double>(iters) * blocks * 256.0 / (ms * 1e-3) / 1e12;
}

}  // namespace asicp
