// GPU-side problem assembly: the SURVEY §8d generators and
// the reference's assembly rules, on the device.
//
//  * cell-centred 5-/7-point diffusion (SURVEY §8d "harmonic face
//    coefficients"; boundary faces use the cell coefficient), row by row;
//  * Q1 plane-strain elasticity with the element formula of
//    proj/src/fem.cpp:53-97 and assemble()'s rules (fem.cpp:99-162): x = 0
//    node column eliminated, duplicate couplings summed in element order the
//    way TripletBuilder::build's stable sort does (sparse.cpp:19-47), body
//    force integrated per element in Gauss-point order;
//  * overlapping partitions: disjoint owners grown by rings of matrix-graph
//    closure (partition.cpp:79-90), lists sorted per subdomain.
//
// Every value is formed with the same operations in the same order as the
// host generator (paper_2106_10913_b200/problems.py, numpy, no contraction):
// explicit __dmul_rn / __dadd_rn / __ddiv_rn, so the device CSR is
// bit-identical to it (tests/test_gpu_assembly.py).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "awg_internal.cuh"

namespace awgb {
namespace {

constexpr int kT = 256;

inline int blocks_for(long long n) { return int(std::max<long long>(1, (n + kT - 1) / kT)); }

// ---------------------------------------------------------------------------
// diffusion
struct Grid {
  int dims, nx, ny, nz;
  long long sx, sy, sz;  // strides of x, y, z
};

__device__ __forceinline__ double face_coef(double lo, double hi) {
  // (2 c_lo c_hi) / (c_lo + c_hi), evaluated as the host: ((2 * lo) * hi) / (lo + hi)
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, lo), hi), __dadd_rn(lo, hi));
}

__device__ __forceinline__ void cell_coords(const Grid& g, long long i, int& x, int& y, int& z) {
  x = int(i % g.nx);
  y = int((i / g.nx) % g.ny);
  z = g.dims == 3 ? int(i / ((long long)g.nx * g.ny)) : 0;
}

__global__ void k_fd_count(Grid g, long long n, int* cnt) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x, y, z;
  cell_coords(g, i, x, y, z);
  int c = 1 + (x > 0) + (x < g.nx - 1) + (y > 0) + (y < g.ny - 1);
  if (g.dims == 3) c += (z > 0) + (z < g.nz - 1);
  cnt[i] = c;
}

__global__ void k_fd_fill(Grid g, long long n, const double* __restrict__ coef, const int* __restrict__ off,
                          int* __restrict__ ci, double* __restrict__ va) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x, y, z;
  cell_coords(g, i, x, y, z);
  const double c0 = coef[i];
  // faces with the -/+ neighbour of each axis (nan-free: existence flags)
  const bool has[3][2] = {{x > 0, x < g.nx - 1}, {y > 0, y < g.ny - 1}, {g.dims == 3 && z > 0, g.dims == 3 && z < g.nz - 1}};
  const long long st[3] = {g.sx, g.sy, g.sz};
  double f[3][2];
  for (int ax = 0; ax < g.dims; ++ax) {
    f[ax][0] = has[ax][0] ? face_coef(coef[i - st[ax]], c0) : 0.0;
    f[ax][1] = has[ax][1] ? face_coef(c0, coef[i + st[ax]]) : 0.0;
  }
  // diagonal: faces in the order -x, +x, -y, +y(, -z, +z); boundary faces use c0
  double diag = 0.0;
  for (int ax = 0; ax < g.dims; ++ax)
    for (int sg = 0; sg < 2; ++sg) diag = __dadd_rn(diag, has[ax][sg] ? f[ax][sg] : c0);
  // columns ascending: -z, -y, -x, self, +x, +y, +z
  int k = off[i];
  for (int ax = g.dims - 1; ax >= 0; --ax)
    if (has[ax][0]) {
      ci[k] = int(i - st[ax]);
      va[k++] = -f[ax][0];
    }
  ci[k] = int(i);
  va[k++] = diag;
  for (int ax = 0; ax < g.dims; ++ax)
    if (has[ax][1]) {
      ci[k] = int(i + st[ax]);
      va[k++] = -f[ax][1];
    }
}

// ---------------------------------------------------------------------------
// Q1 plane-strain elasticity (h = 1)

// 8x8 element stiffness per material (fem.cpp:53-97 restated; the host's
// numpy evaluation order, no contraction)
__global__ void k_element_stiffness(int nmat, const double* __restrict__ young, const double* __restrict__ poisson,
                                    double* __restrict__ ke) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= nmat) return;
  const double e = young[m], nu = poisson[m];
  const double mu = __ddiv_rn(e, __dmul_rn(2.0, __dadd_rn(1.0, nu)));
  const double lam = __ddiv_rn(__dmul_rn(e, nu), __dmul_rn(__dadd_rn(1.0, nu), __dsub_rn(1.0, __dmul_rn(2.0, nu))));
  const double d00 = __dadd_rn(__dmul_rn(2.0, mu), lam), d01 = lam, d22 = mu;
  const double g = __ddiv_rn(1.0, __dsqrt_rn(3.0));
  const double detj = 0.25, ds = 2.0;
  double k[8][8];
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) k[a][b] = 0.0;
  for (int gx = 0; gx < 2; ++gx)
    for (int gy = 0; gy < 2; ++gy) {
      const double xi = gx ? g : -g, eta = gy ? g : -g;
      const double om_e = __dsub_rn(1.0, eta), op_e = __dadd_rn(1.0, eta);
      const double om_x = __dsub_rn(1.0, xi), op_x = __dadd_rn(1.0, xi);
      const double dxi[4] = {__dmul_rn(__ddiv_rn(-om_e, 4.0), ds), __dmul_rn(__ddiv_rn(om_e, 4.0), ds),
                             __dmul_rn(__ddiv_rn(op_e, 4.0), ds), __dmul_rn(__ddiv_rn(-op_e, 4.0), ds)};
      const double deta[4] = {__dmul_rn(__ddiv_rn(-om_x, 4.0), ds), __dmul_rn(__ddiv_rn(-op_x, 4.0), ds),
                              __dmul_rn(__ddiv_rn(op_x, 4.0), ds), __dmul_rn(__ddiv_rn(om_x, 4.0), ds)};
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
          const double kxx = __dadd_rn(__dmul_rn(__dmul_rn(d00, dxi[a]), dxi[b]), __dmul_rn(__dmul_rn(d22, deta[a]), deta[b]));
          const double kxy = __dadd_rn(__dmul_rn(__dmul_rn(d01, dxi[a]), deta[b]), __dmul_rn(__dmul_rn(d22, deta[a]), dxi[b]));
          const double kyx = __dadd_rn(__dmul_rn(__dmul_rn(d01, deta[a]), dxi[b]), __dmul_rn(__dmul_rn(d22, dxi[a]), deta[b]));
          const double kyy = __dadd_rn(__dmul_rn(__dmul_rn(d00, deta[a]), deta[b]), __dmul_rn(__dmul_rn(d22, dxi[a]), dxi[b]));
          k[2 * a][2 * b] = __dadd_rn(k[2 * a][2 * b], __dmul_rn(detj, kxx));
          k[2 * a][2 * b + 1] = __dadd_rn(k[2 * a][2 * b + 1], __dmul_rn(detj, kxy));
          k[2 * a + 1][2 * b] = __dadd_rn(k[2 * a + 1][2 * b], __dmul_rn(detj, kyx));
          k[2 * a + 1][2 * b + 1] = __dadd_rn(k[2 * a + 1][2 * b + 1], __dmul_rn(detj, kyy));
        }
    }
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) ke[(size_t)m * 64 + a * 8 + b] = (b >= a) ? k[a][b] : k[b][a];  // mirror the upper
}

struct Mesh {
  int nodes_x, nodes_y, layer, nmat;
  __device__ int nfx() const { return nodes_x - 1; }  // free nodes per row (x = 0 clamped)
};

// local index of node (x, y) in element (ex, ey): (0,0),(1,0),(1,1),(0,1)
__device__ __forceinline__ int local_node(int dx, int dy) { return dy == 0 ? dx : 3 - dx; }

__global__ void k_el_count(Mesh m, int n, int* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = i >> 1;
  const int ix = f % m.nfx() + 1, iy = f / m.nfx();
  const int nxn = min(ix + 1, m.nodes_x - 1) - max(ix - 1, 1) + 1;
  const int nyn = min(iy + 1, m.nodes_y - 1) - max(iy - 1, 0) + 1;
  cnt[i] = 2 * nxn * nyn;
}

__global__ void k_el_fill(Mesh m, int n, const double* __restrict__ ke, const int* __restrict__ off,
                          int* __restrict__ ci, double* __restrict__ va) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = i >> 1, di = i & 1;
  const int ix = f % m.nfx() + 1, iy = f / m.nfx();
  const int nex = m.nodes_x - 1, ney = m.nodes_y - 1;
  int k = off[i];
  for (int jy = max(iy - 1, 0); jy <= min(iy + 1, m.nodes_y - 1); ++jy)
    for (int jx = max(ix - 1, 1); jx <= min(ix + 1, m.nodes_x - 1); ++jx)
      for (int dj = 0; dj < 2; ++dj) {
        double acc = 0.0;
        // elements holding both nodes, in assembly order (ey outer, ex inner)
        for (int ey = max(max(iy, jy) - 1, 0); ey <= min(min(iy, jy), ney - 1); ++ey)
          for (int ex = max(max(ix, jx) - 1, 0); ex <= min(min(ix, jx), nex - 1); ++ex) {
            const int mat = (ey / m.layer) % m.nmat;
            const int a = local_node(ix - ex, iy - ey), b = local_node(jx - ex, jy - ey);
            acc = __dadd_rn(acc, ke[(size_t)mat * 64 + (2 * a + di) * 8 + 2 * b + dj]);
          }
        ci[k] = 2 * (jy * m.nfx() + jx - 1) + dj;
        va[k++] = acc;
      }
}

// body force: integral of N_a g over every element holding the node, per
// element in Gauss-point order (xi outer, eta inner), 0.25 * N_a * g_d
__global__ void k_el_rhs(Mesh m, int n, double g0, double g1, double* __restrict__ b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = i >> 1, d = i & 1;
  const int ix = f % m.nfx() + 1, iy = f / m.nfx();
  const int nex = m.nodes_x - 1, ney = m.nodes_y - 1;
  const double g = __ddiv_rn(1.0, __dsqrt_rn(3.0));
  const double load = d ? g1 : g0;
  double acc = 0.0;
  for (int ey = max(iy - 1, 0); ey <= min(iy, ney - 1); ++ey)
    for (int ex = max(ix - 1, 0); ex <= min(ix, nex - 1); ++ex) {
      const int a = local_node(ix - ex, iy - ey);
      for (int gx = 0; gx < 2; ++gx)
        for (int gy = 0; gy < 2; ++gy) {
          const double xi = gx ? g : -g, eta = gy ? g : -g;
          const double sx = (a == 0 || a == 3) ? __dsub_rn(1.0, xi) : __dadd_rn(1.0, xi);
          const double sy = (a < 2) ? __dsub_rn(1.0, eta) : __dadd_rn(1.0, eta);
          const double shape = __ddiv_rn(__dmul_rn(sx, sy), 4.0);
          acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(0.25, shape), load));
        }
    }
  b[i] = acc;
}

// ---------------------------------------------------------------------------
// overlapping partition: bitmask per dof (W words of 32 subdomains), grown by
// rings of closure over the stored couplings, then (subdomain, dof) pairs
// stably sorted by subdomain (dofs stay ascending within a subdomain)
__global__ void k_mask_init(int n, int W, const int* __restrict__ owner, unsigned* __restrict__ mask) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int w = 0; w < W; ++w) mask[(size_t)i * W + w] = 0u;
  mask[(size_t)i * W + (owner[i] >> 5)] = 1u << (owner[i] & 31);
}

__global__ void k_mask_ring(int n, int W, const int* __restrict__ rp, const int* __restrict__ ci,
                            const unsigned* __restrict__ in, unsigned* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int w = 0; w < W; ++w) {
    unsigned v = in[(size_t)i * W + w];
    for (int k = rp[i]; k < rp[i + 1]; ++k) v |= in[(size_t)ci[k] * W + w];
    out[(size_t)i * W + w] = v;
  }
}

__global__ void k_mask_count(int n, int W, const unsigned* __restrict__ mask, int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int w = 0; w < W; ++w) c += __popc(mask[(size_t)i * W + w]);
  cnt[i] = c;
}

__global__ void k_mask_pairs(int n, int W, const unsigned* __restrict__ mask, const int* __restrict__ off,
                             int* __restrict__ sub, int* __restrict__ dof) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int k = off[i];
  for (int w = 0; w < W; ++w) {
    unsigned v = mask[(size_t)i * W + w];
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1;
      sub[k] = w * 32 + b;
      dof[k++] = i;
    }
  }
}

template <typename T>
void exclusive_scan(Ctx& c, const T* in, T* out, int n) {
  size_t bytes = 0;
  AWG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c.stream));
  DArr<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(bytes, 1));
  AWG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, c.stream));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

// counts (n) -> row offsets (n + 1) on the host and device
std::vector<int> offsets_from_counts(Ctx& c, DArr<int>& cnt, DArr<int>& off, int n) {
  off.alloc(size_t(n) + 1);
  exclusive_scan(c, cnt.p, off.p, n);
  std::vector<int> h(size_t(n) + 1);
  AWG_CUDA(cudaMemcpy(h.data(), off.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
  int last = 0;
  AWG_CUDA(cudaMemcpy(&last, cnt.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost));
  h[n] = h[n - 1] + last;
  AWG_CUDA(cudaMemcpy(off.p + n, &h[n], sizeof(int), cudaMemcpyHostToDevice));
  return h;
}

}  // namespace

void assemble_fd(Ctx& c, int dims, const int* shape, const double* coef, std::vector<int>& rp, std::vector<int>& ci,
                 std::vector<double>& va) {
  if ((dims != 2 && dims != 3) || !shape || !coef) c.fail(AWG_E_ARG, "assemble_fd: bad arguments");
  Grid g{dims, shape[0], shape[1], dims == 3 ? shape[2] : 1, 1, shape[0], (long long)shape[0] * shape[1]};
  if (g.nx < 1 || g.ny < 1 || g.nz < 1) c.fail(AWG_E_ARG, "assemble_fd: empty grid");
  const long long n = (long long)g.nx * g.ny * g.nz;
  if (n > (1LL << 30)) c.fail(AWG_E_ARG, "assemble_fd: grid too large for int32 indices");
  DArr<double> dcoef;
  dcoef.alloc(size_t(n));
  AWG_CUDA(cudaMemcpyAsync(dcoef.p, coef, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
  DArr<int> cnt, off, dci;
  DArr<double> dva;
  cnt.alloc(size_t(n));
  k_fd_count<<<blocks_for(n), kT, 0, c.stream>>>(g, n, cnt.p);
  ++c.launches;
  rp = offsets_from_counts(c, cnt, off, int(n));
  const int nnz = rp[n];
  dci.alloc(nnz);
  dva.alloc(nnz);
  k_fd_fill<<<blocks_for(n), kT, 0, c.stream>>>(g, n, dcoef.p, off.p, dci.p, dva.p);
  ++c.launches;
  ci.resize(nnz);
  va.resize(nnz);
  AWG_CUDA(cudaMemcpyAsync(ci.data(), dci.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaMemcpyAsync(va.data(), dva.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

void assemble_elasticity(Ctx& c, int nodes_x, int nodes_y, int layer, int nmat, const double* young,
                         const double* poisson, const double* load, std::vector<int>& rp, std::vector<int>& ci,
                         std::vector<double>& va, std::vector<double>& b) {
  if (nodes_x < 2 || nodes_y < 2 || layer < 1 || nmat < 1 || !young || !poisson || !load)
    c.fail(AWG_E_ARG, "assemble_elasticity: bad arguments");
  const long long nl = 2LL * (nodes_x - 1) * nodes_y;
  if (nl > (1LL << 30)) c.fail(AWG_E_ARG, "assemble_elasticity: mesh too large for int32 indices");
  const int n = int(nl);
  Mesh m{nodes_x, nodes_y, layer, nmat};
  DArr<double> E, NU, KE;
  std::vector<double> he(young, young + nmat), hn(poisson, poisson + nmat);
  E.upload(he, c.stream);
  NU.upload(hn, c.stream);
  KE.alloc(size_t(nmat) * 64);
  k_element_stiffness<<<1, 32, 0, c.stream>>>(nmat, E.p, NU.p, KE.p);
  DArr<int> cnt, off, dci;
  DArr<double> dva, db;
  cnt.alloc(n);
  k_el_count<<<blocks_for(n), kT, 0, c.stream>>>(m, n, cnt.p);
  c.launches += 2;
  rp = offsets_from_counts(c, cnt, off, n);
  const int nnz = rp[n];
  dci.alloc(nnz);
  dva.alloc(nnz);
  db.alloc(n);
  k_el_fill<<<blocks_for(n), kT, 0, c.stream>>>(m, n, KE.p, off.p, dci.p, dva.p);
  k_el_rhs<<<blocks_for(n), kT, 0, c.stream>>>(m, n, load[0], load[1], db.p);
  c.launches += 2;
  ci.resize(nnz);
  va.resize(nnz);
  b.resize(n);
  AWG_CUDA(cudaMemcpyAsync(ci.data(), dci.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaMemcpyAsync(va.data(), dva.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaMemcpyAsync(b.data(), db.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

// Omega^s from disjoint owners: `rings` rings of closure over the stored
// couplings of the context matrix (already installed on the device)
void partition_closure(Ctx& c, const std::vector<int>& owner, int nsub, int rings, std::vector<long long>& off,
                       std::vector<int>& idx) {
  const int n = c.n;
  if (int(owner.size()) != n || nsub < 1 || rings < 0) c.fail(AWG_E_ARG, "partition: bad arguments");
  for (int o : owner)
    if (o < 0 || o >= nsub) c.fail(AWG_E_ARG, "partition: owner out of range");
  const int W = (nsub + 31) / 32;
  DArr<int> down;
  down.upload(owner, c.stream);
  DArr<unsigned> m0, m1;
  m0.alloc(size_t(n) * W);
  m1.alloc(size_t(n) * W);
  k_mask_init<<<blocks_for(n), kT, 0, c.stream>>>(n, W, down.p, m0.p);
  ++c.launches;
  for (int r = 0; r < rings; ++r) {
    k_mask_ring<<<blocks_for(n), kT, 0, c.stream>>>(n, W, c.rp.p, c.ci.p, m0.p, m1.p);
    ++c.launches;
    std::swap(m0.p, m1.p);
  }
  DArr<int> cnt, poff;
  cnt.alloc(n);
  k_mask_count<<<blocks_for(n), kT, 0, c.stream>>>(n, W, m0.p, cnt.p);
  ++c.launches;
  const std::vector<int> h = offsets_from_counts(c, cnt, poff, n);
  const int P = h[n];
  DArr<int> sub, dof, sub2, dof2;
  sub.alloc(P);
  dof.alloc(P);
  sub2.alloc(P);
  dof2.alloc(P);
  k_mask_pairs<<<blocks_for(n), kT, 0, c.stream>>>(n, W, m0.p, poff.p, sub.p, dof.p);
  ++c.launches;
  size_t bytes = 0;
  int bits = 1;
  while ((1 << bits) < nsub) ++bits;
  AWG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, sub.p, sub2.p, dof.p, dof2.p, P, 0, bits, c.stream));
  DArr<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(bytes, 1));
  AWG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, sub.p, sub2.p, dof.p, dof2.p, P, 0, bits, c.stream));
  std::vector<int> hs(P);
  idx.resize(P);
  AWG_CUDA(cudaMemcpyAsync(hs.data(), sub2.p, sizeof(int) * P, cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaMemcpyAsync(idx.data(), dof2.p, sizeof(int) * P, cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  off.assign(size_t(nsub) + 1, 0);
  for (int p = 0; p < P; ++p) ++off[size_t(hs[p]) + 1];
  for (int s = 0; s < nsub; ++s) off[s + 1] += off[s];
}

}  // namespace awgb
