// Streamed deterministic generator of the RT/RM-shaped isosurface clouds
// (BASELINE configs[2]/[3]). The reference builds clouds with
// make_volume + marching cubes (volume.hpp:99-145, marching_cubes.hpp:52-109),
// which cannot reach 18.2M / 106.7M points; these clouds sample the analytic
// interface y = h(x, z) directly, one thread per point:
//   * position on a jittered side x side lattice, the jitter drawn with the
//     reference's counter-based hash (hash_combine, rng.hpp:17-20), so point i
//     depends only on (seed, i) and any range of the cloud can be generated
//     on its own;
//   * h = sum over modes of a * cos(kx X + p1) cos(kz Z + p2) (mode table from
//     the host), with a bubble/spike nonlinearity, and its analytic normal;
//   * colour = transfer::normal_matte (marching_cubes.hpp:21-29);
//   * everything rounded to fp32-exact doubles, as scenes.py does.
// paper_2509_12138_b200/scenes.py restates the same definition in numpy.
#include <cmath>

#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

__device__ __forceinline__ uint64_t splitmix(uint64_t s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// hash_combine (rng.hpp:17-20) as a uniform in [0, 1)
__device__ __forceinline__ double hash_uniform(uint64_t seed, uint64_t index) {
  const uint64_t s = seed ^ (0x2545f4914f6cdd1dULL + index * 0x9e3779b97f4a7c15ULL);
  return (double)(splitmix(s) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double f32x(double v) { return (double)(float)v; }

struct HeightArgs {
  int64_t n, side, s0, m;  // cloud size, lattice side, this slice [s0, s0 + m)
  uint64_t seed;
  double span, amp, spikes;
  int nmodes;
  const double* modes;  // [nmodes][5]: kx, kz, ph1, ph2, a
  double* pos;          // [m][3] (slice-local)
  double* col;          // [m][3]
  double* nrm;          // [m][3]
};

__global__ void k_heightfield(HeightArgs a) {
  const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= a.m) return;
  const int64_t i = a.s0 + li;
  const int64_t row = i / a.side, colm = i % a.side;
  const double inv = 1.0 / (double)a.side;
  const double x = ((double)row + 0.5) * inv + (hash_uniform(a.seed, 2 * (uint64_t)i) - 0.5) * 0.8 * inv;
  const double z = ((double)colm + 0.5) * inv + (hash_uniform(a.seed, 2 * (uint64_t)i + 1) - 0.5) * 0.8 * inv;
  const double X = (x - 0.5) * a.span, Z = (z - 0.5) * a.span;
  double h = 0.0, hx = 0.0, hz = 0.0;
  for (int m = 0; m < a.nmodes; ++m) {
    const double* q = a.modes + 5 * m;
    double s1, c1, s2, c2;
    sincos(q[0] * X + q[2], &s1, &c1);
    sincos(q[1] * Z + q[3], &s2, &c2);
    h += q[4] * c1 * c2;
    hx += -q[4] * q[0] * s1 * c2;
    hz += -q[4] * q[1] * c1 * s2;
  }
  const double t = tanh(3.0 * h / a.amp);
  const double h2 = h + a.spikes * t * fabs(h);
  const double ch = cosh(3.0 * h / a.amp);
  const double sg = h > 0.0 ? 1.0 : (h < 0.0 ? -1.0 : 0.0);
  const double d = 1.0 + a.spikes * (t * sg + 3.0 * fabs(h) / a.amp / (ch * ch));
  hx *= d;
  hz *= d;
  double nx = -hx, ny = 1.0, nz = -hz;
  const double nl = fmax(sqrt(nx * nx + ny * ny + nz * nz), 1e-300);
  nx /= nl;
  ny /= nl;
  nz /= nl;
  // transfer::normal_matte (marching_cubes.hpp:21-29)
  const double l1n = sqrt(0.5 * 0.5 + 0.7 * 0.7 + 0.5 * 0.5);
  const double l2n = sqrt(0.6 * 0.6 + 0.2 * 0.2 + 0.75 * 0.75);
  const double lam = 0.25 + 0.55 * fabs((0.5 * nx + 0.7 * ny - 0.5 * nz) / l1n) +
                     0.2 * fabs((-0.6 * nx + 0.2 * ny + 0.75 * nz) / l2n);
  const double b[3] = {0.35 + 0.3 * (0.5 + 0.5 * nx), 0.35 + 0.3 * (0.5 + 0.5 * ny),
                       0.35 + 0.3 * (0.5 + 0.5 * nz)};
  const double p[3] = {X, h2, Z}, nn[3] = {nx, ny, nz};
  for (int k = 0; k < 3; ++k) {
    a.pos[3 * li + k] = f32x(p[k]);
    a.nrm[3 * li + k] = f32x(nn[k]);
    a.col[3 * li + k] = f32x(fmin(fmax(b[k] * lam, 0.0), 1.0));
  }
}

}  // namespace

void heightfield_slice_dev(int64_t n, int64_t s0, int64_t m, uint64_t seed, double span,
                           double amp, double spikes, int nmodes, const double* modes_host,
                           double* pos, double* col, double* nrm, cudaStream_t st) {
  DevBuf<double> modes;
  modes.ensure(5 * (size_t)std::max(nmodes, 1));
  if (nmodes > 0)
    DSG_CUDA_CHECK(cudaMemcpyAsync(modes.get(), modes_host, sizeof(double) * 5 * nmodes,
                                   cudaMemcpyHostToDevice, st));
  HeightArgs a;
  a.n = n;
  a.side = (int64_t)std::ceil(std::sqrt((double)n));  // as scenes.py: ceil(sqrt(n))
  a.s0 = s0;
  a.m = m;
  a.seed = seed;
  a.span = span;
  a.amp = amp;
  a.spikes = spikes;
  a.nmodes = nmodes;
  a.modes = modes.get();
  a.pos = pos;
  a.col = col;
  a.nrm = nrm;
  k_heightfield<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(a);
  count_launch();
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));  // the mode table is freed on return
}

}  // namespace dsg
