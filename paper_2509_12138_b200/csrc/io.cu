// Float64 PLY for splat models and point clouds (ply_io.hpp:89-221).
//
// A device model is written straight from its planar fp32 store: one kernel
// scatters the 14 planes into the PLY's per-vertex property order as doubles
// (x y z f_dc_0..2 opacity scale_0..2 rot_0..3), the bytes cross the bus in
// pinned chunks, and the file is replaced atomically (io_util.hpp:14-29).
// Header and payload are byte-identical to serialize_splat_ply of the same
// model; reading parses the header with parse_ply_header's rules and error
// texts and scatters the payload back into the planar store, so
// save -> load is bit-exact for the device's values.
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

// PLY property j <- planar parameter kPlyParam[j] (adam.hpp:76-98 order)
__constant__ int kPlyParam[kParams] = {0, 1, 2, 11, 12, 13, 10, 3, 4, 5, 6, 7, 8, 9};
constexpr const char* kSplatProps[kParams] = {"x",       "y",       "z",       "f_dc_0", "f_dc_1",
                                             "f_dc_2",  "opacity", "scale_0", "scale_1", "scale_2",
                                             "rot_0",   "rot_1",   "rot_2",   "rot_3"};
constexpr const char* kCloudProps[9] = {"x", "y", "z", "nx", "ny", "nz", "red", "green", "blue"};

__global__ void k_planar_to_ply(const float* __restrict__ P, int64_t pitch, int64_t n,
                                double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one output double
  if (t >= n * kParams) return;
  const int64_t i = t / kParams;
  const int j = (int)(t - i * kParams);
  out[t] = (double)P[kPlyParam[j] * pitch + i];
}

__global__ void k_ply_to_planar(const double* __restrict__ in, int64_t n, float* __restrict__ P,
                                int64_t pitch) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * kParams) return;
  const int64_t i = t / kParams;
  const int j = (int)(t - i * kParams);
  P[kPlyParam[j] * pitch + i] = (float)in[t];
}

}  // namespace

std::string ply_header(const char* const* props, int nprops, int64_t n, const int64_t* iteration,
                       const int32_t* origin) {
  std::ostringstream h;
  h << "ply\nformat binary_little_endian 1.0\n";
  if (iteration) h << "comment iteration " << *iteration << "\n";
  if (origin && *origin >= 0) h << "comment origin_partition " << *origin << "\n";
  h << "element vertex " << n << "\n";
  for (int k = 0; k < nprops; ++k) h << "property double " << props[k] << "\n";
  h << "end_header\n";
  return h.str();
}

void write_file_atomic(const std::string& path, const std::string& head, const char* body,
                       size_t body_bytes) {
  const std::string tmp = path + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) fail(kIoError, "cannot open for writing: " + tmp);
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  if (ok && body_bytes) ok = std::fwrite(body, 1, body_bytes, f) == body_bytes;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) fail(kIoError, "short write: " + tmp);
  if (std::rename(tmp.c_str(), path.c_str()) != 0)
    fail(kIoError, "rename failed for " + path);
}

std::string read_file(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(kIoError, "cannot open: " + path);
  std::string bytes;
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) bytes.append(buf, got);
  std::fclose(f);
  return bytes;
}

// parse_ply_header (ply_io.hpp:47-84): same acceptance rules and messages.
PlyInfo parse_ply(const std::string& bytes, const char* const* props, int nprops,
                  const char* what) {
  const size_t end = bytes.find("end_header\n");
  if (bytes.rfind("ply\n", 0) != 0 || end == std::string::npos)
    fail(kMalformedFile, "not a ply file");
  PlyInfo h;
  h.payload_offset = end + 11;
  std::istringstream header(bytes.substr(0, end));
  std::string line;
  bool little_endian = false;
  std::vector<std::string> names;
  while (std::getline(header, line)) {
    std::istringstream ls(line);
    std::string word;
    ls >> word;
    if (word == "format") {
      std::string fmt;
      ls >> fmt;
      little_endian = fmt == "binary_little_endian";
    } else if (word == "element") {
      std::string name;
      size_t cnt = 0;
      ls >> name >> cnt;
      if (name == "vertex") h.vertex_count = (int64_t)cnt;
    } else if (word == "property") {
      std::string type, name;
      ls >> type >> name;
      if (type != "double") fail(kMalformedFile, "expected double properties, got " + type);
      names.push_back(name);
    } else if (word == "comment") {
      std::string key, value;
      ls >> key;
      std::getline(ls, value);
      if (!value.empty() && value.front() == ' ') value.erase(0, 1);
      if (key == "iteration") {
        h.iteration = std::stoll(value);
      } else if (key == "origin_partition") {
        h.origin = std::stoi(value);
      }
    }
  }
  if (!little_endian) fail(kMalformedFile, "ply must be binary_little_endian");
  if ((int)names.size() != nprops)
    fail(kMalformedFile, std::string(what) + " ply must have " + std::to_string(nprops) +
                             " properties");
  for (int k = 0; k < nprops; ++k)
    if (names[k] != props[k])
      fail(kMalformedFile, std::string("unexpected property order in ") + what + " ply");
  if (bytes.size() < h.payload_offset + (size_t)h.vertex_count * nprops * sizeof(double))
    fail(kMalformedFile, "ply payload truncated");
  return h;
}

void splat_ply_payload_dev(const float* params, int64_t pitch, int64_t n, double* out,
                           cudaStream_t st) {
  if (n <= 0) return;
  const int64_t t = n * kParams;
  k_planar_to_ply<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(params, pitch, n, out);
  count_launch();
}

void splat_ply_scatter_dev(const double* in, int64_t n, float* params, int64_t pitch,
                           cudaStream_t st) {
  if (n <= 0) return;
  const int64_t t = n * kParams;
  k_ply_to_planar<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(in, n, params, pitch);
  count_launch();
}

const char* const* splat_ply_props() { return kSplatProps; }
const char* const* cloud_ply_props() { return kCloudProps; }

}  // namespace dsg
