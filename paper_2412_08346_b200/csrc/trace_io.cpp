// graspmatch::export_trace (io.cpp:691-710) for a B200 solution's trace —
// SURVEY.md §8(f) rank 3.  The per-iteration records are produced on the
// device (record_trace: pre-update pose, loss and collision flag of every
// particle at every iteration, grasp.cpp:197-209) and written here in the
// reference's 13-field text format: a schema header, then one line per
// (iteration, particle) record, doubles in shortest round-trip form
// (std::to_chars, io.cpp:249-254).
#include "asicp.h"

#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

void put_double(std::string& out, double v) {
  char buf[32];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, res.ptr);
}

void put_u64(std::string& out, uint64_t v) {
  char buf[24];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, res.ptr);
}

void set_err(const std::string& msg, char* err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = '\0';
  }
}

}  // namespace

extern "C" int asicp_export_trace(const char* path, int64_t k_max, int64_t n_particles, int64_t k_stein,
                                  const int64_t* particle_preshape, const double* trace_theta,
                                  const double* trace_loss, const int32_t* trace_in_collision, char* err,
                                  size_t errlen) {
  if (!path || k_max < 0 || n_particles < 0) return ASICP_INVALID_ARGUMENT;
  const int64_t rows = k_max * n_particles;
  if (rows > 0 && (!particle_preshape || !trace_theta || !trace_loss || !trace_in_collision))
    return ASICP_INVALID_ARGUMENT;
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    set_err(std::string("cannot write trace: ") + path, err, errlen);
    return ASICP_INVALID_ARGUMENT;
  }
  std::string out;
  out.reserve(static_cast<size_t>(rows) * 160 + 128);
  out += "# graspmatch trace v1: iteration particle preshape phase loss in_collision tx ty tz qw qx qy qz\n";
  for (int64_t k = 0; k < k_max; ++k) {
    const char* phase = k < k_stein ? "stein" : "sgd";
    for (int64_t j = 0; j < n_particles; ++j) {
      const int64_t r = k * n_particles + j;
      put_u64(out, static_cast<uint64_t>(k));
      out += ' ';
      put_u64(out, static_cast<uint64_t>(j));
      out += ' ';
      put_u64(out, static_cast<uint64_t>(particle_preshape[j]));
      out += ' ';
      out += phase;
      out += ' ';
      put_double(out, trace_loss[r]);
      out += trace_in_collision[r] ? " 1" : " 0";
      for (int a = 0; a < 7; ++a) {
        out += ' ';
        put_double(out, trace_theta[7 * r + a]);
      }
      out += '\n';
    }
  }
  const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
  const bool closed = std::fclose(f) == 0;
  if (!ok || !closed) {
    set_err(std::string("trace write failed: ") + path, err, errlen);
    return ASICP_DEVICE_ERROR;
  }
  return ASICP_OK;
}
