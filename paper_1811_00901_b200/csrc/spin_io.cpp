// spin_io.cpp — host-side ingestion of oriented point clouds:
// the paper's `OP = read3DPoints(OF)` (Alg. 3) for the two formats the
// SPEC names (xyzn text, ASCII OFF triangle meshes) and area-weighted vertex normals for
// meshes without normals.  No CUDA: these run on the host before spin_create /
// spin_load_cloud, and are exported through the same C ABI (include/spin.h).
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "spin.h"

namespace spin {
spin_status io_fail(spin_status st, const char* fmt, ...);   // spin_api.cpp (last-error text)
}

namespace {

struct File {
  FILE* f = nullptr;
  explicit File(const char* p) : f(std::fopen(p, "rb")) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

// next non-empty, non-comment line; returns false at EOF
bool next_line(FILE* f, std::string& line, long& lineno) {
  line.clear();
  for (;;) {
    int c;
    line.clear();
    while ((c = std::fgetc(f)) != EOF && c != '\n') line.push_back((char)c);
    if (c == EOF && line.empty()) return false;
    ++lineno;
    size_t i = 0;
    while (i < line.size() && std::isspace((unsigned char)line[i])) ++i;
    if (i == line.size() || line[i] == '#') {
      if (c == EOF) return false;
      continue;
    }
    return true;
  }
}

// parse exactly n reals (double) from s; false if fewer, more, or malformed
bool parse_reals(const std::string& s, double* out, int n) {
  const char* p = s.c_str();
  char* end = nullptr;
  for (int i = 0; i < n; ++i) {
    errno = 0;
    out[i] = std::strtod(p, &end);
    if (end == p || errno == ERANGE) return false;
    p = end;
  }
  while (*p && std::isspace((unsigned char)*p)) ++p;
  return *p == '\0' || *p == '#';
}

}  // namespace

extern "C" {

spin_status spin_read_xyzn(const char* path, float* points, float* normals, int64_t cap,
                           int64_t* n_out) {
  if (!path || !n_out) return spin::io_fail(SPIN_E_INVAL, "null path or n_out");
  File F(path);
  if (!F.f) return spin::io_fail(SPIN_E_INVAL, "cannot open %s", path);
  std::string line;
  long lineno = 0;
  int64_t n = 0;
  while (next_line(F.f, line, lineno)) {
    double v[6];
    if (!parse_reals(line, v, 6))
      return spin::io_fail(SPIN_E_INPUT, "%s:%ld: expected six reals 'x y z nx ny nz'", path, lineno);
    for (double x : v)
      if (!std::isfinite(x)) return spin::io_fail(SPIN_E_INPUT, "%s:%ld: non-finite value", path, lineno);
    const double len = std::sqrt(v[3] * v[3] + v[4] * v[4] + v[5] * v[5]);
    if (!(len > 0.0) || !std::isfinite(len))
      return spin::io_fail(SPIN_E_INPUT, "%s:%ld: point %lld has a zero normal", path, lineno, (long long)n);
    if (points && normals) {
      if (n >= cap) return spin::io_fail(SPIN_E_RANGE, "%s holds more than cap = %lld points", path, (long long)cap);
      for (int a = 0; a < 3; ++a) {
        points[3 * n + a] = (float)v[a];
        normals[3 * n + a] = (float)(v[3 + a] / len);   // normalised once, in double
      }
    }
    ++n;
  }
  if (n == 0) return spin::io_fail(SPIN_E_INPUT, "%s: empty cloud", path);
  *n_out = n;
  return SPIN_OK;
}

spin_status spin_read_off(const char* path, float* vertices, int64_t vcap, int32_t* faces,
                          int64_t fcap, int64_t* nv_out, int64_t* nf_out) {
  if (!path || !nv_out || !nf_out) return spin::io_fail(SPIN_E_INVAL, "null path or count pointer");
  File F(path);
  if (!F.f) return spin::io_fail(SPIN_E_INVAL, "cannot open %s", path);
  std::string line;
  long lineno = 0;
  if (!next_line(F.f, line, lineno)) return spin::io_fail(SPIN_E_INPUT, "%s: empty file", path);
  // header: "OFF" alone, or "OFF nv nf ne" on one line
  size_t i = 0;
  while (i < line.size() && std::isspace((unsigned char)line[i])) ++i;
  if (line.compare(i, 3, "OFF") != 0) return spin::io_fail(SPIN_E_INPUT, "%s:%ld: missing OFF header", path, lineno);
  std::string rest = line.substr(i + 3);
  double cnt[3];
  if (!parse_reals(rest, cnt, 3)) {
    if (!next_line(F.f, line, lineno) || !parse_reals(line, cnt, 3))
      return spin::io_fail(SPIN_E_INPUT, "%s:%ld: expected 'nv nf ne'", path, lineno);
  }
  if (cnt[0] < 1 || cnt[1] < 0 || cnt[0] != std::floor(cnt[0]) || cnt[1] != std::floor(cnt[1]) ||
      cnt[0] > 2147483647.0 || cnt[1] > 2147483647.0)
    return spin::io_fail(SPIN_E_INPUT, "%s:%ld: bad vertex / face counts", path, lineno);
  const int64_t nv = (int64_t)cnt[0], nf = (int64_t)cnt[1];
  *nv_out = nv;
  *nf_out = nf;
  if (!vertices || !faces) return SPIN_OK;   // size query
  if (nv > vcap || nf > fcap) return spin::io_fail(SPIN_E_RANGE, "%s: buffers too small", path);
  for (int64_t v = 0; v < nv; ++v) {
    double x[3];
    if (!next_line(F.f, line, lineno) || !parse_reals(line, x, 3))
      return spin::io_fail(SPIN_E_INPUT, "%s:%ld: expected vertex 'x y z'", path, lineno);
    for (int a = 0; a < 3; ++a) {
      if (!std::isfinite(x[a])) return spin::io_fail(SPIN_E_INPUT, "%s:%ld: non-finite vertex", path, lineno);
      vertices[3 * v + a] = (float)x[a];
    }
  }
  for (int64_t f = 0; f < nf; ++f) {
    double x[4];
    if (!next_line(F.f, line, lineno) || !parse_reals(line, x, 4) || x[0] != 3.0)
      return spin::io_fail(SPIN_E_INPUT, "%s:%ld: expected triangle '3 i j k'", path, lineno);
    for (int a = 0; a < 3; ++a) {
      const double id = x[1 + a];
      if (id < 0 || id >= (double)nv || id != std::floor(id))
        return spin::io_fail(SPIN_E_INPUT, "%s:%ld: face index out of range", path, lineno);
      faces[3 * f + a] = (int32_t)id;
    }
  }
  return SPIN_OK;
}

spin_status spin_vertex_normals(const float* vertices, int64_t nv, const int32_t* faces,
                                int64_t nf, float* normals) {
  if (nv < 1 || nf < 0 || !vertices || !normals || (nf > 0 && !faces))
    return spin::io_fail(SPIN_E_INVAL, "bad vertex normal arguments");
  std::vector<double> acc(3 * (size_t)nv, 0.0);
  std::vector<unsigned char> touched((size_t)nv, 0);
  for (int64_t f = 0; f < nf; ++f) {
    const int32_t a = faces[3 * f], b = faces[3 * f + 1], c = faces[3 * f + 2];
    if (a < 0 || b < 0 || c < 0 || a >= nv || b >= nv || c >= nv)
      return spin::io_fail(SPIN_E_INPUT, "face %lld has an index outside [0, %lld)", (long long)f, (long long)nv);
    double e1[3], e2[3];
    for (int k = 0; k < 3; ++k) {
      e1[k] = (double)vertices[3 * b + k] - vertices[3 * a + k];
      e2[k] = (double)vertices[3 * c + k] - vertices[3 * a + k];
    }
    // un-normalised face normal: |e1 x e2| = twice the area (area weighting is implicit)
    const double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                         e1[0] * e2[1] - e1[1] * e2[0]};
    touched[a] = touched[b] = touched[c] = 1;
    for (int32_t v : {a, b, c})
      for (int k = 0; k < 3; ++k) acc[3 * (size_t)v + k] += n[k];
  }
  for (int64_t v = 0; v < nv; ++v) {
    if (!touched[v]) return spin::io_fail(SPIN_E_INPUT, "vertex %lld has no incident face", (long long)v);
    const double* n = &acc[3 * (size_t)v];
    const double len = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    if (!(len > 0.0)) return spin::io_fail(SPIN_E_INPUT, "vertex %lld has only degenerate faces", (long long)v);
    for (int k = 0; k < 3; ++k) normals[3 * v + k] = (float)(n[k] / len);
  }
  return SPIN_OK;
}

}  // extern "C"
