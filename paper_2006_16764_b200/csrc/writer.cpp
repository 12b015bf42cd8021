// Snapshot and mesh text writers, host C++.
//
// Byte-identical to undercool/vtkio.py:31-86: every number is printed as
// Python's repr(float) prints it -- the shortest digit string that round-trips
// (std::to_chars, same choice rule as CPython's dtoa mode 0) laid out with
// CPython's 'r' format rules (pystrtod.c format_float_short: exponent form
// when decpt <= -4 or decpt > 16, at least two exponent digits, ".0" on
// integral fixed-point values).  Node coordinates are regenerated as
// numpy.linspace builds them (i * (extent / count), last node = extent), so
// no coordinate array is needed.  Rows are formatted by a pool of threads
// into per-chunk buffers and written in order.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/uc_b200.h"

namespace uc {
int set_error(int code, const char* fmt, ...);
}

namespace {

// repr(float(x)) into out (>= 32 bytes); returns the length
int repr_double(double x, char* out) {
  if (std::isnan(x)) {
    std::memcpy(out, "nan", 3);
    return 3;
  }
  if (std::isinf(x)) {
    if (x < 0) {
      std::memcpy(out, "-inf", 4);
      return 4;
    }
    std::memcpy(out, "inf", 3);
    return 3;
  }
  char sci[40];
  const auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
  const char* p = sci;
  const char* end = r.ptr;
  int n = 0;
  if (*p == '-') {
    out[n++] = '-';
    ++p;
  }
  char digits[24];
  int nd = 0;
  while (p < end && *p != 'e') {
    if (*p != '.') digits[nd++] = *p;
    ++p;
  }
  int e10 = 0;
  if (p < end) std::from_chars(p + 1 + (p[1] == '+' ? 1 : 0), end, e10);
  const int decpt = e10 + 1;
  if (decpt <= -4 || decpt > 16) {
    out[n++] = digits[0];
    if (nd > 1) {
      out[n++] = '.';
      std::memcpy(out + n, digits + 1, nd - 1);
      n += nd - 1;
    }
    out[n++] = 'e';
    out[n++] = e10 < 0 ? '-' : '+';
    const int ae = e10 < 0 ? -e10 : e10;
    if (ae < 10) out[n++] = '0';
    const auto q = std::to_chars(out + n, out + n + 8, ae);
    n = (int)(q.ptr - out);
  } else if (decpt <= 0) {
    out[n++] = '0';
    out[n++] = '.';
    for (int i = 0; i < -decpt; ++i) out[n++] = '0';
    std::memcpy(out + n, digits, nd);
    n += nd;
  } else if (decpt >= nd) {
    std::memcpy(out + n, digits, nd);
    n += nd;
    for (int i = 0; i < decpt - nd; ++i) out[n++] = '0';
    out[n++] = '.';
    out[n++] = '0';
  } else {
    std::memcpy(out + n, digits, decpt);
    n += decpt;
    out[n++] = '.';
    std::memcpy(out + n, digits + decpt, nd - decpt);
    n += nd - decpt;
  }
  return n;
}

struct Axes {
  int dim;
  int64_t nn[3];
  double step[3], extent[3];
  int64_t nodes() const { return nn[0] * nn[1] * (dim == 3 ? nn[2] : 1); }
  // numpy.linspace(0, extent, nn): i * (extent / (nn - 1)), last = extent
  double coord(int a, int64_t i) const { return i == nn[a] - 1 ? extent[a] : (double)i * step[a]; }
  void point(int64_t id, double* x) const {
    x[0] = coord(0, id % nn[0]);
    const int64_t r = id / nn[0];
    x[1] = coord(1, dim == 3 ? r % nn[1] : r);
    x[2] = dim == 3 ? coord(2, r / nn[1]) : 0.0;
  }
};

bool make_axes(int dim, const int64_t* counts, const double* extents, Axes& ax) {
  if (dim < 2 || dim > 3 || !counts || !extents) return false;
  ax.dim = dim;
  for (int a = 0; a < 3; ++a) {
    const bool on = a < dim;
    ax.nn[a] = on ? counts[a] + 1 : 1;
    ax.extent[a] = on ? extents[a] : 0.0;
    ax.step[a] = on ? extents[a] / (double)counts[a] : 0.0;
    if (on && counts[a] < 1) return false;
  }
  return true;
}

// format rows [0, n) with fn(i, std::string&) on `threads` workers, write in order
template <class Fn>
bool write_rows(FILE* fh, int64_t n, int threads, Fn fn) {
  if (threads < 1) threads = 1;
  const int64_t chunk = 1 << 16;
  int64_t next = 0;
  while (next < n) {
    const int64_t batch_end = std::min<int64_t>(n, next + chunk * threads);
    const int64_t nb = (batch_end - next + chunk - 1) / chunk;
    std::vector<std::string> bufs((size_t)nb);
    std::vector<std::thread> pool;
    auto work = [&](int64_t b) {
      std::string& s = bufs[(size_t)b];
      const int64_t lo = next + b * chunk, hi = std::min(batch_end, lo + chunk);
      s.reserve((size_t)(hi - lo) * 64);
      for (int64_t i = lo; i < hi; ++i) fn(i, s);
    };
    for (int64_t b = 1; b < nb; ++b) pool.emplace_back(work, b);
    work(0);
    for (auto& t : pool) t.join();
    for (auto& s : bufs)
      if (fwrite(s.data(), 1, s.size(), fh) != s.size()) return false;
    next = batch_end;
  }
  return true;
}

inline void append_repr(std::string& s, double v) {
  char b[40];
  s.append(b, (size_t)repr_double(v, b));
}

}  // namespace

extern "C" int uc_repr_double(double x, char* out32) {
  if (!out32) return UC_ERR_ARG;
  out32[repr_double(x, out32)] = '\0';
  return UC_OK;
}

extern "C" int uc_write_snapshot(const char* path, int format, int dim, const int64_t* counts,
                                 const double* extents, int nfields, const char* const* names,
                                 const double* const* fields, const char* comment, int threads) {
  Axes ax;
  if (!path || !make_axes(dim, counts, extents, ax) || nfields < 0 || (nfields && (!names || !fields)) ||
      format < 0 || format > 1)
    return uc::set_error(UC_ERR_ARG, "uc_write_snapshot: bad argument");
  FILE* fh = fopen(path, "wb");
  if (!fh) return uc::set_error(UC_ERR_ARG, "uc_write_snapshot: cannot open %s", path);
  const int64_t n = ax.nodes();
  bool ok = true;
  if (format == 0) {  // write_snapshot_csv (vtkio.py:76-86)
    std::string head = dim == 3 ? "x,y,z" : "x,y";
    for (int f = 0; f < nfields; ++f) head += std::string(",") + names[f];
    head += "\n";
    ok = fwrite(head.data(), 1, head.size(), fh) == head.size();
    ok = ok && write_rows(fh, n, threads, [&](int64_t i, std::string& s) {
      double x[3];
      ax.point(i, x);
      for (int a = 0; a < dim; ++a) {
        if (a) s.push_back(',');
        append_repr(s, x[a]);
      }
      for (int f = 0; f < nfields; ++f) {
        s.push_back(',');
        append_repr(s, fields[f][i]);
      }
      s.push_back('\n');
    });
  } else {  // write_snapshot_vtk (vtkio.py:54-73)
    std::string head = "# vtk DataFile Version 3.0\n";
    head += (comment && *comment) ? comment : "solidification snapshot";
    head += "\nASCII\nDATASET STRUCTURED_GRID\n";
    head += "DIMENSIONS " + std::to_string(ax.nn[0]) + " " + std::to_string(ax.nn[1]) + " " +
            std::to_string(dim == 3 ? ax.nn[2] : 1) + "\n";
    head += "POINTS " + std::to_string(n) + " double\n";
    ok = fwrite(head.data(), 1, head.size(), fh) == head.size();
    ok = ok && write_rows(fh, n, threads, [&](int64_t i, std::string& s) {
      double x[3];
      ax.point(i, x);
      append_repr(s, x[0]);
      s.push_back(' ');
      append_repr(s, x[1]);
      s.push_back(' ');
      append_repr(s, x[2]);
      s.push_back('\n');
    });
    const std::string pd = "POINT_DATA " + std::to_string(n) + "\n";
    ok = ok && fwrite(pd.data(), 1, pd.size(), fh) == pd.size();
    for (int f = 0; f < nfields && ok; ++f) {
      const std::string sh = std::string("SCALARS ") + names[f] + " double 1\nLOOKUP_TABLE default\n";
      ok = fwrite(sh.data(), 1, sh.size(), fh) == sh.size();
      const double* v = fields[f];
      ok = ok && write_rows(fh, n, threads, [&](int64_t i, std::string& s) {
        append_repr(s, v[i]);
        s.push_back('\n');
      });
    }
  }
  ok = (fclose(fh) == 0) && ok;
  return ok ? UC_OK : uc::set_error(UC_ERR_ARG, "uc_write_snapshot: write failed for %s", path);
}

// write_mesh_vtk (vtkio.py:31-51): points, VTK-ordered Q1 cells, cell types
extern "C" int uc_write_mesh_vtk(const char* path, int dim, const int64_t* counts,
                                 const double* extents, int threads) {
  Axes ax;
  if (!path || !make_axes(dim, counts, extents, ax))
    return uc::set_error(UC_ERR_ARG, "uc_write_mesh_vtk: bad argument");
  FILE* fh = fopen(path, "wb");
  if (!fh) return uc::set_error(UC_ERR_ARG, "uc_write_mesh_vtk: cannot open %s", path);
  const int64_t n = ax.nodes();
  const int64_t ne = counts[0] * counts[1] * (dim == 3 ? counts[2] : 1);
  const int nloc = dim == 3 ? 8 : 4;
  // tensor local order -> VTK order (vtkio.py:20-24)
  static const int o2[4] = {0, 1, 3, 2};
  static const int o3[8] = {0, 1, 3, 2, 4, 5, 7, 6};
  const int* ord = dim == 3 ? o3 : o2;
  std::string head = "# vtk DataFile Version 3.0\nstructured solidification mesh\nASCII\n"
                     "DATASET UNSTRUCTURED_GRID\nPOINTS " + std::to_string(n) + " double\n";
  bool ok = fwrite(head.data(), 1, head.size(), fh) == head.size();
  ok = ok && write_rows(fh, n, threads, [&](int64_t i, std::string& s) {
    double x[3];
    ax.point(i, x);
    append_repr(s, x[0]);
    s.push_back(' ');
    append_repr(s, x[1]);
    s.push_back(' ');
    append_repr(s, x[2]);
    s.push_back('\n');
  });
  const std::string ch = "CELLS " + std::to_string(ne) + " " + std::to_string(ne * (nloc + 1)) + "\n";
  ok = ok && fwrite(ch.data(), 1, ch.size(), fh) == ch.size();
  ok = ok && write_rows(fh, ne, threads, [&](int64_t e, std::string& s) {
    const int64_t ex = e % counts[0], r = e / counts[0];
    const int64_t ey = dim == 3 ? r % counts[1] : r, ez = dim == 3 ? r / counts[1] : 0;
    s += std::to_string(nloc);
    for (int k = 0; k < nloc; ++k) {
      const int l = ord[k];
      const int64_t id = (ex + (l & 1)) + ax.nn[0] * ((ey + ((l >> 1) & 1)) + ax.nn[1] * (ez + (l >> 2)));
      s.push_back(' ');
      s += std::to_string(id);
    }
    s.push_back('\n');
  });
  const std::string ct = "CELL_TYPES " + std::to_string(ne) + "\n";
  ok = ok && fwrite(ct.data(), 1, ct.size(), fh) == ct.size();
  const std::string tline = dim == 3 ? "12\n" : "9\n";
  ok = ok && write_rows(fh, ne, threads, [&](int64_t, std::string& s) { s += tline; });
  ok = (fclose(fh) == 0) && ok;
  return ok ? UC_OK : uc::set_error(UC_ERR_ARG, "uc_write_mesh_vtk: write failed for %s", path);
}
