// obj.cpp -- native Wavefront OBJ ingest with the
// semantics of the reference's load_obj (mesh.py:112-163): `v` and `f`
// records, `#` comments, polygons fan-triangulated, negative indices relative
// to the vertex count at the point of use, every other record ignored.
// Tokens parse like Python's float() / int() on ASCII input (underscores
// between digits allowed, inf / nan spellings); errors carry the 1-based
// line number and the reference's message.  Host code only (no GPU).
#include <stdint.h>

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gdist.h"

namespace gd {

void set_error(const std::string& msg);

struct ObjData {
  std::vector<double> v;   // 3 per vertex
  std::vector<int64_t> t;  // 3 per triangle
};

namespace {

// str.split() whitespace on ASCII: \t \n \v \f \r, \x1c-\x1f and space
inline bool is_space(unsigned char c) { return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f); }

// Python's underscore rule: a single '_' only between two digits
bool strip_underscores(const std::string& s, std::string& out) {
  out.clear();
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i] == '_') {
      if (i == 0 || i + 1 >= s.size() || !isdigit((unsigned char)s[i - 1]) || !isdigit((unsigned char)s[i + 1]))
        return false;
      continue;
    }
    out.push_back(s[i]);
  }
  return true;
}

bool parse_float(const std::string& tok, double& out) {
  std::string s;
  if (!strip_underscores(tok, s) || s.empty()) return false;
  // Python accepts inf / infinity / nan with an optional sign, any case
  std::string low;
  for (char c : s) low.push_back((char)tolower((unsigned char)c));
  size_t k = (low[0] == '+' || low[0] == '-') ? 1 : 0;
  const std::string body = low.substr(k);
  if (body == "inf" || body == "infinity" || body == "nan") {
    out = body == "nan" ? NAN : INFINITY;
    if (low[0] == '-') out = -out;
    return true;
  }
  // otherwise a decimal literal: digits, '.', exponent (no hex, no spaces)
  for (char c : body)
    if (!(isdigit((unsigned char)c) || c == '.' || c == 'e' || c == '+' || c == '-')) return false;
  errno = 0;
  char* end = nullptr;
  out = strtod(s.c_str(), &end);
  return end == s.c_str() + s.size() && end != s.c_str();
}

// int(): optional sign, digits (underscores between digits); *big = the
// value does not fit 64 bits (the reference then reports it out of range)
bool parse_int(const std::string& tok, long long& out, bool* big, std::string& canon) {
  std::string s;
  *big = false;
  if (!strip_underscores(tok, s) || s.empty()) return false;
  size_t i = (s[0] == '+' || s[0] == '-') ? 1 : 0;
  if (i >= s.size()) return false;
  for (size_t j = i; j < s.size(); ++j)
    if (!isdigit((unsigned char)s[j])) return false;
  size_t nz = s.find_first_not_of('0', i);
  canon = nz == std::string::npos ? std::string("0") : s.substr(nz);
  if (s[0] == '-' && canon != "0") canon = "-" + canon;  // str(int(...))
  errno = 0;
  out = strtoll(s.c_str(), nullptr, 10);
  if (errno == ERANGE) *big = true;
  return true;
}

// Python's repr of an ASCII string (the reference formats tokens with !r)
std::string py_repr(const std::string& s) {
  const bool has_sq = s.find('\'') != std::string::npos, has_dq = s.find('"') != std::string::npos;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string r(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') {
      r.push_back('\\');
      r.push_back((char)c);
    } else if (c == '\t') {
      r += "\\t";
    } else if (c == '\n') {
      r += "\\n";
    } else if (c == '\r') {
      r += "\\r";
    } else if (c < 0x20 || c == 0x7f) {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", c);
      r += buf;
    } else {
      r.push_back((char)c);
    }
  }
  r.push_back(q);
  return r;
}

struct ParseError {
  long long line;
  std::string msg;
};

}  // namespace

ObjData* obj_parse(const char* path, long long* err_line) {
  FILE* fh = fopen(path, "rb");
  if (!fh) {
    set_error(std::string("cannot open ") + path + ": " + strerror(errno));
    *err_line = 0;
    return nullptr;
  }
  std::string text;
  {
    char buf[1 << 16];
    size_t n;
    while ((n = fread(buf, 1, sizeof buf, fh)) > 0) text.append(buf, n);
    fclose(fh);
  }
  ObjData* d = new ObjData();
  std::vector<std::string> tok;
  std::vector<int64_t> idx;
  long long line_no = 0;
  try {
    size_t pos = 0;
    const size_t n = text.size();
    while (pos < n) {
      // universal newlines, as Python's text mode: \n, \r\n and a lone \r
      size_t end = pos;
      while (end < n && text[end] != '\n' && text[end] != '\r') ++end;
      size_t next = end;
      if (next < n) next += (text[next] == '\r' && next + 1 < n && text[next + 1] == '\n') ? 2 : 1;
      ++line_no;
      size_t stop = end;
      for (size_t c = pos; c < end; ++c)
        if (text[c] == '#') {
          stop = c;
          break;
        }
      tok.clear();
      size_t i = pos;
      while (i < stop) {
        while (i < stop && is_space((unsigned char)text[i])) ++i;
        size_t j = i;
        while (j < stop && !is_space((unsigned char)text[j])) ++j;
        if (j > i) tok.emplace_back(text, i, j - i);
        i = j;
      }
      pos = next;
      if (tok.empty()) continue;
      if (tok[0] == "v") {
        if (tok.size() < 4) throw ParseError{line_no, "vertex needs 3 coordinates"};
        for (int c = 1; c <= 3; ++c) {
          double x;
          if (!parse_float(tok[c], x))
            throw ParseError{line_no, "bad vertex coordinate: could not convert string to float: " + py_repr(tok[c])};
          d->v.push_back(x);
        }
      } else if (tok[0] == "f") {
        if (tok.size() < 4) throw ParseError{line_no, "face needs at least 3 vertices"};
        idx.clear();
        const long long nv = (long long)(d->v.size() / 3);
        for (size_t k = 1; k < tok.size(); ++k) {
          const std::string head = tok[k].substr(0, tok[k].find('/'));
          long long ref;
          bool big;
          std::string canon;
          if (!parse_int(head, ref, &big, canon)) throw ParseError{line_no, "bad face index " + py_repr(tok[k])};
          if (!big && ref == 0) throw ParseError{line_no, "face index 0 is not valid OBJ"};
          const long long r = big ? -1 : (ref > 0 ? ref - 1 : nv + ref);
          if (r < 0 || r >= nv)
            throw ParseError{line_no, "face index " + canon + " out of range (have " + std::to_string(nv) + " vertices)"};
          idx.push_back(r);
        }
        for (size_t k = 1; k + 1 < idx.size(); ++k) {  // fan (mesh.py:108-109)
          d->t.push_back(idx[0]);
          d->t.push_back(idx[k]);
          d->t.push_back(idx[k + 1]);
        }
      }
    }
  } catch (const ParseError& e) {
    delete d;
    set_error(e.msg);
    *err_line = e.line;
    return nullptr;
  }
  return d;
}

}  // namespace gd

extern "C" {

int gd_obj_open(const char* path, void** handle, int64_t* n_vertices, int64_t* n_triangles, int64_t* err_line) {
  if (!path || !handle || !n_vertices || !n_triangles || !err_line) return GD_ERR_INVALID;
  long long line = 0;
  gd::ObjData* d = gd::obj_parse(path, &line);
  *err_line = line;
  if (!d) return GD_ERR_INVALID;
  *handle = d;
  *n_vertices = (int64_t)(d->v.size() / 3);
  *n_triangles = (int64_t)(d->t.size() / 3);
  return GD_OK;
}

int gd_obj_read(void* handle, double* vertices, int64_t* triangles) {
  if (!handle) return GD_ERR_INVALID;
  const gd::ObjData* d = static_cast<const gd::ObjData*>(handle);
  if (!d->v.empty()) memcpy(vertices, d->v.data(), d->v.size() * sizeof(double));
  if (!d->t.empty()) memcpy(triangles, d->t.data(), d->t.size() * sizeof(int64_t));
  return GD_OK;
}

void gd_obj_close(void* handle) { delete static_cast<gd::ObjData*>(handle); }

}  // extern "C"
