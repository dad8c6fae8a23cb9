// Native fast path of parse_msms (mesh.py; reference pbbem/mesh.py:141-185):
// MSMS .vert/.face text -> vertex rows and 0-based faces, with the record
// rules of the Python parser (a vertex record is a line, '#' comment removed,
// with >= 6 tokens whose first token is a real; a face record has >= 3 tokens
// whose first three are integers).  strtod/strtoll are correctly rounded like
// Python's float()/int(); any line where the two could disagree (non-ASCII
// bytes, '_' or hex or nan/inf spellings, an int64 overflow) or where the
// Python parser would raise (a broken record, an index < 1) makes the scan
// report "irregular", and the caller re-runs the Python parser, which then
// produces the reference's exact error or result.  Host code only.
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hobi_internal.cuh"

namespace {

struct Tok {
  const char* p;
  int n;
};

inline bool space(char c) { return c == ' ' || c == '\t'; }

// Tokens of one line [b, e) (no line terminator) with the '#' comment
// removed; false if the line holds bytes where Python's splitlines()/split()
// could cut differently (control characters, non-ASCII).
bool tokens(const char* b, const char* e, std::vector<Tok>& out) {
  out.clear();
  for (const char* p = b; p < e; ++p) {
    const unsigned char c = static_cast<unsigned char>(*p);
    if (c >= 0x80 || (c < 0x20 && c != '\t')) return false;
  }
  const char* h = static_cast<const char*>(memchr(b, '#', e - b));
  if (h) e = h;
  const char* p = b;
  while (p < e) {
    while (p < e && space(*p)) ++p;
    if (p >= e) break;
    const char* q = p;
    while (q < e && !space(*q)) ++q;
    out.push_back({p, (int)(q - p)});
    p = q;
  }
  return true;
}

// 1 = a real for both strtod and Python float(), 0 = for neither,
// -1 = the two could disagree (underscores, hex, nan payloads, long tokens)
int as_double(const Tok& t, double* v) {
  char buf[64];
  if (t.n >= (int)sizeof(buf)) return -1;
  bool odd = false;
  for (int i = 0; i < t.n; ++i) {
    const char c = t.p[i];
    if (c == '_') return -1;
    odd |= c == 'x' || c == 'X' || c == '(';
  }
  memcpy(buf, t.p, t.n);
  buf[t.n] = '\0';
  char* end = nullptr;
  *v = strtod(buf, &end);
  const bool full = end != buf && *end == '\0';
  if (full && odd) return -1;
  return full ? 1 : 0;
}

// 1 = an int for both strtoll and Python int(), 0 = for neither, -1 = unsure
int as_int(const Tok& t, long long* v) {
  char buf[32];
  if (t.n >= (int)sizeof(buf)) return -1;
  for (int i = 0; i < t.n; ++i)
    if (t.p[i] == '_') return -1;
  memcpy(buf, t.p, t.n);
  buf[t.n] = '\0';
  char* end = nullptr;
  errno = 0;
  *v = strtoll(buf, &end, 10);
  if (end == buf || *end != '\0') return 0;
  if (errno == ERANGE) return -1;
  return 1;
}

// One line [b, le) of a text; `next` is where the following line starts.
inline const char* line_end(const char* b, const char* e, const char** next) {
  const char* nl = static_cast<const char*>(memchr(b, '\n', e - b));
  const char* le = nl ? nl : e;
  *next = nl ? nl + 1 : e;
  if (le > b && le[-1] == '\r') --le;  // CRLF
  return le;
}

// Scan (and, with outputs, fill).  Returns 0 on a regular text, 1 if irregular.
int scan(const char* vert, int64_t vlen, const char* face, int64_t flen, int64_t* nv, int64_t* nf,
         double* vdata, int64_t vcap, int64_t* faces, int64_t fcap) {
  std::vector<Tok> tk;
  int64_t rows = 0, tris = 0;
  const char* e = vert + vlen;
  for (const char* b = vert; b < e;) {
    const char* next;
    const char* le = line_end(b, e, &next);
    if (!tokens(b, le, tk)) return 1;
    b = next;
    if (tk.size() < 6) continue;  // the Python parser skips short lines whatever they hold
    double v[6];
    const int first = as_double(tk[0], &v[0]);
    if (first < 0) return 1;
    if (first == 0) continue;  // header / other record
    for (int k = 1; k < 6; ++k)
      if (as_double(tk[k], &v[k]) != 1) return 1;  // the Python parser raises (or might) here
    if (vdata) {
      if (rows >= vcap) return 1;
      for (int k = 0; k < 6; ++k) vdata[6 * rows + k] = v[k];
    }
    ++rows;
  }
  e = face + flen;
  for (const char* b = face; b < e;) {
    const char* next;
    const char* le = line_end(b, e, &next);
    if (!tokens(b, le, tk)) return 1;
    b = next;
    if (tk.size() < 3) continue;
    long long ijk[3];
    bool all = true;
    for (int k = 0; k < 3; ++k) {
      const int r = as_int(tk[k], &ijk[k]);
      if (r < 0) return 1;
      all = all && r == 1;
    }
    if (!all) continue;
    if (ijk[0] < 1 || ijk[1] < 1 || ijk[2] < 1) return 1;  // the Python parser raises here
    if (faces) {
      if (tris >= fcap) return 1;
      for (int k = 0; k < 3; ++k) faces[3 * tris + k] = ijk[k] - 1;
    }
    ++tris;
  }
  *nv = rows;
  *nf = tris;
  return 0;
}

}  // namespace

extern "C" {

int hobi_msms_parse(const char* vert, int64_t vlen, const char* face, int64_t flen, double* vdata,
                    int64_t vcap, int64_t* faces, int64_t fcap, int64_t* n_vert, int64_t* n_face) {
  *n_vert = *n_face = 0;
  if (scan(vert, vlen, face, flen, n_vert, n_face, vdata, vcap, faces, fcap))
    return hobi::fail(HOBI_ERR_VALUE, "irregular MSMS text: use the line-by-line parser");
  return 0;
}

}  // extern "C"
