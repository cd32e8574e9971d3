// Host input pipeline: JSONL sample records ->
// the CSR index arrays of one Batch, parsed natively on several threads.
//
// Reference: data.py:293-311 (write_samples / read_samples: one JSON object
// per line with the SAMPLE_KEYS user, scenario, ad, ad_category, ad_image,
// behavior_items, behavior_images, label, day) followed by encode_batch
// (model.py:158-198), whose per-sample Python loops dominate at production
// batch sizes (SURVEY.md 7 hard part 7).  Here the bytes go straight to
// columns: scalar keys -> int32 [n], list keys -> (flat int32, offsets [n+1])
// keeping the most recent b_max entries (model.py:168, 176), labels -> f32.
//
// The buffer is split at line boundaries into one chunk per thread; each
// thread parses its chunk into private columns, which are concatenated in
// chunk order, so the result does not depend on the thread count.
#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dicm_b200.h"

namespace dicm {
int fail(int code, const char* fmt, ...);
}

namespace {

// A persistent worker pool for the per-step host copies: pool_run(n, fn)
// calls fn(0..n-1), fn(0) on the caller, the rest on pool threads created
// once (a step no longer pays thread creation).  One caller at a time.
class Pool {
 public:
  void run(int n, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> call(call_m_);
    {
      std::unique_lock<std::mutex> lk(m_);
      while ((int)th_.size() < n - 1) {
        const int id = (int)th_.size() + 1;
        th_.emplace_back([this, id] { loop(id); });
        th_.back().detach();
      }
      fn_ = &fn;
      n_ = n;
      left_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return left_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= n_) continue;
        f = fn_;
      }
      (*f)(id);
      std::unique_lock<std::mutex> lk(m_);
      if (--left_ == 0) done_.notify_one();
    }
  }
  std::mutex call_m_, m_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> th_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, left_ = 0;
  uint64_t gen_ = 0;
};

void pool_run(int n, const std::function<void(int)>& fn) {
  static Pool* pool = new Pool();  // never destroyed: detached workers outlive static destructors
  pool->run(n, fn);
}

struct Col {
  bool list = false;
  std::vector<int64_t> vals;   // scalars, or the flat list entries
  std::vector<int32_t> lens;   // list lengths per record (lists only)
};

struct Parsed {
  std::vector<std::string> keys;
  std::vector<bool> is_list;
  int label_key = -1;
  int b_max = 0;
  std::vector<Col> cols;
  int64_t n = 0;
};

struct Chunk {
  std::vector<Col> cols;
  int64_t n = 0, lines = 0, bad_line = -1;
  std::string err;
};

inline const char* skip_ws(const char* p, const char* e) {
  while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  return p;
}

// number: int, or a float (labels); returns false on malformed input
inline bool parse_num(const char*& p, const char* e, double& out, bool& is_int) {
  const char* s = p;
  if (p < e && (*p == '-' || *p == '+')) ++p;
  bool digits = false;
  while (p < e && *p >= '0' && *p <= '9') ++p, digits = true;
  is_int = true;
  if (p < e && (*p == '.' || *p == 'e' || *p == 'E')) {
    is_int = false;
    while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '-' || *p == '+'))
      ++p, digits = true;
  }
  if (!digits) return false;
  char buf[64];
  const size_t n = std::min<size_t>(p - s, sizeof(buf) - 1);
  memcpy(buf, s, n);
  buf[n] = 0;
  out = strtod(buf, nullptr);
  return true;
}

void parse_chunk(const Parsed& P, const char* b, const char* e, Chunk& C) {
  const size_t nk = P.keys.size();
  C.cols.assign(nk, Col());
  for (size_t k = 0; k < nk; ++k) C.cols[k].list = P.is_list[k];
  std::vector<int64_t> tmp;
  std::vector<char> seen(nk);
  const char* p = b;
  while (p < e) {
    const char* eol = static_cast<const char*>(memchr(p, '\n', e - p));
    if (!eol) eol = e;
    ++C.lines;
    const char* q = skip_ws(p, eol);
    if (q == eol) {  // blank line: skipped like the reference
      p = eol + 1;
      continue;
    }
    auto bad = [&](const char* why) {
      C.bad_line = C.lines;
      C.err = why;
    };
    if (*q != '{') return bad("expected a JSON object");
    ++q;
    std::fill(seen.begin(), seen.end(), 0);
    bool ok = true;
    while (ok) {
      q = skip_ws(q, eol);
      if (q < eol && *q == '}') {
        ++q;
        break;
      }
      if (q >= eol || *q != '"') {
        bad("expected a key");
        ok = false;
        break;
      }
      const char* ks = ++q;
      while (q < eol && *q != '"') ++q;
      if (q >= eol) {
        bad("unterminated key");
        ok = false;
        break;
      }
      const std::string key(ks, q - ks);
      ++q;
      q = skip_ws(q, eol);
      if (q >= eol || *q != ':') {
        bad("expected ':'");
        ok = false;
        break;
      }
      q = skip_ws(q + 1, eol);
      int k = -1;
      for (size_t i = 0; i < nk; ++i)
        if (P.keys[i] == key) k = (int)i;
      if (q < eol && *q == '[') {  // list of ints
        ++q;
        tmp.clear();
        while (true) {
          q = skip_ws(q, eol);
          if (q < eol && *q == ']') {
            ++q;
            break;
          }
          double v;
          bool is_int;
          if (!parse_num(q, eol, v, is_int) || !is_int) {
            bad("expected an integer list");
            ok = false;
            break;
          }
          tmp.push_back((int64_t)v);
          q = skip_ws(q, eol);
          if (q < eol && *q == ',') ++q;
        }
        if (!ok) break;
        if (k >= 0) {
          if (!P.is_list[k]) {
            bad("list where an integer was expected");
            ok = false;
            break;
          }
          const size_t keep = std::min<size_t>(tmp.size(), (size_t)P.b_max);  // most recent b_max
          Col& c = C.cols[k];
          c.vals.insert(c.vals.end(), tmp.end() - keep, tmp.end());
          c.lens.push_back((int32_t)keep);
          seen[k] = 1;
        }
      } else {
        double v;
        bool is_int;
        if (q < eol && *q == '"') {  // a string value (ignored key)
          ++q;
          while (q < eol && *q != '"') ++q;
          ++q;
          if (k >= 0) {
            bad("string where a number was expected");
            ok = false;
            break;
          }
        } else if (!parse_num(q, eol, v, is_int)) {
          bad("expected a number");
          ok = false;
          break;
        } else if (k >= 0) {
          if (P.is_list[k]) {
            bad("integer where a list was expected");
            ok = false;
            break;
          }
          if (k != P.label_key && !is_int) {
            bad("non-integer id");
            ok = false;
            break;
          }
          C.cols[k].vals.push_back(k == P.label_key ? (int64_t)(v * 1e6) : (int64_t)v);  // label in micro-units
          seen[k] = 1;
        }
      }
      q = skip_ws(q, eol);
      if (q < eol && *q == ',') ++q;
    }
    if (!ok) return;
    for (size_t i = 0; i < nk; ++i)
      if (!seen[i]) {
        static thread_local std::string msg;
        msg = "missing key '" + P.keys[i] + "'";
        C.bad_line = C.lines;
        C.err = msg;
        return;
      }
    ++C.n;
    p = eol + 1;
  }
}

}  // namespace

extern "C" {

void* dicm_jsonl_parse(const char* buf, int64_t len, const dicm_jsonl_spec_t* spec, int nthreads, int64_t* n_records,
                       int64_t* bad_line) {
  using namespace dicm;
  *bad_line = -1;
  auto* P = new Parsed();
  P->b_max = spec->b_max > 0 ? spec->b_max : 1 << 30;
  for (int i = 0; i < spec->n_keys; ++i) {
    P->keys.emplace_back(spec->keys[i]);
    P->is_list.push_back(spec->key_is_list[i] != 0);
    if (P->keys.back() == "label") P->label_key = i;
  }
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, len / (1 << 16) + 1));
  std::vector<const char*> cut(nt + 1);
  cut[0] = buf;
  cut[nt] = buf + len;
  for (int i = 1; i < nt; ++i) {  // chunk boundaries just after a newline
    const char* c = buf + len * i / nt;
    if (c < cut[i - 1]) c = cut[i - 1];
    const char* nl = static_cast<const char*>(memchr(c, '\n', buf + len - c));
    cut[i] = nl ? nl + 1 : buf + len;
  }
  std::vector<Chunk> ch(nt);
  std::vector<std::thread> th;
  for (int i = 0; i < nt; ++i) th.emplace_back([&, i] { parse_chunk(*P, cut[i], cut[i + 1], ch[i]); });
  for (auto& t : th) t.join();
  int64_t line0 = 0;
  for (int i = 0; i < nt; ++i) {
    if (ch[i].bad_line >= 0) {
      *bad_line = line0 + ch[i].bad_line;
      fail(DICM_ERR_VALUE, "line %lld: bad sample record: %s", (long long)*bad_line, ch[i].err.c_str());
      delete P;
      return nullptr;
    }
    line0 += ch[i].lines;
  }
  P->cols.assign(P->keys.size(), Col());
  for (size_t k = 0; k < P->keys.size(); ++k) {
    Col& c = P->cols[k];
    c.list = P->is_list[k];
    for (auto& x : ch) {
      c.vals.insert(c.vals.end(), x.cols[k].vals.begin(), x.cols[k].vals.end());
      c.lens.insert(c.lens.end(), x.cols[k].lens.begin(), x.cols[k].lens.end());
    }
  }
  for (auto& x : ch) P->n += x.n;
  *n_records = P->n;
  return P;
}

int64_t dicm_jsonl_list_total(void* h, int key) {
  auto* P = static_cast<Parsed*>(h);
  return (int64_t)P->cols[key].vals.size();
}

int dicm_jsonl_export(void* h, int key, int32_t* vals, int32_t* offsets, float* labels) {
  using namespace dicm;
  auto* P = static_cast<Parsed*>(h);
  const Col& c = P->cols[key];
  if (key == P->label_key) {
    for (size_t i = 0; i < c.vals.size(); ++i) labels[i] = (float)((double)c.vals[i] * 1e-6);
    return DICM_OK;
  }
  for (size_t i = 0; i < c.vals.size(); ++i) {
    const int64_t v = c.vals[i];
    if (v < INT32_MIN || v > INT32_MAX)
      return fail(DICM_ERR_KEY, "id %lld outside the int32 id range of this build", (long long)v);
    vals[i] = (int32_t)v;
  }
  if (c.list && offsets) {
    offsets[0] = 0;
    for (size_t i = 0; i < c.lens.size(); ++i) offsets[i + 1] = offsets[i] + c.lens[i];
  }
  return DICM_OK;
}

void dicm_jsonl_free(void* h) { delete static_cast<Parsed*>(h); }

// Packs n host segments into one buffer (the pinned upload staging of a
// batch): segment i = bytes[i] bytes from srcs[i] to dst + dst_off[i].  The
// total is cut into equal byte ranges, one per thread, so a batch of a few
// large columns still spreads over every thread.
int dicm_host_pack(void* dst, const void* const* srcs, const int64_t* bytes, const int64_t* dst_off, int n,
                   int nthreads) {
  int64_t total = 0;
  for (int i = 0; i < n; ++i) total += bytes[i];
  // a handful of threads saturate a host's memcpy bandwidth; more only add
  // contention when every GPU's rank packs at once (DICM_HOST_THREADS overrides)
  static const int def_threads = [] {
    const char* e = getenv("DICM_HOST_THREADS");
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    return e && atoi(e) > 0 ? atoi(e) : std::min(hw, 4);
  }();
  int nt = nthreads > 0 ? nthreads : def_threads;
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, total / (256 << 10) + 1));
  auto work = [&](int64_t lo, int64_t hi) {  // byte range [lo, hi) of the concatenated segments
    int64_t pos = 0;
    for (int i = 0; i < n && pos < hi; ++i) {
      const int64_t a = std::max(lo, pos), b = std::min(hi, pos + bytes[i]);
      if (a < b)
        memcpy(static_cast<char*>(dst) + dst_off[i] + (a - pos), static_cast<const char*>(srcs[i]) + (a - pos), b - a);
      pos += bytes[i];
    }
  };
  if (nt == 1) {
    work(0, total);
    return DICM_OK;
  }
  pool_run(nt, [&](int t) { work(total * t / nt, total * (t + 1) / nt); });
  return DICM_OK;
}

}  // extern "C"
