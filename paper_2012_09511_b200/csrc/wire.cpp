// The reference's coordinator-worker wire protocol and a GPU worker that speaks it
// (SURVEY.md §8(f) next #3): a B200 pool joins the reference's multi-box runtime as a worker.
//
//   frames        src/protocol.cpp:104-177, protocol.hpp:16-52: u32 big-endian length (tag byte +
//                 payload), u8 tag (1 WORK, 2 BEST, 3 END); WORK from a worker = u32 worker_id,
//                 u64 nodes_since_checkpoint, u32 kmax, intervals; WORK from the coordinator =
//                 intervals; intervals = u32 count, then per interval two BigCounts, each a u16
//                 big-endian byte count and that many big-endian magnitude bytes (zero = none);
//                 BEST / END = u64 makespan (UINT64_MAX = none), u32 length, u32 jobs
//   transport     src/transport.cpp:108-341: blocking TCP, TCP_NODELAY, frames read exactly,
//                 a length above 64 MiB is refused
//   worker role   src/worker.cpp:138-296: NEH + 2000-iteration insertion search seed, initial
//                 bound offered, then rounds of apply_work_update -> run_round -> BEST on an
//                 improved schedule -> WORK checkpoint (steals >= K/5, checkpoint timer, or
//                 exhaustion) until END. The reference's comm agent runs the request / reply
//                 exchange beside the pool with a single-slot outbox; here it runs inline between
//                 rounds (one outstanding message either way; a GPU round is milliseconds).
//
// Interval endpoints are decimal BigCounts on the wire and factoradic digit vectors at the
// pool's C-ABI; the conversion is done here with a small limb integer (no GMP).
// Built into libpbbgpu.so on top of the pool's C-ABI (include/pbbgpu.h) only.
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pbbgpu.h"

namespace {

struct TransportError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ limb integer
struct Big {
  std::vector<uint32_t> w;  // little-endian limbs, no leading zero limb
  void trim() {
    while (!w.empty() && !w.back()) w.pop_back();
  }
  void mul_add(uint32_t mul, uint32_t add) {
    uint64_t carry = add;
    for (uint32_t& x : w) {
      const uint64_t v = static_cast<uint64_t>(x) * mul + carry;
      x = static_cast<uint32_t>(v);
      carry = v >> 32;
    }
    if (carry) w.push_back(static_cast<uint32_t>(carry));
    trim();
  }
  uint32_t div_small(uint32_t d) {  // *this /= d, returns the remainder
    uint64_t rem = 0;
    for (size_t i = w.size(); i-- > 0;) {
      const uint64_t cur = (rem << 32) | w[i];
      w[i] = static_cast<uint32_t>(cur / d);
      rem = cur % d;
    }
    trim();
    return static_cast<uint32_t>(rem);
  }
};

int cmp(const Big& a, const Big& b) {
  if (a.w.size() != b.w.size()) return a.w.size() < b.w.size() ? -1 : 1;
  for (size_t i = a.w.size(); i-- > 0;)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

Big factorial(int n) {
  Big f;
  f.w = {1};
  for (int i = 2; i <= n; ++i) f.mul_add(static_cast<uint32_t>(i), 0);
  return f;
}

// to_decimal (src/factoradic.cpp:18-33): Horner over radices n, n-1, ..., 1
Big from_digits(const uint16_t* d, int n) {
  Big x;
  for (int l = 0; l < n; ++l) x.mul_add(static_cast<uint32_t>(n - l), d[l]);
  return x;
}

// from_decimal (src/factoradic.cpp:35-49): least significant digit first; x < n! required
void to_digits(Big x, int n, uint16_t* d) {
  for (int l = n - 1; l >= 0; --l) d[l] = static_cast<uint16_t>(x.div_small(static_cast<uint32_t>(n - l)));
  if (!x.w.empty()) throw std::invalid_argument("interval endpoint beyond n!");
}

Big from_bytes(const uint8_t* p, size_t len) {
  Big x;
  for (size_t i = 0; i < len; ++i) x.mul_add(256, p[i]);
  return x;
}

std::vector<uint8_t> to_bytes(const Big& x) {  // minimal big-endian magnitude, zero = no bytes
  std::vector<uint8_t> out;
  for (size_t i = x.w.size(); i-- > 0;)
    for (int s = 24; s >= 0; s -= 8) out.push_back(static_cast<uint8_t>(x.w[i] >> s));
  size_t z = 0;
  while (z < out.size() && !out[z]) ++z;
  out.erase(out.begin(), out.begin() + static_cast<std::ptrdiff_t>(z));
  return out;
}

// ------------------------------------------------------------------ frames
enum : uint8_t { kTagWork = 1, kTagBest = 2, kTagEnd = 3 };
enum Kind { WorkRequest, WorkReply, Best, End };

struct Msg {
  Kind kind = Best;
  uint32_t worker_id = 0;
  uint64_t nodes = 0;
  uint32_t kmax = 0;
  std::vector<std::pair<Big, Big>> ivs;
  uint64_t makespan = UINT64_MAX;
  std::vector<uint32_t> sched;
};

void put_u16(std::vector<uint8_t>& b, uint16_t v) {
  b.push_back(static_cast<uint8_t>(v >> 8));
  b.push_back(static_cast<uint8_t>(v));
}
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int s = 24; s >= 0; s -= 8) b.push_back(static_cast<uint8_t>(v >> s));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
  for (int s = 56; s >= 0; s -= 8) b.push_back(static_cast<uint8_t>(v >> s));
}
void put_big(std::vector<uint8_t>& b, const Big& x) {
  const std::vector<uint8_t> m = to_bytes(x);
  if (m.size() > UINT16_MAX) throw std::length_error("BigCount too large for the wire");
  put_u16(b, static_cast<uint16_t>(m.size()));
  b.insert(b.end(), m.begin(), m.end());
}

std::vector<uint8_t> encode(const Msg& m) {
  std::vector<uint8_t> pl;
  if (m.kind == WorkRequest) {
    put_u32(pl, m.worker_id);
    put_u64(pl, m.nodes);
    put_u32(pl, m.kmax);
  }
  if (m.kind == WorkRequest || m.kind == WorkReply) {
    put_u32(pl, static_cast<uint32_t>(m.ivs.size()));
    for (const auto& iv : m.ivs) {
      put_big(pl, iv.first);
      put_big(pl, iv.second);
    }
  } else {
    put_u64(pl, m.makespan);
    put_u32(pl, static_cast<uint32_t>(m.sched.size()));
    for (uint32_t j : m.sched) put_u32(pl, j);
  }
  std::vector<uint8_t> fr;
  put_u32(fr, static_cast<uint32_t>(pl.size() + 1));
  fr.push_back(m.kind == Best ? kTagBest : (m.kind == End ? kTagEnd : kTagWork));
  fr.insert(fr.end(), pl.begin(), pl.end());
  return fr;
}

struct Reader {
  const uint8_t* p;
  size_t n, i = 0;
  uint64_t take(int k) {
    if (i + static_cast<size_t>(k) > n) throw std::runtime_error("truncated frame");
    uint64_t v = 0;
    for (int t = 0; t < k; ++t) v = v << 8 | p[i++];
    return v;
  }
  Big big() {
    const size_t len = static_cast<size_t>(take(2));
    if (i + len > n) throw std::runtime_error("truncated frame");
    Big x = from_bytes(p + i, len);
    i += len;
    return x;
  }
};

// sender_is_worker disambiguates the two WORK layouts (PeerRole, protocol.hpp:43)
Msg decode(const uint8_t* fr, size_t len, bool sender_is_worker) {
  Reader h{fr, len};
  const uint32_t L = static_cast<uint32_t>(h.take(4));
  if (len != static_cast<size_t>(L) + 4 || L < 1) throw std::runtime_error("frame length mismatch");
  const uint8_t tag = static_cast<uint8_t>(h.take(1));
  Reader r{fr + 5, len - 5};
  Msg m;
  if (tag == kTagWork) {
    m.kind = sender_is_worker ? WorkRequest : WorkReply;
    if (sender_is_worker) {
      m.worker_id = static_cast<uint32_t>(r.take(4));
      m.nodes = r.take(8);
      m.kmax = static_cast<uint32_t>(r.take(4));
    }
    const uint32_t cnt = static_cast<uint32_t>(r.take(4));
    for (uint32_t k = 0; k < cnt; ++k) {
      Big a = r.big(), b = r.big();
      if (cmp(a, b) >= 0) throw std::runtime_error("malformed interval on the wire (a >= b)");
      m.ivs.emplace_back(std::move(a), std::move(b));
    }
  } else if (tag == kTagBest || tag == kTagEnd) {
    m.kind = tag == kTagBest ? Best : End;
    m.makespan = r.take(8);
    const uint32_t cnt = static_cast<uint32_t>(r.take(4));
    for (uint32_t k = 0; k < cnt; ++k) m.sched.push_back(static_cast<uint32_t>(r.take(4)));
  } else {
    throw std::runtime_error("unknown message tag " + std::to_string(tag));
  }
  if (r.i != r.n) throw std::runtime_error("trailing bytes in frame");
  return m;
}

// ------------------------------------------------------------------ TCP worker side
struct Conn {
  int fd = -1;
  ~Conn() {
    if (fd >= 0) ::close(fd);
  }
  void connect_to(const char* host, int port) {
    addrinfo hints{}, *res = nullptr;
    hints.ai_family = AF_INET;
    hints.ai_socktype = SOCK_STREAM;
    const std::string ps = std::to_string(port);
    if (::getaddrinfo(host, ps.c_str(), &hints, &res) != 0 || !res) throw TransportError("cannot resolve coordinator host");
    fd = ::socket(AF_INET, SOCK_STREAM, 0);
    const int rc = fd >= 0 ? ::connect(fd, res->ai_addr, res->ai_addrlen) : -1;
    ::freeaddrinfo(res);
    if (rc != 0) throw TransportError(std::string("connect to coordinator failed: ") + std::strerror(errno));
    const int one = 1;
    ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
  }
  void send(const Msg& m) {
    const std::vector<uint8_t> fr = encode(m);
    size_t off = 0;
    while (off < fr.size()) {
      const ssize_t w = ::send(fd, fr.data() + off, fr.size() - off, MSG_NOSIGNAL);
      if (w < 0) {
        if (errno == EINTR) continue;
        throw TransportError(std::string("send failed: ") + std::strerror(errno));
      }
      off += static_cast<size_t>(w);
    }
  }
  void read_exact(uint8_t* p, size_t len) {
    size_t got = 0;
    while (got < len) {
      const ssize_t r = ::recv(fd, p + got, len - got, 0);
      if (r < 0) {
        if (errno == EINTR) continue;
        throw TransportError(std::string("recv failed: ") + std::strerror(errno));
      }
      if (r == 0) throw TransportError("coordinator closed the connection");
      got += static_cast<size_t>(r);
    }
  }
  Msg receive() {
    uint8_t head[4];
    read_exact(head, 4);
    const uint32_t L = static_cast<uint32_t>(head[0]) << 24 | static_cast<uint32_t>(head[1]) << 16 |
                       static_cast<uint32_t>(head[2]) << 8 | head[3];
    if (L < 1 || L > (64u << 20)) throw TransportError("unreasonable frame length");
    std::vector<uint8_t> fr(static_cast<size_t>(L) + 4);
    std::memcpy(fr.data(), head, 4);
    read_exact(fr.data() + 4, L);
    return decode(fr.data(), fr.size(), false);
  }
};

}  // namespace

void pbbgpu_internal_set_error(const char* msg);  // pool.cu: the C-ABI's pbbgpu_last_error()

namespace {

int set_err(const std::exception& e) {
  pbbgpu_internal_set_error(e.what());
  if (dynamic_cast<const TransportError*>(&e)) return PBBGPU_ERR_TRANSPORT;
  if (dynamic_cast<const std::invalid_argument*>(&e) || dynamic_cast<const std::length_error*>(&e)) return PBBGPU_ERR_ARG;
  return PBBGPU_ERR_TRANSPORT;  // protocol violations (malformed frames) are transport failures
}

void pcheck(int rc) {
  if (rc != PBBGPU_OK) throw std::runtime_error(std::string("pool: ") + pbbgpu_last_error());
}

}  // namespace

extern "C" {

int pbbgpu_wire_reencode(const uint8_t* frame, int64_t len, int sender_is_worker, int n, uint8_t* out, int64_t cap,
                         int64_t* out_len) {
  try {
    Msg m = decode(frame, static_cast<size_t>(len), sender_is_worker != 0);
    if (n > 0) {  // through the pool boundary's representation: factoradic digits, n! as a flag
      const Big nf = factorial(n);
      std::vector<uint16_t> d(static_cast<size_t>(n));
      for (auto& iv : m.ivs) {
        to_digits(iv.first, n, d.data());
        iv.first = from_digits(d.data(), n);
        if (cmp(iv.second, nf) != 0) {
          to_digits(iv.second, n, d.data());
          iv.second = from_digits(d.data(), n);
        }
      }
    }
    const std::vector<uint8_t> fr = encode(m);
    *out_len = static_cast<int64_t>(fr.size());
    if (static_cast<int64_t>(fr.size()) > cap) throw std::length_error("output buffer too small");
    std::memcpy(out, fr.data(), fr.size());
    return PBBGPU_OK;
  } catch (const std::exception& e) {
    return set_err(e);
  }
}

int pbbgpu_worker_run(pbbgpu_pool* pool, const char* host, int port, const pbbgpu_worker_config_t* cfg_in,
                      pbbgpu_worker_result_t* out) {
  using clock = std::chrono::steady_clock;
  try {
    if (!pool || !host || !out) throw std::invalid_argument("pbbgpu_worker_run: null argument");
    pbbgpu_worker_config_t cfg{};
    if (cfg_in) cfg = *cfg_in;
    if (cfg.checkpoint_period_s <= 0) cfg.checkpoint_period_s = 30.0;
    if (cfg.rng_seed == 0) cfg.rng_seed = 1;
    if (cfg.ils_iterations == 0) cfg.ils_iterations = 2000;
    cfg.send_initial_best = cfg.send_initial_best >= 0 ? 1 : 0;
    std::memset(out, 0, sizeof(*out));
    int n = 0, m = 0;
    pcheck(pbbgpu_pool_shape(pool, &n, &m));
    std::vector<int32_t> p(static_cast<size_t>(n) * m), seed(static_cast<size_t>(n)), perm(static_cast<size_t>(n));
    pcheck(pbbgpu_pool_times(pool, p.data()));
    // seed schedule (src/worker.cpp:144-152): NEH refined by an insertion descent
    int64_t cmax = pbbgpu_neh(n, m, p.data(), seed.data());
    if (cmax < 0) throw std::runtime_error(pbbgpu_last_error());
    if (n > 1 && cfg.ils_iterations > 0) {
      cmax = pbbgpu_insertion_ls(n, m, p.data(), seed.data(), static_cast<uint64_t>(cfg.ils_iterations), 0.0,
                                 cfg.rng_seed, perm.data());
      if (cmax < 0) throw std::runtime_error(pbbgpu_last_error());
      seed = perm;
    }
    pcheck(pbbgpu_set_initial_bound(pool, cmax, seed.data(), n));
    if (cfg.initial_ub > 0) pcheck(pbbgpu_offer_bound(pool, cfg.initial_ub));
    int dummy = 0;
    pcheck(pbbgpu_improved_since_mark(pool, &dummy));  // the seed is not an improvement to report

    Conn conn;
    conn.connect_to(host, port);
    const int K = pbbgpu_K(pool);
    const Big nfact = factorial(n);
    std::vector<uint16_t> a(static_cast<size_t>(K) * n), b(static_cast<size_t>(K) * n);
    std::vector<uint8_t> nf(static_cast<size_t>(K));
    bool have_work = false, done = false;
    std::vector<std::pair<Big, Big>> work;

    auto best_msg = [&](Kind kind) {
      Msg msg;
      msg.kind = kind;
      int64_t v = 0;
      int has = 0;
      pcheck(pbbgpu_best_schedule(pool, &v, perm.data(), &has));
      if (has) {
        msg.makespan = static_cast<uint64_t>(v);
        for (int i = 0; i < n; ++i) msg.sched.push_back(static_cast<uint32_t>(perm[static_cast<size_t>(i)]));
      }
      return msg;
    };
    auto exchange = [&](const Msg& msg) {  // the comm agent's loop body (src/worker.cpp:158-202)
      conn.send(msg);
      ++out->messages;
      Msg r = conn.receive();
      if (r.kind == Best) {
        if (r.makespan != UINT64_MAX) pcheck(pbbgpu_offer_bound(pool, static_cast<int64_t>(r.makespan)));
      } else if (r.kind == WorkReply) {
        work = std::move(r.ivs);
        have_work = true;
      } else if (r.kind == End) {
        if (r.makespan != UINT64_MAX) pcheck(pbbgpu_offer_bound(pool, static_cast<int64_t>(r.makespan)));
        conn.send(best_msg(End));  // the worker's final message, not answered
        ++out->messages;
        done = true;
      } else {
        throw TransportError("unexpected message from coordinator");
      }
    };

    const uint64_t steal_threshold = std::max<uint64_t>(1, (static_cast<uint64_t>(K) + 4) / 5);
    auto last_checkpoint = clock::time_point{};
    uint64_t nodes_at_last = 0;
    bool pending_best = cfg.send_initial_best != 0;
    while (!done) {
      if (have_work) {
        std::vector<uint16_t> wa(work.size() * static_cast<size_t>(n)), wb(work.size() * static_cast<size_t>(n), 0);
        std::vector<uint8_t> wnf(work.size(), 0);
        for (size_t i = 0; i < work.size(); ++i) {
          to_digits(work[i].first, n, wa.data() + i * static_cast<size_t>(n));
          if (cmp(work[i].second, nfact) == 0) wnf[i] = 1;
          else to_digits(work[i].second, n, wb.data() + i * static_cast<size_t>(n));
        }
        pcheck(pbbgpu_apply_work_update(pool, wa.data(), wb.data(), wnf.data(), static_cast<int>(work.size())));
        have_work = false;
        ++out->updates_applied;
      }
      int active = 0;
      pcheck(pbbgpu_run_round(pool, &active));
      int improved = 0;
      pcheck(pbbgpu_improved_since_mark(pool, &improved));
      if (improved) pending_best = true;
      if (pending_best) {
        Msg msg = best_msg(Best);
        if (!msg.sched.empty()) {
          exchange(msg);
          ++out->bests_sent;
        }
        pending_best = false;
        if (done) break;
      }
      uint64_t steals = 0;
      pcheck(pbbgpu_steals_since_mark(pool, &steals));
      const double since = std::chrono::duration<double>(clock::now() - last_checkpoint).count();
      if (steals >= steal_threshold || since >= cfg.checkpoint_period_s || active == 0) {
        int cnt = 0;
        uint64_t recount = 0;
        pcheck(pbbgpu_snapshot_ex(pool, a.data(), b.data(), nf.data(), K, &cnt, &recount));
        pbbgpu_stats_t st{};
        pcheck(pbbgpu_stats(pool, &st));
        Msg req;
        req.kind = WorkRequest;
        req.worker_id = cfg.worker_id;
        req.nodes = st.decomposed - nodes_at_last;
        req.kmax = static_cast<uint32_t>(K);
        for (int i = 0; i < cnt; ++i) {
          Big lo = from_digits(a.data() + static_cast<size_t>(i) * n, n);
          Big hi = nf[static_cast<size_t>(i)] ? nfact : from_digits(b.data() + static_cast<size_t>(i) * n, n);
          if (cmp(lo, hi) < 0) req.ivs.emplace_back(std::move(lo), std::move(hi));
        }
        std::sort(req.ivs.begin(), req.ivs.end(), [](const auto& x, const auto& y) { return cmp(x.first, y.first) < 0; });
        exchange(req);
        nodes_at_last = st.decomposed;
        pcheck(pbbgpu_reset_steal_mark(pool));
        last_checkpoint = clock::now();
        ++out->checkpoints_sent;
        if (active == 0 && !have_work && !done) std::this_thread::sleep_for(std::chrono::microseconds(200));
      }
    }
    int has = 0;
    pcheck(pbbgpu_best_schedule(pool, &out->local_best, nullptr, &has));
    out->has_schedule = has;
    return PBBGPU_OK;
  } catch (const std::exception& e) {
    return set_err(e);
  }
}

}  // extern "C"
