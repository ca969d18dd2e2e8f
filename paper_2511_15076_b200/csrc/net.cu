// net.cu -- the Proxy backend's socket transport: the path
// for peers the fabric cannot reach with loads and stores (another box, a
// NIC), built from the reference's GIN1 framing (wire.h; the reference's
// SocketTransport, proj/core/src/socket_transport.cpp:498-590).
//
// Between every ordered pair of ranks (a, b) one TCP connection: a's Put and
// Signal frames travel a -> b, b's Acks for a's puts travel back on the same
// connection (socket_transport.cpp:557-560).  Per rank:
//   * the proxy agent (proxy.cu) hands every descriptor toward a socket peer
//     here instead of issuing a peer-mapped copy: a put's source bytes are
//     copied device -> pinned staging on the peer's copy stream and queued
//     with an event; an inline value or a signal is queued as is;
//   * the sender thread sends the queue in order -- a put once its staging
//     copy completed (header from a small buffer, payload straight from the
//     pinned staging, one writev) -- so a signal frame always follows the
//     puts queued before it (its watermark = the last put's sequence);
//   * the receiver thread parses inbound frames: a put is copied into this
//     rank's window on the receive stream, a signal adds to the running value
//     of sub-cell [src][id] and writes it with a stream memop on the same
//     stream (after the puts that preceded it: the watermark rule,
//     fabric.cpp:63-79); once the stream has drained a batch it acks the
//     highest put sequence per source; an ack from a peer advances
//     acked[peer] in pinned, device-mapped memory;
//   * local completion (counters, flush words) waits for the acks: the
//     agent's completion stream holds a stream wait on acked[peer] >= the
//     last sequence posted to that peer before it writes them.
// The transport only uses this rank's own windows and signal table; the
// peers' VMM mappings are never touched for socket peers.
#include <arpa/inet.h>
#include <fcntl.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/uio.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>

#include "runtime_internal.h"
#include "wire.h"

namespace ginsim_b200 {

static uint64_t mono_ms() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000ull + (uint64_t)ts.tv_nsec / 1000000ull;
}

// ------------------------------------------------------------- TCP helpers
static std::string errno_str() { return std::string(std::strerror(errno)); }

static void set_nodelay(int fd) {
  int one = 1;
  setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
}

static in_addr_t parse_host(const std::string& host) {
  in_addr a{};
  if (inet_pton(AF_INET, host.c_str(), &a) != 1) fail(GINSIM_E_USAGE, "socket transport: host must be an IPv4 address, got '" + host + "'");
  return a.s_addr;
}

static int tcp_listen(in_addr_t addr, uint16_t port, uint16_t* bound, int backlog) {
  int fd = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (fd < 0) fail(GINSIM_E_GENERIC, "socket(): " + errno_str());
  int one = 1;
  setsockopt(fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
  sockaddr_in sa{};
  sa.sin_family = AF_INET;
  sa.sin_addr.s_addr = addr;
  sa.sin_port = htons(port);
  if (::bind(fd, reinterpret_cast<sockaddr*>(&sa), sizeof(sa)) != 0 || ::listen(fd, backlog) != 0) {
    const std::string e = errno_str();
    ::close(fd);
    fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "socket transport: bind/listen on port " + std::to_string(port) + ": " + e);
  }
  socklen_t len = sizeof(sa);
  getsockname(fd, reinterpret_cast<sockaddr*>(&sa), &len);
  if (bound) *bound = ntohs(sa.sin_port);
  return fd;
}

static int tcp_connect(in_addr_t addr, uint16_t port, uint64_t timeout_ms) {
  const uint64_t t0 = mono_ms();
  for (;;) {
    int fd = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (fd < 0) fail(GINSIM_E_GENERIC, "socket(): " + errno_str());
    sockaddr_in sa{};
    sa.sin_family = AF_INET;
    sa.sin_addr.s_addr = addr;
    sa.sin_port = htons(port);
    if (::connect(fd, reinterpret_cast<sockaddr*>(&sa), sizeof(sa)) == 0) {
      set_nodelay(fd);
      return fd;
    }
    ::close(fd);
    if (mono_ms() - t0 > timeout_ms)
      fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "socket transport: connect to port " + std::to_string(port) + " timed out");
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
}

static int tcp_accept(int lfd, uint64_t timeout_ms) {
  pollfd p{lfd, POLLIN, 0};
  const int r = ::poll(&p, 1, (int)std::min<uint64_t>(timeout_ms, 1u << 30));
  if (r <= 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "socket transport: no peer connected in time");
  int fd = ::accept4(lfd, nullptr, nullptr, SOCK_CLOEXEC);
  if (fd < 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "accept(): " + errno_str());
  set_nodelay(fd);
  return fd;
}

static void send_all(int fd, const void* data, size_t n) {
  const char* p = static_cast<const char*>(data);
  while (n) {
    const ssize_t w = ::send(fd, p, n, MSG_NOSIGNAL);
    if (w < 0) {
      if (errno == EINTR) continue;
      if (errno == EAGAIN || errno == EWOULDBLOCK) {
        pollfd pf{fd, POLLOUT, 0};
        ::poll(&pf, 1, 100);
        continue;
      }
      fail(GINSIM_E_GENERIC, "socket transport: send: " + errno_str());
    }
    p += w;
    n -= (size_t)w;
  }
}

static void sendv_all(int fd, iovec* iov, int cnt) {
  while (cnt > 0) {
    const ssize_t w = ::writev(fd, iov, cnt);
    if (w < 0) {
      if (errno == EINTR) continue;
      if (errno == EAGAIN || errno == EWOULDBLOCK) {
        pollfd pf{fd, POLLOUT, 0};
        ::poll(&pf, 1, 100);
        continue;
      }
      fail(GINSIM_E_GENERIC, "socket transport: writev: " + errno_str());
    }
    size_t left = (size_t)w;
    while (cnt > 0 && left >= iov->iov_len) {
      left -= iov->iov_len;
      ++iov;
      --cnt;
    }
    if (cnt > 0) {
      iov->iov_base = static_cast<char*>(iov->iov_base) + left;
      iov->iov_len -= left;
    }
  }
}

static void recv_exact(int fd, void* data, size_t n, uint64_t timeout_ms) {
  char* p = static_cast<char*>(data);
  const uint64_t t0 = mono_ms();
  while (n) {
    pollfd pf{fd, POLLIN, 0};
    const int r = ::poll(&pf, 1, 100);
    if (r < 0 && errno != EINTR) fail(GINSIM_E_GENERIC, "socket transport: poll: " + errno_str());
    if (r > 0) {
      const ssize_t g = ::recv(fd, p, n, 0);
      if (g == 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "socket transport: peer closed the connection");
      if (g < 0) {
        if (errno == EINTR || errno == EAGAIN) continue;
        fail(GINSIM_E_GENERIC, "socket transport: recv: " + errno_str());
      }
      p += g;
      n -= (size_t)g;
    }
    if (n && mono_ms() - t0 > timeout_ms) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "socket transport: receive timed out");
  }
}

// The first frame on a connection: CONTROL from `rank` carrying the rank.
static void send_hello(int fd, uint32_t rank) {
  uint8_t buf[wire::kControlPrefixBytes + 4];
  const size_t h = wire::encode_control_prefix(buf, rank, 4);
  std::memcpy(buf + h, &rank, 4);
  send_all(fd, buf, sizeof(buf));
}
static uint32_t recv_hello(int fd, uint64_t timeout_ms) {
  uint8_t buf[wire::kControlPrefixBytes + 4];
  recv_exact(fd, buf, sizeof(buf), timeout_ms);
  wire::Parser p;
  p.feed(buf, sizeof(buf));
  wire::Frame f;
  if (!p.next(f) || f.type != wire::kControl || f.body.size() != 4)
    fail(GINSIM_E_MALFORMED_FRAME, "socket transport: expected a hello frame");
  uint32_t r;
  std::memcpy(&r, f.body.data(), 4);
  return r;
}

// ------------------------------------------------------ socket bootstrap
// comm_init_socket's rendezvous (socket_transport.cpp:178-231): rank 0
// listens on host:port, every other rank connects and says hello; an
// allgather is a gather to rank 0 and a broadcast back.
struct SocketBoot {
  uint32_t world = 0, rank = 0;
  uint64_t timeout_ms = 30000;
  int root_fd = -1;            // rank != 0: the connection to rank 0
  std::vector<int> fds;        // rank 0: [rank] connection
};

static int sock_allgather(void* ctx, const void* send, void* recv, size_t bytes) {
  auto* b = static_cast<SocketBoot*>(ctx);
  try {
    char* out = static_cast<char*>(recv);
    if (b->rank == 0) {
      std::memcpy(out, send, bytes);
      for (uint32_t r = 1; r < b->world; ++r) recv_exact(b->fds[r], out + (size_t)r * bytes, bytes, b->timeout_ms);
      for (uint32_t r = 1; r < b->world; ++r) send_all(b->fds[r], out, (size_t)b->world * bytes);
    } else {
      send_all(b->root_fd, send, bytes);
      recv_exact(b->root_fd, out, (size_t)b->world * bytes, b->timeout_ms);
    }
    return 0;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 1;
  }
}

// ------------------------------------------------------ the transport
struct NetTransport {
  Comm* c = nullptr;
  uint32_t world = 0, rank = 0;
  std::vector<int> out_fd, in_fd;  // [peer]: my frames to peer / peer's frames to me
  std::vector<wire::Parser> out_parser, in_parser;

  // pinned staging ring for put payloads (device -> host before the send)
  static constexpr uint64_t kChunk = 4ull << 20;
  char* staging = nullptr;
  uint64_t staging_bytes = 0, st_head = 0, st_tail = 0;  // byte counters (mod staging_bytes)
  std::mutex st_mu;
  std::condition_variable st_cv;

  struct Op {
    uint8_t kind;  // wire::kPut / kSignal
    uint32_t peer;
    uint16_t ctx;
    uint64_t seq;
    uint32_t id;
    uint64_t offset, len;
    bool add;
    uint64_t operand;
    char* payload;          // staging (put from a window) or inline bytes
    uint64_t st_release;    // staging bytes to release after the send (0: inline)
    cudaEvent_t ready;      // the staging copy (null: inline)
    uint8_t inline_bytes[8];
  };
  std::mutex q_mu;
  std::condition_variable q_cv;
  std::deque<Op> q;
  std::vector<uint64_t> tx_seq;     // [peer] last put sequence posted (agent thread)

  uint64_t* acked = nullptr;        // pinned, device-mapped: [peer] highest put sequence acked
  uint64_t* acked_dev = nullptr;

  // receive side
  cudaStream_t rx_stream = nullptr;
  std::mutex sig_mu;
  std::vector<uint64_t> sig_rx;     // [src][cell] running value of sub-cell (src, cell) in my table
  std::atomic<uint64_t> rx_puts{0}, rx_bytes{0}, tx_frames{0};

  std::thread tx_th, rx_th;
  std::atomic<bool> stop{false};
  std::mutex fail_mu;
  std::string failure;
  std::atomic<bool> failed{false};

  void set_failed(const std::string& what) {
    std::lock_guard<std::mutex> lk(fail_mu);
    if (!failed.exchange(true)) failure = what;
  }

  // ---- staging ring: FIFO allocation, released in send order
  // (agent thread) a contiguous block of n bytes; *release = the bytes the
  // sender frees after sending it, including the padding skipped to avoid a wrap
  char* st_alloc(uint64_t n, uint64_t* release) {
    std::unique_lock<std::mutex> lk(st_mu);
    for (;;) {
      const uint64_t used = st_head - st_tail;
      const uint64_t pos = st_head % staging_bytes;
      const uint64_t pad = pos + n > staging_bytes ? staging_bytes - pos : 0;  // never wrap a block
      if (used + pad + n <= staging_bytes) {
        st_head += pad;
        char* p = staging + st_head % staging_bytes;
        st_head += n;
        *release = pad + n;
        return p;
      }
      if (failed.load()) {
        std::lock_guard<std::mutex> fl(fail_mu);  // (never taken before st_mu elsewhere)
        fail(GINSIM_E_GENERIC, "socket transport failed: " + failure);
      }
      st_cv.wait_for(lk, std::chrono::milliseconds(50));
    }
  }
  void st_free(uint64_t n) {
    {
      std::lock_guard<std::mutex> lk(st_mu);
      st_tail += n;
    }
    st_cv.notify_all();
  }

  void enqueue(Op&& op) {
    {
      std::lock_guard<std::mutex> lk(q_mu);
      q.push_back(std::move(op));
    }
    q_cv.notify_one();
  }

  // ---- sender thread
  void tx_main() {
    DeviceGuard g(c->device);
    uint8_t hdr[64];
    for (;;) {
      Op op;
      {
        std::unique_lock<std::mutex> lk(q_mu);
        q_cv.wait_for(lk, std::chrono::milliseconds(20), [&] { return !q.empty() || stop.load(); });
        if (q.empty()) {
          if (stop.load()) return;
          continue;
        }
        op = q.front();
        q.pop_front();
      }
      try {
        if (op.kind == wire::kPut) {
          const bool staged = op.ready != nullptr;
          if (staged) {
            GIN_CUDA(cudaEventSynchronize(op.ready));
            GIN_CUDA(cudaEventDestroy(op.ready));
          }
          const size_t h = wire::encode_put_prefix(hdr, rank, op.ctx, op.seq, op.id, op.offset, op.len);
          iovec iov[2] = {{hdr, h}, {staged ? (void*)op.payload : (void*)op.inline_bytes, (size_t)op.len}};
          sendv_all(out_fd[op.peer], iov, op.len ? 2 : 1);
          if (op.st_release) st_free(op.st_release);
        } else {
          const size_t h = wire::encode_signal(hdr, rank, op.ctx, op.seq, op.id, op.add, op.operand);
          send_all(out_fd[op.peer], hdr, h);
        }
        tx_frames.fetch_add(1, std::memory_order_relaxed);
      } catch (const std::exception& e) {
        if (!stop.load()) set_failed(e.what());
        if (op.st_release) st_free(op.st_release);
      }
    }
  }

  // ---- receiver thread
  void apply_put(uint32_t src, wire::Frame& f) {
    const GinDevCommView& v = c->host_view;
    // window registration is collective, but a peer may return from it and
    // put before this rank has recorded the window: give it the comm timeout
    const uint64_t t0 = mono_ms();
    while (f.id < GIN_MAX_WINDOWS && !((__atomic_load_n(&v.win_live, __ATOMIC_ACQUIRE) >> f.id) & 1ull) &&
           mono_ms() - t0 < c->cfg.timeout_ms && !stop.load())
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    if (f.id >= GIN_MAX_WINDOWS || !((__atomic_load_n(&v.win_live, __ATOMIC_ACQUIRE) >> f.id) & 1ull))
      fail(GINSIM_E_UNKNOWN_WINDOW, "socket transport: put into unknown window " + std::to_string(f.id));
    const GinWindowView& w = v.win[f.id];
    if (f.offset > w.size[rank] || f.body.size() > w.size[rank] - f.offset)
      fail(GINSIM_E_OUT_OF_BOUNDS, "socket transport: put exceeds the window");
    if (!f.body.empty())  // (pageable source: the call returns once the bytes are staged)
      GIN_CUDA(cudaMemcpyAsync(w.base[rank] + f.offset, f.body.data(), f.body.size(), cudaMemcpyHostToDevice, rx_stream));
    rx_puts.fetch_add(1, std::memory_order_relaxed);
    rx_bytes.fetch_add(f.body.size(), std::memory_order_relaxed);
    (void)src;
  }
  void apply_signal(uint32_t src, const wire::Frame& f) {
    const GinDevCommView& v = c->host_view;
    if (f.id >= v.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "socket transport: signal id out of range");
    uint64_t val;
    {
      std::lock_guard<std::mutex> lk(sig_mu);
      uint64_t& cell = sig_rx[(size_t)src * v.signal_cells + f.id];
      cell += f.add ? f.operand : 1ull;
      val = cell;
    }
    CUstreamBatchMemOpParams op{};
    op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
    op.writeValue.address = (CUdeviceptr)(v.signals[rank] + (uint64_t)src * v.signal_cells + f.id);
    op.writeValue.value64 = val;
    op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    GIN_CU(cuapi().cuStreamBatchMemOp((CUstream)rx_stream, 1, &op, 0));
  }

  void rx_main() {
    DeviceGuard g(c->device);
    std::vector<pollfd> pfd;
    std::vector<std::pair<uint32_t, bool>> who;  // (peer, inbound)
    for (uint32_t p = 0; p < world; ++p) {
      if (p == rank) continue;
      pfd.push_back(pollfd{in_fd[p], POLLIN, 0});
      who.emplace_back(p, true);
      pfd.push_back(pollfd{out_fd[p], POLLIN, 0});
      who.emplace_back(p, false);
    }
    std::vector<uint64_t> ack_due(world, 0);
    std::vector<uint8_t> open(pfd.size(), 1);
    std::vector<char> buf(1 << 20);
    while (!stop.load()) {
      const int r = ::poll(pfd.data(), pfd.size(), 5);
      if (r <= 0) continue;
      bool any_put = false;
      try {
        for (size_t i = 0; i < pfd.size(); ++i) {
          if (!open[i] || !(pfd[i].revents & (POLLIN | POLLHUP | POLLERR))) continue;
          const uint32_t peer = who[i].first;
          const bool inbound = who[i].second;
          for (;;) {
            const ssize_t n = ::recv(pfd[i].fd, buf.data(), buf.size(), MSG_DONTWAIT);
            if (n > 0) {
              (inbound ? in_parser[peer] : out_parser[peer]).feed(buf.data(), (size_t)n);
              if ((size_t)n < buf.size()) break;
              continue;
            }
            if (n == 0) {  // the peer tore down (anything still owed surfaces as a timeout)
              open[i] = 0;
              pfd[i].fd = -1;  // (poll skips it: a hung-up socket would report POLLHUP forever)
              break;
            }
            if (errno == EINTR) continue;
            if (errno != EAGAIN && errno != EWOULDBLOCK) {  // reset by a peer that left
              open[i] = 0;
              pfd[i].fd = -1;  // (poll skips it: a hung-up socket would report POLLHUP forever)
            }
            break;
          }
          wire::Frame f;
          wire::Parser& ps = inbound ? in_parser[peer] : out_parser[peer];
          while (ps.next(f)) {
            if (f.src != peer) fail(GINSIM_E_MALFORMED_FRAME, "socket transport: frame from rank " + std::to_string(f.src) +
                                                                  " on rank " + std::to_string(peer) + "'s connection");
            if (inbound && f.type == wire::kPut) {
              apply_put(peer, f);
              ack_due[peer] = std::max(ack_due[peer], f.seq);
              any_put = true;
            } else if (inbound && f.type == wire::kSignal) {
              apply_signal(peer, f);
            } else if (!inbound && f.type == wire::kAck) {
              uint64_t cur = __atomic_load_n(acked + peer, __ATOMIC_ACQUIRE);
              if (f.seq > cur) __atomic_store_n(acked + peer, f.seq, __ATOMIC_RELEASE);
            } else {
              fail(GINSIM_E_MALFORMED_FRAME, "socket transport: unexpected frame type " + std::to_string(f.type) +
                                                 (inbound ? " on an inbound connection" : " on an outbound connection"));
            }
          }
        }
        if (any_put) {
          // the batch's puts are performed in this rank's memory: ack the
          // highest sequence per source on the connection they came on
          GIN_CUDA(cudaStreamSynchronize(rx_stream));
          uint8_t a[wire::kAckBytes];
          for (uint32_t p = 0; p < world; ++p) {
            if (!ack_due[p]) continue;
            wire::encode_ack(a, rank, 0, ack_due[p]);
            send_all(in_fd[p], a, sizeof(a));
            ack_due[p] = 0;
          }
        }
      } catch (const std::exception& e) {
        if (!stop.load()) set_failed(e.what());
        return;
      }
    }
  }

  ~NetTransport() {
    stop.store(true);
    q_cv.notify_all();
    st_cv.notify_all();
    if (tx_th.joinable()) tx_th.join();
    if (rx_th.joinable()) rx_th.join();
    for (int fd : out_fd)
      if (fd >= 0) ::close(fd);
    for (int fd : in_fd)
      if (fd >= 0) ::close(fd);
    DeviceGuard g(c->device);
    if (rx_stream) cudaStreamDestroy(rx_stream);
    if (staging) cudaFreeHost(staging);
    if (acked) cudaFreeHost(acked);
  }
};

void NetDeleter::operator()(NetTransport* t) const { delete t; }

// Collective: every rank listens, the addresses are exchanged through the
// comm's bootstrap, then every rank connects to every peer and accepts the
// peers' connections.  GINSIM_NET_HOST (default 127.0.0.1) is the address
// this rank listens on and publishes.
NetPtr net_start(Comm* c) {
  NetPtr t(new NetTransport);
  t->c = c;
  t->world = c->world;
  t->rank = c->rank;
  const uint64_t tmo = c->cfg.timeout_ms;
  const char* h = std::getenv("GINSIM_NET_HOST");
  const in_addr_t addr = parse_host(h && *h ? h : "127.0.0.1");
  uint16_t port = 0;
  const int lfd = tcp_listen(addr, 0, &port, (int)c->world + 4);
  struct Addr {
    uint32_t ip;
    uint32_t port;
  } mine{(uint32_t)addr, port};
  std::vector<Addr> all(c->world);
  try {
    c->allgather(&mine, all.data(), sizeof(Addr));
    t->out_fd.assign(c->world, -1);
    t->in_fd.assign(c->world, -1);
    for (uint32_t p = 0; p < c->world; ++p) {
      if (p == c->rank) continue;
      t->out_fd[p] = tcp_connect(all[p].ip, (uint16_t)all[p].port, tmo);
      send_hello(t->out_fd[p], c->rank);
    }
    for (uint32_t i = 0; i + 1 < c->world; ++i) {
      const int fd = tcp_accept(lfd, tmo);
      const uint32_t r = recv_hello(fd, tmo);
      if (r >= c->world || r == c->rank || t->in_fd[r] >= 0) {
        ::close(fd);
        fail(GINSIM_E_DUPLICATE_ENDPOINT, "socket transport: unexpected hello from rank " + std::to_string(r));
      }
      t->in_fd[r] = fd;
    }
  } catch (...) {
    ::close(lfd);
    throw;
  }
  ::close(lfd);
  for (int fd : t->out_fd)
    if (fd >= 0) fcntl(fd, F_SETFL, fcntl(fd, F_GETFL) | O_NONBLOCK);
  for (int fd : t->in_fd)
    if (fd >= 0) fcntl(fd, F_SETFL, fcntl(fd, F_GETFL) | O_NONBLOCK);
  t->out_parser.resize(c->world);
  t->in_parser.resize(c->world);
  t->tx_seq.assign(c->world, 0);
  t->sig_rx.assign((size_t)c->world * c->cfg.signal_cells, 0);
  DeviceGuard g(c->device);
  const char* mb = std::getenv("GINSIM_NET_STAGING_MB");
  t->staging_bytes = (mb ? std::max<uint64_t>(8, std::strtoull(mb, nullptr, 10)) : 64ull) << 20;
  GIN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->staging), t->staging_bytes, cudaHostAllocDefault));
  GIN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->acked), c->world * sizeof(uint64_t), cudaHostAllocMapped));
  std::memset(t->acked, 0, c->world * sizeof(uint64_t));
  GIN_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t->acked_dev), t->acked, 0));
  GIN_CUDA(cudaStreamCreateWithFlags(&t->rx_stream, cudaStreamNonBlocking));
  NetTransport* raw = t.get();
  t->tx_th = std::thread([raw] { raw->tx_main(); });
  t->rx_th = std::thread([raw] { raw->rx_main(); });
  return t;
}

uint64_t net_put(NetTransport* t, uint32_t peer, uint32_t ctx, uint32_t win, uint64_t off, const char* dev_src,
                 uint64_t bytes, cudaStream_t stream) {
  net_check_failed(t);
  for (uint64_t done = 0; done < bytes;) {
    const uint64_t n = std::min(bytes - done, std::min(NetTransport::kChunk, t->staging_bytes / 4));
    uint64_t rel = 0;
    char* st = t->st_alloc(n, &rel);
    GIN_CUDA(cudaMemcpyAsync(st, dev_src + done, n, cudaMemcpyDeviceToHost, stream));
    cudaEvent_t ev;
    GIN_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    GIN_CUDA(cudaEventRecord(ev, stream));
    NetTransport::Op op{};
    op.kind = wire::kPut;
    op.peer = peer;
    op.ctx = (uint16_t)ctx;
    op.seq = ++t->tx_seq[peer];
    op.id = win;
    op.offset = off + done;
    op.len = n;
    op.payload = st;
    op.st_release = rel;
    op.ready = ev;
    t->enqueue(std::move(op));
    done += n;
  }
  return t->tx_seq[peer];
}

uint64_t net_put_inline(NetTransport* t, uint32_t peer, uint32_t ctx, uint32_t win, uint64_t off, uint64_t value,
                        uint32_t bytes) {
  net_check_failed(t);
  NetTransport::Op op{};
  op.kind = wire::kPut;
  op.peer = peer;
  op.ctx = (uint16_t)ctx;
  op.seq = ++t->tx_seq[peer];
  op.id = win;
  op.offset = off;
  op.len = bytes;
  std::memcpy(op.inline_bytes, &value, 8);  // little-endian: the value's low bytes first
  t->enqueue(std::move(op));
  return op.seq;
}

void net_signal(NetTransport* t, uint32_t peer, uint32_t ctx, uint32_t id, bool add, uint64_t operand) {
  net_check_failed(t);
  NetTransport::Op op{};
  op.kind = wire::kSignal;
  op.peer = peer;
  op.ctx = (uint16_t)ctx;
  op.seq = t->tx_seq[peer];  // watermark: the last put on this connection
  op.id = id;
  op.add = add;
  op.operand = operand;
  t->enqueue(std::move(op));
}

uint64_t* net_acked_device(NetTransport* t, uint32_t peer) { return t->acked_dev + peer; }
uint64_t net_last_seq(NetTransport* t, uint32_t peer) { return t->tx_seq[peer]; }

void net_release_waits(NetTransport* t) {
  for (uint32_t p = 0; p < t->world; ++p) __atomic_store_n(t->acked + p, ~0ull, __ATOMIC_RELEASE);
}

void net_reset_cells(NetTransport* t, uint32_t first, uint32_t span) {
  std::lock_guard<std::mutex> lk(t->sig_mu);
  const uint32_t cells = t->c->cfg.signal_cells;
  for (uint32_t s = 0; s < t->world; ++s)
    for (uint32_t i = first; i < first + span && i < cells; ++i) t->sig_rx[(size_t)s * cells + i] = 0;
}

void net_check_failed(NetTransport* t) {
  if (t->failed.load()) {
    std::lock_guard<std::mutex> lk(t->fail_mu);
    fail(GINSIM_E_GENERIC, "socket transport failed: " + t->failure);
  }
}

void net_stats(NetTransport* t, uint64_t* tx_frames, uint64_t* rx_puts, uint64_t* rx_bytes) {
  if (tx_frames) *tx_frames = t->tx_frames.load();
  if (rx_puts) *rx_puts = t->rx_puts.load();
  if (rx_bytes) *rx_bytes = t->rx_bytes.load();
}

}  // namespace ginsim_b200

using namespace ginsim_b200;

extern "C" {

int ginsim_cuda_socket_bootstrap_create(const char* host, uint16_t port, uint32_t world, uint32_t rank,
                                        uint64_t timeout_ms, ginsim_cuda_bootstrap* out) {
  GIN_API_BEGIN
  if (!out || !host) fail(GINSIM_E_USAGE, "socket bootstrap: null host or output");
  if (world == 0 || world > GIN_MAX_RANKS || rank >= world) fail(GINSIM_E_USAGE, "socket bootstrap: bad world / rank");
  auto b = std::make_unique<SocketBoot>();
  b->world = world;
  b->rank = rank;
  b->timeout_ms = timeout_ms ? timeout_ms : 30000;
  const in_addr_t addr = parse_host(host);
  if (rank == 0) {
    const int lfd = tcp_listen(addr, port, nullptr, (int)world + 4);
    b->fds.assign(world, -1);
    try {
      for (uint32_t i = 1; i < world; ++i) {
        const int fd = tcp_accept(lfd, b->timeout_ms);
        const uint32_t r = recv_hello(fd, b->timeout_ms);
        if (r == 0 || r >= world || b->fds[r] >= 0) {
          ::close(fd);
          fail(GINSIM_E_DUPLICATE_ENDPOINT, "socket bootstrap: duplicate or out-of-range rank " + std::to_string(r));
        }
        b->fds[r] = fd;
      }
    } catch (...) {
      ::close(lfd);
      throw;
    }
    ::close(lfd);
  } else {
    b->root_fd = tcp_connect(addr, port, b->timeout_ms);
    send_hello(b->root_fd, rank);
  }
  out->ctx = b.release();
  out->allgather = &sock_allgather;
  GIN_API_END
}

int ginsim_cuda_socket_bootstrap_destroy(ginsim_cuda_bootstrap* boot) {
  if (!boot || !boot->ctx) return GINSIM_OK;
  auto* b = static_cast<SocketBoot*>(boot->ctx);
  if (b->root_fd >= 0) ::close(b->root_fd);
  for (int fd : b->fds)
    if (fd >= 0) ::close(fd);
  delete b;
  boot->ctx = nullptr;
  return GINSIM_OK;
}

int ginsim_cuda_reserve_loopback_port(uint16_t* port) {
  GIN_API_BEGIN
  if (!port) fail(GINSIM_E_USAGE, "reserve_loopback_port: null output");
  const int fd = tcp_listen(htonl(INADDR_LOOPBACK), 0, port, 1);
  ::close(fd);
  GIN_API_END
}

int ginsim_cuda_net_stats(ginsim_cuda_comm_t comm, uint64_t* tx_frames, uint64_t* rx_puts, uint64_t* rx_bytes) {
  GIN_API_BEGIN
  if (!comm) fail(GINSIM_E_USAGE, "net_stats: null comm");
  NetTransport* t = proxy_net(&comm->impl);
  if (!t) fail(GINSIM_E_USAGE, "net_stats: the comm does not use the socket transport");
  net_stats(t, tx_frames, rx_puts, rx_bytes);
  GIN_API_END
}

}  // extern "C"
