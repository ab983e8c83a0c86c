// Test-infrastructure stub (NOT product code): just enough of cpp-httplib's
// surface for the reference's embedding.cpp / engine_service.cpp to compile.
// Every client call fails with a transport error; servers never bind.  The
// reference's HTTP paths are out of scope.
#pragma once
#include <functional>
#include <map>
#include <memory>
#include <string>

namespace httplib {
using Headers = std::multimap<std::string, std::string>;
enum class Error { Success = 0, Connection = 2 };
inline std::string to_string(Error) { return "connection (stub)"; }

struct Request {
  std::string body;
  Headers headers;
};
struct Response {
  int status = 200;
  std::string body;
  void set_content(const std::string& b, const std::string&) { body = b; }
};
class Result {
 public:
  explicit operator bool() const { return false; }
  const Response* operator->() const { return &r_; }
  const Response& operator*() const { return r_; }
  Error error() const { return Error::Connection; }

 private:
  Response r_;
};
class Client {
 public:
  explicit Client(const std::string&) {}
  Client(const std::string&, int) {}
  void set_connection_timeout(int, int) {}
  void set_read_timeout(int, int) {}
  void set_write_timeout(int, int) {}
  Result Post(const std::string&, const Headers&, const std::string&, const std::string&) {
    return Result();
  }
  Result Post(const std::string&, const std::string&, const std::string&) { return Result(); }
  Result Get(const std::string&) { return Result(); }
};
using Handler = std::function<void(const Request&, Response&)>;
class Server {
 public:
  Server& Post(const std::string&, Handler) { return *this; }
  Server& Get(const std::string&, Handler) { return *this; }
  bool bind_to_port(const std::string&, int) { return false; }
  int bind_to_any_port(const std::string&) { return -1; }
  bool listen_after_bind() { return false; }
  bool listen(const std::string&, int) { return false; }
  void stop() {}
  bool is_running() const { return false; }
  void wait_until_ready() const {}
};
}  // namespace httplib
