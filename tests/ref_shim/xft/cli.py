from paper_0912_1379_b200.cli import entrypoint, main  # noqa: F401

if __name__ == "__main__":
    entrypoint()
